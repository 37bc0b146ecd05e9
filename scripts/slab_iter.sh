# 3D plane-walk kernel iteration: parity tests, variant sweep (C4: 3D p=8, 100k patches), ncu capture.
TAG=${1:-slab}
mkdir -p gpurun_out
LOG=gpurun_out/$TAG.log
{
echo "== pytest 3D"; timeout 900 python -m pytest tests -x -q -m gpu -k "3d or c4 or golden" 2>&1 | tail -15
for v in ${VARIANTS:-0 1 2 3}; do
  FVB_TUNE_SLAB_VARIANT=$v timeout 300 python bench.py --dim 3 --p 8 --patches 100000 --steps 30 --warmup 3 --no-e2e --no-cpu 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('slab variant $v', round(d['value']/1e9,2), 'Gcell/s', round(d['roofline']['frac'],3), 'of HBM', d['ms_per_step'], 'ms', d['clocks'])"
done
echo "== ncu full"; timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused3d -s 3 -c 1 -o gpurun_out/$TAG.slab python bench.py --dim 3 --p 8 --patches 100000 --steps 3 --warmup 3 --warmup-seconds 0 --no-e2e --no-cpu > gpurun_out/$TAG.ncu.log 2>&1; echo rc=$?
} > $LOG 2>&1
tail -40 $LOG
