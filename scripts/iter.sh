# GPU iteration: all parity tests, device-only benches of C3 (2D p16 2^20) and
# C4 (3D p8 100k) and C2 (2D p3 100k), one ncu --set full capture per fused kernel.
TAG=${1:-it}
mkdir -p gpurun_out
LOG=gpurun_out/$TAG.log
b() { timeout 300 python bench.py "$@" --steps 30 --warmup 3 --no-e2e --no-cpu 2>/dev/null \
  | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['value']/1e9,2), 'Gcell/s', round(d['roofline']['frac'],3), 'of HBM', round(d['ms_per_step'],4), 'ms', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
{
echo "== pytest -m gpu"; timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
echo "== bench"
b --dim 2 --p 16
b --dim 3 --p 8 --patches 100000
b --dim 2 --p 3 --patches 100000
for v in ${PV:-}; do FVB_TUNE_PENCIL_VARIANT=$v b --dim 2 --p 16; done
for v in ${SV:-}; do FVB_TUNE_SLAB_VARIANT=$v b --dim 3 --p 8 --patches 100000; done
echo "== ncu"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused2d -s 3 -c 1 -o gpurun_out/$TAG.p16 python bench.py --steps 3 --warmup 3 --warmup-seconds 0 --no-e2e --no-cpu > gpurun_out/$TAG.ncu2.log 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused3d -s 3 -c 1 -o gpurun_out/$TAG.p8 python bench.py --dim 3 --p 8 --patches 100000 --steps 3 --warmup 3 --warmup-seconds 0 --no-e2e --no-cpu > gpurun_out/$TAG.ncu3.log 2>&1; echo rc=$?
} > $LOG 2>&1
tail -40 $LOG
