# Fast GPU iteration: parity tests, variant sweep, one ncu capture of the default kernel.
TAG=${1:-it}
mkdir -p gpurun_out
LOG=gpurun_out/$TAG.log
{
echo "== pytest -m gpu"; timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
echo "== sweep"; bash scripts/sweep_variants.sh $TAG
echo "== ncu full"; timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused2d -s 3 -c 1 -o gpurun_out/$TAG.fused python bench.py --steps 3 --warmup 3 --warmup-seconds 0 --no-e2e --no-cpu > gpurun_out/$TAG.ncu.log 2>&1; echo rc=$?
} > $LOG 2>&1
tail -40 $LOG
