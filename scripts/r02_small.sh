TAG=${1:-r02}
mkdir -p gpurun_out
LOG=gpurun_out/$TAG.small.log
{
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_physics.py -x -q -m gpu -k "p3 or p2 or p4 or 3-1000 or 2-129 or golden" 2>&1 | tail -3
for p in 2 3 4; do echo "== p=$p"; timeout 300 python scripts/small_ab.py --p $p --variants 0,6; done
echo "== p=3 exhaustive"; timeout 300 python scripts/small_ab.py --p 3 --variants 0,6 --filter 0
} > $LOG 2>&1
cat $LOG
