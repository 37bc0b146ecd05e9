TAG=${1:-r02}
mkdir -p gpurun_out
LOG=gpurun_out/$TAG.small.log
{
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "tile" 2>&1 | tail -2
echo "== p=3"; timeout 300 python scripts/small_ab.py --p 3 --variants 0,7,3,6 --flush 2
echo "== p=3 exhaustive"; timeout 300 python scripts/small_ab.py --p 3 --variants 0 --filter 0 --flush 2
} > $LOG 2>&1
cat $LOG
