TAG=${1:-r02}
mkdir -p gpurun_out
LOG=gpurun_out/$TAG.3d.log
{
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_physics.py tests/test_gpu_layouts.py -x -q -m gpu -k "3d or 3-" 2>&1 | tail -3
FVB_TUNE_REDUCE_FILTER=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "slab_sizes or 3d" 2>&1 | tail -2
bash scripts/p3d_sweep.sh
} > $LOG 2>&1
cat $LOG
