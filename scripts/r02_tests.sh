# GPU pass: new launch tests first, then the whole -m gpu suite, then sanitizers.
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,driver_version --format=csv > gpurun_out/$TAG.tests.log
nproc >> gpurun_out/$TAG.tests.log; lscpu | grep "Model name" >> gpurun_out/$TAG.tests.log
timeout 900 python -m pytest tests/test_gpu_launch.py -x -q -m gpu >> gpurun_out/$TAG.tests.log 2>&1
echo "launch rc=$?" >> gpurun_out/$TAG.tests.log
timeout 1500 python -m pytest tests -q -m gpu -x --deselect tests/test_gpu_launch.py >> gpurun_out/$TAG.tests.log 2>&1
echo "suite rc=$?" >> gpurun_out/$TAG.tests.log
tail -30 gpurun_out/$TAG.tests.log
