# GPU pass: run_launch drop-in tests + whole-batch full-size parity
TAG=${1:-r02}
mkdir -p gpurun_out
free -g > gpurun_out/$TAG.full.log
timeout 900 python -m pytest tests/test_gpu_launch.py -x -q >> gpurun_out/$TAG.full.log 2>&1
echo "launch rc=$?" >> gpurun_out/$TAG.full.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q --durations=0 >> gpurun_out/$TAG.full.log 2>&1
echo "full rc=$?" >> gpurun_out/$TAG.full.log
tail -40 gpurun_out/$TAG.full.log
