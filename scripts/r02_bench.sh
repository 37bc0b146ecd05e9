# GPU pass: run_launch tests, then the default bench (+ reference arm).
TAG=${1:-r02}
mkdir -p gpurun_out
LOG=gpurun_out/$TAG.log
{
timeout 900 python -m pytest tests/test_gpu_launch.py tests/test_bench.py -x -q -m gpu 2>&1 | tail -30
echo "== bench"; timeout 900 python bench.py > gpurun_out/$TAG.bench.json 2> gpurun_out/$TAG.bench.err; echo rc=$?; tail -5 gpurun_out/$TAG.bench.err
echo "== reference"; timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/$TAG.ref.json 2> gpurun_out/$TAG.ref.err; echo rc=$?; tail -3 gpurun_out/$TAG.ref.err
} > $LOG 2>&1
tail -40 $LOG
