# GPU pass: the whole -m gpu suite, then a short device-only bench line.
TAG=${1:-r02}
mkdir -p gpurun_out
LOG=gpurun_out/$TAG.all.log
timeout 2400 python -m pytest tests -x -q -m gpu --durations=15 > $LOG 2>&1
echo "suite rc=$?" >> $LOG
timeout 600 python bench.py --no-e2e --no-cpu --no-extras --steps 50 > gpurun_out/$TAG.quick.json 2> gpurun_out/$TAG.quick.err
echo "bench rc=$?" >> $LOG
tail -30 $LOG
cat gpurun_out/$TAG.quick.json | head -c 600
