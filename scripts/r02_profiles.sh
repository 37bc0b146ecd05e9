# Round-2 profile set: smoke, bench (+ reference arm), flavour + layout sweeps,
# launch list, ncu --set full of the three top kernels.
TAG=${1:-r02}
mkdir -p gpurun_out
LOG=gpurun_out/$TAG.log
{
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,driver_version --format=csv
nproc; free -g | head -2; lscpu | grep "Model name"
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
echo "== bench"; timeout 900 python bench.py > gpurun_out/$TAG.bench.json 2> gpurun_out/$TAG.bench.err; tail -3 gpurun_out/$TAG.bench.err
echo "== bench reference arm"; timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/$TAG.ref.json 2>&1; tail -c 300 gpurun_out/$TAG.ref.json
echo "== flavour sweep"; timeout 900 python scripts/flavour_sweep.py --out gpurun_out/$TAG.flavours.csv 2>&1 | tail -30
echo "== layout sweep"; timeout 900 python scripts/layout_sweep.py --out gpurun_out/$TAG.layouts.csv 2>&1 | tail -12
echo "== launches"; timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$TAG.launches.csv python bench.py --steps 5 --warmup 3 --warmup-seconds 0 --no-e2e --no-cpu --no-extras --no-exhaustive > /dev/null 2>&1; echo rc=$?
echo "== ncu p16"; timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused2d -s 3 -c 1 -o gpurun_out/$TAG.fused python bench.py --steps 3 --warmup 3 --warmup-seconds 0 --no-e2e --no-cpu --no-extras --no-exhaustive > gpurun_out/$TAG.ncu.log 2>&1; echo rc=$?
echo "== ncu 3D"; timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused3d -s 3 -c 1 -o gpurun_out/$TAG.fused3d python bench.py --dim 3 --p 8 --patches 100000 --steps 3 --warmup 3 --warmup-seconds 0 --no-e2e --no-cpu --no-extras --no-exhaustive > gpurun_out/$TAG.ncu3.log 2>&1; echo rc=$?
echo "== ncu C2"; timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused2d_tile -s 8 -c 1 -o gpurun_out/$TAG.tile_p3 python scripts/small_ab.py --p 3 --variants 0 --steps 10 > gpurun_out/$TAG.ncu2.log 2>&1; echo rc=$?
} > $LOG 2>&1
tail -60 $LOG
