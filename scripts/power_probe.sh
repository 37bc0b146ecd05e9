# Sustained vs cold behaviour of the fused 2D kernel: clocks, power, temperatures during 100-step benches.
TAG=${1:-pw}
mkdir -p gpurun_out
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,temperature.memory,clocks_event_reasons.active --format=csv -lms 100 > gpurun_out/$TAG.smi.csv &
SMI=$!
for mode in filtered exhaustive filtered; do
  if [ $mode = exhaustive ]; then export FVB_TUNE_REDUCE_FILTER=0; else unset FVB_TUNE_REDUCE_FILTER; fi
  echo "== $mode $(date +%T.%N)"
  timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,2), 'Gcell/s', round(d['ms_per_step'],4), 'ms', d['clocks'])"
  sleep 5
done
unset FVB_TUNE_REDUCE_FILTER
echo "== 3D exhaustive vs filtered"
FVB_TUNE_REDUCE_FILTER=0 timeout 300 python bench.py --dim 3 --p 8 --patches 100000 --steps 30 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('3D all', round(d['ms_per_step'],4), 'ms')"
FVB_TUNE_REDUCE_FILTER=1 timeout 300 python bench.py --dim 3 --p 8 --patches 100000 --steps 30 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('3D filtered', round(d['ms_per_step'],4), 'ms')"
kill $SMI
