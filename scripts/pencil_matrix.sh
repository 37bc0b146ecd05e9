# 2D p16 sustained bench: launch variant x reduction mode (same box, back to back)
for cfg in "0 1" "3 0" "3 1" "0 0" "0 1"; do
  set -- $cfg
  FVB_TUNE_PENCIL_VARIANT=$1 FVB_TUNE_REDUCE_FILTER=$2 timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('variant $1 filter $2', round(d['ms_per_step'],4), 'ms', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
