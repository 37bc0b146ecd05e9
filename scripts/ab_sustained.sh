# Sustained (power-capped) A/B of builds / variants: bench.py 2D p=16 default
# workload, alternating A B A B on one box so clocks and caps are shared.
# usage: bash scripts/ab_sustained.sh "<bench args>" A.so[:VAR=val] B.so[:VAR=val] ...
ARGS=$1; shift
for round in 1 2; do
  for spec in "$@"; do
    lib=${spec%%:*}; env=""; [ "$spec" != "$lib" ] && env=${spec#*:}
    env $env FVB_LIBRARY=$lib timeout 300 python bench.py $ARGS --no-e2e --no-cpu 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$spec', round(d['ms_per_step'],4), 'ms', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
