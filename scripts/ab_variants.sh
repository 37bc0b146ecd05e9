# ncu A/B of launch variants of one build (cold single-launch device time + instruction count).
# usage: VAR=FVB_TUNE_PENCIL_VARIANT bash scripts/ab_variants.sh "<bench args>" regex v1 v2 ...
ARGS=$1; RX=$2; shift 2
for v in "$@"; do
  env ${VAR:-FVB_TUNE_PENCIL_VARIANT}=$v timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,launch__registers_per_thread --clock-control none -k regex:$RX -s 3 -c 1 python bench.py $ARGS --steps 3 --warmup 3 --warmup-seconds 0 --no-e2e --no-cpu 2>/dev/null | grep -E "gpu__time|inst_exec|registers" | sed "s|^|v$v |"
done
