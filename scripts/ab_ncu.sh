# A/B of two builds of libfvb.so with ncu (cold single-launch device time, no power-cap noise).
# usage: bash scripts/ab_ncu.sh "<bench args>" regex A.so B.so ...
ARGS=$1; RX=$2; shift 2
for lib in "$@"; do
  for rep in 1 2; do
    FVB_LIBRARY=$lib timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:$RX -s 3 -c 2 python bench.py $ARGS --steps 3 --warmup 3 --warmup-seconds 0 --no-e2e --no-cpu 2>/dev/null | grep -E "gpu__time|inst_exec" | sed "s|^|$(basename $lib) |"
  done
done
