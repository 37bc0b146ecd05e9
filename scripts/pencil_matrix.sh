# 2D p16 sustained bench: launch variants (same box, back to back) + cold ncu launch list of each
for v in ${PV:-0 4 0 4}; do
  FVB_TUNE_PENCIL_VARIANT=$v timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('variant $v', round(d['ms_per_step'],4), 'ms', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
for v in ${NV:-0 4}; do
  FVB_TUNE_PENCIL_VARIANT=$v timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:fused2d -s 3 -c 1 python bench.py --steps 3 --warmup 3 --warmup-seconds 0 --no-e2e --no-cpu 2>/dev/null | grep -E "gpu__time|inst_executed|fp64|issue_active" | sed "s/^/v$v /"
done
