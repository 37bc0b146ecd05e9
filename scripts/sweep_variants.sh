# Bench every FVB_TUNE_PENCIL_VARIANT of the p=16 fused kernel (device time only).
TAG=${1:-sweep}
mkdir -p gpurun_out
for v in ${VARIANTS:-0 1 2 3 4 5 6}; do
  FVB_TUNE_PENCIL_VARIANT=$v timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('variant $v', round(d['value']/1e9,2), 'Gcell/s', round(d['roofline']['frac'],3), 'of HBM', d['clocks'])"
done
