# A/B of two builds of libfvb.so on the sustained bench (interleaved A B A B)
# usage: bash scripts/ab_lib.sh TAG LIB_B [bench args...]
TAG=$1; B=$2; shift 2
mkdir -p gpurun_out
LOG=gpurun_out/$TAG.ablib.log
: > $LOG
for i in 1 2; do
  for lib in paper_2306_16731_b200/libfvb.so $B; do
    FVB_LIBRARY=$lib timeout 300 python bench.py --no-e2e --no-cpu --no-extras "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); x=d.get('exhaustive') or {}
print('$lib'.split('/')[-2], 'value %.4g frac %.4f ms %.4f mhz %s | exh frac %s ms %s mhz %s' % (d['value'], d['roofline']['frac'], d['ms_per_step'], d['clocks']['sm_mhz'], x.get('roofline_frac'), x.get('ms_per_step'), (x.get('clocks') or {}).get('sm_mhz')))" >> $LOG
  done
done
cat $LOG
