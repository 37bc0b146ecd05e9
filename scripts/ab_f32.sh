# A/B of the fp32 eigenvalue filter build: parity tests under it, then the sustained bench interleaved
TAG=$1; B=${2:-paper_2306_16731_b200/_ab/f32/libfvb.so}
mkdir -p gpurun_out
LOG=gpurun_out/$TAG.f32.log
{
FVB_LIBRARY=$B timeout 1500 python -m pytest tests -x -q -m gpu -k "filtered or degenerate or fullsize or golden or slab" 2>&1 | tail -3
bash scripts/ab_lib.sh $TAG $B --steps 100
for lib in paper_2306_16731_b200/libfvb.so $B; do
  echo -n "$lib C4: "; FVB_LIBRARY=$lib python scripts/small_ab.py --dim 3 --p 8 --patches 100000 --variants 0 --flush 0 --steps 30 | tail -1
done
} > $LOG 2>&1
cat $LOG
