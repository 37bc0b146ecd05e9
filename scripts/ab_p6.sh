# 3D p=6 / p=8: parity tests of the one-warp kernel, then device time vs the baseline build
TAG=$1; B=${2:-paper_2306_16731_b200/_ab/base/libfvb.so}
mkdir -p gpurun_out
LOG=gpurun_out/$TAG.p6.log
{
timeout 1200 python -m pytest tests -x -q -m gpu -k "slab or degenerate or filtered or p6 or c4_whole or 3d or acceptance" 2>&1 | tail -3
for i in 1 2; do
  for p in 6 8; do
    echo -n "base p=$p: "; FVB_LIBRARY=$B python scripts/small_ab.py --dim 3 --p $p --patches 100000 --variants 0 --flush 0 --steps 20 | tail -1
    echo -n "new  p=$p: "; python scripts/small_ab.py --dim 3 --p $p --patches 100000 --variants 0,5 --flush 0 --steps 20 | tr '\n' ' '; echo
  done
done
} > $LOG 2>&1
cat $LOG
