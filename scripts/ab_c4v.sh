# C4 A/B: current build (variants given) vs a baseline build, interleaved, plus the 3D parity tests
# usage: bash scripts/ab_c4v.sh TAG "0,6" [BASE_LIB]
TAG=$1; V=${2:-0}; B=${3:-paper_2306_16731_b200/_ab/base/libfvb.so}
mkdir -p gpurun_out
LOG=gpurun_out/$TAG.c4.log
{
timeout 900 python -m pytest tests -x -q -m gpu -k "3d or fullsize and c4 or warp or slab" 2>&1 | tail -2
for i in 1 2 3; do
  echo -n "base: "; FVB_LIBRARY=$B python scripts/small_ab.py --dim 3 --p 8 --patches 100000 --variants 0 --flush 0 --steps 30 | tail -1
  echo "new:"; python scripts/small_ab.py --dim 3 --p 8 --patches 100000 --variants $V --flush 0 --steps 30
done
} > $LOG 2>&1
cat $LOG
