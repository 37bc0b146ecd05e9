# slot-kernel A/B (3D p != 8, AoS, p = 8 variant 5): 3D parity tests, then device time per p vs a baseline build
TAG=$1; B=${2:-paper_2306_16731_b200/_ab/base/libfvb.so}
mkdir -p gpurun_out
LOG=gpurun_out/$TAG.slot.log
{
timeout 1500 python -m pytest tests -x -q -m gpu -k "slab or 3d or layout or degenerate or random or physics or acceptance" 2>&1 | tail -3
for p in 2 3 4 5 6 7 9 10; do
  T=100000; [ $p -ge 9 ] && T=50000
  echo -n "p=$p base: "; FVB_LIBRARY=$B python scripts/small_ab.py --dim 3 --p $p --patches $T --variants 0 --flush 0 --steps 20 | tail -1
  echo -n "p=$p new:  "; python scripts/small_ab.py --dim 3 --p $p --patches $T --variants 0 --flush 0 --steps 20 | tail -1
done
echo -n "p=8 v5 base: "; FVB_LIBRARY=$B python scripts/small_ab.py --dim 3 --p 8 --patches 100000 --variants 5 --flush 0 --steps 20 | tail -1
echo -n "p=8 v5 new:  "; python scripts/small_ab.py --dim 3 --p 8 --patches 100000 --variants 5 --flush 0 --steps 20 | tail -1
echo -n "p=8 v0 new:  "; python scripts/small_ab.py --dim 3 --p 8 --patches 100000 --variants 0 --flush 0 --steps 20 | tail -1
} > $LOG 2>&1
cat $LOG
