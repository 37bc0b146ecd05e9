# 3D patch sizes: fused kernel device time per step, 100k patches (p <= 8) / fewer for p > 8
for p in 2 3 4 5 6 7 8 9 10; do
  T=100000; [ $p -ge 9 ] && T=50000
  echo -n "p=$p T=$T: "; python scripts/small_ab.py --dim 3 --p $p --patches $T --variants 0 --flush 0 --steps 20 | tail -1
done
