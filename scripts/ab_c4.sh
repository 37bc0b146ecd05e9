# A/B of the current build vs a baseline build on C4 (3D p=8, 100k patches; interleaved)
B=${1:-paper_2306_16731_b200/_ab/base/libfvb.so}
for i in 1 2 3; do
  for lib in paper_2306_16731_b200/libfvb.so $B; do
    echo -n "$lib: "; FVB_LIBRARY=$lib python scripts/small_ab.py --dim 3 --p 8 --patches 100000 --variants 0 --flush 0 --steps 30 | tail -1
  done
done
