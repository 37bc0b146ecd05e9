# A/B of two libfvb builds on C2 (interleaved)
B=$1
for i in 1 2 3; do
  for lib in paper_2306_16731_b200/libfvb.so $B; do
    echo -n "$lib: "; FVB_LIBRARY=$lib python scripts/small_ab.py --p 3 --variants 0 --flush 2 --steps 100 | tail -1
  done
done
