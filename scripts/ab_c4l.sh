# C4 A/B of builds, interleaved: bash scripts/ab_c4l.sh TAG LIB...
TAG=$1; shift
mkdir -p gpurun_out
LOG=gpurun_out/$TAG.c4l.log
{
for i in 1 2 3; do
  for lib in "$@"; do
    echo -n "$lib: "; FVB_LIBRARY=$lib python scripts/small_ab.py --dim 3 --p 8 --patches 100000 --variants 0 --flush 0 --steps 30 | tail -1
  done
done
} > $LOG 2>&1
cat $LOG
