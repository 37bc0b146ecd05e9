# ncu --set full of the 3D slot kernel at p = 6 and p = 4 (100k patches), one cold launch each
TAG=${1:-r02}
mkdir -p gpurun_out
for p in 6 4; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused3d -s 2 -c 1 \
    -o gpurun_out/$TAG.slab_p$p -f python scripts/small_ab.py --dim 3 --p $p --patches 100000 --variants 0 --flush 0 --steps 1 \
    > gpurun_out/$TAG.slab_p$p.log 2>&1
  tail -3 gpurun_out/$TAG.slab_p$p.log
done
