TAG=${1:-r02}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused2d_tile -s 8 -c 1 -o gpurun_out/$TAG.tile_p3 python scripts/small_ab.py --p 3 --variants 0 --steps 10 --flush 2 > gpurun_out/$TAG.ncu2.log 2>&1; echo rc=$?
