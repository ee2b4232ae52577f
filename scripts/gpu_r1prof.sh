# ncu capture of the cube r = 1 collect with the round-1 library and the current one
set -u
mkdir -p gpurun_out
for v in libcmgpu_r1.so libcmgpu.so; do
  CMGPU_ALLOW_MISSING=1 CMGPU_LIB=$v timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:radius_tile_kernel -s 2 -c 1 -o gpurun_out/prof_cube_$v \
    python scripts/sweep.py --configs 1 --flavors mixed --radii 1 --kernels 1 --sample 50 > gpurun_out/ncu_cube_$v.log 2>&1
  echo "$v rc=$?"
done
