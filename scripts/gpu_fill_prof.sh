# ncu capture of the wide FILL launch at config-1 mixed sphere r = 2.5 (current and round-1 library)
set -u
mkdir -p gpurun_out
for v in ${VARIANTS:-libcmgpu.so libcmgpu_r1.so}; do
  CMGPU_ALLOW_MISSING=1 CMGPU_LIB=$v timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:radius_tile_kernel -s 3 -c 1 -o gpurun_out/prof_fill_$v \
    python scripts/sweep.py --configs 1 --flavors mixed --radii 2.5 --kernels 0 --sample 20 > gpurun_out/ncu_fill_$v.log 2>&1
  echo "$v rc=$?"
done
