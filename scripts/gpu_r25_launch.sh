# launch lists of config-1 mixed sphere r = 2.5 with the round-1 and the current library
set -u
mkdir -p gpurun_out
for v in libcmgpu_r1.so libcmgpu.so; do
  CMGPU_ALLOW_MISSING=1 CMGPU_LIB=$v timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch25_$v.csv python scripts/sweep.py --configs 1 --flavors mixed --radii 2.5 --kernels ${K:-0} --sample 20 > /dev/null 2>&1
  echo "$v rc=$?"
done
