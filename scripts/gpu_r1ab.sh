# round-1 library vs current on config-1 mixed cases (regression check)
set -u
mkdir -p gpurun_out
for v in libcmgpu_r1.so libcmgpu.so; do
  echo "== $v"
  CMGPU_ALLOW_MISSING=1 CMGPU_LIB=$v timeout 1200 python scripts/sweep.py --configs 1 --flavors mixed --radii ${RADII:-1,2.5} --sample 200 > gpurun_out/ab_sweep_$v.json 2> gpurun_out/ab_sweep_$v.log
  grep "cfg" gpurun_out/ab_sweep_$v.log
done
