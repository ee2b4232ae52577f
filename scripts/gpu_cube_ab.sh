# cube-kernel A/B (config 1 mixed r = 1 and 2.5) over library variants
set -u
for v in ${VARIANTS}; do
  echo "== $v"
  CMGPU_ALLOW_MISSING=1 CMGPU_LIB=$v timeout 1200 python scripts/sweep.py --configs 1 --flavors mixed --radii ${RADII:-1,2.5} --kernels ${KERNELS:-1} --sample 200 2>&1 >/dev/null | grep cfg
done
