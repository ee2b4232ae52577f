# tile counters accumulated per warp: tests, bench, count probe, large radii
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
VARIANTS="libcmgpu.so ${OTHER:-}" bash scripts/gpu_split_ab.sh
for v in libcmgpu.so ${OTHER:-}; do
  echo "== $v"
  CMGPU_LIB=$v python scripts/count_probe.py 2>&1 | grep cfg | cut -c1-80
  CMGPU_LIB=$v timeout 900 python scripts/sweep.py --configs 1 --flavors mixed --radii 2.5,5 2>&1 >/dev/null | grep cfg | cut -c1-200
  CMGPU_LIB=$v timeout 900 python scripts/sweep.py --configs 2 2>&1 >/dev/null | grep cfg | cut -c1-120
done
