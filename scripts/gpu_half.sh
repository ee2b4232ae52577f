# half tiles: GPU parity tests, then A/B on the headline and config-1 sweeps
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
VARIANTS="libcmgpu.so libcmgpu_nohalf.so" bash scripts/gpu_ab2.sh
for v in libcmgpu.so libcmgpu_nohalf.so; do
  echo "== $v"
  CMGPU_LIB=$v timeout 1200 python scripts/sweep.py --configs 1 --flavors mixed --radii 0.5,1,2.5 --sample 200 2>&1 >/dev/null | grep cfg
done
