# GPU tests, then A/B of the build (onesweep vs per-pass upsweep radix)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for v in ${VARIANTS:-libcmgpu.so}; do
  CMGPU_LIB=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python -c "
import json
d=json.load(open('gpurun_out/ab_$v.json'))
print('$v', round(d['value']/1e6,1), 'Mq/s build', d['build_ms'], d['build_detail']['mixed'])
" || tail -3 gpurun_out/ab_$v.err
done
