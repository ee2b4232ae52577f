# cluster ABI + concurrency tests, then compute-sanitizer over the probe
set -x
mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_concurrency.py tests/test_gpu_parity.py -x -q 2>&1 | tail -15
python scripts/sanitize_probe.py 2>&1 | tail -3
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_probe.py > gpurun_out/r02/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/r02/sanitizer_$tool.log
done
