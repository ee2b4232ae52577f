# Row-sort probe: config-1 mixed at large radii, bucket vs bitonic row sort
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
S="python scripts/sweep.py --configs 1 --flavors mixed --radii 2.5,5 --sample 500"
timeout 900 $S > gpurun_out/rs_bucket.json 2> gpurun_out/rs_bucket.log; echo "bucket rc=$?"
grep cfg1 gpurun_out/rs_bucket.log
CMGPU_ROWSORT=radix timeout 900 $S > gpurun_out/rs_radix.json 2> gpurun_out/rs_radix.log; echo "radix rc=$?"; grep cfg1 gpurun_out/rs_radix.log
grep cfg1 gpurun_out/rs_bitonic.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  -k regex:"sort|radius_tile|gather" --log-file gpurun_out/rs_launches.csv \
  python scripts/sweep.py --configs 1 --flavors mixed --radii 2.5 --kernels 0 --sample 100 > /dev/null 2>gpurun_out/rs_ncu.log
echo "ncu rc=$?"
