set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
S="python scripts/sweep.py --configs 1 --flavors mixed --radii 2.5,5 --sample 500"
timeout 900 $S > gpurun_out/split.json 2> gpurun_out/split.log; echo "split rc=$?"
grep cfg1 gpurun_out/split.log
touch paper_2502_11602_b200/csrc/query.cu
make -C paper_2502_11602_b200/csrc EXTRA="-DCM_ROWSORT_PADDED" > /dev/null 2>&1
timeout 900 $S --kernels 0 > gpurun_out/padded.json 2> gpurun_out/padded.log; echo "padded rc=$?"
grep cfg1 gpurun_out/padded.log
