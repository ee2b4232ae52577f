# full-population parity (every query of configs 1-4 vs the CPU oracle)
set -x
mkdir -p gpurun_out/r02
timeout 600 python -m pytest tests/test_gpu_full.py tests/test_gpu_parity.py -x -q 2>&1 | tail -5
timeout 5400 python scripts/verify_full.py --configs 1,3,2,4 --out gpurun_out/r02/verify_full.json 2> gpurun_out/r02/verify_full.log
tail -40 gpurun_out/r02/verify_full.log
