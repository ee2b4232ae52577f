# full-population parity of the current build (every query of configs 1-4 vs the CPU oracle)
set -u
mkdir -p gpurun_out/r02
timeout 5400 python scripts/verify_full.py --configs 1,3,2,4 --out gpurun_out/r02/verify_full.json 2> gpurun_out/r02/verify_full.log
echo "verify rc=$?"
tail -8 gpurun_out/r02/verify_full.log
