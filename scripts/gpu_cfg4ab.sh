set -u
mkdir -p gpurun_out
S="python scripts/sweep.py --configs 4 --radii 1"
timeout 900 $S > /dev/null 2> gpurun_out/c4a.log; grep cfg4 gpurun_out/c4a.log
touch paper_2502_11602_b200/csrc/query.cu
make -C paper_2502_11602_b200/csrc EXTRA="-DCM_LANE_BITONIC" > /dev/null 2>&1
timeout 900 $S > /dev/null 2> gpurun_out/c4b.log; grep cfg4 gpurun_out/c4b.log
