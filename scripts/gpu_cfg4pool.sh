set -u
mkdir -p gpurun_out
S="python scripts/sweep.py --configs 4 --radii 1"
for R in 0 96; do
  CMGPU_POOL_RESERVE_GB=$R timeout 900 $S > /dev/null 2> gpurun_out/c4p$R.log; echo "reserve=$R"; grep -E "cfg4|free" gpurun_out/c4p$R.log
done
