set -u
mkdir -p gpurun_out
S="python scripts/sweep.py --configs 4 --radii 1"
for K in 0.5 0.75 0.9 0.5 0.75 0.9; do
  CMGPU_POOL_KEEP_FRAC=$K timeout 900 $S > /dev/null 2> gpurun_out/c4k.log; echo "keep=$K $(grep cfg4 gpurun_out/c4k.log)"
done
