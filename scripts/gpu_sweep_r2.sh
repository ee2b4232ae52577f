# round-2 sweep refresh: config 1 (both flavours, all radii), config 3 kNN, config 2 digests
set -u
mkdir -p gpurun_out
timeout 2400 python scripts/sweep.py --configs ${CFGS:-1,3,2} ${SWEEP_ARGS:-} > gpurun_out/sweep_r2.json 2> gpurun_out/sweep_r2.log; echo "sweep rc=$?"
grep "cfg" gpurun_out/sweep_r2.log
