# One GPU session: plain bench, then the ncu launch list, then one full capture
# each of the collect and gather kernels (each ncu only after the same command
# exited 0 without ncu).
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_info.txt
nproc > gpurun_out/host_cores.txt
BENCH="python bench.py --steps 5 --warmup 3"
$BENCH > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
cat gpurun_out/bench.json
SMALL="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$SMALL > gpurun_out/small.json 2> gpurun_out/small.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launches.log 2>&1
echo "ncu launches rc=$?"
$SMALL > gpurun_out/small2.json 2> gpurun_out/small2.err && \
ncu --set full --clock-control none --import-source on -k regex:"radius_tile_kernel|gather_rows" -s 1 -c 2 \
    -o gpurun_out/prof_collect $SMALL > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
tail -3 gpurun_out/ncu_full.log
