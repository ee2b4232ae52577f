# r = 2.5 m evidence: bench line (two-pass path) + ncu full of count, fill, 257..512 row sort
set -u
mkdir -p gpurun_out
python bench.py --radius 2.5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_r25.json 2> gpurun_out/bench_r25.err
echo "bench rc=$?"; cat gpurun_out/bench_r25.json | cut -c1-400
SMALL="python bench.py --radius 2.5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$SMALL > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"radius_tile_kernel|sort_blocked_rows_kernel" -s 4 -c 4 \
    -o gpurun_out/prof_wide $SMALL > gpurun_out/ncu_wide.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_wide.log
