# bench + one ncu --set full capture of the tile kernels (count + fill)
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
SMALL="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-}"
$SMALL > gpurun_out/small.json 2> gpurun_out/small.err && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-radius_tile_kernel} -s 1 -c 2 \
    -o gpurun_out/prof_tile $SMALL > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_full.log
