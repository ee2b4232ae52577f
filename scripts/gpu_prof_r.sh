# ncu capture of the collect kernel at a given radius (default 2.5)
mkdir -p gpurun_out
R=${R:-2.5}
SMALL="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --radius $R"
$SMALL > gpurun_out/small.json 2> gpurun_out/small.err && \
ncu --set full --clock-control none --import-source on -k regex:radius_tile_kernel -s 1 -c 1 \
    -o gpurun_out/prof_r $SMALL > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_full.log; cat gpurun_out/small.json | head -c 600
