# one ncu --set full capture (source-level) of one kernel of a short bench run
set -u
mkdir -p gpurun_out
SMALL="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-}"
$SMALL > gpurun_out/small.json 2> gpurun_out/small.err && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-radius_tile_kernel} -s ${SKIP:-1} -c ${COUNT:-1} \
    -o gpurun_out/${OUT:-prof} $SMALL > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_full.log
