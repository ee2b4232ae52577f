# quick device-only bench line (no e2e / cpu baseline) -> gpurun_out/x.json
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/x.json 2> gpurun_out/x.err
python -c 'import json; d = json.load(open("gpurun_out/x.json")); print(d["value"], d["phases_ms"], d["tile_stats"])'
