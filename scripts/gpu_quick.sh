# bench only (no CPU baseline, no e2e): phase times of the headline step
set -u
mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
d=json.load(open("gpurun_out/bench.json"))
print("value", d["value"], "ms", d["ms_per_step"], "phases", d.get("phases_ms"), "general", d.get("general_centres",{}).get("ms_per_step"))
PY
