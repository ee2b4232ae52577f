set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q -k "parity or golden or property or edge or configs" > gpurun_out/pytest_c.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_c.log
for rep in 1 2; do
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/v.json 2>/dev/null; python -c 'import json; d=json.load(open("gpurun_out/v.json")); print(round(d["value"]/1e6,1), d["phases_ms"])'
python bench.py --kernel cube --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/v.json 2>/dev/null; python -c 'import json; d=json.load(open("gpurun_out/v.json")); print("cube", round(d["value"]/1e6,1), d["phases_ms"])'
done
