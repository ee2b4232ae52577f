set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q > gpurun_out/pytest_self.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_self.log
for rep in 1 2; do
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/v.json 2>/dev/null; python -c 'import json; d=json.load(open("gpurun_out/v.json")); print(round(d["value"]/1e6,1), d["phases_ms"], d["build_ms"])'
done
KNN_REPS=2 python scripts/knn_probe.py
