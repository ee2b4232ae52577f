set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/v.json 2>/dev/null; python -c 'import json; d=json.load(open("gpurun_out/v.json")); print(round(d["value"]/1e6,1), d["phases_ms"], d["build_detail"]["mixed"])'
timeout 900 python scripts/sweep.py --configs 4 --radii 1 > /dev/null 2> gpurun_out/c4r.log; grep -E "cfg4" gpurun_out/c4r.log
