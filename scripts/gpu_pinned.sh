set -u
mkdir -p gpurun_out
python scripts/pinned_probe.py 2>&1 | tail -12
timeout 900 python -m pytest tests/ -m gpu -x -q > /dev/null 2>&1; echo "pytest rc=$?"
python scripts/pinned_probe.py 2>&1 | tail -12
python bench.py --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("e2e", d["e2e"]["ms_steps"])'
