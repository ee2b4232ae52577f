# GPU tests, bench, config-1/3 sweep
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('bench', d['value'], d['ms_per_step'], d['phases_ms'], d['build_ms'], 'e2e', d['e2e']['value'])"
timeout 2400 python scripts/sweep.py --configs 1,3 > gpurun_out/sweep_r2.json 2> gpurun_out/sweep_r2.log; echo "sweep rc=$?"
grep "cfg" gpurun_out/sweep_r2.log
