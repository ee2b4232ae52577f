set -u
mkdir -p gpurun_out
CMGPU_TRACE=1 timeout 600 python scripts/e2e_probe.py > gpurun_out/trace.log 2>&1; echo "trace rc=$?"
grep -v "^\s*$" gpurun_out/trace.log | tail -40
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
