set -x
mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_gpu_checked.py tests/test_bench_contract.py -x -q -m gpu 2>&1 | tail -15
CMGPU_LIB=libcmgpu_checked.so timeout 600 python scripts/checked_probe.py > gpurun_out/r02/checked_probe.log 2>&1; echo "probe rc=$?"; tail -3 gpurun_out/r02/checked_probe.log
timeout 900 python bench.py --config 4 --layout slabs --flavor sparse --steps 3 --warmup 2 > gpurun_out/r02/bench_cfg4_slabs_n1.json 2> gpurun_out/r02/bench_cfg4_slabs_n1.err; tail -2 gpurun_out/r02/bench_cfg4_slabs_n1.err; cat gpurun_out/r02/bench_cfg4_slabs_n1.json
