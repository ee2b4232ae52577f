set -x
mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "knn" 2>&1 | tail -5
timeout 600 python scripts/knn_bench.py > gpurun_out/r02/knn_v2.jsonl 2> gpurun_out/r02/knn_v2.err; tail -3 gpurun_out/r02/knn_v2.err
cat gpurun_out/r02/knn_v2.jsonl
CMGPU_KNN_LEGACY=1 timeout 600 python scripts/knn_bench.py > gpurun_out/r02/knn_legacy.jsonl 2>&1
cat gpurun_out/r02/knn_legacy.jsonl
