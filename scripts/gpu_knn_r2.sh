# kNN: GPU parity tests + config-3 timing (per-thread kernel vs the round-1 path)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q -k "knn or Knn or KNN" > gpurun_out/pytest_knn.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_knn.log
KNN_SAMPLE=${KNN_SAMPLE:-20000} timeout 900 python scripts/knn_bench.py ${KS:-8,16,32,64} 2>&1 | grep '^{' | tee gpurun_out/knn_new.jsonl
if [ -n "${LEGACY:-}" ]; then
CMGPU_KNN_LEGACY=1 KNN_SAMPLE=2000 timeout 900 python scripts/knn_bench.py ${KS:-8,16,32,64} 2>&1 | grep '^{' | tee gpurun_out/knn_legacy.jsonl
fi
