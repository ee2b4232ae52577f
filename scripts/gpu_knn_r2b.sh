# kNN round-2b check: parity tests, then config-3 timing under env A/B
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q -k "knn or Knn or KNN" > gpurun_out/pytest_knn.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_knn.log
echo "== default"; KNN_SAMPLE=${KNN_SAMPLE:-20000} timeout 900 python scripts/knn_bench.py ${KS:-8,16,32,64} 2>&1 | grep '^{' | tee gpurun_out/knn_new.jsonl
for e in ${ENVS:-}; do
  echo "== $e"; env $e KNN_SAMPLE=2000 timeout 900 python scripts/knn_bench.py ${KS2:-8,16,32} 2>&1 | grep '^{'
done
