set -u
mkdir -p gpurun_out
KNN_REPS=3 python scripts/knn_probe.py
timeout 900 python -m pytest tests/ -m gpu -x -q -k "knn or property or edge or golden or configs" > gpurun_out/pytest_knn.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_knn.log
