set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q -k "knn or property or edge" > gpurun_out/pytest_knn.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_knn.log
timeout 1200 python scripts/sweep.py --configs 3 --sample 2000 > gpurun_out/knn.json 2> gpurun_out/knn.log; echo "knn rc=$?"
grep cfg3 gpurun_out/knn.log
