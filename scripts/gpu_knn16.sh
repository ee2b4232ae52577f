set -u
mkdir -p gpurun_out
KNN_REPS=3 python scripts/knn_probe.py
touch paper_2502_11602_b200/csrc/knn.cu
make -C paper_2502_11602_b200/csrc EXTRA="-DCM_KNN_TILE_MAX=16" > /dev/null 2>&1
KNN_REPS=3 python scripts/knn_probe.py
timeout 900 python -m pytest tests/ -m gpu -x -q -k "knn or property or edge or golden" > gpurun_out/pytest_knn.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_knn.log
