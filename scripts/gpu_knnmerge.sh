set -u
for V in "" "-DCM_KNN_MERGE_MIN=2" "-DCM_KNN_MERGE_MIN=4" "-DCM_KNN_MERGE_MIN=8"; do
  touch paper_2502_11602_b200/csrc/knn.cu
  make -C paper_2502_11602_b200/csrc EXTRA="$V" > /dev/null 2>&1 || { echo "build failed $V"; continue; }
  echo "[$V]"; KNN_REPS=3 python scripts/knn_probe.py
done
timeout 600 python -m pytest tests/ -m gpu -x -q -k "knn" 2>&1 | tail -1
