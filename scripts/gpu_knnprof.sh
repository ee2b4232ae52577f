set -u
mkdir -p gpurun_out
KNN_REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:knn \
  --log-file gpurun_out/knn_launches.csv python scripts/knn_probe.py > gpurun_out/knn_l.log 2>&1; echo "launches rc=$?"
KNN_K=16 KNN_REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:knn_warp -c 1 \
  -o gpurun_out/prof_knn16 python scripts/knn_probe.py > gpurun_out/knn_full.log 2>&1; echo "full rc=$?"
KNN_K=8 KNN_REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:knn_tile -c 1 \
  -o gpurun_out/prof_knn8 python scripts/knn_probe.py > gpurun_out/knn_full8.log 2>&1; echo "full8 rc=$?"
