set -u
mkdir -p gpurun_out
timeout 1200 python scripts/sweep.py --configs 3 --sample 2000 > gpurun_out/knn.json 2> gpurun_out/knn.log; echo "knn rc=$?"
grep cfg3 gpurun_out/knn.log
