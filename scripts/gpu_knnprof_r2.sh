# ncu --set full capture of the per-thread kNN kernel (pass 1 and 2) at one k
set -u
mkdir -p gpurun_out
KNN_SAMPLE=100 timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-knn_thread_kernel} -s 0 -c ${COUNT:-2} \
  -o gpurun_out/${OUT:-prof_knn} python scripts/knn_bench.py ${KS:-8} > gpurun_out/ncu_knn.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_knn.log
