# launch list + one ncu full capture of a named kNN kernel
set -u
mkdir -p gpurun_out
KS=${KS:-32,64} bash scripts/gpu_knn_launches.sh | grep -v "radix\|scan_\|query_keys" | tail -${TAILN:-12}
KNN_SAMPLE=100 timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-knn_hist_kernel} -s 0 -c ${COUNT:-1} \
  -o gpurun_out/${OUT:-prof_knn_hist} python scripts/knn_bench.py ${KPROF:-32} > gpurun_out/ncu_knn.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_knn.log
