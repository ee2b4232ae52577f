# Round-2 final evidence: bench, launch list, ncu full capture of collect +
# gather, then the kNN kernels (launch list at k = 8..64, full captures).
# The .ncu-rep files are reduced to CSV / line summaries on the box
# (gpurun_out/ is capped at 64 MiB).
set -u
bash scripts/gpu_bench.sh
summ() {  # rep-stem
  ncu -i gpurun_out/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  python scripts/ncu_lines.py gpurun_out/$1.ncu-rep 60 --stalls > gpurun_out/$1_lines.txt 2>/dev/null
}
summ prof_collect
KS=8,16,32,64 TAILN=400 bash scripts/gpu_knn_launches.sh > gpurun_out/knn_launch_tail.txt 2>&1
KNN_SAMPLE=100 timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:'knn_thread_kernel|knn_warp_reg_kernel' -s 0 -c 2 -o gpurun_out/prof_knn_k8_v5 \
  python scripts/knn_bench.py 8 > gpurun_out/ncu_knn8.log 2>&1
echo "ncu knn8 rc=$?"; summ prof_knn_k8_v5
KNN_SAMPLE=100 timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:'knn_hist_kernel|knn_warp_kernel' -s 0 -c 2 -o gpurun_out/prof_knn_k64_v5 \
  python scripts/knn_bench.py 64 > gpurun_out/ncu_knn64.log 2>&1
echo "ncu knn64 rc=$?"; summ prof_knn_k64_v5
ls -la gpurun_out/*.ncu-rep
rm -f gpurun_out/prof_knn_k8_v5.ncu-rep gpurun_out/prof_knn_k64_v5.ncu-rep
du -sh gpurun_out
