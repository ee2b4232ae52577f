# kNN A/B of library variants on config 3 (timing + a small parity sample)
set -u
mkdir -p gpurun_out
for v in ${VARIANTS:-libcmgpu.so}; do
  echo "== $v ${KNNENV:-}"
  env ${KNNENV:-} CMGPU_LIB=$v KNN_SAMPLE=${KNN_SAMPLE:-3000} timeout 900 python scripts/knn_bench.py ${KS:-8,16,32,64} 2>&1 | grep '^{'
done
