set -x
export KNN_SAMPLE=20000
CMGPU_KNN_TRACE=1 timeout 300 python scripts/knn_bench.py 8,64 2>&1 | grep -v "^\[knn\]   phase" | awk '!seen[$0]++' | head -40
echo "== legacy, cell order"; CMGPU_KNN_LEGACY=1 CMGPU_KNN_CELL_ORDER=1 timeout 300 python scripts/knn_bench.py 8,16,32,64 2>/dev/null
echo "== legacy, morton"; CMGPU_KNN_LEGACY=1 timeout 300 python scripts/knn_bench.py 8,16,32,64 2>/dev/null
for R in 1 2 6; do for M in 1.0 1.5; do
  echo "== rounds $R r0x $M"; CMGPU_KNN_ROUNDS=$R CMGPU_KNN_R0=$M timeout 300 python scripts/knn_bench.py 8,16,32,64 2>/dev/null
done; done
