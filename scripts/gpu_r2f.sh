set -x
mkdir -p gpurun_out/r02
export KNN_SAMPLE=20000
CMGPU_KNN_TRACE=1 CMGPU_KNN_ROUNDS=6 timeout 300 python scripts/knn_bench.py 8,64 > gpurun_out/r02/knn_trace.out 2> gpurun_out/r02/knn_trace.err
grep -A12 "round 0" gpurun_out/r02/knn_trace.err | head -60
cat gpurun_out/r02/knn_trace.out
for R in 1 2 3; do for M in 1.0 1.5 2.0; do
  echo "== rounds $R r0x $M"; CMGPU_KNN_ROUNDS=$R CMGPU_KNN_R0=$M timeout 300 python scripts/knn_bench.py 8,16,64 2>/dev/null
done; done
