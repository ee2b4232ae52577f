# ncu launch list of one kNN bench run (kernel durations per launch)
set -u
mkdir -p gpurun_out
CMGPU_LIB=${LIB:-libcmgpu.so} KNN_SAMPLE=100 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/knn_launches.csv python scripts/knn_bench.py ${KS:-8,16} > gpurun_out/ncu_knn_launches.log 2>&1
echo "ncu rc=$?"
python - <<'PY'
import csv, collections
rows = list(csv.reader(l for l in open("gpurun_out/knn_launches.csv") if l.startswith('"')))
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
seq = []
for r in rows[1:]:
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    ms = v / 1e6 if u in ("ns", "nsecond") else v / 1e3 if u in ("us", "usecond") else v
    seq.append((r[ki][:70], ms))
# print the last 40 launches (the last timed kNN call of the last k and what precedes it)
for n, ms in seq[-60:]:
    print(f"{ms:9.3f} ms  {n}")
PY
