set -u
mkdir -p gpurun_out
S="python scripts/sweep.py --configs 4 --radii 1"
timeout 900 $S > /dev/null 2> gpurun_out/c4c.log; grep cfg4 gpurun_out/c4c.log
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/v.json 2>/dev/null; python -c 'import json; d=json.load(open("gpurun_out/v.json")); print(round(d["value"]/1e6,1), d["phases_ms"], d["build_ms"])'
KNN_REPS=2 python scripts/knn_probe.py
touch paper_2502_11602_b200/csrc/query.cu paper_2502_11602_b200/csrc/knn.cu
make -C paper_2502_11602_b200/csrc EXTRA="-DCM_GATHER_ROW=80 -DCM_GATHER_MINB=5 -DCM_KNN_TILE_MAX=0" > /dev/null 2>&1
timeout 900 $S > /dev/null 2> gpurun_out/c4d.log; grep cfg4 gpurun_out/c4d.log
KNN_REPS=2 python scripts/knn_probe.py
