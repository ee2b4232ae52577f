set -u
mkdir -p gpurun_out
for V in "" "-DCM_LANE_ROW_CAP=104 -DCM_QTILE_MINB=6"; do
  touch paper_2502_11602_b200/csrc/query.cu
  make -C paper_2502_11602_b200/csrc EXTRA="$V" > /dev/null 2>&1 || { echo "build failed $V"; continue; }
  echo "[$V]"
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/v.json 2>/dev/null; python -c 'import json; d=json.load(open("gpurun_out/v.json")); print(round(d["value"]/1e6,1), d["phases_ms"], d["tile_stats"]["fill_long_rows"])'
  python bench.py --kernel cube --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/v.json 2>/dev/null; python -c 'import json; d=json.load(open("gpurun_out/v.json")); print("cube", round(d["value"]/1e6,1), d["phases_ms"], d["tile_stats"]["fill_long_rows"])'
  timeout 600 python scripts/sweep.py --configs 1 --flavors mixed --radii 0.5,2.5 --kernels 0 --sample 200 > /dev/null 2> gpurun_out/occ.log; grep cfg1 gpurun_out/occ.log | sed 's/parity=True all_rows=True//'
done
timeout 900 python -m pytest tests/ -m gpu -x -q -k "parity or property or edge" 2>&1 | tail -1
