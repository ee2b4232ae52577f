set -u
mkdir -p gpurun_out
for K in 0.75 0.5 0.75; do
  CMGPU_POOL_KEEP_FRAC=$K python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e.json 2>/dev/null
  python -c 'import json,sys; d=json.load(open("gpurun_out/e.json")); print(sys.argv[1], round(d["value"]/1e6,1), "e2e", d["e2e"]["ms_per_step"])' "keep=$K"
done
