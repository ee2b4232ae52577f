set -u
mkdir -p gpurun_out
: > gpurun_out/ab.log
for args in "--no-e2e --no-cpu-baseline" "--no-cpu-baseline" "--no-e2e --no-cpu-baseline"; do
  python bench.py --steps 5 --warmup 3 $args > gpurun_out/v.json 2> gpurun_out/v.err
  python -c 'import json,sys; d=json.load(open("gpurun_out/v.json")); print(sys.argv[1], round(d["value"]/1e6,1), d["phases_ms"])' "[$args]" >> gpurun_out/ab.log
done
cat gpurun_out/ab.log
