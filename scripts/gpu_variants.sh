# A/B of compile-time variants: device-only bench per EXTRA flag set
set -u
mkdir -p gpurun_out
: > gpurun_out/variants.log
for V in "" "-DCM_RADIX_BALLOT"; do
  touch paper_2502_11602_b200/csrc/query.cu paper_2502_11602_b200/csrc/build.cu
  make -C paper_2502_11602_b200/csrc EXTRA="$V" > /dev/null 2>&1 || { echo "build failed $V" >> gpurun_out/variants.log; continue; }
  for rep in 1 2; do
    python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/v.json 2> gpurun_out/v.err
    python -c 'import json,sys; d=json.load(open("gpurun_out/v.json")); print(sys.argv[1], round(d["value"]/1e6,1), d["phases_ms"]["order_ms"], d["build_detail"]["mixed"]["sort_ms"], d["build_ms"])' "[$V]" >> gpurun_out/variants.log
  done
done
cat gpurun_out/variants.log
