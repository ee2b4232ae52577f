# round-2 evidence: bench line, launch list, one ncu --set full capture of collect + gather
set -u
mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
  > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
SMALL="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"radius_tile_kernel|gather_rows_kernel" -s 2 -c 2 \
    -o gpurun_out/prof_cg $SMALL > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
