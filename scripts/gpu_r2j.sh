# Re-entry check of the tip: GPU tests, smoke, bench (both arms), launch list
set -u
bash scripts/gpu_round.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
  > gpurun_out/ncu_launch.log 2>&1
echo "ncu rc=$?"
