set -u
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  -k regex:"sort|radius_tile|gather_rows" --log-file gpurun_out/wide_launches.csv \
  python scripts/sweep.py --configs 1 --flavors mixed --radii 2.5 --sample 50 > /dev/null 2>gpurun_out/wide_ncu.log
echo "ncu rc=$?"
