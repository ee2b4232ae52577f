set -u
mkdir -p gpurun_out
for V in "" "-DCM_MID_MIN=512" "-DCM_MID_MIN=256"; do
  touch paper_2502_11602_b200/csrc/query.cu
  make -C paper_2502_11602_b200/csrc EXTRA="$V" > /dev/null 2>&1 || { echo "build failed $V"; continue; }
  timeout 900 python scripts/sweep.py --configs 1 --flavors mixed --radii 2.5,5 --sample 200 > /dev/null 2> gpurun_out/mm.log; grep -c "all_rows=True" gpurun_out/mm.log
  echo "[$V]"; grep cfg1 gpurun_out/mm.log | sed 's/parity=True all_rows=True//'
done
