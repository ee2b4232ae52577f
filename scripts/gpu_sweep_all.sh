set -u
mkdir -p gpurun_out
timeout 2400 python scripts/sweep.py --configs 0,1,2,3 > gpurun_out/sweep_cfg0-3.json 2> gpurun_out/sweep_cfg0-3.log; echo "sweep03 rc=$?"
timeout 1800 python scripts/sweep.py --configs 4 > gpurun_out/sweep_cfg4.json 2> gpurun_out/sweep_cfg4.log; echo "sweep4 rc=$?"
grep "cfg" gpurun_out/sweep_cfg0-3.log gpurun_out/sweep_cfg4.log
