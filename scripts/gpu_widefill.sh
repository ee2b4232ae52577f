set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q -k "wide or big or tall or property or csr or slabs" > gpurun_out/pytest_w.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_w.log
timeout 900 python scripts/sweep.py --configs 1 --flavors mixed --radii 2.5,5 --sample 300 > /dev/null 2> gpurun_out/wf.log
grep cfg1 gpurun_out/wf.log | sed 's/parity=True all_rows=True//'; grep -c "all_rows=True" gpurun_out/wf.log
