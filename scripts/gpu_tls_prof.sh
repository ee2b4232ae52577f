# ncu full capture of the DIGEST tile kernel on config 2 (TLS), reduced to CSV on the box
set -u
mkdir -p gpurun_out
timeout 600 python scripts/tls_probe.py > gpurun_out/tls_probe.log 2>&1; echo "probe rc=$?"; cat gpurun_out/tls_probe.log | cut -c1-200
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radius_tile_kernel -s 2 -c 1 \
  -o gpurun_out/prof_tls_digest python scripts/tls_probe.py > gpurun_out/ncu_tls.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/prof_tls_digest.ncu-rep --page details --csv > gpurun_out/prof_tls_digest_details.csv 2>/dev/null
ncu -i gpurun_out/prof_tls_digest.ncu-rep --page raw --csv > gpurun_out/prof_tls_digest_raw.csv 2>/dev/null
python scripts/ncu_lines.py gpurun_out/prof_tls_digest.ncu-rep 40 --stalls > gpurun_out/prof_tls_digest_lines.txt 2>/dev/null
rm -f gpurun_out/prof_tls_digest.ncu-rep
