# e2e (host buffers) vs the to_host chunk count -> gpurun_out/chunks.txt
mkdir -p gpurun_out
for c in ${CHUNKS:-default 1 2 3 4}; do
  env $( [ "$c" = default ] || echo CMGPU_CHUNKS=$c ) python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c$c.json 2> gpurun_out/c$c.err
  python -c "import json; d=json.load(open('gpurun_out/c$c.json')); print('chunks=$c', d['value']/1e6, d['e2e']['value']/1e6, d['e2e']['ms_per_step'])"
done | tee gpurun_out/chunks.txt
