# A/B of library variants on the headline bench (phase times), twice each
set -u
mkdir -p gpurun_out
for rep in 1 2; do
for v in ${VARIANTS:-libcmgpu.so}; do
  CMGPU_LIB=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python -c "
import json,sys
d=json.load(open('gpurun_out/ab_$v.json'))
print('$v', round(d['value']/1e6,1), 'Mq/s', d['ms_per_step'], d.get('phases_ms'))
" || tail -3 gpurun_out/ab_$v.err
done; done
