# same-box A/B of library variants on the bench (device rate + e2e)
set -u
mkdir -p gpurun_out
for v in ${VARIANTS:-libcmgpu.so}; do
  echo "== $v"
  CMGPU_LIB=$v python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), d['ms_per_step'], d['phases_ms']['pass1_ms'], d['phases_ms']['pass2_ms'], 'e2e', d['e2e']['ms_steps'], 'general', d['general_centres']['ms_per_step'], (d['tile_stats'] if isinstance(d['tile_stats'], str) else d['tile_stats']['fill_fallback_tiles']))"
done
