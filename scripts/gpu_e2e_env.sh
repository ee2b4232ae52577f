# e2e under environment variants (same box): ENVS="A=1 B=2|C=3" (| separates sets)
set -u
IFS='|' read -ra SETS <<< "${ENVS:-X=1}"
for e in "${SETS[@]}"; do
  echo "== $e"
  env $e python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), 'e2e', d['e2e']['ms_steps'])"
done
