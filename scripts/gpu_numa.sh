set -u
for m in default local remote; do timeout 300 python scripts/numa_probe.py $m 2>&1 | grep -E "D2H|gpu-local|affinity|GPU0" ; done
