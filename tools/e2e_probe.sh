#!/bin/bash
# End-to-end (host in / host out) rate of one config for several host-thread counts of the float32
# transfer + host widening (FBGPU_HOST_THREADS; 0 = float64 rows over PCIe).
cfg=${1:-c4}; shift
for t in "$@"; do
  echo "== FBGPU_HOST_THREADS=$t"
  FBGPU_HOST_THREADS=$t python bench.py --config $cfg --no-cpu-baseline --no-extra-legs --steps 5 --warmup 3 \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value', round(d['value'],1), 'e2e', d['e2e'])"
done
