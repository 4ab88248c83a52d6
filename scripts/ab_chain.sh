#!/bin/bash
# Alternating A/B of the split-K chain workloads across tree copies given as arguments.
set -u
for r in 1 2 3; do
  for d in "$@"; do
    for w in square4096 square4096_fp32 sign4096; do
      (cd $d && timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-extra 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']['ms_per_step']; print('$d $w', round(d['value'],1), round(d['ms_per_step'],3), {a: round(b,3) for a,b in k.items()})")
    done
  done
done
