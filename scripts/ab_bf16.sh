#!/bin/bash
# Alternating A/B of the BF16 polar workloads across tree copies given as arguments.
set -u
for r in 1 2 3; do
  for d in "$@"; do
    for w in gpt2 square4096 gpt1b; do
      (cd $d && timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-extra 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']['ms_per_step']; print('$d $w', round(d['value'],1), round(d['ms_per_step'],3), {a: round(b,3) for a,b in k.items()})")
    done
  done
done
