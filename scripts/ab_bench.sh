#!/bin/bash
# Alternating A/B of the GPT-2 and 4096^2 bench steps across tree copies given as arguments
# (e.g. ab_old . ab_x): each runs its own bench.py against its own libprism.so.
set -u
for r in 1 2; do
  for d in "$@"; do
    (cd $d && python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extra 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']['ms_per_step']; print('$d gpt2', round(d['value']), round(d['ms_per_step'],4), {a: round(b,3) for a,b in k.items()})")
    (cd $d && python bench.py --workload square4096 --steps 10 --warmup 3 --no-cpu-baseline --no-extra 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']['ms_per_step']; print('$d 4096', round(d['value'],1), round(d['ms_per_step'],4), {a: round(b,3) for a,b in k.items()})")
  done
done
