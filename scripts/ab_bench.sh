#!/bin/bash
# Alternating A/B of the GPT-2 and 4096^2 bench steps: ab_old/ (a previous commit's tree) vs the working tree.
set -u
for r in 1 2; do
  for side in old new; do
    if [ $side = old ]; then d=ab_old; else d=.; fi
    (cd $d && python bench.py --steps 20 --warmup 5 --no-cpu-baseline $( [ $side = new ] && echo --no-extra ) 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$side gpt2', round(d['value']), round(d['ms_per_step'],4), {k: round(v['ms'] if isinstance(v,dict) else v,3) for k,v in d['kernels']['ms_per_step'].items()})")
    (cd $d && python bench.py --workload square4096 --steps 10 --warmup 3 --no-cpu-baseline $( [ $side = new ] && echo --no-extra ) 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$side 4096', round(d['value'],1), round(d['ms_per_step'],4), {k: round(v,3) for k,v in d['kernels']['ms_per_step'].items()})")
  done
done
