#!/bin/bash
# Round-end measurement pass (run under gpurun, one GPU): every bench workload (default
# options: cpu_baseline on the headline workload, extra block on the default run), the
# reference arm, then the judged profile captures (scripts/profile_round.sh).
# usage: bash scripts/final_round.sh r2
set -u
R=${1:-r2}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${R}_bench_default.log 2>&1
for W in square4096 square4096_fp32 gpt1b rowblock8192 shampoo sign4096 invroot cheb4096 dbnewton; do
  timeout 600 python bench.py --workload $W --no-extra --no-cpu-baseline > gpurun_out/${R}_bench_$W.log 2>&1
done
timeout 900 python bench.py --impl reference > gpurun_out/${R}_bench_reference.log 2>&1
echo finished
