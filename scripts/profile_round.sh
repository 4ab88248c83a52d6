#!/bin/bash
# Round profile capture (run under gpurun, one GPU): the plain bench, the ncu launch list of
# the same command (cold-cache, serialised: compare SHARES), then one full-set capture of
# each hot kernel of the iteration from a direct-launch solve: the role-named tcgen05 GEMMs
# (Gram, square, apply), one sketch-chain pass and the alpha solve.  Outputs go to
# gpurun_out/ (scratch); scripts/summarize_profiles.py writes the judged summaries to profiles/.
# usage: bash scripts/profile_round.sh r2 gpt2
set -u
R=${1:-r2}
W=${2:-gpt2}
O=gpurun_out
python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline --no-extra > $O/${R}_${W}_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file $O/${R}_${W}_launches.csv python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline \
    --no-extra > $O/${R}_${W}_ncu_bench.log 2>&1
python scripts/profile_step.py --workload $W --direct > $O/${R}_${W}_plain2.log 2>&1
# skip the first launches of a kind (iteration 0 of the warm-up solve), capture one
for K in prism_gram_kernel prism_square_kernel prism_apply_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
      -o $O/${R}_${W}_${K} -f python scripts/profile_step.py --workload $W --direct > $O/${R}_${W}_${K}.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:prism_chaint_kernel -s 7 -c 1 \
    -o $O/${R}_${W}_chain -f python scripts/profile_step.py --workload $W --direct > $O/${R}_${W}_chain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_alpha -s 2 -c 1 \
    -o $O/${R}_${W}_alpha -f python scripts/profile_step.py --workload $W --direct > $O/${R}_${W}_alpha.log 2>&1
echo done
