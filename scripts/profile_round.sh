#!/bin/bash
# Round profile capture (run under gpurun): plain bench, then the ncu launch list of the
# same command, then one full capture of the dominant kernel (apply GEMM, iteration 1).
# Outputs in gpurun_out/ (scratch); scripts/summarize_profiles.py writes profiles/.
set -u
R=${1:-r1}
W=${2:-gpt2}
python bench.py --workload $W --steps 2 --warmup 3 > gpurun_out/${R}_${W}_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/${R}_${W}_launches.csv python bench.py --workload $W --steps 2 --warmup 3 \
    > gpurun_out/${R}_${W}_ncu_bench.log 2>&1
python scripts/profile_step.py --workload $W --direct > gpurun_out/${R}_${W}_plain2.log 2>&1 &&
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:Li0ELb0ELi0ELb1 \
    -s 5 -c 1 -o gpurun_out/${R}_${W}_apply -f python scripts/profile_step.py --workload $W --direct \
    > gpurun_out/${R}_${W}_ncu_full.log 2>&1
echo done
