# A/B of the early square GEMM (PRISM_EARLY_SQUARE=0 disables), same box, alternating
for rep in 1 2; do
for E in 0 1; do
for W in ${WORKLOADS:-gpt2 square4096 shampoo}; do
  PRISM_EARLY_SQUARE=$E timeout 300 python bench.py --workload $W --no-cpu-baseline --steps 20 > gpurun_out/ab_${W}_${E}_${rep}.log 2>&1
done; done; done
