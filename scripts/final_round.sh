set -u
mkdir -p gpurun_out
for W in gpt2 square4096 gpt1b shampoo sign4096 invroot cheb4096 dbnewton; do
  timeout 600 python bench.py --workload $W > gpurun_out/final_bench_$W.log 2>&1
done
timeout 300 python bench.py --impl reference > gpurun_out/final_bench_reference_gpt2.log 2>&1
bash scripts/profile_round.sh r1 gpt2
bash scripts/profile_round.sh r1 square4096
echo finished
