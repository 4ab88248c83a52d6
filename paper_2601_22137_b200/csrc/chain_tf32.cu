// Sketch-chain kernels (chaint.cuh), tf32 instantiation: one kernel per pass code.
#include "chain_launch.cuh"

namespace prism {
cudaError_t launch_chain_tf32(int pass, const GemmLaunch& L, cudaStream_t st) {
  return launch_chain_cfg<ChainTCfg<1, false>>(pass, L, st);
}
cudaError_t set_chain_trace_tf32(unsigned long long* buf) {
  return cudaMemcpyToSymbol(g_chain_trace, &buf, sizeof(buf));
}
}  // namespace prism
