// Sketch-chain kernels (chaint.cuh), f32x3 instantiation: one kernel per pass code.
#include "chain_launch.cuh"

namespace prism {
cudaError_t launch_chain_f32x3(int pass, const GemmLaunch& L, cudaStream_t st) {
  if (L.chain_bn == 128) return launch_chain_cfg<ChainTCfg<1, true, 128>>(pass, L, st);
  return launch_chain_cfg<ChainTCfg<1, true>>(pass, L, st);
}
cudaError_t set_chain_trace_f32x3(unsigned long long* buf) {
  return cudaMemcpyToSymbol(g_chain_trace, &buf, sizeof(buf));
}
}  // namespace prism
