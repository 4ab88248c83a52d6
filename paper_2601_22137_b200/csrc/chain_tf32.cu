// Sketch-chain kernels (chaint.cuh), tf32 instantiation: one kernel per pass code.
#include "chain_launch.cuh"

namespace prism {
cudaError_t launch_chain_tf32(int pass, const GemmLaunch& L, cudaStream_t st) {
  return launch_chain_cfg<ChainTCfg<1, false>>(pass, L, st);
}
}  // namespace prism
