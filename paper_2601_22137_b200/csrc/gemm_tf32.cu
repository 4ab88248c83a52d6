// tcgen05 GEMM kernels (gemm.cuh), tf32 instantiation: one kernel symbol per role.
#include "launch.h"

namespace prism {
cudaError_t launch_gemm_tf32(int role, const GemmLaunch& L, cudaStream_t st) {
  return launch_gemm_cfg<GemmCfg<1, false>>(role, L, st);
}
}  // namespace prism
