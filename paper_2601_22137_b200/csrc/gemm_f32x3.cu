// tcgen05 GEMM kernels (gemm.cuh), f32x3 instantiation: one kernel symbol per role.
#include "launch.h"

namespace prism {
cudaError_t launch_gemm_f32x3(int role, const GemmLaunch& L, cudaStream_t st) {
  return launch_gemm_cfg<GemmCfg<1, true>>(role, L, st);
}
}  // namespace prism
