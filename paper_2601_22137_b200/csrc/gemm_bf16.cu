// tcgen05 GEMM kernels (gemm.cuh), bf16 instantiation: one kernel symbol per role.
#include "launch.h"

namespace prism {
cudaError_t launch_gemm_bf16(int role, const GemmLaunch& L, cudaStream_t st) {
  return launch_gemm_cfg<GemmCfg<0, false>>(role, L, st);
}
}  // namespace prism
