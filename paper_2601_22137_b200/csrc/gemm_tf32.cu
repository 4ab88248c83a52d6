// tcgen05 GEMM kernels (gemm.cuh), tf32 instantiation: one kernel symbol per role.
#include "launch.h"

namespace prism {
cudaError_t launch_gemm_tf32(int role, const GemmLaunch& L, cudaStream_t st) {
  return launch_gemm_cfg<GemmCfg<1, false>>(role, L, st);
}
}  // namespace prism

namespace prism {
// diagnostics: this translation unit's copy of the GEMM k-block timeline hook (gemm.cuh)
cudaError_t set_gemm_trace_tf32(unsigned long long* buf, int mode) {
  cudaError_t e = cudaMemcpyToSymbol(g_gemm_trace2, &buf, sizeof(buf));
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(g_trace_mode, &mode, sizeof(mode));
}
}  // namespace prism
