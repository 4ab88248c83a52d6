// Launch helpers shared by the translation units of libprism.so.  The tcgen05 GEMM and
// sketch-chain kernels are instantiated per precision in their own .cu files (compiled in
// parallel); prism.cu (host side, SIMT kernels) reaches them through the launchers below.
#pragma once
#include "gemm.cuh"

#include <algorithm>
#include <array>

namespace prism {

constexpr int kMaxDevices = 64;

// Current CUDA device (the library runs on whatever device is current on the calling
// thread; every per-device cache below is indexed by it).
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return (d >= 0 && d < kMaxDevices) ? d : 0;
}

// SM count of the current device (cached per device).
inline int device_sms() {
  static std::array<int, kMaxDevices> sms{};
  const int d = current_device();
  if (sms[d] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    sms[d] = v > 0 ? v : 148;
  }
  return sms[d];
}

// Opt a kernel into `bytes` of dynamic shared memory on the current device (once per
// kernel and device: the attribute is per-context state).
template <typename K>
cudaError_t ensure_smem_attr(K kernel, int bytes, std::array<char, kMaxDevices>& done) {
  const int d = current_device();
  if (done[d]) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done[d] = 1;
  return e;
}

// Launch `k` with programmatic dependent launch (every kernel of the solve calls
// griddep_wait() before reading its predecessors' results, ptx.cuh) and, for
// cluster > 1, a 1-D thread-block cluster.
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cluster,
                     Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int n = 0;
  at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[n].val.programmaticStreamSerializationAllowed = 1;
  ++n;
  if (cluster > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cluster;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// ---- per-precision launchers (gemm_<prec>.cu, chain_<prec>.cu); precision 0 bf16,
// 1 fp32 (3xTF32), 2 tf32.  ntiles == 0 only sets the kernels' smem attributes.
cudaError_t launch_gemm_bf16(int role, const GemmLaunch& L, cudaStream_t st);
cudaError_t launch_gemm_f32x3(int role, const GemmLaunch& L, cudaStream_t st);
cudaError_t launch_gemm_tf32(int role, const GemmLaunch& L, cudaStream_t st);
cudaError_t set_gemm_trace_bf16(unsigned long long* buf, int mode);
cudaError_t set_chain_trace_bf16(unsigned long long* buf);
cudaError_t set_chain_trace_f32x3(unsigned long long* buf);
cudaError_t set_chain_trace_tf32(unsigned long long* buf);
cudaError_t set_gemm_trace_f32x3(unsigned long long* buf, int mode);
cudaError_t set_gemm_trace_tf32(unsigned long long* buf, int mode);
cudaError_t launch_chain_bf16(int pass, const GemmLaunch& L, cudaStream_t st);
cudaError_t launch_chain_f32x3(int pass, const GemmLaunch& L, cudaStream_t st);
cudaError_t launch_chain_tf32(int pass, const GemmLaunch& L, cudaStream_t st);

inline cudaError_t launch_gemm(int precision, int role, const GemmLaunch& L, cudaStream_t st) {
  if (precision == 0) return launch_gemm_bf16(role, L, st);
  if (precision == 1) return launch_gemm_f32x3(role, L, st);
  return launch_gemm_tf32(role, L, st);
}
inline cudaError_t launch_chain(int precision, int pass, const GemmLaunch& L, cudaStream_t st) {
  if (precision == 0) return launch_chain_bf16(pass, L, st);
  if (precision == 1) return launch_chain_f32x3(pass, L, st);
  return launch_chain_tf32(pass, L, st);
}

// GEMM launch of one role for configuration Cfg: persistent over the tile list, CTA
// pairs (clusters of 2) for cta_group::2 tiles.
template <class Cfg>
cudaError_t launch_gemm_cfg(int role, const GemmLaunch& L, cudaStream_t st) {
  static std::array<char, kMaxDevices> d0{}, d1{}, d2{}, d3{};
  void (*k)(const GemmLaunch) = role == ROLE_GRAM     ? prism_gram_kernel<Cfg>
                                : role == ROLE_SQUARE ? prism_square_kernel<Cfg>
                                : role == ROLE_APPLY  ? prism_apply_kernel<Cfg>
                                                      : prism_gemm_kernel<Cfg>;
  std::array<char, kMaxDevices>& done = role == ROLE_GRAM ? d0 : role == ROLE_SQUARE ? d1 : role == ROLE_APPLY ? d2 : d3;
  cudaError_t e = ensure_smem_attr(k, Cfg::SMEM_BYTES, done);
  if (e != cudaSuccess) return e;
  if (L.ntiles <= 0) return cudaSuccess;
  const int sms = device_sms();
  if constexpr (Cfg::CTA2) {
    const int pairs = std::min(L.ntiles, (L.max_ctas > 0 ? std::min(sms, L.max_ctas) : sms) / 2);
    return launch_k(k, dim3(2 * pairs), dim3(Cfg::THREADS), Cfg::SMEM_BYTES, st, 2, L);
  } else {
    const int grid = std::min(L.ntiles, L.max_ctas > 0 ? std::min(sms, L.max_ctas) : sms);
    return launch_k(k, dim3(grid), dim3(Cfg::THREADS), Cfg::SMEM_BYTES, st, 1, L);
  }
}

}  // namespace prism
