// Launcher of the sketch-chain kernel (chaint.cuh), one kernel per pass code (each carries
// only its own epilogue: a chain pass's code runs once per CTA per launch, from a cold
// instruction cache).  Included by chain_<precision>.cu.
#pragma once
#include "launch.h"
#include "chaint.cuh"

namespace prism {

template <class Cfg, int PASS>
cudaError_t launch_chain_pass(const GemmLaunch& L, cudaStream_t st) {
  static std::array<char, kMaxDevices> done{};
  cudaError_t e = ensure_smem_attr(prism_chaint_kernel<Cfg, PASS>, Cfg::SMEM_BYTES, done);
  if (e != cudaSuccess) return e;
  if (L.ntiles <= 0) return cudaSuccess;
  const int C = std::max(1, L.ksplit);   // split chains: clusters of C CTAs (reduce-scatter)
  const int grid = std::min(L.ntiles, device_sms() / C * C);
  return launch_k(prism_chaint_kernel<Cfg, PASS>, dim3(grid), dim3(Cfg::THREADS), Cfg::SMEM_BYTES, st, C, L);
}

template <class Cfg>
cudaError_t launch_chain_cfg(int pass, const GemmLaunch& L, cudaStream_t st) {
  switch (pass) {
    case CH2_P1: return launch_chain_pass<Cfg, CH2_P1>(L, st);
    case CH2_P2: return launch_chain_pass<Cfg, CH2_P2>(L, st);
    case CH2_P3: return launch_chain_pass<Cfg, CH2_P3>(L, st);
    case CH2_P4: return launch_chain_pass<Cfg, CH2_P4>(L, st);
    case CH2_P5: return launch_chain_pass<Cfg, CH2_P5>(L, st);
    case CH1_P1: return launch_chain_pass<Cfg, CH1_P1>(L, st);
    case CH1_P2: return launch_chain_pass<Cfg, CH1_P2>(L, st);
    case CH1_P3: return launch_chain_pass<Cfg, CH1_P3>(L, st);
    case CHI_K2: return launch_chain_pass<Cfg, CHI_K2>(L, st);
    case CHI_L1: return launch_chain_pass<Cfg, CHI_L1>(L, st);
    case CHI_L2: return launch_chain_pass<Cfg, CHI_L2>(L, st);
    case CHI_L3: return launch_chain_pass<Cfg, CHI_L3>(L, st);
    case CHI_L4: return launch_chain_pass<Cfg, CHI_L4>(L, st);
    case CHC_P1: return launch_chain_pass<Cfg, CHC_P1>(L, st);
    case CHC_P2: return launch_chain_pass<Cfg, CHC_P2>(L, st);
    case CHC_P3: return launch_chain_pass<Cfg, CHC_P3>(L, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace prism
