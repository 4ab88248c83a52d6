// Transposed sketch-chain pass for matrices that do not split K (PRISM §4.2, the
// sketched-trace chain of DESIGN.md §4.6): D = W · Rᵀ, i.e. D[c][n] = (R W)[n][c].
//
// One tcgen05.mma costs the same ~138 cycles for any N ≤ 256 (measured, scripts/
// mma_probe.cu), so the thin product R·W (W has 2w ≤ 32 columns) is issued with W as
// the A operand (M = 128, of which the first 32 rows are the W rows; rows 32..127
// read the B bytes that follow in smem and give TMEM lanes nobody reads) and 256 rows
// of R as the B operand (N = 256): half the MMAs of the N = 32 form (gemm.cuh,
// BN = 32), one 256-row tile of R per CTA.
//
// Both operands are K-major in their natural layouts: W is stored [c][ldS] (the
// previous pass's output) and R row-major.  Epilogue: the two warps that may read
// TMEM lanes 0..31 (warp % 4 == 0) copy D (32 x 256 fp32) to shared memory, then the
// 256 epilogue threads take one row n of R each and run the same per-row chain
// epilogue as the N = 32 kernel (epi_chain, gemm.cuh) — identical arithmetic per
// element, so both kernels produce the same K / L / <Va,Vb> definitions.
#pragma once

#include "gemm.cuh"

namespace prism {

template <int KIND_, bool SPLIT_>
struct ChainTCfg {
  static constexpr int KIND = KIND_;
  static constexpr bool SPLIT = SPLIT_;   // 3xTF32: B carries R_hi and R_lo (W holds its own hi/lo rows)
  static constexpr int ESZ = KIND == 0 ? 2 : 4;
  static constexpr int BK = 128 / ESZ;      // one 128-B swizzle row of K
  static constexpr int UK = 32 / ESZ;       // K per tcgen05.mma
  static constexpr int BN = 256;            // rows of R per tile (MMA N)
  static constexpr int WROWS = 32;          // W rows loaded per stage (MMA M = 128)
  static constexpr int A_BYTES = WROWS * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int STAGE_BYTES = A_BYTES + (SPLIT ? 2 : 1) * B_BYTES;
  static constexpr int DSTRIDE = 257;       // D staging row stride (floats): conflict-free both ways
  static constexpr int DSM_BYTES = 32 * DSTRIDE * 4;
  static constexpr int STAGES_RAW = (227 * 1024 - 2048 - DSM_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 6 ? 6 : STAGES_RAW;
  static constexpr int EPI_WARPS = 8;
  static constexpr int THREADS = 64 + 32 * EPI_WARPS;
  static constexpr int PROMO_KB = KIND == 0 ? (1 << 30) : (SPLIT ? 1 : 4);
  static constexpr uint32_t IDESC = idesc_make(KIND == 0 ? 1u : 2u, 0u, 128, BN);
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 1024 /*barriers*/ + DSM_BYTES;
  static_assert(STAGES >= 2, "chainT pipeline needs two stages");
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1) prism_chaint_kernel(const __grid_constant__ GemmLaunch L) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
  uint8_t* stage_base = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + Cfg::STAGES;
  uint64_t* tfull = bars + 2 * Cfg::STAGES;   // [2]
  uint64_t* tempty = tfull + 2;               // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  double* dred = reinterpret_cast<double*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES + 256);   // [8][6]
  float* dsm = reinterpret_cast<float*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES + 1024);     // [32][DSTRIDE]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2);   // the two TMEM-reading warps
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<1>(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (threadIdx.x == 0 && (int)blockIdx.x < L.ntiles) {
    const uint32_t code = __ldg(L.tiles + blockIdx.x);
    tma_prefetch(L.probs[code >> 20].tmA);
    tma_prefetch(L.probs[code >> 20].tmB);
  }
  griddep_launch();
  griddep_wait();
  const GemmProblem* __restrict__ probs = L.probs;
  bool run = true;
  if (L.iter) {
    const int k = *L.iter;
    run = k >= L.iter_lo && k < L.iter_hi;
    if (L.probs_odd && (k & 1)) probs = L.probs_odd;
  }

  if (!run) {
  } else if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < L.ntiles; t += gridDim.x) {
        const uint32_t code = L.tiles[t];
        const GemmProblem& P = probs[code >> 20];
        if (L.done && L.done[P.matrix * L.done_stride]) continue;
        const int n0 = ((code >> 10) & 1023) * Cfg::BN;
        const int nkb = (P.K + Cfg::BK - 1) / Cfg::BK;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sA = stage_base + stage * Cfg::STAGE_BYTES;
          uint8_t* sB = sA + Cfg::A_BYTES;
          mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
          tma_load_2d(sA, P.tmA, &full[stage], kb * Cfg::BK, 0);    // W rows 0..31 (OOB rows zero)
          tma_load_2d(sB, P.tmB, &full[stage], kb * Cfg::BK, n0);   // R rows n0 .. n0+255
          if constexpr (Cfg::SPLIT) tma_load_2d(sB + Cfg::B_BYTES, P.tmB_lo, &full[stage], kb * Cfg::BK, n0);
          if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < L.ntiles; t += gridDim.x) {
        const uint32_t code = L.tiles[t];
        const GemmProblem& P = probs[code >> 20];
        if (L.done && L.done[P.matrix * L.done_stride]) continue;
        const int nkb = (P.K + Cfg::BK - 1) / Cfg::BK;
        for (int kb0 = 0; kb0 < nkb; kb0 += Cfg::PROMO_KB) {
          const int kb1 = min(nkb, kb0 + Cfg::PROMO_KB);
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t dt = tmem_base + acc * Cfg::BN;
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t aA = smem_u32(stage_base + stage * Cfg::STAGE_BYTES);
            const uint32_t aB = aA + Cfg::A_BYTES;
#pragma unroll
            for (int k = 0; k < Cfg::BK / Cfg::UK; ++k) {
              const uint64_t da = sdesc_rt(aA + k * 32, 16, 1024, 2u);
              umma<Cfg::KIND, 1>(dt, da, sdesc_rt(aB + k * 32, 16, 1024, 2u), Cfg::IDESC,
                                 (kb != kb0 || k != 0) ? 1u : 0u);
              if constexpr (Cfg::SPLIT)
                umma<Cfg::KIND, 1>(dt, da, sdesc_rt(aB + Cfg::B_BYTES + k * 32, 16, 1024, 2u), Cfg::IDESC, 1u);
            }
            umma_commit<1>(&empty[stage]);
            if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
          }
          umma_commit<1>(&tfull[acc]);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
      }
    }
  } else {
    // ===================== epilogue (warps 2..9) =====================
    const int e = warp - 2;
    const int et = threadIdx.x - 64;             // 0..255: row n0 + et of R
    const bool reader = (warp & 3) == 0;         // warps 4 and 8 own TMEM lanes 0..31
    const int h = e >> 2;                        // reader column half
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < L.ntiles; t += gridDim.x) {
      const uint32_t code = L.tiles[t];
      const GemmProblem& P = probs[code >> 20];
      if (L.done && L.done[P.matrix * L.done_stride]) continue;
      const int tn = (code >> 10) & 1023;
      const int nkb = (P.K + Cfg::BK - 1) / Cfg::BK;
      for (int kb0 = 0; kb0 < nkb; kb0 += Cfg::PROMO_KB) {
        if (reader) {
          mbar_wait(&tfull[acc], acc_phase);
          tc_fence_after();
#pragma unroll 1
          for (int x = 0; x < 4; ++x) {
            uint32_t r[32];
            const int col = h * 128 + x * 32;
            tmem_ld32(tmem_base + acc * Cfg::BN + col, r);
            tmem_ld_wait();
            float* row = dsm + lane * Cfg::DSTRIDE + col;
            if (kb0 == 0) {
#pragma unroll
              for (int u = 0; u < 32; ++u) row[u] = __uint_as_float(r[u]);
            } else {
#pragma unroll
              for (int u = 0; u < 32; ++u) row[u] += __uint_as_float(r[u]);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      named_bar_sync(1, 32 * Cfg::EPI_WARPS);   // D staged
      float d[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) d[c] = dsm[c * Cfg::DSTRIDE + et];
      named_bar_sync(1, 32 * Cfg::EPI_WARPS);   // staging free for the next tile
      epi_chain<Cfg>(P, tn * Cfg::BN + et, tn, d, dred, e, lane, et, 2);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem_base, 512);
  }
}

}  // namespace prism
