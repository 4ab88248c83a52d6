// Sketch-chain pass (PRISM §4.2 — the sketched-trace chain; device form DESIGN.md §4.4,
// §4.6): D = W · Rᵀ, i.e. D[c][n] = (R W)[n][c], for every matrix of the batch.
//
// A kind::f16 tcgen05.mma (M = 128, K = 16) costs ≈ 50 cycles for N ≤ 64 and 128 for
// N = 256 (scripts/mma_probe.cu), so the thin product R·W (W has
// 2w ≤ 32 columns) is issued with W as the A operand (M = 128, of which the first 32
// rows are the W rows; rows 32..127 read the B bytes that follow in smem and give TMEM
// lanes nobody reads) and 256 rows of R as the B operand (N = 256): 32 x 256 useful
// MACs per 128 cycles, against 128 x 32 per 50 for the untransposed form.  Both operands are K-major in their natural
// layouts: W is stored [c][ldS] (the previous pass's output) and R row-major.
//
// Large matrices split K over a cluster of C = L.ksplit CTAs (the tile code's low bits
// carry the slice; a matrix whose own factor P.ksplit is smaller leaves the trailing
// slices empty, i.e. zeros).  The fp32 partials are combined by a reduce-scatter over
// distributed shared memory: CTA r owns rows [r·256/C, (r+1)·256/C) of the tile; every
// CTA st.async's its partial of those rows into the owner's smem (complete_tx on the
// owner's mbarrier), the owner sums the C slices in fixed order (deterministic) and
// runs the per-row chain epilogue for its rows.  C = 1: the two warps that may read
// TMEM lanes 0..31 stage D (32 x 256 fp32) in smem and every epilogue thread takes a row.
#pragma once

#include "gemm.cuh"

namespace prism {

template <int KIND_, bool SPLIT_, int BN_ = 256>
struct ChainTCfg {
  static constexpr int KIND = KIND_;
  static constexpr bool SPLIT = SPLIT_;   // 3xTF32: B carries R_hi and R_lo (W holds its own hi/lo rows)
  static constexpr int ESZ = KIND == 0 ? 2 : 4;
  static constexpr int BK = 128 / ESZ;      // one 128-B swizzle row of K
  static constexpr int UK = 32 / ESZ;       // K per tcgen05.mma
  // rows of R per tile (MMA N): 256, or 128 for launches with few row tiles (a 4096^2
  // matrix: 32 x 4 split CTAs instead of 16 x 4 — half the MMA time and epilogue rows each)
  static constexpr int BN = BN_;
  static constexpr int WROWS = 32;          // W rows loaded per stage (MMA M = 128)
  static constexpr int A_BYTES = WROWS * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int STAGE_BYTES = A_BYTES + (SPLIT ? 2 : 1) * B_BYTES;
  // receive / staging buffer: [C sources][32 c][BN/C + 4] fp32 (padded rows: conflict-free)
  static constexpr int recv_bytes(int C) { return C * 32 * (BN / C + 4) * 4; }
  static constexpr int DSM_BYTES = recv_bytes(4) > recv_bytes(1) ? recv_bytes(4) : recv_bytes(1);
  static constexpr int STAGES_RAW = (227 * 1024 - 2048 - DSM_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 6 ? 6 : STAGES_RAW;
  static constexpr int EPI_WARPS = 8;
  // warpgroup 0: TMA producer, MMA issuer, two idle warps (REG_LO registers); warpgroups
  // 1-2: the epilogue warps 4..11 (REG_HI)
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  static constexpr int REG_LO = 72, REG_HI = 216;   // 128 x 72 + 256 x 216 = 384 x 168
  static constexpr uint32_t IDESC = idesc_make(KIND == 0 ? 1u : 2u, 0u, 128, BN);
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 1024 /*barriers*/ + DSM_BYTES;
  static_assert(STAGES >= 2, "chain pipeline needs two stages");
};

// K-block range of slice `ks` of a matrix split `own` ways (empty past its own factor)
__device__ __forceinline__ void chain_krange(int K, int BK, int own, int ks, int& lo, int& hi) {
  const int nkb = (K + BK - 1) / BK;
  lo = ks < own ? ks * nkb / own : nkb;
  hi = ks < own ? (ks + 1) * nkb / own : nkb;
}

// Slices of a tile this CTA computes: in a split launch (C > 1) the one at its cluster
// rank (the tile code's low bits); in a C = 1 launch all P.ksplit slices of the matrix,
// in order (each accumulated separately and summed in the same order as the split
// launch's reduce-scatter, so the bits do not depend on C).
__device__ __forceinline__ void chain_slices(const GemmProblem& P, uint32_t code, int C, int& s_lo, int& s_hi) {
  s_lo = C > 1 ? (int)(code & 1023) : 0;
  s_hi = C > 1 ? s_lo + 1 : (P.ksplit > 1 ? P.ksplit : 1);
}

// Pass timeline (prism_debug_trace_chain, scripts/trace_chain.py): per iteration k < 16, pass
// code and CTA, globaltimer at entry, after the PDL wait, when the first tile's accumulator is
// ready and when its epilogue ends.  Null (the default): no recording.
__device__ unsigned long long* g_chain_trace = nullptr;

template <class Cfg, int PASS>
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
  uint64_t* recv_full = tempty + 2;           // split: remote slices landed (complete_tx)
  uint64_t* recv_free = recv_full + 1;        // split: every owner consumed this CTA's slices
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(recv_free + 1);
  float* dsm = reinterpret_cast<float*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES + 1024);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int C = L.ksplit > 1 ? L.ksplit : 1;           // cluster size (1, 2, 4, 8)
  const uint32_t krank = C > 1 ? cluster_ctarank() : 0u;
  const int rows_per = Cfg::BN / C;                    // rows of the tile this CTA finishes
  const int rstride = rows_per + 4;                    // receive-buffer row stride (floats)
  // every tile / slice accumulates in TMEM as one chunk (no tf32 promotion chunks): the
  // same partial whether or not the launch splits K, so a matrix's bits never depend on
  // the batch; the tf32 accumulation error (~1e-5 relative) is immaterial for alpha
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2);   // the two TMEM-reading warps
    }
    mbar_init(recv_full, 1);                 // own expect_tx arrival; remote bytes complete_tx
    mbar_init(recv_free, C > 1 ? C - 1 : 1); // one arrival per other owner
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<1>(tmem_slot, 512);
  tc_fence_before();
  if (C > 1) cluster_sync_all();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // Before the predecessor (the previous pass) completes, everything this launch reads
  // except W is already final: the iteration counter, the done flags and R were written
  // at least two launches back, and every kernel of the solve calls launch_dependents only
  // after its own griddepcontrol.wait (so kernels two launches back have completed).  The
  // producer therefore stages the R half of its first stages now and adds W after the wait.
  const GemmProblem* __restrict__ probs = L.probs;
  bool run = true;
  unsigned long long* tr = nullptr;
  if (g_chain_trace && L.iter && *L.iter < 16)
    tr = g_chain_trace + ((size_t)(*L.iter * 32 + PASS) * 160 + blockIdx.x) * 32;
  if (tr && threadIdx.x == 0) tr[0] = globaltimer_ns();
  if (L.iter) {
    const int k = *L.iter;
    run = k >= L.iter_lo && k < L.iter_hi;
    if (L.probs_odd && (k & 1)) probs = L.probs_odd;
  }
  // The first tile's skip decision is taken once, before the wait, and shared by every role
  // and every CTA of a cluster: skip only matrices stopped in an EARLIER iteration
  // (stop_iter < k, final long before this launch).  A matrix stopped by this iteration's
  // residual stage (the launch just before the first pass) has its first tile computed and
  // ignored, so producer, MMA, epilogue and the cluster's partial exchange stay in step.
  __shared__ int s_first_active;
  int pre_n = 0;   // producer: leading k-blocks of its first tile whose R is in flight
  if (threadIdx.x == 0) s_first_active = 1;
  if (run && warp == 0 && lane == 0 && (int)blockIdx.x < L.ntiles) {
    const uint32_t code = (int)blockIdx.x < kFirstCodes ? L.first_code[blockIdx.x] : L.tiles[blockIdx.x];
    const int q = (int)(code >> 20);
    // the matrix from the problem index (matrix-major, probs_per_matrix each), so its stop
    // iteration loads together with the problem's fields instead of after them (a late CTA's
    // prologue is on the pass's critical path)
    const int* stop_p = (L.done && L.iter)
                            ? L.done + (size_t)(L.probs_per_matrix ? q / L.probs_per_matrix : probs[q].matrix) *
                                           L.done_stride + kStopIterOffset
                            : nullptr;
    const int stop_it = stop_p ? *stop_p : 0x7fffffff;
    const GemmProblem& P = probs[q];
    tma_prefetch(P.tmA);
    tma_prefetch(P.tmB);
    s_first_active = !(stop_p && stop_it < *L.iter);
    if (s_first_active) {
      const int n0 = ((code >> 10) & 1023) * Cfg::BN;
      int s_lo, s_hi, kb_lo, kb_hi, dummy;
      chain_slices(P, code, C, s_lo, s_hi);
      chain_krange(P.K, Cfg::BK, P.ksplit, s_lo, kb_lo, dummy);
      chain_krange(P.K, Cfg::BK, P.ksplit, s_hi - 1, dummy, kb_hi);
      pre_n = min(Cfg::STAGES, kb_hi - kb_lo);
      for (int j = 0; j < pre_n; ++j) {
        uint8_t* sB = stage_base + j * Cfg::STAGE_BYTES + Cfg::A_BYTES;
        mbar_arrive_expect_tx(&full[j], Cfg::STAGE_BYTES);
        tma_load_2d(sB, P.tmB, &full[j], (kb_lo + j) * Cfg::BK, n0);
        if constexpr (Cfg::SPLIT) tma_load_2d(sB + Cfg::B_BYTES, P.tmB_lo, &full[j], (kb_lo + j) * Cfg::BK, n0);
      }
    }
  }
  griddep_wait();
  griddep_launch();
  __syncthreads();   // s_first_active
  if (tr && threadIdx.x == 0) tr[1] = globaltimer_ns();
  auto skip = [&](int t, int matrix) -> bool {
    if (t == (int)blockIdx.x) return !s_first_active;
    return L.done && L.done[matrix * L.done_stride];
  };

  if (warp < 4) {
    setmaxnreg_dec<Cfg::REG_LO>();
    if (!run) {
    } else if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < L.ntiles; t += gridDim.x) {
        const uint32_t code = L.tiles[t];
        const GemmProblem& P = probs[code >> 20];
        if (skip(t, P.matrix)) continue;
        const int n0 = ((code >> 10) & 1023) * Cfg::BN;
        int s_lo, s_hi, kb_lo, kb_hi, dummy;   // the slices' k-blocks are contiguous
        chain_slices(P, code, C, s_lo, s_hi);
        chain_krange(P.K, Cfg::BK, P.ksplit, s_lo, kb_lo, dummy);
        chain_krange(P.K, Cfg::BK, P.ksplit, s_hi - 1, dummy, kb_hi);
        for (int kb = kb_lo; kb < kb_hi; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sA = stage_base + stage * Cfg::STAGE_BYTES;
          uint8_t* sB = sA + Cfg::A_BYTES;
          const bool staged = t == (int)blockIdx.x && kb - kb_lo < pre_n;   // R already in flight
          if (!staged) mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
          tma_load_2d(sA, P.tmA, &full[stage], kb * Cfg::BK, 0);    // W rows 0..31 (OOB rows zero)
          if (tr && t == (int)blockIdx.x && kb - kb_lo < 8) tr[24 + kb - kb_lo] = globaltimer_ns();
          if (!staged) {
            tma_load_2d(sB, P.tmB, &full[stage], kb * Cfg::BK, n0);   // R rows n0 .. n0+255
            if constexpr (Cfg::SPLIT) tma_load_2d(sB + Cfg::B_BYTES, P.tmB_lo, &full[stage], kb * Cfg::BK, n0);
          }
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
        if (skip(t, P.matrix)) continue;
        int s_lo, s_hi;
        chain_slices(P, code, C, s_lo, s_hi);
        for (int sl = s_lo; sl < s_hi; ++sl) {   // one TMEM chunk per slice
          int kb0, kb1;
          chain_krange(P.K, Cfg::BK, P.ksplit, sl, kb0, kb1);
          if (kb0 >= kb1) continue;
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t dt = tmem_base + acc * Cfg::BN;
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(&full[stage], phase);
            if (tr && t == (int)blockIdx.x && kb - kb0 < 16 && sl == s_lo) tr[8 + kb - kb0] = globaltimer_ns();
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
    }
  } else {
    setmaxnreg_inc<Cfg::REG_HI>();
    if (run) {
    // ===================== epilogue (warps 4..11) =====================
    const int e = warp - 4;
    const int et = threadIdx.x - 128;            // 0..255
    const bool reader = (warp & 3) == 0;         // warps 4 and 8 own TMEM lanes 0..31
    const int h = e >> 2;                        // reader column half
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t rphase = 0;   // split: receive-buffer round parity
    for (int t = blockIdx.x; t < L.ntiles; t += gridDim.x) {
      const uint32_t code = L.tiles[t];
      const GemmProblem& P = probs[code >> 20];
      if (skip(t, P.matrix)) continue;
      const int tn = (code >> 10) & 1023;
      int s_lo, s_hi;
      chain_slices(P, code, C, s_lo, s_hi);
      // this thread's row of the pass output, and its operands loaded ahead (chain_prefetch)
      const bool mine = et < rows_per;   // whole warps (rows_per = BN / C, a multiple of 32)
      const int i = !mine ? P.M : tn * Cfg::BN + (C == 1 ? 0 : (int)krank * rows_per) + et;   // P.M: no row
      const int row0 = tn * Cfg::BN + (C == 1 ? 0 : (int)krank * rows_per) + (et & ~31);
      const int grp = (mine && row0 < P.M) ? row0 >> 5 : -1;   // this warp's 32-row group
      ChainPre pre;
      chain_prefetch<Cfg, PASS>(P, i, 2, pre);
      // the accumulator (32 x 256, TMEM lanes 0..31) to the owners of its rows: CTA r of
      // the cluster owns rows [r·rows_per, (r+1)·rows_per); C = 1: all rows stay here
      if (C == 1) {
        // every slice here: staged in order (first slice written, later ones added)
        bool first = true;
        for (int sl = s_lo; sl < s_hi; ++sl) {
          int k0, k1;
          chain_krange(P.K, Cfg::BK, P.ksplit, sl, k0, k1);
          if (k0 >= k1) continue;
          if (reader) {
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            if (tr && t == (int)blockIdx.x && et == 0) tr[2] = globaltimer_ns();
#pragma unroll 1
            for (int x0 = 0; x0 < Cfg::BN / 64; x0 += 2) {   // two 32-column loads in flight per wait
              uint32_t r[2][32];
              tmem_ld32(tmem_base + acc * Cfg::BN + h * (Cfg::BN / 2) + x0 * 32, r[0]);
              tmem_ld32(tmem_base + acc * Cfg::BN + h * (Cfg::BN / 2) + (x0 + 1) * 32, r[1]);
              tmem_ld_wait();
#pragma unroll
              for (int x = 0; x < 2; ++x) {
                float* dst = dsm + (size_t)lane * rstride + h * (Cfg::BN / 2) + (x0 + x) * 32;
                if (first) {
#pragma unroll
                  for (int u = 0; u < 32; ++u) dst[u] = __uint_as_float(r[x][u]);
                } else {
#pragma unroll
                  for (int u = 0; u < 32; ++u) dst[u] += __uint_as_float(r[x][u]);
                }
              }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (tr && t == (int)blockIdx.x && et == 0) tr[4] = globaltimer_ns();
          }
          first = false;
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
      } else {
      int kb_lo, kb_hi;
      chain_krange(P.K, Cfg::BK, P.ksplit, s_lo, kb_lo, kb_hi);
      const bool have = kb_lo < kb_hi;
      if (reader) {
        if (have) {
          mbar_wait(&tfull[acc], acc_phase);
          tc_fence_after();
          if (tr && t == (int)blockIdx.x && et == 0) tr[2] = globaltimer_ns();
        }
        // every owner consumed the previous round's slices: send this round's
        mbar_wait(recv_free, rphase ^ 1);
#pragma unroll 1
        for (int x = 0; x < Cfg::BN / 64; ++x) {
          const int col = h * (Cfg::BN / 2) + x * 32;   // 32 rows n of the tile
          uint32_t r[32];
          if (have) {
            tmem_ld32(tmem_base + acc * Cfg::BN + col, r);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int u = 0; u < 32; ++u) r[u] = 0x80000000u;   // -0.0: x + (-0) == x for every x
          }
          const uint32_t owner = (uint32_t)(col / rows_per);
          const int nl = col - (int)owner * rows_per;  // row offset within the owner's range
          float* dst = dsm + ((size_t)krank * 32 + lane) * rstride + nl;   // source krank's slot
#pragma unroll
          for (int u = 0; u < 32; u += 4) {
            const float4 v = make_float4(__uint_as_float(r[u]), __uint_as_float(r[u + 1]),
                                         __uint_as_float(r[u + 2]), __uint_as_float(r[u + 3]));
            if (owner == krank) *reinterpret_cast<float4*>(dst + u) = v;
            else st_async_v4(dst + u, recv_full, owner, v);
          }
        }
        if (have) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        if (tr && t == (int)blockIdx.x && et == 0) tr[4] = globaltimer_ns();
      }
      if (have && ++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      if (C > 1 && et == 0) mbar_arrive_expect_tx(recv_full, (uint32_t)(C - 1) * 32 * rows_per * 4);
      named_bar_sync(1, 32 * Cfg::EPI_WARPS);    // own slice written locally
      if (tr && t == (int)blockIdx.x && et == 0) tr[5] = globaltimer_ns();
      if (C > 1) {
        mbar_wait(recv_full, rphase);            // the other C-1 slices landed
        if (et < rows_per) {
          // sum the C slices in fixed order (deterministic; -0.0 identity: one real slice
          // sums to itself exactly) into this thread's column of slot 0; 32 independent
          // accumulators keep each source's loads in flight together
          float v[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) v[c] = -0.f;
          for (int src = 0; src < C; ++src) {
#pragma unroll
            for (int c = 0; c < 32; ++c) v[c] += dsm[((size_t)src * 32 + c) * rstride + et];
          }
#pragma unroll
          for (int c = 0; c < 32; ++c) dsm[(size_t)c * rstride + et] = v[c];
        }
      }
      if (tr && t == (int)blockIdx.x && et == 0) tr[6] = globaltimer_ns();
      epi_chain<Cfg, PASS>(pre, i, grp, dsm + et, rstride, lane, 2);
      if (tr && t == (int)blockIdx.x && et == 0) tr[7] = globaltimer_ns();
      named_bar_sync(1, 32 * Cfg::EPI_WARPS);    // buffer consumed
      if (tr && t == (int)blockIdx.x && et == 0) tr[3] = globaltimer_ns();
      if (C > 1) {
        rphase ^= 1;
        // hand the slots back (gates only a later round's sends: off the critical path)
        if (et == 32)
          for (int x = 0; x < C; ++x)
            if (x != (int)krank) mbar_arrive_release_cluster(recv_free, (uint32_t)x);
      }
    }
  }

  }
  tc_fence_before();
  if (C > 1) cluster_sync_all();   // no CTA leaves while a peer may still write into its smem
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem_base, 512);
  }
}

}  // namespace prism
