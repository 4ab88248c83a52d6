// Persistent, warp-specialised, grouped tcgen05 GEMM for the PRISM iteration.
//
// One launch runs a list of tiles drawn from many independent problems (the
// matrices of a Muon/Shampoo batch): D = A·B with
//   A  : M x K, K-major (row-major A), fed by TMA with 128-B swizzle
//   B  : K-major (B stored N x K, i.e. A·Bᵀ) or MN-major (B stored K x N)
//   D  : fp32 accumulator in TMEM (two accumulator buffers, so the epilogue
//        of tile t overlaps the MMAs of tile t+1)
// and a fused epilogue that forms the PRISM quantity directly:
//   RESID  out = I − D            (residual R_k, P:252-254 / P:274), ‖R‖² partial,
//                                 fp32 diag(D) (= diag G, for the sketch)
//   POLY   out = c1·C + α·D       (P = ½R + αR², d=2)
//   APPLY  out = C + s·D          (X ← X + X·P, or X + α·X·R for d=1)
//   STORE  out = D                (tests)
// `sym` schedules only tiles touching the upper triangle and mirrors the
// stores, so XᵀX and R·R cost half a dense GEMM and R, P are exactly symmetric.
//
// Roles (192 threads, one CTA per SM):
//   warp 0      TMA producer  (one elected lane)
//   warp 1      TMEM allocator + MMA issuer (one elected lane)
//   warps 2..5  epilogue: tcgen05.ld → registers → fused math → global
// Precisions: KIND 0 = bf16 (kind::f16), KIND 1 = tf32 (kind::tf32); SPLIT
// adds the 3xTF32 correction D += A·B_lo + A_lo·B with hi parts stored
// pre-truncated to tf32 (so hardware rounding mode is irrelevant).
#pragma once
#include "ptx.cuh"

namespace prism {

enum EpiMode : int { EPI_RESID = 0, EPI_POLY = 1, EPI_APPLY = 2, EPI_STORE = 3 };

struct GemmProblem {
  const CUtensorMap* tmA;
  const CUtensorMap* tmB;
  const CUtensorMap* tmA_lo;
  const CUtensorMap* tmB_lo;
  void* out;
  void* out_lo;
  const void* C;
  const void* C_lo;
  float* norm_part;      // [tiles_m * tiles_n] per-tile Σ out² (RESID) or null
  float* gdiag;          // [M] diag of D (RESID) or null
  const double* alpha;   // device scalar α (POLY, APPLY with scale_by_alpha)
  long long ldo, ldc;    // leading dimensions (elements)
  int M, N, K;
  int mode, sym, matrix, scale_by_alpha, tiles_n;
  float c1;
  int pad_;
};

struct GemmLaunch {
  const GemmProblem* probs;
  const uint32_t* tiles;   // (problem << 20) | (tm << 10) | tn
  const int* done;         // per matrix (stride done_stride ints): 1 = stopped, skip its tiles
  int done_stride;
  int ntiles;
};

template <int KIND_, bool SPLIT_, bool BMN_>
struct GemmCfg {
  static constexpr int KIND = KIND_;
  static constexpr bool SPLIT = SPLIT_;
  static constexpr bool BMN = BMN_;
  static constexpr int ESZ = KIND == 0 ? 2 : 4;
  static constexpr int BM = 128;
  static constexpr int BN = KIND == 0 ? 256 : 128;
  static constexpr int BK = 128 / ESZ;          // one 128-B swizzle row of K
  static constexpr int UK = 32 / ESZ;           // K per tcgen05.mma (32 bytes)
  static constexpr int A_BYTES = BM * BK * ESZ;
  static constexpr int B_BYTES = BN * BK * ESZ;
  static constexpr int NOPS = SPLIT ? 2 : 1;
  static constexpr int STAGE_BYTES = NOPS * (A_BYTES + B_BYTES);
  static constexpr int STAGES_RAW = (192 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int B_ATOMS = BN * ESZ / 128;  // MN-major: 128-B wide boxes along N
  static constexpr int B_ATOM_BYTES = BK * 128;
  // MN-major B: bf16 uses the 128-B swizzle (8-row K groups, SBO 1024); tf32 must use
  // the 128-B/32-B-atom swizzle (layout type 1, 4-row K groups, SBO 512).
  static constexpr uint32_t BMN_LAYOUT = KIND == 0 ? 2u : 1u;
  static constexpr uint32_t BMN_SBO = KIND == 0 ? 1024u : 512u;
  static constexpr uint32_t IDESC = idesc_make(KIND == 0 ? 1u : 2u, BMN ? 1u : 0u, BM, BN);
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int THREADS = 192;
  // k-blocks per TMEM accumulation chunk: tf32 partials are promoted to fp32
  // registers every k-block (3xTF32, K = 32: 12 MMAs per chunk) or every 4
  // (1xTF32); bf16 keeps one accumulator per tile (products exact, 2^-9 output).
  static constexpr int PROMO_KB = KIND == 0 ? (1 << 30) : (SPLIT ? 1 : 4);
};

// ---------------------------------------------------------------- epilogue helpers

__device__ __forceinline__ float tf32_trunc(float v) {
  return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
}

template <int KIND, bool SPLIT>
__device__ __forceinline__ void load_row32(const void* base, const void* base_lo, long long ld, int i, int j0,
                                           int N, float (&c)[32]) {
  if constexpr (KIND == 0) {
    const __nv_bfloat16* p = static_cast<const __nv_bfloat16*>(base) + (long long)i * ld + j0;
    if (j0 + 32 <= N) {
      const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint4 w = __ldg(q + u);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 f = __bfloat1622float2(h[e]);
          c[u * 8 + 2 * e] = f.x;
          c[u * 8 + 2 * e + 1] = f.y;
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < 32; ++u) c[u] = (j0 + u < N) ? __bfloat162float(p[u]) : 0.f;
    }
  } else {
    const float* p = static_cast<const float*>(base) + (long long)i * ld + j0;
    const float* pl = SPLIT ? static_cast<const float*>(base_lo) + (long long)i * ld + j0 : nullptr;
    if (j0 + 32 <= N) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        float4 w = __ldg(reinterpret_cast<const float4*>(p) + u);
        c[4 * u] = w.x; c[4 * u + 1] = w.y; c[4 * u + 2] = w.z; c[4 * u + 3] = w.w;
        if constexpr (SPLIT) {
          float4 l = __ldg(reinterpret_cast<const float4*>(pl) + u);
          c[4 * u] += l.x; c[4 * u + 1] += l.y; c[4 * u + 2] += l.z; c[4 * u + 3] += l.w;
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        float x = 0.f;
        if (j0 + u < N) {
          x = p[u];
          if constexpr (SPLIT) x += pl[u];
        }
        c[u] = x;
      }
    }
  }
}

template <int KIND, bool SPLIT>
__device__ __forceinline__ void store_elem(void* out, void* out_lo, long long idx, float v) {
  if constexpr (KIND == 0) {
    static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(v);
  } else if constexpr (SPLIT) {
    float hi = tf32_trunc(v);
    static_cast<float*>(out)[idx] = hi;
    static_cast<float*>(out_lo)[idx] = v - hi;
  } else {
    static_cast<float*>(out)[idx] = v;
  }
}

// full 32-wide row segment, all in bounds, 16-B aligned
template <int KIND, bool SPLIT>
__device__ __forceinline__ void store_row32(void* out, void* out_lo, long long off, const float (&v)[32]) {
  if constexpr (KIND == 0) {
    uint4* q = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(out) + off);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint4 w;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
      for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[u * 8 + 2 * e], v[u * 8 + 2 * e + 1]);
      q[u] = w;
    }
  } else {
    float4* q = reinterpret_cast<float4*>(static_cast<float*>(out) + off);
    float4* ql = SPLIT ? reinterpret_cast<float4*>(static_cast<float*>(out_lo) + off) : nullptr;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if constexpr (SPLIT) {
        float4 h = make_float4(tf32_trunc(v[4 * u]), tf32_trunc(v[4 * u + 1]), tf32_trunc(v[4 * u + 2]),
                               tf32_trunc(v[4 * u + 3]));
        q[u] = h;
        ql[u] = make_float4(v[4 * u] - h.x, v[4 * u + 1] - h.y, v[4 * u + 2] - h.z, v[4 * u + 3] - h.w);
      } else {
        q[u] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
      }
    }
  }
}

// Fused epilogue for one 32-column row segment [j0, j0+32) of output row i,
// given the fp32 accumulator values d[] of D = A·B.
template <class Cfg>
__device__ __forceinline__ void epi_segment(const GemmProblem& P, int mode, bool sym, int i, int j0, float coefA,
                                            float coefC, const float (&d)[32], float& sumsq) {
  if (i >= P.M || j0 >= P.N) return;
  if (sym && j0 + 31 < i) return;           // whole segment below the diagonal
  float v[32];
  if (mode == EPI_POLY || mode == EPI_APPLY) {
    float c[32];
    load_row32<Cfg::KIND, Cfg::SPLIT>(P.C, P.C_lo, P.ldc, i, j0, P.N, c);
#pragma unroll
    for (int u = 0; u < 32; ++u) v[u] = coefC * c[u] + coefA * d[u];
  } else if (mode == EPI_RESID) {
#pragma unroll
    for (int u = 0; u < 32; ++u) v[u] = ((j0 + u == i) ? 1.f : 0.f) - d[u];
    if (P.gdiag && i >= j0 && i < j0 + 32) {
#pragma unroll
      for (int u = 0; u < 32; ++u)
        if (j0 + u == i) P.gdiag[i] = d[u];
    }
  } else {
#pragma unroll
    for (int u = 0; u < 32; ++u) v[u] = d[u];
  }
  const long long off = (long long)i * P.ldo + j0;
  if (!sym) {
    if (j0 + 32 <= P.N) {
      store_row32<Cfg::KIND, Cfg::SPLIT>(P.out, P.out_lo, off, v);
      if (mode == EPI_RESID) {
#pragma unroll
        for (int u = 0; u < 32; ++u) sumsq += v[u] * v[u];
      }
    } else {
      for (int u = 0; u < 32; ++u)
        if (j0 + u < P.N) {
          store_elem<Cfg::KIND, Cfg::SPLIT>(P.out, P.out_lo, off + u, v[u]);
          if (mode == EPI_RESID) sumsq += v[u] * v[u];
        }
    }
  } else {
    // upper triangle (j >= i) written directly, (j > i) mirrored to (j, i)
    if (j0 >= i && j0 + 32 <= P.N) {
      store_row32<Cfg::KIND, Cfg::SPLIT>(P.out, P.out_lo, off, v);
    } else {
      for (int u = 0; u < 32; ++u) {
        const int j = j0 + u;
        if (j >= i && j < P.N) store_elem<Cfg::KIND, Cfg::SPLIT>(P.out, P.out_lo, off + u, v[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const int j = j0 + u;
      if (j > i && j < P.N) {
        store_elem<Cfg::KIND, Cfg::SPLIT>(P.out, P.out_lo, (long long)j * P.ldo + i, v[u]);
        if (mode == EPI_RESID) sumsq += 2.f * v[u] * v[u];
      } else if (j == i && mode == EPI_RESID) {
        sumsq += v[u] * v[u];
      }
    }
  }
}

// ---------------------------------------------------------------- the kernel

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1) prism_gemm_kernel(const __grid_constant__ GemmLaunch L) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment for the 128-B swizzle atoms
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
  uint8_t* stage_base = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* full = bars;                       // [STAGES]
  uint64_t* empty = bars + Cfg::STAGES;        // [STAGES]
  uint64_t* tfull = bars + 2 * Cfg::STAGES;    // [2]
  uint64_t* tempty = tfull + 2;                // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* red = reinterpret_cast<float*>(tmem_slot + 4);   // [4] epilogue reduction scratch

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < L.ntiles; t += gridDim.x) {
        const uint32_t code = L.tiles[t];
        const GemmProblem& P = L.probs[code >> 20];
        if (L.done && L.done[P.matrix * L.done_stride]) continue;
        const int tm = (code >> 10) & 1023, tn = code & 1023;
        const int nkb = (P.K + Cfg::BK - 1) / Cfg::BK;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sA = stage_base + stage * Cfg::STAGE_BYTES;
          uint8_t* sB = sA + Cfg::A_BYTES;
          mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
          tma_load_2d(sA, P.tmA, &full[stage], kb * Cfg::BK, tm * Cfg::BM);
          if constexpr (Cfg::BMN) {
#pragma unroll
            for (int q = 0; q < Cfg::B_ATOMS; ++q)
              tma_load_2d(sB + q * Cfg::B_ATOM_BYTES, P.tmB, &full[stage], tn * Cfg::BN + q * (128 / Cfg::ESZ),
                          kb * Cfg::BK);
          } else {
            tma_load_2d(sB, P.tmB, &full[stage], kb * Cfg::BK, tn * Cfg::BN);
          }
          if constexpr (Cfg::SPLIT) {
            uint8_t* sA2 = sB + Cfg::B_BYTES;
            uint8_t* sB2 = sA2 + Cfg::A_BYTES;
            tma_load_2d(sA2, P.tmA_lo, &full[stage], kb * Cfg::BK, tm * Cfg::BM);
            if constexpr (Cfg::BMN) {
#pragma unroll
              for (int q = 0; q < Cfg::B_ATOMS; ++q)
                tma_load_2d(sB2 + q * Cfg::B_ATOM_BYTES, P.tmB_lo, &full[stage],
                            tn * Cfg::BN + q * (128 / Cfg::ESZ), kb * Cfg::BK);
            } else {
              tma_load_2d(sB2, P.tmB_lo, &full[stage], kb * Cfg::BK, tn * Cfg::BN);
            }
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
        const GemmProblem& P = L.probs[code >> 20];
        if (L.done && L.done[P.matrix * L.done_stride]) continue;
        const int nkb = (P.K + Cfg::BK - 1) / Cfg::BK;
        // tf32: one TMEM accumulation chunk per PROMO_KB k-blocks, promoted to fp32
        // registers by the epilogue (bounds the truncation of the MMA accumulator add)
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
              const uint64_t da = sdesc_sw128(aA + k * 32, 16, 1024);
              const uint64_t db =
                  Cfg::BMN ? sdesc_sw128<Cfg::BMN_LAYOUT>(aB + k * Cfg::UK * 128, Cfg::B_ATOM_BYTES, Cfg::BMN_SBO)
                           : sdesc_sw128(aB + k * 32, 16, 1024);
              umma<Cfg::KIND>(dt, da, db, Cfg::IDESC, (kb != kb0 || k != 0) ? 1u : 0u);
              if constexpr (Cfg::SPLIT) {
                const uint32_t aA2 = aB + Cfg::B_BYTES;
                const uint32_t aB2 = aA2 + Cfg::A_BYTES;
                const uint64_t da2 = sdesc_sw128(aA2 + k * 32, 16, 1024);
                const uint64_t db2 =
                    Cfg::BMN ? sdesc_sw128<Cfg::BMN_LAYOUT>(aB2 + k * Cfg::UK * 128, Cfg::B_ATOM_BYTES, Cfg::BMN_SBO)
                             : sdesc_sw128(aB2 + k * 32, 16, 1024);
                umma<Cfg::KIND>(dt, da, db2, Cfg::IDESC, 1u);   // A_hi · B_lo
                umma<Cfg::KIND>(dt, da2, db, Cfg::IDESC, 1u);   // A_lo · B_hi
              }
            }
            umma_commit(&empty[stage]);     // smem slot free once these MMAs retire
            if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
          }
          umma_commit(&tfull[acc]);          // accumulator (chunk) ready for the epilogue
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
      }
    }
  } else {
    // ===================== epilogue (warps 2..5) =====================
    const int q = warp & 3;                 // TMEM lane quarter this warp may access
    const int et = threadIdx.x - 64;        // 0..127
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < L.ntiles; t += gridDim.x) {
      const uint32_t code = L.tiles[t];
      const GemmProblem& P = L.probs[code >> 20];
      if (L.done && L.done[P.matrix * L.done_stride]) continue;
      const int tm = (code >> 10) & 1023, tn = code & 1023;
      const int mode = P.mode;
      const bool sym = P.sym != 0;
      const int i = tm * Cfg::BM + q * 32 + lane;   // output row of this thread
      float coefA = 1.f, coefC = 1.f;
      if (mode == EPI_POLY) { coefA = static_cast<float>(*P.alpha); coefC = P.c1; }
      if (mode == EPI_APPLY && P.scale_by_alpha) coefA = static_cast<float>(*P.alpha);
      float sumsq = 0.f;

      if constexpr (Cfg::PROMO_KB >= (1 << 20)) {
        // bf16: one TMEM accumulator per tile, consumed 32 columns at a time
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * Cfg::BN;
#pragma unroll 1
        for (int ch = 0; ch < Cfg::BN / 32; ++ch) {
          __syncwarp();
          uint32_t r[32];
          tmem_ld32(tbase + ch * 32, r);
          tmem_ld_wait();
          float d[32];
#pragma unroll
          for (int u = 0; u < 32; ++u) d[u] = __uint_as_float(r[u]);
          epi_segment<Cfg>(P, mode, sym, i, tn * Cfg::BN + ch * 32, coefA, coefC, d, sumsq);
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      } else {
        // tf32: sum the K-chunk partials from TMEM in fp32 registers (round-to-nearest)
        float d[Cfg::BN / 32][32];
#pragma unroll
        for (int ch = 0; ch < Cfg::BN / 32; ++ch)
#pragma unroll
          for (int u = 0; u < 32; ++u) d[ch][u] = 0.f;
        const int nkb = (P.K + Cfg::BK - 1) / Cfg::BK;
        for (int kb0 = 0; kb0 < nkb; kb0 += Cfg::PROMO_KB) {
          mbar_wait(&tfull[acc], acc_phase);
          tc_fence_after();
          const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * Cfg::BN;
#pragma unroll
          for (int ch = 0; ch < Cfg::BN / 32; ++ch) {
            uint32_t r[32];
            tmem_ld32(tbase + ch * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int u = 0; u < 32; ++u) d[ch][u] += __uint_as_float(r[u]);
          }
          tc_fence_before();
          mbar_arrive(&tempty[acc]);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
#pragma unroll
        for (int ch = 0; ch < Cfg::BN / 32; ++ch)
          epi_segment<Cfg>(P, mode, sym, i, tn * Cfg::BN + ch * 32, coefA, coefC, d[ch], sumsq);
      }

      if (mode == EPI_RESID && P.norm_part) {
        // deterministic per-tile Σ out²: fixed shuffle tree, then 4 warps in order
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sumsq += __shfl_xor_sync(0xffffffffu, sumsq, o);
        if (lane == 0) red[q] = sumsq;
        named_bar_sync(1, 128);
        if (et == 0) P.norm_part[tm * P.tiles_n + tn] = (red[0] + red[1]) + (red[2] + red[3]);
        named_bar_sync(1, 128);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

}  // namespace prism
