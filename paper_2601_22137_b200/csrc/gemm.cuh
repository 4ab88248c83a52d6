// Persistent, warp-specialised, grouped tcgen05 GEMM for the PRISM iteration.
//
// One launch runs a list of tiles drawn from many independent problems (the
// matrices of a Muon/Shampoo batch): D = A·B with operands
// fed by TMA with 128-B swizzle, each either K-major (A stored M x K / B stored
// N x K) or MN-major (A stored K x M / B stored K x N) — a per-problem runtime
// choice, so XᵀX of a tall row-major X needs no transpose.
//   D  : fp32 accumulator in TMEM (two accumulator buffers, so the epilogue
//        of tile t overlaps the MMAs of tile t+1)
// and a fused epilogue that forms the PRISM quantity directly:
//   RESID  out = I − D            (residual R_k, P:252-254 / P:274), ‖R‖² partial,
//                                 fp32 diag(D) (= diag G, for the sketch)
//   POLY   out = c1·C + α·D       (P = ½R + αR², d=2)
//   APPLY  out = C + s·D          (X ← X + X·P, or X + α·X·R for d=1)
//          (general form of both: out = (κ_C α^{e_C} + λ_C)·C + (κ_A α^{e_A} + λ_A)·D,
//          which also builds the inverse-Newton polynomials (I + αR)^q − I, P:560-561,
//          the DB Newton updates (1−α)X + αX·M⁻¹, and its Schur sweeps)
//   STORE  out = D                (tests)
//   GRAM32 out = D as fp32 packed upper-triangle panels (row-block partial Gram, summed
//                                 across ranks)
//   APPLY2 out = C + ½·D, out2 = D  (row-block d = 2: X_r + ½Y_r and Y_r = X_r R)
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

enum EpiMode : int { EPI_RESID = 0, EPI_POLY = 1, EPI_APPLY = 2, EPI_STORE = 3, EPI_CHAIN = 4, EPI_GRAM32 = 5,
                     EPI_APPLY2 = 6 };

// Sketch-chain pass codes (EPI_CHAIN).  The thin GEMM computes
// D = R · [W_hi | W_lo] (N = 2w) and the epilogue forms out = D_hi + D_lo, then
//   d=2: P1 K1 -> Q (diag trick) -> next [K1|Q];  P2 [K2|L1] keep K2 -> next [K2|L1];
//        P3 [K3|L2] keep K3,L2 -> next L2;  P4 L3 keep -> next L3;  P5 L4 -> <Va,Vb>
//   d=1: P1 K1 keep -> next Q;  P2 L1 keep -> next L1;  P3 L2 -> <Va,Vb>
//   inverse Newton, root q: CH1_P1 (K1 = R S^T keep, next Q = M S^T),
//        then Z_j = R Z_{j-1}: CH1_P2 (slot 1), CHI_K2 (slot 2), CH2_P4 (slot 3) for
//        j < q, and CHI_L<q> for j = q: <V_i, V_j>, V_0 = K1, V_i = -C(q,i) Z_i
//   Chebyshev inverse (R stored transposed, so a pass gives the rows of W R):
//        CHC_P1 S R -> next;  CHC_P2 S R^2 keep -> next;  CHC_P3 S R^3: U = S R^2,
//        V = U - S R^3 = U G (G = I - R) by the diagonal trick, <U,U>, <U,V>, <V,V>
enum ChainPassCode : int { CH2_P1 = 0, CH2_P2, CH2_P3, CH2_P4, CH2_P5, CH1_P1, CH1_P2, CH1_P3,
                           CHI_K2, CHI_L1, CHI_L2, CHI_L3, CHI_L4, CHC_P1, CHC_P2, CHC_P3, CH_NCODES };
constexpr int kChainG = 15;   // doubles per 32-row group in chain_part (<V_i,V_j>, i <= j <= 4)
__host__ __device__ constexpr bool chain_is_last(int pass) {
  return pass == CH2_P5 || pass == CH1_P3 || pass == CHC_P3 || (pass >= CHI_L1 && pass <= CHI_L4);
}
// kept slots the last pass reads
__host__ __device__ constexpr int chain_last_slots(int pass) {
  return pass == CH2_P5 ? 4 : pass == CH1_P3 ? 2 : pass == CHC_P3 ? 1 : pass - CHI_L1 + 1;
}
// <Va,Vb> values the last pass writes
__host__ __device__ constexpr int chain_ng(int pass) {
  return (pass >= CHI_L1 && pass <= CHI_L4) ? (pass - CHI_L1 + 2) * (pass - CHI_L1 + 3) / 2 : pass == CHC_P3 ? 3 : 6;
}

// Per-matrix solver state (device memory, one per matrix of the batch).
struct MatState {
  double c;          // ||A||_F
  double inv_c;      // 1 / c   (folded normalisation: iteration 0 reads A itself)
  double inv_c2;     // 1 / c^2
  double alpha;      // current alpha_k (read by GEMM epilogues)
  double r_prev;     // ||R_{k-1}||_F
  float resid;       // ||R_final||_F / sqrt(s)
  int done;          // 1 once the matrix stopped (skip all further work)
  int iters;         // updates applied
  int status;        // PRISM_CONVERGED ...
  int incr;          // consecutive residual increases
  int stop_iter;     // iteration k at which the matrix stopped (INT_MAX while active; -1: zero input)
  int arrivals;      // residual stage: norm partials landed this iteration (the last one decides)
  int flip;          // folded polar, this solve: the caller's Q holds the odd iterates X_1, X_3, ...
                     // (else the even ones); chosen by k_init_state
};

// Stop test of iteration k (R12), run once per matrix by the last residual-stage
// block (GEMM tile or SIMT block) whose norm partial lands: ||R_k||_F from the nparts
// partials (fixed order: lane-strided fp64 sums, a fixed xor tree, lane 0's value), then the
// state update.  Converged when ||R_k||_F <= tol sqrt(s); non-finite; diverged after 5
// consecutive increases; max_iters when k = max_iters.  Every later kernel of iteration k
// (sketch, chain, alpha, square, apply) sees `done` and skips the matrix.  Warp-collective.
__device__ __forceinline__ void residual_stop_warp(MatState* S, const float* norm_part, int nparts, int k,
                                                   double tol, int s, int max_iters, float* hist, int lane) {
  double part = 0.0;
  for (int t = lane; t < nparts; t += 32) part += (double)__ldcg(norm_part + t);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane != 0) return;
  const double r = sqrt(part);
  int stop = 0, status = 1, incr = 0;
  if (!isfinite(r)) { stop = 1; status = 3; }
  else if (r <= tol * sqrt((double)s)) { stop = 1; status = 0; }
  else {
    incr = (k >= 1 && r > S->r_prev) ? S->incr + 1 : 0;
    if (incr >= 5) { stop = 1; status = 2; }
    else if (k >= max_iters) { stop = 1; status = 1; }
  }
  hist[k] = (float)(r / sqrt((double)s));
  if (isfinite(r) && !(r <= tol * sqrt((double)s))) S->incr = incr;
  S->r_prev = r;
  S->resid = (float)(r / sqrt((double)s));
  S->iters = k;
  S->arrivals = 0;   // next iteration's residual stage counts from zero
  if (stop) {
    S->stop_iter = k;
    S->status = status;
    __threadfence();
    S->done = 1;
  }
}

// Residual-stage arrival: called by one thread after its block's norm partial is stored;
// returns true for the last of `expect` arrivals of the matrix this iteration.
__device__ __forceinline__ bool residual_arrive(MatState* S, int expect) {
  __threadfence();
  return atomicAdd(&S->arrivals, 1) == expect - 1;
}

// ints from MatState::done to MatState::stop_iter (chain kernel's first-tile snapshot)
constexpr int kStopIterOffset = (int)((offsetof(MatState, stop_iter) - offsetof(MatState, done)) / sizeof(int));

struct GemmProblem {
  const CUtensorMap* tmA;
  const CUtensorMap* tmB;
  const CUtensorMap* tmA_lo;
  const CUtensorMap* tmB_lo;
  const CUtensorMap* tmC;   // bf16 epilogue: 32 x 32 blocks of C (TMA load) and of out (TMA store)
  const CUtensorMap* tmO;
  const CUtensorMap* tmO2;  // EPI_APPLY2: second output (bf16 TMA store)
  void* out;
  void* out_lo;
  void* out2;               // EPI_APPLY2: out2 = D (same leading dimension as out)
  void* out2_lo;
  const void* C;
  const void* C_lo;
  float* norm_part;      // [tiles_m * tiles_n] per-tile Σ out² (RESID) or null
  float* gdiag;          // [M] diag of D (RESID) or null
  const double* alpha;   // device scalar α (POLY, APPLY with scale_by_alpha)
  long long ldo, ldc;    // leading dimensions (elements)
  int M, N, K;
  int mode, sym, matrix, scale_by_alpha, tiles_n;
  float c1;              // POLY / APPLY: out = (c1 α^eC + lC) · C + (kA α^eA + lA) · D
  float kA;
  int eA, eC;
  float lA, lC;
  int pass;              // EPI_CHAIN pass code
  int a_mn, b_mn;        // operand major-ness: 0 K-major, 1 MN-major
  int ksplit;            // EPI_CHAIN split-K slices (tile code tn = slice index) or 1
  // EPI_CHAIN operands (row i of R = row i of the output)
  const float* S;        // [p][ldS] sketch (fp32)
  const void* Rg;        // R (for R_ii), compute dtype (+ R_lo in 3xTF32)
  const void* Rg_lo;
  void* Wn;              // next pass B operand: [2w'][ldS] hi rows then lo rows, compute dtype
  const void* Wi;        // this pass's input W (same layout; CHC_P3 reads the values the MMA used)
  float* keep;           // [4][M][p] fp32 kept chain columns
  double* chain_part;    // [row groups][kChainG] per-group <Va,Vb> partials
  long long ldS, ldr;
  int p;
  int pad2_;
};

constexpr int kFirstCodes = 160;
// tile code bit 9: a BN/2-column tile (bf16 applies only: the last, partial wave of a launch
// is split in N so it runs on twice the CTA pairs; prism.cu).  tn then counts BN/2 columns.
constexpr uint32_t kHalfTile = 512;
struct GemmLaunch {
  const GemmProblem* probs;      // problem table (even iterations)
  const GemmProblem* probs_odd;  // problem table for odd iterations (ping-pong buffers) or null
  const GemmProblem* probs_k0;   // problem table of iteration 0 (folded normalisation) or null
  const uint32_t* tiles;         // (problem << 20) | (tm << 10) | tn
  // per-iteration compacted tile list (tiles of matrices still active, plan order; written by
  // k_alpha's compaction blocks) and its length, used from iteration c_from on; null: `tiles` only
  const uint32_t* ctiles;
  const int* ccount;
  int c_from;
  const int* done;               // per matrix (stride done_stride ints): 1 = stopped, skip its tiles
  const int* iter;               // device iteration counter k (or null): run only if iter_lo <= k < iter_hi
  int done_stride;
  int ntiles;
  int iter_lo, iter_hi;
  int ksplit;                    // chain split-K: cluster size (the CTAs of one row tile), else 1
  // operands final before the predecessor completes (the square GEMM after k_alpha): the
  // producer and MMA warps run the mainloop without waiting; only the epilogue waits (for
  // alpha).  Tiles are then skipped by stop_iter < k (final for earlier iterations; a
  // matrix stopping at k, decided concurrently, is computed by every role alike)
  int early;
  int max_ctas;                  // > 0: persistent grid capped (row-block Gram: SMs left to NCCL)
  int probs_per_matrix;          // chain: problems per matrix (sketch chunks, matrix-major order), else 0
  int chain_bn;                  // chain: rows of R per tile (256, or 128 for launches with few row tiles)
  // chain: the first tile code of CTA b (b < kFirstCodes) as a kernel parameter, so a CTA
  // that starts late needs no dependent load of the tile list before staging its R
  uint32_t first_code[kFirstCodes];
};

// The problem fields the tile epilogue needs, held in registers for the tile: read
// through `const GemmProblem&` they are reloaded from global memory after every store
// (the compiler cannot rule out aliasing).
struct EpiArgs {
  void* out;
  void* out_lo;
  float* gdiag;
  long long ldo;
  int M, N;
  void* out2;
  void* out2_lo;
};

template <int KIND_, bool SPLIT_, int BN_ = 0, bool CTA2_ = (BN_ == 0)>
struct GemmCfg {
  static constexpr int KIND = KIND_;
  static constexpr bool SPLIT = SPLIT_;
  // CTA pair (cta_group::2): a cluster of 2 CTAs computes a 256 x BN tile; each CTA
  // loads its 128 rows of A and half of B (BN/2 rows), holds 128 x BN of the
  // accumulator, and only the even CTA issues the MMAs.  Cuts the L2 -> SMEM operand
  // traffic per FLOP by a third versus 128 x BN single-CTA tiles.
  static constexpr bool CTA2 = CTA2_;
  static constexpr int CG = CTA2 ? 2 : 1;
  static constexpr int ESZ = KIND == 0 ? 2 : 4;
  static constexpr int BM = 128;                  // rows per CTA
  static constexpr int TILE_M = BM * CG;          // rows per (pair) tile
  static constexpr int BN = BN_ ? BN_ : (KIND == 0 ? 256 : 128);
  static constexpr int B_ROWS = BN / CG;          // B rows (along N) loaded per CTA
  static constexpr bool LOB = SPLIT;            // 3xTF32: B carries a lo plane too
  static constexpr int BK = 128 / ESZ;          // one 128-B swizzle row of K
  static constexpr int UK = 32 / ESZ;           // K per tcgen05.mma (32 bytes)
  static constexpr int A_BYTES = BM * BK * ESZ;
  static constexpr int B_BYTES = B_ROWS * BK * ESZ;
  static constexpr int STAGE_BYTES = (SPLIT ? 2 * A_BYTES : A_BYTES) + (LOB ? 2 * B_BYTES : B_BYTES);
  static constexpr int TB_BYTES = 8 * 32 * 33 * 4;   // tf32: per-epilogue-warp staging / transpose buffers
  // bf16: per epilogue warp two C blocks and two output blocks (32 x 32 bf16, TMA-swizzled)
  static constexpr int EPI_BYTES = KIND == 0 ? 8 * 4 * 2048 : TB_BYTES;
  static constexpr int STAGES_RAW =
      KIND == 0 ? (227 * 1024 - 2048 - EPI_BYTES) / STAGE_BYTES : (192 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int AE = 128 / ESZ;           // elements per 128-B atom along MN (MN-major)
  static constexpr int ATOM_BYTES = BK * 128;    // one MN-major atom column: BK rows of 128 B
  // MN-major: bf16 uses the 128-B swizzle (8-row K groups, SBO 1024); tf32 must use
  // the 128-B/32-B-atom swizzle (layout type 1, 4-row K groups, SBO 512).
  static constexpr uint32_t MN_LAYOUT = KIND == 0 ? 2u : 1u;
  static constexpr uint32_t MN_SBO = KIND == 0 ? 1024u : 512u;
  static constexpr uint32_t IDESC = idesc_make(KIND == 0 ? 1u : 2u, 0u, TILE_M, BN);
  static constexpr int EPI_WARPS = 8;   // two per TMEM lane quarter, each owning half the columns
  static constexpr int NCH = BN / 32;   // 32-column chunks per tile
  static constexpr int CH_PER = NCH >= 2 ? NCH / 2 : 1;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 1024 /*barriers, scratch*/ + EPI_BYTES;
  // warpgroup 0: TMA producer (warp 0), MMA issuer (warp 1), two idle warps — shrunk to
  // REG_LO registers; warpgroups 1-2: the epilogue warps 4..11, grown to REG_HI
  // (setmaxnreg: the epilogue keeps accumulator, C and output rows in registers)
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  static constexpr int REG_LO = 72, REG_HI = 216;   // 128 x 72 + 256 x 216 = 384 x 168 (the launch allocation)
  // k-blocks per TMEM accumulation chunk: tf32 partials are promoted to fp32
  // registers every k-block (3xTF32, K = 32: 12 MMAs per chunk) or every 4
  // (1xTF32); bf16 keeps one accumulator per tile (products exact, 2^-9 output).
  static constexpr int PROMO_KB = KIND == 0 ? (1 << 30) : (SPLIT ? 1 : 4);
  static constexpr int TMEM_ALLOC = TMEM_COLS < 32 ? 32 : TMEM_COLS;
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

// bf16 C row segment as raw 16-byte words (converted only when used, so the
// load latency overlaps the previous chunk's work)
__device__ __forceinline__ void load_raw_bf16(const void* base, long long ld, int i, int j0, int N, uint4 (&w)[4]) {
  const __nv_bfloat16* p = static_cast<const __nv_bfloat16*>(base) + (long long)i * ld + j0;
  if (j0 + 32 <= N) {
#pragma unroll
    for (int u = 0; u < 4; ++u) w[u] = __ldg(reinterpret_cast<const uint4*>(p) + u);
  } else {
    __nv_bfloat16 t[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) t[u] = (j0 + u < N) ? p[u] : __float2bfloat16_rn(0.f);
#pragma unroll
    for (int u = 0; u < 4; ++u) w[u] = reinterpret_cast<const uint4*>(t)[u];
  }
}
__device__ __forceinline__ void decode_bf16(const uint4 (&w)[4], float (&c)[32]) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w[u]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(h[e]);
      c[u * 8 + 2 * e] = f.x;
      c[u * 8 + 2 * e + 1] = f.y;
    }
  }
}

// ---- coalesced 32 x 32 bf16 block moves for an epilogue warp (one row per lane in
// registers).  A lane-per-row access makes every warp instruction touch 32 lines with
// 16-B pieces; restaging through the warp's smem buffer (32 rows x 64 B, 16-B chunks
// XOR-swizzled: conflict-free both ways) lets each instruction move 8 rows x 64 B.
__device__ __forceinline__ uint32_t stg_off(int row, int ch) { return (uint32_t)(row * 64 + ((ch ^ ((row >> 1) & 3)) << 4)); }

// this lane's row v[32] as bf16 into the staging block (row `lane`)
__device__ __forceinline__ void stage_row_bf16(const float (&v)[32], uint8_t* stg, int lane) {
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) {
    uint4 w;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
    for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[ch * 8 + 2 * e], v[ch * 8 + 2 * e + 1]);
    *reinterpret_cast<uint4*>(stg + stg_off(lane, ch)) = w;
  }
}
// staged block -> rows [r0, r0 + 32) x cols [c0, c0 + 32) of out, 8 rows x 64 B per instruction
__device__ __forceinline__ void store_staged_bf16(void* out, long long ld, long long r0, long long c0,
                                                  const uint8_t* stg, int lane) {
  __nv_bfloat16* o = static_cast<__nv_bfloat16*>(out);
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int row = u * 8 + (lane >> 2), ch = lane & 3;
    *reinterpret_cast<uint4*>(o + (r0 + row) * ld + c0 + ch * 8) = *reinterpret_cast<const uint4*>(stg + stg_off(row, ch));
  }
}
// dst = src^T for a staged 32 x 32 bf16 block: the 16 8x8 tiles are read transposed
// (ldmatrix .trans) and written to the mirrored tile positions (stmatrix)
__device__ __forceinline__ void transpose_staged_bf16(const uint8_t* src, uint8_t* dst, int lane) {
  const int i = lane >> 3, j = lane & 7;   // this lane addresses row j of tile i of the x4 group
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    uint32_t r0, r1, r2, r3;
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(smem_u32(src + stg_off(8 * a + j, i))));
    // tile (a, b = i) transposed goes to tile position (b, a)
    asm volatile("stmatrix.sync.aligned.m8n8.x4.shared.b16 [%0], {%1, %2, %3, %4};" ::"r"(
                     smem_u32(dst + stg_off(8 * i + j, a))),
                 "r"(r0), "r"(r1), "r"(r2), "r"(r3)
                 : "memory");
  }
}
// this lane's row v[32] -> rows [r0, r0 + 32) x cols [c0, c0 + 32) of out (block fully in bounds)
__device__ __forceinline__ void warp_store_bf16_block(void* out, long long ld, long long r0, long long c0,
                                                      const float (&v)[32], uint8_t* stg, int lane) {
  stage_row_bf16(v, stg, lane);
  __syncwarp();
  store_staged_bf16(out, ld, r0, c0, stg, lane);
  __syncwarp();
}
// coalesced global read of a 32 x 32 bf16 block (registers, in flight) ...
__device__ __forceinline__ void warp_load_bf16_block(const void* base, long long ld, long long r0, long long c0,
                                                     uint4 (&g)[4], int lane) {
  const __nv_bfloat16* p = static_cast<const __nv_bfloat16*>(base);
#pragma unroll
  for (int u = 0; u < 4; ++u)
    g[u] = __ldg(reinterpret_cast<const uint4*>(p + (r0 + u * 8 + (lane >> 2)) * ld + c0 + (lane & 3) * 8));
}
// ... then redistributed so that this lane holds its row as 32 floats
__device__ __forceinline__ void warp_rows_from_block(const uint4 (&g)[4], uint8_t* stg, int lane, float (&c)[32]) {
#pragma unroll
  for (int u = 0; u < 4; ++u) *reinterpret_cast<uint4*>(stg + stg_off(u * 8 + (lane >> 2), lane & 3)) = g[u];
  __syncwarp();
  uint4 w[4];
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) w[ch] = *reinterpret_cast<const uint4*>(stg + stg_off(lane, ch));
  __syncwarp();
  decode_bf16(w, c);
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

// fp32 / 3xTF32 32 x 32 blocks moved with coalesced 16-B accesses (each instruction covers
// 4 rows x 128 B) through the warp's 32 x 33 staging tile tb (conflict-free both ways),
// instead of one row per lane (32 rows, i.e. 32 lines, per instruction).
// Load: lane l receives row r0 + l of C (+ C_lo) as 32 floats.
template <bool SPLIT>
__device__ __forceinline__ void warp_load_f32_block(const void* base, const void* base_lo, long long ld, int r0,
                                                    int c0, float (&c)[32], float* tb, int lane) {
  const int rr = lane >> 3, c4 = (lane & 7) * 4;
  float4 h[8], l[8];
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const long long off = (long long)(r0 + it * 4 + rr) * ld + c0 + c4;
    h[it] = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(base) + off));
    if constexpr (SPLIT) l[it] = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(base_lo) + off));
  }
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    float* t = tb + (it * 4 + rr) * 33 + c4;
    if constexpr (SPLIT) {
      t[0] = h[it].x + l[it].x; t[1] = h[it].y + l[it].y; t[2] = h[it].z + l[it].z; t[3] = h[it].w + l[it].w;
    } else {
      t[0] = h[it].x; t[1] = h[it].y; t[2] = h[it].z; t[3] = h[it].w;
    }
  }
  __syncwarp();
#pragma unroll
  for (int u = 0; u < 32; ++u) c[u] = tb[lane * 33 + u];
  __syncwarp();
}
// Store the staged tile (tb[row][col] = value at (r0 + row, c0 + col)), or its transpose
// when TR (value at (r0 + row, c0 + col) = tb[col][row]); SPLIT: tf32 hi + fp32 remainder.
template <bool SPLIT, bool TR>
__device__ __forceinline__ void warp_store_f32_staged(void* out, void* out_lo, long long ld, int r0, int c0,
                                                      const float* tb, int lane) {
  const int rr = lane >> 3, c4 = (lane & 7) * 4;
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int row = it * 4 + rr;
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = TR ? tb[(c4 + e) * 33 + row] : tb[row * 33 + c4 + e];
    const long long off = (long long)(r0 + row) * ld + c0 + c4;
    if constexpr (SPLIT) {
      const float4 hi = make_float4(tf32_trunc(v[0]), tf32_trunc(v[1]), tf32_trunc(v[2]), tf32_trunc(v[3]));
      *reinterpret_cast<float4*>(static_cast<float*>(out) + off) = hi;
      *reinterpret_cast<float4*>(static_cast<float*>(out_lo) + off) =
          make_float4(v[0] - hi.x, v[1] - hi.y, v[2] - hi.z, v[3] - hi.w);
    } else {
      *reinterpret_cast<float4*>(static_cast<float*>(out) + off) = make_float4(v[0], v[1], v[2], v[3]);
    }
  }
}

// Row-block partial Gram (EPI_GRAM32): D in plain fp32 whatever the compute dtype (the
// partial Grams are summed across ranks), upper triangle only, packed by 256-row panels:
// panel t holds rows [256t, 256t + 256) x columns [256t, N), row-major with leading
// dimension N - 256t, at float offset 256 (t N - 128 t (t - 1)) (= prism_rowblock_layout).
__device__ __forceinline__ long long gram_panel_off(long long t, long long N) { return 256 * (t * N - 128 * t * (t - 1)); }
__device__ __forceinline__ void epi_gram32(const EpiArgs& P, int i0, int lane, int j0, const float (&d)[32],
                                           float* tb) {
  if (i0 >= P.M || j0 >= P.N || j0 + 31 < i0) return;   // warp-uniform: strictly lower blocks are not stored
  const long long t = i0 >> 8, w = P.N - 256 * t;
  float* base = static_cast<float*>(P.out) + gram_panel_off(t, P.N);
  const int r0 = i0 - 256 * (int)t, c0 = j0 - 256 * (int)t;
  if (j0 >= i0 + 32 && j0 + 32 <= P.N && i0 + 32 <= P.M && (w & 3) == 0) {
    // whole block above the diagonal: staged, 16-B coalesced stores (4 rows x 128 B per instruction)
#pragma unroll
    for (int u = 0; u < 32; ++u) tb[lane * 33 + u] = d[u];
    __syncwarp();
    warp_store_f32_staged<false, false>(base, nullptr, w, r0, c0, tb, lane);
    __syncwarp();
    return;
  }
  const int i = i0 + lane;
  if (i < P.M) {
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const int j = j0 + u;
      if (j >= i && j < P.N) base[(long long)(r0 + lane) * w + c0 + u] = d[u];
    }
  }
}

// Row-block APPLY2, fp32 / 3xTF32 kernels: out = coefC C + coefA D and out2 = D.
template <class Cfg>
__device__ __forceinline__ void epi_apply2(const EpiArgs& P, int i0, int lane, int j0, float coefA, float coefC,
                                           const float (&d)[32], const float (&c)[32], float* tb) {
  if (i0 >= P.M || j0 >= P.N) return;
  float v[32];
#pragma unroll
  for (int u = 0; u < 32; ++u) v[u] = coefC * c[u] + coefA * d[u];
  const int i = i0 + lane;
  if (j0 + 32 <= P.N && i0 + 32 <= P.M && (P.ldo & 3) == 0) {
#pragma unroll
    for (int u = 0; u < 32; ++u) tb[lane * 33 + u] = v[u];
    __syncwarp();
    warp_store_f32_staged<Cfg::SPLIT, false>(P.out, P.out_lo, P.ldo, i0, j0, tb, lane);
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 32; ++u) tb[lane * 33 + u] = d[u];
    __syncwarp();
    warp_store_f32_staged<Cfg::SPLIT, false>(P.out2, P.out2_lo, P.ldo, i0, j0, tb, lane);
    __syncwarp();
    return;
  }
  if (i >= P.M) return;
  const long long off = (long long)i * P.ldo + j0;
  for (int u = 0; u < 32; ++u)
    if (j0 + u < P.N) {
      store_elem<Cfg::KIND, Cfg::SPLIT>(P.out, P.out_lo, off + u, v[u]);
      store_elem<Cfg::KIND, Cfg::SPLIT>(P.out2, P.out2_lo, off + u, d[u]);
    }
}

// Fused epilogue for one 32 x 32 block: rows i0 + lane (one row per lane of an
// epilogue warp), columns [j0, j0 + 32), given the fp32 accumulators d[] of
// D = A·B and (POLY / APPLY) the prefetched row segment c[] of C.  Called by all
// 32 lanes of the warp (warp-collective: the symmetric mirror goes through a
// per-warp 32 x 33 shared-memory transpose tb so that both the direct and the
// mirrored stores are 16-byte vectors).
template <class Cfg>
__device__ __forceinline__ void epi_segment(const EpiArgs& P, int mode, bool sym, int i0, int lane, int j0,
                                            float coefA, float coefC, const float (&d)[32], const float (&c)[32],
                                            float* tb, float& sumsq) {
  if (mode == EPI_GRAM32) { epi_gram32(P, i0, lane, j0, d, tb); return; }
  if (mode == EPI_APPLY2) { epi_apply2<Cfg>(P, i0, lane, j0, coefA, coefC, d, c, tb); return; }
  if (i0 >= P.M || j0 >= P.N) return;            // warp-uniform
  if (sym && j0 + 31 < i0) return;               // block strictly below the diagonal
  const int i = i0 + lane;
  const bool row_ok = i < P.M;
  float v[32];
  if (mode == EPI_POLY || mode == EPI_APPLY) {
#pragma unroll
    for (int u = 0; u < 32; ++u) v[u] = coefC * c[u] + coefA * d[u];
  } else if (mode == EPI_RESID) {
#pragma unroll
    for (int u = 0; u < 32; ++u) v[u] = ((j0 + u == i) ? 1.f : 0.f) - coefA * d[u];
    if (P.gdiag && row_ok && i >= j0 && i < j0 + 32) {
#pragma unroll
      for (int u = 0; u < 32; ++u)
        if (j0 + u == i) P.gdiag[i] = coefA * d[u];
    }
  } else {
#pragma unroll
    for (int u = 0; u < 32; ++u) v[u] = d[u];
  }
  const long long off = (long long)i * P.ldo + j0;
  const bool full_n = j0 + 32 <= P.N;
  const bool full_blk = full_n && i0 + 32 <= P.M;   // warp-uniform
  uint8_t* stg = reinterpret_cast<uint8_t*>(tb);
  if (Cfg::KIND != 0 && full_blk && ((P.ldo & 3) == 0)) {
    // fp32 / 3xTF32 whole block: staged once, stored coalesced (the mirror from the same tile)
    const bool diag = sym && j0 < i0 + 32;
    if (mode == EPI_RESID) {
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        if (!sym) sumsq = fmaf(v[u], v[u], sumsq);
        else if (!diag || u > lane) sumsq = fmaf(2.f * v[u], v[u], sumsq);
        else if (u == lane) sumsq = fmaf(v[u], v[u], sumsq);
      }
    }
#pragma unroll
    for (int u = 0; u < 32; ++u) tb[lane * 33 + u] = v[u];
    __syncwarp();
    if (diag) {
      // own values on / above the diagonal, transposed ones below (exact symmetry)
      float w[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) w[u] = tb[u * 33 + lane];
      __syncwarp();
#pragma unroll
      for (int u = 0; u < 32; ++u)
        if (u < lane) tb[lane * 33 + u] = w[u];
      __syncwarp();
    }
    warp_store_f32_staged<Cfg::SPLIT, false>(P.out, P.out_lo, P.ldo, i0, j0, tb, lane);
    if (sym && !diag) warp_store_f32_staged<Cfg::SPLIT, true>(P.out, P.out_lo, P.ldo, j0, i0, tb, lane);
    __syncwarp();
    return;
  }
  if (!sym) {
    if (Cfg::KIND == 0 && full_blk) {
      warp_store_bf16_block(P.out, P.ldo, i0, j0, v, stg, lane);
      if (mode == EPI_RESID) {
#pragma unroll
        for (int u = 0; u < 32; ++u) sumsq = fmaf(v[u], v[u], sumsq);
      }
    } else if (row_ok) {
      if (full_n) {
        store_row32<Cfg::KIND, Cfg::SPLIT>(P.out, P.out_lo, off, v);
        if (mode == EPI_RESID) {
#pragma unroll
          for (int u = 0; u < 32; ++u) sumsq = fmaf(v[u], v[u], sumsq);
        }
      } else {
        for (int u = 0; u < 32; ++u)
          if (j0 + u < P.N) {
            store_elem<Cfg::KIND, Cfg::SPLIT>(P.out, P.out_lo, off + u, v[u]);
            if (mode == EPI_RESID) sumsq = fmaf(v[u], v[u], sumsq);
          }
      }
    }
    return;
  }
  // symmetric: upper triangle (j >= i) written directly, (j > i) mirrored to (j, i)
  const bool diag = j0 < i0 + 32;                // 32-aligned blocks: the diagonal block (j0 == i0)
  if (Cfg::KIND == 0 && full_blk) {
    // bf16 rows staged once; the mirror is the staged block transposed by 8x8 tiles
    // (ldmatrix.trans / stmatrix) — same bf16 values, exact symmetry
    uint8_t* stg2 = stg + 2048;
    stage_row_bf16(v, stg, lane);
    __syncwarp();
    if (!diag) store_staged_bf16(P.out, P.ldo, i0, j0, stg, lane);
    transpose_staged_bf16(stg, stg2, lane);
    __syncwarp();
    if (mode == EPI_RESID) {
#pragma unroll
      for (int u = 0; u < 32; ++u)
        if (!diag || u >= lane) sumsq = fmaf((diag && u == lane) ? v[u] : 2.f * v[u], v[u], sumsq);
    }
    if (!diag) {
      store_staged_bf16(P.out, P.ldo, j0, i0, stg2, lane);
    } else {
      // diagonal block: row lane = own values on/above the diagonal, transposed below
      uint4 wr[4];
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) wr[ch] = *reinterpret_cast<const uint4*>(stg2 + stg_off(lane, ch));
      float w[32];
      decode_bf16(wr, w);
#pragma unroll
      for (int u = 0; u < 32; ++u) w[u] = u >= lane ? v[u] : w[u];
      __syncwarp();
      stage_row_bf16(w, stg, lane);
      __syncwarp();
      store_staged_bf16(P.out, P.ldo, i0, j0, stg, lane);
    }
    __syncwarp();
    return;
  }
  // transpose through shared memory: lane l obtains column j0 + l, rows i0 .. i0+31
#pragma unroll
  for (int u = 0; u < 32; ++u) tb[lane * 33 + u] = v[u];
  __syncwarp();
  float w[32];
#pragma unroll
  for (int u = 0; u < 32; ++u) w[u] = tb[u * 33 + lane];
  __syncwarp();
  if (diag) {
    // whole symmetric block at once: own values on and above the diagonal, transposed
    // ones below (exact symmetry), written as full rows — no partial-sector stores
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      if (mode == EPI_RESID && u >= lane && j0 + u < P.N && row_ok) sumsq = fmaf(u > lane ? 2.f * v[u] : v[u], v[u], sumsq);
      v[u] = u >= lane ? v[u] : w[u];
    }
    if (Cfg::KIND == 0 && full_blk) {
      warp_store_bf16_block(P.out, P.ldo, i0, j0, v, stg, lane);
    } else if (row_ok) {
      if (full_n) {
        store_row32<Cfg::KIND, Cfg::SPLIT>(P.out, P.out_lo, off, v);
      } else {
        for (int u = 0; u < 32; ++u)
          if (j0 + u < P.N) store_elem<Cfg::KIND, Cfg::SPLIT>(P.out, P.out_lo, off + u, v[u]);
      }
    }
    return;
  }
  if (Cfg::KIND == 0 && full_blk) {
    warp_store_bf16_block(P.out, P.ldo, i0, j0, v, stg, lane);
  } else if (row_ok) {
    if (full_n) {
      store_row32<Cfg::KIND, Cfg::SPLIT>(P.out, P.out_lo, off, v);
    } else {
      for (int u = 0; u < 32; ++u)
        if (j0 + u < P.N) store_elem<Cfg::KIND, Cfg::SPLIT>(P.out, P.out_lo, off + u, v[u]);
    }
  }
  if (mode == EPI_RESID && row_ok) {
#pragma unroll
    for (int u = 0; u < 32; ++u)
      if (j0 + u < P.N) sumsq = fmaf(2.f * v[u], v[u], sumsq);
  }
  // mirror: lane l writes row j0 + l, columns i0 .. i0+31 (all below the diagonal)
  const int j = j0 + lane;
  if (Cfg::KIND == 0 && full_blk) {
    warp_store_bf16_block(P.out, P.ldo, j0, i0, w, stg, lane);
  } else if (j < P.N) {
    const long long moff = (long long)j * P.ldo + i0;
    if (i0 + 32 <= P.M) {
      store_row32<Cfg::KIND, Cfg::SPLIT>(P.out, P.out_lo, moff, w);
    } else {
#pragma unroll
      for (int u = 0; u < 32; ++u)
        if (i0 + u < P.M) store_elem<Cfg::KIND, Cfg::SPLIT>(P.out, P.out_lo, moff + u, w[u]);
    }
  }
}

// bf16 fused epilogue for one 32 x 32 block through TMA: rows i0 + lane (one row per
// lane), columns [j0, j0 + 32), accumulators d[] of D = A·B and (POLY / APPLY) the C
// row c[].  The block is staged as bf16 rows in ob (64-B swizzle = the TMA box layout)
// and stored by lane 0 (TMA clips rows >= M / columns >= N).  Symmetric outputs: the
// upper triangle of blocks is computed; an off-diagonal block is also stored transposed
// (ldmatrix.trans / stmatrix into ob2), a diagonal block is stored whole (own values on /
// above the diagonal, transposed ones below).  Warp-collective; ob / ob2 must be free.
template <class Cfg>
__device__ __forceinline__ void epi_block_tma(const EpiArgs& P, const CUtensorMap* tmO, int mode, bool sym, int i0,
                                              int lane, int j0, float coefA, float coefC, const float (&d)[32],
                                              const float (&c)[32], uint8_t* ob, uint8_t* ob2, float& sumsq) {
  if (sym && j0 + 31 < i0) return;               // block strictly below the diagonal
  const int i = i0 + lane;
  const bool row_ok = i < P.M;
  float v[32];
  if (mode == EPI_POLY || mode == EPI_APPLY) {
#pragma unroll
    for (int u = 0; u < 32; ++u) v[u] = coefC * c[u] + coefA * d[u];
  } else if (mode == EPI_RESID) {
    if (j0 == i0) {   // warp-uniform: the 32 x 32 block holding the diagonal (square R)
#pragma unroll
      for (int u = 0; u < 32; ++u) v[u] = (u == lane ? 1.f : 0.f) - coefA * d[u];
      if (P.gdiag && row_ok) {
        float g = 0.f;   // this lane's diagonal entry, by selects (no divergent branch per column)
#pragma unroll
        for (int u = 0; u < 32; ++u) g = u == lane ? d[u] : g;
        P.gdiag[i] = coefA * g;
      }
    } else {
#pragma unroll
      for (int u = 0; u < 32; ++u) v[u] = -coefA * d[u];
    }
  } else {
#pragma unroll
    for (int u = 0; u < 32; ++u) v[u] = d[u];
  }
  const bool diag = sym && j0 < i0 + 32;         // 32-aligned: the diagonal block (j0 == i0)
  if (mode == EPI_RESID && row_ok) {
    // ||R||_F^2 from this block: an off-diagonal block of a symmetric R stands for itself
    // and its mirror (weight 2); a diagonal block is summed whole (both of its triangles:
    // the computed values, equal to the stored mirror up to the rounding of the products).
    // No lane-dependent test per element: the first form's branches diverged on every
    // element and its select form still cost ~1 us per 32 x 32 block (scripts/trace_gemm.py)
    float ss = 0.f;
    if (j0 + 32 <= P.N) {
#pragma unroll
      for (int u = 0; u < 32; ++u) ss = fmaf(v[u], v[u], ss);
    } else {
#pragma unroll
      for (int u = 0; u < 32; ++u) ss = j0 + u < P.N ? fmaf(v[u], v[u], ss) : ss;
    }
    sumsq += (sym && !diag) ? 2.f * ss : ss;
  }
  stage_row_bf16(v, ob, lane);
  __syncwarp();
  if (!sym) {
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(tmO, ob, j0, i0);
      bulk_commit();
    }
    return;
  }
  transpose_staged_bf16(ob, ob2, lane);          // ob2 = block^T (same bf16 values)
  __syncwarp();
  if (diag) {
    uint4 wr[4];
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) wr[ch] = *reinterpret_cast<const uint4*>(ob2 + stg_off(lane, ch));
    float w[32];
    decode_bf16(wr, w);
#pragma unroll
    for (int u = 0; u < 32; ++u) w[u] = u >= lane ? v[u] : w[u];
    __syncwarp();
    stage_row_bf16(w, ob, lane);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(tmO, ob, j0, i0);
      bulk_commit();
    }
    return;
  }
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(tmO, ob, j0, i0);    // the block
    tma_store_2d(tmO, ob2, i0, j0);   // its mirror
    bulk_commit();
  }
}

// Sketch-chain epilogue (thin GEMM, BN = 32): d[c] + d[w + c] = (R W)[i][c].
template <class Cfg>
__device__ __forceinline__ void store_w(const GemmProblem& P, int c, int wn, int i, float v) {
  // next-pass B operand, hi row c and lo row wn + c (K-major: [2w'][ldS])
  if constexpr (Cfg::KIND == 0) {
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    static_cast<__nv_bfloat16*>(P.Wn)[(long long)c * P.ldS + i] = h;
    static_cast<__nv_bfloat16*>(P.Wn)[(long long)(wn + c) * P.ldS + i] = __float2bfloat16_rn(v - __bfloat162float(h));
  } else {
    const float h = tf32_trunc(v);
    static_cast<float*>(P.Wn)[(long long)c * P.ldS + i] = h;
    static_cast<float*>(P.Wn)[(long long)(wn + c) * P.ldS + i] = v - h;
  }
}

// Everything the per-row chain epilogue reads besides the accumulator, loaded by
// chain_prefetch before the accumulator is ready (the loads then overlap the MMAs /
// the partial exchange; the values are consumed by epi_chain).  P is a local copy:
// read through a reference every field would be reloaded after each store.
struct ChainPre {
  GemmProblem P;
  float rii, gii;     // pass 1 (and CHC_P3): R_ii and G_ii
  float v[32];        // pass 1: S[c][i] (c < 8); last pass: kept columns kv[slot][c]
                      // (CHC_P3: kv[0] = U, v[8 + c] / v[16 + c] = the input's hi / lo W[c][i])
};

template <class Cfg, int PASS>
__device__ __forceinline__ void chain_prefetch(const GemmProblem& Pin, int i, int h, ChainPre& pre) {
  pre.P = Pin;
  const GemmProblem& P = pre.P;
  const int p = P.p;
  const int c0 = h == 1 ? (p + 1) / 2 : 0;
  const int c1 = h == 0 ? (p + 1) / 2 : p;
  const bool valid = i < P.M;
#pragma unroll
  for (int u = 0; u < 32; ++u) pre.v[u] = 0.f;
  pre.rii = pre.gii = 0.f;
  if (!valid) return;
  if constexpr (PASS == CH2_P1 || PASS == CH1_P1 || PASS == CHC_P3) {
    if constexpr (Cfg::KIND == 0) pre.rii = __bfloat162float(static_cast<const __nv_bfloat16*>(P.Rg)[(long long)i * P.ldr + i]);
    else pre.rii = static_cast<const float*>(P.Rg)[(long long)i * P.ldr + i] +
                   (P.Rg_lo ? static_cast<const float*>(P.Rg_lo)[(long long)i * P.ldr + i] : 0.f);
    pre.gii = P.gdiag[i];
  }
  if constexpr (PASS == CH2_P1 || PASS == CH1_P1) {
#pragma unroll
    for (int c = 0; c < 8; ++c) pre.v[c] = (c >= c0 && c < c1) ? __ldg(P.S + (long long)c * P.ldS + i) : 0.f;
  } else if constexpr (chain_is_last(PASS)) {
    const int ns = chain_last_slots(PASS);
    const long long M = P.M;
    if (p == 8 && c0 == 0 && c1 == 8) {   // full chunk: two 16-B loads per kept row
#pragma unroll
      for (int sl = 0; sl < 4; ++sl) {
        if (sl < ns) {
          const float4* q = reinterpret_cast<const float4*>(P.keep + ((long long)sl * M + i) * 8);
          const float4 a = __ldcg(q), b = __ldcg(q + 1);
          pre.v[sl * 8 + 0] = a.x; pre.v[sl * 8 + 1] = a.y; pre.v[sl * 8 + 2] = a.z; pre.v[sl * 8 + 3] = a.w;
          pre.v[sl * 8 + 4] = b.x; pre.v[sl * 8 + 5] = b.y; pre.v[sl * 8 + 6] = b.z; pre.v[sl * 8 + 7] = b.w;
        }
      }
    } else {
#pragma unroll
      for (int sl = 0; sl < 4; ++sl)
#pragma unroll
        for (int c = 0; c < 8; ++c)
          pre.v[sl * 8 + c] = (sl < ns && c >= c0 && c < c1) ? __ldcg(P.keep + ((long long)sl * M + i) * p + c) : 0.f;
    }
    if constexpr (PASS == CHC_P3) {   // the hi / lo input rows the MMA multiplied (written by CHC_P2)
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c < c0 || c >= c1 || c >= p) continue;
        if constexpr (Cfg::KIND == 0) {
          const __nv_bfloat16* w = static_cast<const __nv_bfloat16*>(P.Wi);
          pre.v[8 + c] = __bfloat162float(w[(long long)c * P.ldS + i]);
          pre.v[16 + c] = __bfloat162float(w[(long long)(p + c) * P.ldS + i]);
        } else {
          const float* w = static_cast<const float*>(P.Wi);
          pre.v[8 + c] = __ldcg(w + (long long)c * P.ldS + i);
          pre.v[16 + c] = __ldcg(w + (long long)(p + c) * P.ldS + i);
        }
      }
    }
  }
}

// Kept chain columns of row i: p consecutive floats ([slot][M][p]); a full chunk (p = 8,
// 32-B aligned rows) as two 16-B stores — eight scalar stores per row made each warp
// instruction touch 32 sectors, and the row epilogue of a pass took up to 2.8 us
__device__ __forceinline__ void keep_row(float* dst, const float (&v)[8], int p) {
  if (p == 8) {
    float4* d4 = reinterpret_cast<float4*>(dst);
    d4[0] = make_float4(v[0], v[1], v[2], v[3]);
    d4[1] = make_float4(v[4], v[5], v[6], v[7]);
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c < p) dst[c] = v[c];
  }
}

template <class Cfg, int PASS>   // one pass code per launch: only its epilogue is compiled in
__device__ __forceinline__ void epi_chain(const ChainPre& pre, int i, int grp, const float* col, int cs, int lane,
                                          int h) {
  const GemmProblem& P = pre.P;
  // Row i of the pass output: D[c] = col[c * cs] (this thread's column of the staged
  // accumulator in smem).  The two warps sharing a TMEM lane quarter may split the p
  // sketch rows c (h = 0: c < p/2, h = 1: the rest; h = 2: all).
  const int p = P.p;
  const int w = P.N / 2;          // columns of this pass's output
  const bool valid = i < P.M;
  const int c0 = h == 1 ? (p + 1) / 2 : 0;       // h = 2: one thread per row, every c
  const int c1 = h == 0 ? (p + 1) / 2 : p;
  constexpr int NG = chain_ng(PASS);
  double g[NG];
#pragma unroll
  for (int j = 0; j < NG; ++j) g[j] = 0.0;
  // o[c] = D[c] + D[w + c] (hi + lo halves of the pass output), op[c] = o[p + c]
  float o[8], op[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    o[c] = (c < w) ? col[c * cs] + col[(w + c) * cs] : 0.f;
    op[c] = (p + c < w) ? col[(p + c) * cs] + col[(w + p + c) * cs] : 0.f;
  }
  float* __restrict__ keep = P.keep;
  const long long M = P.M;
  constexpr int pass = PASS;
  if (valid) {
    if constexpr (pass == CH2_P1 || pass == CH1_P1) {
      const float rii = pre.rii, gii = pre.gii;
      const float* sc = pre.v;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c < c0 || c >= c1) continue;
        const float qv = gii * sc[c] - (o[c] - rii * sc[c]);   // Q = G S^T, G_ii exact (fp32 from the Gram)
        if constexpr (pass == CH2_P1) {
          store_w<Cfg>(P, c, 2 * p, i, o[c]);
          store_w<Cfg>(P, p + c, 2 * p, i, qv);
        } else {
          store_w<Cfg>(P, c, p, i, qv);
        }
      }
      if constexpr (pass == CH1_P1)
        if (h == 2) keep_row(keep + (long long)i * p, o, p);
    } else if constexpr (pass == CH2_P2) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c < c0 || c >= c1) continue;
        store_w<Cfg>(P, c, 2 * p, i, o[c]);
        store_w<Cfg>(P, p + c, 2 * p, i, op[c]);
      }
      keep_row(keep + (long long)i * p, o, p);
    } else if constexpr (pass == CH2_P3) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c < c0 || c >= c1) continue;
        store_w<Cfg>(P, c, p, i, op[c]);
      }
      keep_row(keep + (M + i) * p, o, p);
      keep_row(keep + (2 * M + i) * p, op, p);
    } else if constexpr (pass == CH2_P4 || pass == CH1_P2 || pass == CHI_K2) {
      constexpr long long slot = pass == CH2_P4 ? 3 : pass == CHI_K2 ? 2 : 1;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c < c0 || c >= c1) continue;
        store_w<Cfg>(P, c, p, i, o[c]);
      }
      keep_row(keep + (slot * M + i) * p, o, p);
    } else if constexpr (pass == CHC_P1 || pass == CHC_P2) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c < c0 || c >= c1) continue;
        store_w<Cfg>(P, c, p, i, o[c]);
      }
      if constexpr (pass == CHC_P2) keep_row(keep + (long long)i * p, o, p);
    } else if constexpr (pass == CHC_P3) {
      // V = U - U R = U G with G = I - R: R ~ I in the compute dtype loses G_ii, so the
      // diagonal term is replaced exactly as for Q in pass 1: V_i = G_ii U_i - (UR_i - R_ii U_i),
      // per hi / lo half (the products the MMA formed are exact in fp32, so subtracting them
      // leaves the off-diagonal sum)
      const float(&kv)[4][8] = *reinterpret_cast<const float(*)[4][8]>(pre.v);
      const float rii = pre.rii, gii = pre.gii;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c < c0 || c >= c1) continue;
        const float uh = pre.v[8 + c], ul = pre.v[16 + c];
        const float off = (col[c * cs] - uh * rii) + (col[(w + c) * cs] - ul * rii);
        const double u = (double)kv[0][c];
        const double v = (double)gii * ((double)uh + (double)ul) - (double)off;
        g[0] += u * u; g[1] += u * v; g[2] += v * v;
      }
    } else if constexpr (pass >= CHI_L1 && pass <= CHI_L4) {
      // inverse Newton: m(a) = ||sum_i a^i V_i||^2, V_0 = K1, V_i = -C(q,i) Z_i (Z_q = this
      // pass's output); <V_i, V_j> for i <= j in row-major upper-triangle order
      constexpr int q = pass - CHI_L1 + 1;
      const float(&kv)[4][8] = *reinterpret_cast<const float(*)[4][8]>(pre.v);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c < c0 || c >= c1) continue;
        double v[q + 1];
        v[0] = (double)kv[0][c];
#pragma unroll
        for (int j = 1; j < q; ++j) {
          const double bin = (q == 4 && j == 2) ? 6.0 : (double)q;   // C(q, j), 1 <= j < q <= 4
          v[j] = -bin * (double)kv[j][c];
        }
        v[q] = -(double)o[c];
        int idx = 0;
#pragma unroll
        for (int a = 0; a <= q; ++a)
#pragma unroll
          for (int b = a; b <= q; ++b) g[idx++] += v[a] * v[b];
      }
    } else {
      // CH2_P5 / CH1_P3: inner products <Va, Vb> (fp64 products of widened factors)
      const float(&kv)[4][8] = *reinterpret_cast<const float(*)[4][8]>(pre.v);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c < c0 || c >= c1) continue;
        double v0, v1, v2;
        if constexpr (pass == CH2_P5) {
          v0 = 0.25 * (3.0 * (double)kv[0][c] + (double)kv[1][c]);   // 1/4 (3 K2 + K3)
          v1 = -((double)kv[3][c] + 2.0 * (double)kv[2][c]);         // -(L3 + 2 L2)
          v2 = -(double)o[c];                                        // -L4
        } else {
          v0 = (double)kv[0][c];                                     // K1
          v1 = -2.0 * (double)kv[1][c];                              // -2 L1
          v2 = -(double)o[c];                                        // -L2
        }
        g[0] += v0 * v0; g[1] += v0 * v1; g[2] += v0 * v2;
        g[3] += v1 * v1; g[4] += v1 * v2; g[5] += v2 * v2;
      }
    }
  }
  if constexpr (chain_is_last(pass)) {
    // <Va, Vb> partial of this warp's 32 rows (one aligned row group): a fixed shuffle
    // tree, written per group — the grouping never depends on the launch (split factor,
    // batch), so k_alpha's fixed-order sum over groups is reproducible bit for bit
#pragma unroll
    for (int j = 0; j < NG; ++j) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) g[j] += __shfl_xor_sync(0xffffffffu, g[j], off);
    }
    if (lane == 0 && grp >= 0)
#pragma unroll
      for (int j = 0; j < NG; ++j) P.chain_part[grp * kChainG + j] = g[j];
  }
}


// TMA load of one operand tile (rows = BM or BN along MN, BK along K) into smem.
template <class Cfg>
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  if constexpr (Cfg::CTA2) tma_load_2d_pair(dst, map, bar, c0, c1);
  else tma_load_2d(dst, map, bar, c0, c1);
}

template <class Cfg>
__device__ __forceinline__ void load_operand(uint8_t* dst, const CUtensorMap* map, uint64_t* bar, int mn0, int k0,
                                             int rows, int mn_major) {
  if (mn_major) {
    for (int q = 0; q < rows / Cfg::AE; ++q)
      tma2d<Cfg>(dst + q * Cfg::ATOM_BYTES, map, bar, mn0 + q * Cfg::AE, k0);
  } else {
    tma2d<Cfg>(dst, map, bar, k0, mn0);
  }
}

// UMMA smem descriptor of the k-th K-step (UK elements) of an operand tile.
template <class Cfg>
__device__ __forceinline__ uint64_t operand_desc(uint32_t base, int k, int mn_major) {
  return mn_major ? sdesc_rt(base + k * Cfg::UK * 128, Cfg::ATOM_BYTES, Cfg::MN_SBO, Cfg::MN_LAYOUT)
                  : sdesc_rt(base + k * 32, 16, 1024, 2u);
}

// ---------------------------------------------------------------- the kernel

// Main-GEMM k-block timeline (prism_debug_trace_gemm): for launches whose first problem has
// epilogue mode g_trace_mode, each CTA's first tile records [0,64) producer issue (after
// its empty wait), [64,128) MMA full arrival, [128,192) MMA issue done, per k-block, and
// [192 + 4 j ..] tile j MMA start / end, epilogue start / end.  Kept compiled in: with the
// hooks removed the MMA-issue and producer loops schedule differently and the GEMMs ran
// 8-10 % slower on B200 (A/B on one box).
__device__ unsigned long long* g_gemm_trace2 = nullptr;
__device__ int g_trace_mode = -1;
constexpr int TRACE2_W = 376;

template <class Cfg>
__device__ __forceinline__ void gemm_body(const GemmLaunch& L) {
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
  uint64_t* cbar = tempty + 2;                 // [16] bf16 epilogue: C block landed (warp e, buffer b)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cbar + 16);
  float* red = reinterpret_cast<float*>(tmem_slot + 4);   // [8] epilogue reduction scratch
  float* tbuf = reinterpret_cast<float*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES + 1024);    // [8][32*33] (tf32)
  uint8_t* ebuf = smem + Cfg::STAGES * Cfg::STAGE_BYTES + 1024;   // bf16: [8 warps][C0, C1, O0, O1] 2 KB each

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = Cfg::CTA2 ? cluster_ctarank() : 0u;   // CTA within the pair
  const bool leader = rank == 0;
  const int cid = Cfg::CTA2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;   // tile-loop index / stride
  const int ncl = Cfg::CTA2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const GemmProblem* __restrict__ probs = L.probs;
  unsigned long long* trace2 = nullptr;
  if (g_gemm_trace2 && L.probs[0].mode == g_trace_mode) trace2 = g_gemm_trace2 + (size_t)blockIdx.x * TRACE2_W;

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], Cfg::CG * Cfg::EPI_WARPS);   // one arrival per epilogue warp (of both CTAs)
    }
    for (int x = 0; x < 16; ++x) mbar_init(&cbar[x], 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<Cfg::CG>(tmem_slot, Cfg::TMEM_ALLOC);
  tc_fence_before();
  if constexpr (Cfg::CTA2) cluster_sync_all();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // before the predecessor is done: the tile list, problem tables and tensor maps are
  // plan constants, so warm them; then wait for the predecessor's results
  if (threadIdx.x == 0 && cid < L.ntiles) {
    const uint32_t code = __ldg(L.tiles + cid);
    tma_prefetch(L.probs[code >> 20].tmA);
    tma_prefetch(L.probs[code >> 20].tmB);
    if (L.probs_odd) {
      tma_prefetch(L.probs_odd[code >> 20].tmA);
      tma_prefetch(L.probs_odd[code >> 20].tmB);
    }
  }
  // wait, then let dependents launch: a launch's predecessor-of-predecessor is then always
  // complete, which the chain kernel relies on for reads before its own wait (chaint.cuh).
  // An early launch's producer / MMA warps neither wait nor trigger (its epilogue does both).
  const bool early_role = L.early && warp < 4;
  if (!early_role) {
    griddep_wait();
    griddep_launch();
  }
  // device-side loop control (CUDA-graph WHILE body): uniform skip / parity select
  bool run = true;
  int kcur = 0;
  if (L.iter) {
    const int k = *L.iter;
    kcur = k;
    run = k >= L.iter_lo && k < L.iter_hi;
    if (L.probs_odd && (k & 1)) probs = L.probs_odd;
    if (L.probs_k0 && k == 0) probs = L.probs_k0;
  }
  // this iteration's tile list: the compacted one once it exists (read after the wait)
  const uint32_t* __restrict__ tiles = L.tiles;
  int ntiles = L.ntiles;
  if constexpr (Cfg::KIND == 0) {   // bf16 plans only (prism.cu)
    if (L.ctiles && !L.early && L.iter && kcur >= L.c_from) {
      tiles = L.ctiles;
      ntiles = *L.ccount;
    }
  }
  // tiles of stopped matrices are skipped (the same decision in every role)
  auto skip_tile = [&](int matrix) -> bool {
    if (!L.done) return false;
    const int* st = L.done + (size_t)matrix * L.done_stride;
    return st[0] != 0;   // the stop test ran in this iteration's residual stage (final here)
  };

  if (warp < 4) {
    setmaxnreg_dec<Cfg::REG_LO>();
    if (!run) {
      // this launch is outside its iteration window: nothing to do
    } else if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < ntiles; t += ncl) {
        const uint32_t code = tiles[t];
        const GemmProblem& P = probs[code >> 20];
        if (skip_tile(P.matrix)) continue;
        const int tm = (code >> 10) & 1023;
        const int tn = code & 511;
        const bool half = (code & kHalfTile) != 0;   // BN/2-column tile (last wave of an apply)
        const int kb_lo = 0, kb_hi = (P.K + Cfg::BK - 1) / Cfg::BK;
        // warm the TMA descriptor cache with this tile's maps (they live in global memory)
        tma_prefetch(P.tmA);
        tma_prefetch(P.tmB);
        if constexpr (Cfg::SPLIT) {
          tma_prefetch(P.tmA_lo);
          if constexpr (Cfg::LOB) tma_prefetch(P.tmB_lo);
        }
        const int am0 = tm * Cfg::TILE_M + (int)rank * Cfg::BM;      // this CTA's rows of A
        // this CTA's half of B (a half tile: the first B_ROWS/2 rows of the box are used)
        const int bn0 = half ? tn * (Cfg::BN / 2) + (int)rank * (Cfg::B_ROWS / 2) : tn * Cfg::BN + (int)rank * Cfg::B_ROWS;
        for (int kb = kb_lo; kb < kb_hi; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sA = stage_base + stage * Cfg::STAGE_BYTES;
          uint8_t* sB = sA + Cfg::A_BYTES;
          // the leader's full barrier counts the bytes of both CTAs of the pair
          if (leader) mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES * Cfg::CG);
          load_operand<Cfg>(sA, P.tmA, &full[stage], am0, kb * Cfg::BK, Cfg::BM, P.a_mn);
          load_operand<Cfg>(sB, P.tmB, &full[stage], bn0, kb * Cfg::BK, Cfg::B_ROWS, P.b_mn);
          if constexpr (Cfg::SPLIT) {
            uint8_t* sA2 = sB + Cfg::B_BYTES;
            uint8_t* sB2 = sA2 + Cfg::A_BYTES;
            load_operand<Cfg>(sA2, P.tmA_lo, &full[stage], am0, kb * Cfg::BK, Cfg::BM, P.a_mn);
            if constexpr (Cfg::LOB)
              load_operand<Cfg>(sB2, P.tmB_lo, &full[stage], bn0, kb * Cfg::BK, Cfg::B_ROWS, P.b_mn);
          }
          if (trace2 && t == cid && kb < 64) trace2[kb] = globaltimer_ns();
          if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA of the pair) =====================
    if (lane == 0 && leader) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int tcount = 0;
      for (int t = cid; t < ntiles; t += ncl) {
        const uint32_t code = tiles[t];
        const GemmProblem& P = probs[code >> 20];
        if (skip_tile(P.matrix)) continue;
        const bool half = (code & kHalfTile) != 0;
        const int kb_lo = 0, kb_hi = (P.K + Cfg::BK - 1) / Cfg::BK;
        // tf32: one TMEM accumulation chunk per PROMO_KB k-blocks, promoted to fp32
        // registers by the epilogue (bounds the truncation of the MMA accumulator add)
        for (int kb0 = kb_lo; kb0 < kb_hi; kb0 += Cfg::PROMO_KB) {
          const int kb1 = min(kb_hi, kb0 + Cfg::PROMO_KB);
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t dt = tmem_base + acc * Cfg::BN;
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(&full[stage], phase);
            if (trace2 && t == cid && kb < 64) trace2[64 + kb] = globaltimer_ns();
            if (trace2 && kb == kb_lo && tcount < 8) trace2[192 + 4 * tcount] = globaltimer_ns();
            tc_fence_after();
            const uint32_t aA = smem_u32(stage_base + stage * Cfg::STAGE_BYTES);
            const uint32_t aB = aA + Cfg::A_BYTES;
            uint32_t idesc = Cfg::IDESC | ((uint32_t)P.a_mn << 15) | ((uint32_t)P.b_mn << 16);
            if (half) idesc = (idesc & ~(0x3Fu << 17)) | ((uint32_t)(Cfg::BN / 2 / 8) << 17);   // N = BN/2
#pragma unroll
            for (int k = 0; k < Cfg::BK / Cfg::UK; ++k) {
              const uint64_t da = operand_desc<Cfg>(aA, k, P.a_mn);
              const uint64_t db = operand_desc<Cfg>(aB, k, P.b_mn);
              umma<Cfg::KIND, Cfg::CG>(dt, da, db, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
              if constexpr (Cfg::SPLIT) {
                const uint32_t aA2 = aB + Cfg::B_BYTES;
                const uint32_t aB2 = aA2 + Cfg::A_BYTES;
                const uint64_t da2 = operand_desc<Cfg>(aA2, k, P.a_mn);
                if constexpr (Cfg::LOB) umma<Cfg::KIND, Cfg::CG>(dt, da, operand_desc<Cfg>(aB2, k, P.b_mn), idesc, 1u);   // A_hi · B_lo
                umma<Cfg::KIND, Cfg::CG>(dt, da2, db, idesc, 1u);                                                          // A_lo · B_hi
              }
            }
            umma_commit<Cfg::CG>(&empty[stage]);     // smem slots (of both CTAs) free once these MMAs retire
            if (trace2 && t == cid && kb < 64) trace2[128 + kb] = globaltimer_ns();
            if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
          }
          umma_commit<Cfg::CG>(&tfull[acc]);          // accumulator (chunk) ready for both epilogues
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        if (trace2 && tcount < 8) trace2[192 + 4 * tcount + 1] = globaltimer_ns();
        ++tcount;
      }
    }
    }
  } else {
    setmaxnreg_inc<Cfg::REG_HI>();
    if (run) {
    // ===================== epilogue (warps 4..11) =====================
    const int q = warp & 3;                 // TMEM lane quarter this warp may access
    const int e = warp - 4;                 // 0..7
    const int h = e >> 2;                   // column half of the tile owned by this warp
    const int et = threadIdx.x - 128;       // 0..255
    const int c_begin0 = h * Cfg::CH_PER;
    const int c_end0 = min(Cfg::NCH, c_begin0 + Cfg::CH_PER);
    float* tb = tbuf + e * 32 * 33;
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t cph = 0;       // bf16: phase bits of this warp's two C-block barriers
    int etcount = 0;
    // accumulator release: one arrival per epilogue warp on the leader's tempty barrier
    auto release_acc = [&](uint64_t* bar) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (Cfg::CTA2 && !leader) mbar_arrive_cluster(bar, 0u);
        else mbar_arrive(bar);
      }
    };
    for (int t = cid; t < ntiles; t += ncl) {
      const uint32_t code = tiles[t];
      const GemmProblem& P = probs[code >> 20];
      if (skip_tile(P.matrix)) continue;
      const int tm = (code >> 10) & 1023;
      const int tn = code & 511;
      const bool half = (code & kHalfTile) != 0;
      const int mode = P.mode;
      const bool sym = P.sym != 0;
      const EpiArgs ea{P.out, P.out_lo, P.gdiag, P.ldo, P.M, P.N, P.out2, P.out2_lo};
      const void* const Cp = P.C;
      const long long ldc = P.ldc;
      const int i0 = tm * Cfg::TILE_M + (int)rank * Cfg::BM + q * 32;
      const int i = i0 + lane;                     // output row of this thread
      float coefA = 1.f, coefC = 1.f;
      // (RESID: coefA = 1, or 1/c^2 through `alpha` in a folded iteration 0: R = I - D/c^2)
      if (mode == EPI_POLY || mode == EPI_APPLY || mode == EPI_APPLY2 || mode == EPI_RESID) {
        const double al = (P.eA | P.eC) ? *P.alpha : 1.0;
        const double pa = P.eA == 0 ? 1.0 : P.eA == 1 ? al : P.eA == 2 ? al * al : al * al * al;
        const double pc = P.eC == 0 ? 1.0 : P.eC == 1 ? al : P.eC == 2 ? al * al : al * al * al;
        coefA = static_cast<float>((double)P.kA * pa + (double)P.lA);
        coefC = static_cast<float>((double)P.c1 * pc + (double)P.lC);
      }
      const bool needC = (mode == EPI_POLY || mode == EPI_APPLY || mode == EPI_APPLY2);
      float sumsq = 0.f;

      if constexpr (Cfg::KIND == 0) {
        // bf16: one TMEM accumulator per tile; per 32-column chunk: C block by TMA (two
        // chunks ahead, per-warp buffers C0/C1), next chunk's tcgen05.ld in flight
        // (ping-pong registers), output block staged and TMA-stored (O0/O1 alternate)
        uint8_t* wb = ebuf + e * 8192;
        // a half tile: BN/2 columns, half the chunks per warp
        const int c_begin = half ? h * (Cfg::CH_PER / 2) : c_begin0;
        const int c_end = half ? c_begin + Cfg::CH_PER / 2 : c_end0;
        const int jb = half ? tn * (Cfg::BN / 2) : tn * Cfg::BN;
        const CUtensorMap* tmC = P.tmC;
        const CUtensorMap* tmO = P.tmO;
        auto c_fetch = [&](int ch) {   // lane 0
          const int b = (ch - c_begin) & 1;
          mbar_arrive_expect_tx(&cbar[e * 2 + b], 2048);
          tma_load_2d(wb + b * 2048, tmC, &cbar[e * 2 + b], jb + ch * 32, i0);
        };
        if (needC && lane == 0) {
          c_fetch(c_begin);
          if (c_begin + 1 < c_end) c_fetch(c_begin + 1);
        }
        mbar_wait(&tfull[acc], acc_phase);
        if (trace2 && et == 0 && leader && etcount < 8) trace2[192 + 4 * etcount + 2] = globaltimer_ns();
        tc_fence_after();
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * Cfg::BN;
        uint32_t ra[32], rb[32];
        tmem_ld32(tbase + c_begin * 32, ra);
        tmem_ld_wait_dep(ra);
        auto step = [&](int ch, uint32_t (&rc)[32], uint32_t (&rn)[32]) {
          const int b = (ch - c_begin) & 1;
          const bool more = ch + 1 < c_end;
          if (more) tmem_ld32(tbase + (ch + 1) * 32, rn);
          float d[32], c[32];
          if (needC) {
            mbar_wait(&cbar[e * 2 + b], (cph >> b) & 1u);
            cph ^= 1u << b;
            uint4 w[4];
#pragma unroll
            for (int x = 0; x < 4; ++x) w[x] = *reinterpret_cast<const uint4*>(wb + b * 2048 + stg_off(lane, x));
            decode_bf16(w, c);
            __syncwarp();
            if (lane == 0 && ch + 2 < c_end) c_fetch(ch + 2);
          } else {
#pragma unroll
            for (int u = 0; u < 32; ++u) c[u] = 0.f;
          }
#pragma unroll
          for (int u = 0; u < 32; ++u) d[u] = __uint_as_float(rc[u]);
          // output buffers: non-symmetric blocks alternate O0 / O1 (the previous store may
          // still be reading the other one); symmetric blocks use both (block + mirror)
          if (mode == EPI_GRAM32) {
            // row-block partial Gram: plain fp32 stores (the warp's buffers as transpose scratch)
            epi_gram32(ea, i0, lane, jb + ch * 32, d, reinterpret_cast<float*>(wb));
          } else if (mode == EPI_APPLY2) {
            // row-block d = 2: X + Y/2 and Y = X R, both staged as bf16 blocks and TMA-stored
            if (lane == 0) bulk_wait_read<0>();
            __syncwarp();
            float v[32];
#pragma unroll
            for (int u = 0; u < 32; ++u) v[u] = coefC * c[u] + coefA * d[u];
            stage_row_bf16(v, wb + 4096, lane);
            stage_row_bf16(d, wb + 6144, lane);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(tmO, wb + 4096, jb + ch * 32, i0);
              tma_store_2d(P.tmO2, wb + 6144, jb + ch * 32, i0);
              bulk_commit();
            }
          } else {
            // output blocks: non-symmetric ones alternate O0 / O1; symmetric ones need a block
            // and its mirror — without C (the Gram) they alternate the pairs (C0, C1) and
            // (O0, O1), so a chunk never waits for the previous chunk's stores to drain
            const bool pairs2 = sym && !needC;
            if (lane == 0) {
              if (sym && !pairs2) bulk_wait_read<0>();
              else bulk_wait_read<1>();
            }
            __syncwarp();
            uint8_t* ob = pairs2 ? wb + b * 4096 : wb + 4096 + (sym ? 0 : b * 2048);
            epi_block_tma<Cfg>(ea, tmO, mode, sym, i0, lane, jb + ch * 32, coefA, coefC, d, c, ob, ob + 2048, sumsq);
          }
          if (more) tmem_ld_wait_dep(rn);
        };
#pragma unroll 1
        for (int ch = c_begin; ch < c_end; ch += 2) {
          step(ch, ra, rb);
          if (ch + 1 < c_end) step(ch + 1, rb, ra);
        }
        release_acc(&tempty[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      } else {
        // tf32: sum the K-chunk partials from TMEM in fp32 registers (round-to-nearest)
        float d[Cfg::CH_PER][32];
#pragma unroll
        for (int x = 0; x < Cfg::CH_PER; ++x)
#pragma unroll
          for (int u = 0; u < 32; ++u) d[x][u] = 0.f;
        const int nkb = (P.K + Cfg::BK - 1) / Cfg::BK;
        for (int kb0 = 0; kb0 < nkb; kb0 += Cfg::PROMO_KB) {
          mbar_wait(&tfull[acc], acc_phase);
          tc_fence_after();
          const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * Cfg::BN;
#pragma unroll
          for (int x = 0; x < Cfg::CH_PER; ++x) {
            uint32_t r[32];
            tmem_ld32(tbase + (c_begin0 + x) * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int u = 0; u < 32; ++u) d[x][u] += __uint_as_float(r[u]);
          }
          release_acc(&tempty[acc]);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
#pragma unroll
        for (int x = 0; x < Cfg::CH_PER; ++x) {
          float c[32];
#pragma unroll
          for (int u = 0; u < 32; ++u) c[u] = 0.f;
          const int j0 = tn * Cfg::BN + (c_begin0 + x) * 32;
          if (needC && i0 + 32 <= P.M && j0 + 32 <= P.N && (P.ldc & 3) == 0)
            warp_load_f32_block<Cfg::SPLIT>(P.C, P.C_lo, P.ldc, i0, j0, c, tb, lane);   // warp-uniform
          else if (needC && i < P.M && j0 < P.N) load_row32<Cfg::KIND, Cfg::SPLIT>(P.C, P.C_lo, P.ldc, i, j0, P.N, c);
          epi_segment<Cfg>(ea, mode, sym, i0, lane, j0, coefA, coefC, d[x], c, tb, sumsq);
        }
      }

      if (mode == EPI_RESID && P.norm_part) {
        // deterministic per-tile sum of out^2: fixed shuffle tree, then the 8 warps in order
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sumsq += __shfl_xor_sync(0xffffffffu, sumsq, o);
        if (lane == 0) red[e] = sumsq;
        named_bar_sync(1, 32 * Cfg::EPI_WARPS);
        if (et == 0 && (tm * Cfg::CG + (int)rank) * Cfg::BM < P.M) {
          float tsum = 0.f;
#pragma unroll
          for (int x = 0; x < Cfg::EPI_WARPS; ++x) tsum += red[x];
          P.norm_part[(tm * Cfg::CG + (int)rank) * P.tiles_n + tn] = tsum;
        }
        named_bar_sync(1, 32 * Cfg::EPI_WARPS);
      }
      if (trace2 && et == 0 && leader && etcount < 8) trace2[192 + 4 * etcount + 3] = globaltimer_ns();
      ++etcount;
    }
    if (Cfg::KIND == 0 && lane == 0) bulk_wait_all();   // this warp's TMA stores are complete
  }

  }
  tc_fence_before();
  if constexpr (Cfg::CTA2) cluster_sync_all();   // no CTA leaves while its peer may still touch its smem
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<Cfg::CG>(tmem_base, Cfg::TMEM_ALLOC);
  }
}

// One GEMM body, one kernel symbol per role in the iteration, so ncu launch lists and
// per-kernel profiles separate the residual (Gram) product, the square R.R, the apply
// X + X.P and the other products (DB Newton sweep, test hook).
enum GemmRole : int { ROLE_GRAM = 0, ROLE_SQUARE = 1, ROLE_APPLY = 2, ROLE_OTHER = 3 };

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1) prism_gram_kernel(const __grid_constant__ GemmLaunch L) {
  gemm_body<Cfg>(L);
}
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1) prism_square_kernel(const __grid_constant__ GemmLaunch L) {
  gemm_body<Cfg>(L);
}
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1) prism_apply_kernel(const __grid_constant__ GemmLaunch L) {
  gemm_body<Cfg>(L);
}
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1) prism_gemm_kernel(const __grid_constant__ GemmLaunch L) {
  gemm_body<Cfg>(L);
}

}  // namespace prism
