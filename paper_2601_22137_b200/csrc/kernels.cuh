// SIMT kernels of the PRISM iteration (everything that is not a dense
// contraction): Frobenius pre-scaling, layout/cast, the Philox sketch, the
// thin sketch chain, the single-CTA fp64 coefficient solve, and the output
// write-back.  All reductions are fixed-order (no float atomics), so results
// are bit-reproducible run to run.
#pragma once
#include "ptx.cuh"
#include "gemm.cuh"   // kChainG (chain_part layout)

namespace prism {


// Per-matrix static description (device memory).
struct MatDesc {
  const void* A;       // user input (row-major, lda)
  void* Q;             // polar output / sqrt output
  void* Q2;            // inv-sqrt output (sqrt path) or null
  long long lda, ldq;
  long long ldx0;      // leading dimension of X[0] (= ldq when X[0] is the caller's output Q)
  int fold;            // folded normalisation for this matrix (BF16 / TF32 polar, TMA-legal A, Q)
  int flip_ok;         // folded and Q does not overlap A: Q may hold the odd iterates (MatState.flip)
  int pad0_;
  int m, n;            // user shape
  int s, L;            // small side / large side (polar); n, n (sqrt)
  int trans;           // polar: 1 if the compute layout Xt (s x L) is A^T (tall A)
  int sketch_id;       // global matrix index b of the Philox counter
  // compute buffers (compute dtype, + lo planes in 3xTF32 mode), leading dim ldx / ldr
  void* X[2]; void* X_lo[2];
  void* Y[2]; void* Y_lo[2];
  void* R; void* R_lo;
  long long ldx, ldr;
  float* gdiag;        // [s]
  float* norm_part;    // Gram per-tile partials
  int tiles_m, tiles_n, sym;
  int pad_;
  float* S;            // [p x ldS] sketch S_k (fp32)
  void* W[2];          // chain B operands [4p x ldS] (compute dtype), hi rows then lo rows
  float* keep;         // [4][s][p] kept chain columns (fp32)
  double* chain_part;  // [tiles_m][6] per-tile <Va,Vb>
  long long ldS;
  int chain_tiles;     // <Va,Vb> partial groups: nchunk x ceil(s / 32)
  int nchunk;          // sketch column chunks (p <= 8: 1; else ceil(p / 8), W / keep per chunk)
  // DB Newton (fp32 3xTF32 only): M_k (plain fp32, ld ldx), Gauss-Jordan sweep temporaries
  // (E = row block of W, T = D E, D = pivot inverse; hi + lo planes), W = R / R_lo,
  // per-tile (<E1,E1>, <E1,E2>, <E2,E2>) for the alpha fit
  float* Mst;
  void* E; void* E_lo;
  void* T; void* T_lo;
  void* Dp; void* Dp_lo;
  double* dbpart;
};

// Tile list compacted per iteration to the matrices still active (plan order kept): the plan
// describes the list as runs of consecutive tiles of one matrix (start, length, matrix).
struct CompactList {
  const int* runs;        // [nruns][3] (plan constants)
  int nruns;
  const uint32_t* src;    // the launch's full tile list
  uint32_t* dst;          // compacted list (plan memory)
  int* count;             // its length
};
constexpr int kMaxCompactRuns = 1024;

struct SolveParams {
  MatDesc* mats;
  MatState* st;
  int* iter;            // device iteration counter k (workspace)
  double* alpha_hist;   // [batch * max_iters] (workspace; copied to the user's report)
  float* resid_hist;    // [batch * (max_iters+1)] (workspace)
  int32_t* rep_iters;   // user report (device) or null — only used by k_report
  float* rep_resid;
  int32_t* rep_status;
  double* rep_alphas;
  float* rep_resid_hist;
  double* fro_part;     // [batch * kFroParts]
  const int* tile_off;  // [batch + 1] prefix of 64x64 layout tiles (normalise: Xt; finalise: output)
  const int* out_tile_off;
  const int* tile_mat;  // [n_tiles] matrix of each layout tile (same tiling for normalise / finalise)
  const int* fro_off;   // [batch + 1] prefix of the per-matrix ||A||_F partial counts (fro_parts)
  int n_tiles, n_out_tiles, n_fro_blocks;
  double* fro2_out;     // row-block begin: local sum of squares (else null)
  const double* fro2_in;   // row-block: all-reduced sum of squares (else null)
  int batch, p, d, max_iters, warmup, fit, precision, kind_sqrt;
  int inv_q;            // coupled inverse Newton root order (0: polar / sqrt / sign)
  int kind_cheb;        // Chebyshev inverse (A' in Y[0], X_0 = A'^T, output X / c)
  int kind_db;          // DB Newton (M_k in Mst, W = R: M_k then -M_k^{-1}; output X, Y unscaled)
  int* parity;          // [batch] (plan-owned): final parity of each matrix's last solve (k_finalize)
  int* flip_cur;        // [batch] (plan-owned): parity the ping-pong tables hold for each matrix
  // folded polar: the tables whose entry b (matrix b) is swapped to flip matrix b's parity:
  // gram[0] <-> gram[1], apply[0] <-> apply[1], apply0 <-> apply0f
  GemmProblem* flip_tab[6];
  // tile lists of the Gram / square / apply launches compacted by k_alpha's compaction blocks
  int ncompact;
  CompactList clist[3];
  double tol, alo, ahi, ataylor;
  unsigned long long seed;
};

constexpr int kFroParts = 256;   // max ||A||_F partials per matrix (fixed order)
// partials of an m x n matrix: one per 32 K elements, 1 .. kFroParts (size-only rule)
__host__ __device__ inline int fro_parts(long long m, long long n) {
  const long long q = (m * n + 32767) / 32768;
  return (int)(q < 1 ? 1 : q > kFroParts ? kFroParts : q);
}

// ----------------------------------------------------------------- helpers
__device__ __forceinline__ float load_val(const void* base, long long idx, int prec_bf16) {
  if (prec_bf16) return __bfloat162float(static_cast<const __nv_bfloat16*>(base)[idx]);
  return static_cast<const float*>(base)[idx];
}

template <typename T, int NT>
__device__ __forceinline__ T block_sum(T v, T* scratch) {
  // fixed-order: warp tree, then warp 0 sums the per-warp values in order
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) scratch[w] = v;
  __syncthreads();
  T t = T(0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NT / 32; ++i) t += scratch[i];
    scratch[0] = t;
  }
  __syncthreads();
  t = scratch[0];
  __syncthreads();
  return t;
}

// matrix owning flat block t of a per-matrix prefix table off[0..batch]
__device__ __forceinline__ int find_matrix(const int* off, int batch, int t) {
  int lo = 0, hi = batch - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (off[mid] <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// ----------------------------------------------------------------- a1: ||A||_F partials
// One block per partial; a matrix gets fro_parts(m, n) blocks (a function of its size only,
// so its bits do not depend on the batch), listed by the prefix P.fro_off.  Block j sums a
// fixed contiguous share of the matrix with 16-byte vector loads when the layout allows it.
__global__ void __launch_bounds__(256) k_fro_partials(SolveParams P) {
  griddep_wait();
  griddep_launch();
  __shared__ double scratch[8];
  const int b = find_matrix(P.fro_off, P.batch, blockIdx.x);
  const int jp = blockIdx.x - P.fro_off[b], parts = P.fro_off[b + 1] - P.fro_off[b];
  const MatDesc& D = P.mats[b];
  const int bf16 = P.precision == 0;
  const int esz = bf16 ? 2 : 4, vec = 16 / esz;
  const bool vok = ((D.lda * esz) % 16 == 0) && ((reinterpret_cast<uintptr_t>(D.A) & 15) == 0);
  const long long nv = vok ? D.n / vec : 0;       // 16-B vectors per row
  // block jp sums a fixed contiguous share of the flattened (row, vector) index space,
  // eight independent 16-B loads in flight per thread (fixed assignment: deterministic)
  const long long total = (long long)D.m * nv;
  const long long per = (total + parts - 1) / parts;
  const long long beg = jp * per, end = min(total, beg + per);
  const char* A = static_cast<const char*>(D.A);
  double acc = 0.0;
  // (row, vector) of the thread's first index; later indices advance by 256 vectors with an
  // incremental carry instead of a 64-bit division per load
  long long jr = 0, jc = 0;
  if (nv > 0) {
    const long long j0 = beg + threadIdx.x;
    jr = j0 / nv;
    jc = j0 - jr * nv;
  }
  if (nv > 0 && D.lda * esz == nv * 16) {
    // dense rows (lda = n, n a whole number of vectors): the block's share is one contiguous
    // range of memory — plain strided vector loads, no (row, column) bookkeeping
    const uint4* q = reinterpret_cast<const uint4*>(A);
    for (long long base = beg + threadIdx.x; base < end; base += 8 * 256) {
      uint4 w[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const long long j = base + (long long)u * 256;
        w[u] = j < end ? __ldg(q + j) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (bf16) {
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w[u]);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(h[e]);
            acc += (double)f.x * f.x + (double)f.y * f.y;
          }
        } else {
          const float* f = reinterpret_cast<const float*>(&w[u]);
#pragma unroll
          for (int e = 0; e < 4; ++e) acc += (double)f[e] * f[e];
        }
      }
    }
  } else
  for (long long base = beg + threadIdx.x; base < end; base += 8 * 256) {
    uint4 w[8];
    long long r = jr, c = jc;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const long long j = base + (long long)u * 256;
      w[u] = make_uint4(0, 0, 0, 0);
      if (j < end) w[u] = __ldg(reinterpret_cast<const uint4*>(A + r * D.lda * esz) + c);
      c += 256;
      while (c >= nv && nv > 0) { c -= nv; ++r; }
    }
    jr = r;
    jc = c;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (bf16) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w[u]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h[e]);
          acc += (double)f.x * f.x + (double)f.y * f.y;
        }
      } else {
        const float* f = reinterpret_cast<const float*>(&w[u]);
#pragma unroll
        for (int e = 0; e < 4; ++e) acc += (double)f[e] * f[e];
      }
    }
  }
  // columns past the last whole vector (n % vec, or every column when unaligned)
  const int c0 = (int)(nv * vec);
  if (c0 < D.n) {
    for (int r = jp; r < D.m; r += parts)
      for (int c = c0 + threadIdx.x; c < D.n; c += 256) {
        const double x = (double)load_val(D.A, (long long)r * D.lda + c, bf16);
        acc += x * x;
      }
  }
  acc = block_sum<double, 256>(acc, scratch);
  if (threadIdx.x == 0) P.fro_part[b * kFroParts + jp] = acc;
}

// c = ||A||_F per matrix from its partials (fixed-order tree); one block per matrix
__global__ void __launch_bounds__(256) k_fro_final(SolveParams P) {
  griddep_wait();
  griddep_launch();
  __shared__ double scratch[8];
  const int b = blockIdx.x;
  const int parts = P.fro_off[b + 1] - P.fro_off[b];
  double v = (threadIdx.x < parts) ? P.fro_part[b * kFroParts + threadIdx.x] : 0.0;
  v = block_sum<double, 256>(v, scratch);
  if (threadIdx.x == 0) {
    if (P.fro2_out) {
      P.fro2_out[b] = v;   // row-block: the caller all-reduces it
    } else {
      const double c = sqrt(v);
      P.st[b].c = c;
      P.st[b].inv_c = c > 0.0 ? 1.0 / c : 0.0;
      P.st[b].inv_c2 = c > 0.0 ? 1.0 / v : 0.0;
    }
  }
}

// End of a residual-stage SIMT block (R = I - M, DB Newton's begin, the row-block unpack):
// store this block's norm partial; the last block of the matrix runs the stop test (R12).
__device__ __forceinline__ void residual_stage_end(const SolveParams& P, int b, int slot, double acc) {
  __shared__ int s_last;
  const MatDesc& D = P.mats[b];
  if (threadIdx.x == 0) {
    D.norm_part[slot] = (float)acc;
    s_last = residual_arrive(&P.st[b], D.tiles_m * D.tiles_n) ? 1 : 0;
  }
  __syncthreads();
  if (s_last && threadIdx.x < 32) {
    __threadfence();
    residual_stop_warp(&P.st[b], D.norm_part, D.tiles_m * D.tiles_n, *P.iter, P.tol, D.s, P.max_iters,
                       P.resid_hist + (size_t)b * (P.max_iters + 1), threadIdx.x);
  }
}

// row-block: c = sqrt(all-reduced sum of squares)
__global__ void k_set_c(SolveParams P) {
  griddep_wait();
  griddep_launch();
  if (threadIdx.x == 0) {
    const double v = P.fro2_in[blockIdx.x], c = sqrt(v);
    P.st[blockIdx.x].c = c;
    P.st[blockIdx.x].inv_c = c > 0.0 ? 1.0 / c : 0.0;
    P.st[blockIdx.x].inv_c2 = c > 0.0 ? 1.0 / v : 0.0;
  }
}

__device__ __forceinline__ void store_x(void* hi, void* lo, long long idx, float v, int precision);

// Row-block: R = I - G from the all-reduced packed fp32 Gram (upper-triangle
// panels, gemm.cuh epi_gram32), diag(G) in fp32, and the per-64x64-tile sum of R^2 that
// k_alpha reads as the norm partials (tiles_m = tiles_n = ceil(n / 64), sym = 0).  The source
// block of an R block below the diagonal is the transposed upper block, staged through smem so
// both the packed reads and the R writes are coalesced.  grid (ceil(n/64), ceil(n/64)).
template <int PREC>
__global__ void __launch_bounds__(256) k_resid_packed(SolveParams P, const float* Gp) {
  griddep_wait();
  griddep_launch();
  __shared__ float tile[64][65];
  __shared__ double scratch[8];
  const MatDesc& D = P.mats[0];
  if (P.st[0].done) return;
  const int n = D.s;
  const int bx = blockIdx.x, by = blockIdx.y;    // R rows [64 by, +64), columns [64 bx, +64)
  const bool upper = bx >= by;
  const int rs = 64 * (upper ? by : bx), cs = 64 * (upper ? bx : by);   // upper source block
  for (int e = threadIdx.x; e < 64 * 64; e += 256) {
    const int r = e >> 6, c = e & 63;
    const long long i = rs + r, j = cs + c;
    float g = 0.f;
    if (i < n && j < n && j >= i) {
      const long long t = i >> 8;
      g = Gp[gram_panel_off(t, n) + (i - 256 * t) * (n - 256 * t) + (j - 256 * t)];
    }
    tile[r][c] = g;
  }
  __syncthreads();
  double acc = 0.0;
  for (int e = threadIdx.x; e < 64 * 64; e += 256) {
    const int rr = e >> 6, cc = e & 63;
    const int i = 64 * by + rr, j = 64 * bx + cc;
    if (i >= n || j >= n) continue;
    const float g = (upper && j >= i) ? tile[rr][cc] : tile[cc][rr];
    const float rv = (i == j ? 1.f : 0.f) - g;
    store_x(D.R, D.R_lo, (long long)i * D.ldr + j, rv, PREC);
    if (i == j) D.gdiag[i] = g;
    acc += (double)rv * rv;
  }
  acc = block_sum<double, 256>(acc, scratch);
  if (threadIdx.x == 0) D.norm_part[by * D.tiles_n + bx] = (float)acc;
}

__device__ __forceinline__ void store_x(void* hi, void* lo, long long idx, float v, int precision) {
  if (precision == 0) {
    static_cast<__nv_bfloat16*>(hi)[idx] = __float2bfloat16_rn(v);
  } else if (precision == 1) {   // 3xTF32 split
    float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    static_cast<float*>(hi)[idx] = h;
    static_cast<float*>(lo)[idx] = v - h;
  } else {
    static_cast<float*>(hi)[idx] = v;
  }
}

// Layout tiles (normalise / finalise): 32 rows x 32 16-byte vectors, one block
// (256 threads, 4 vectors each, a warp = one 512-B row segment) per tile over a
// batch-wide flat list.  X keeps A's row-major layout, so both are scaled copies.
// One 16-byte vector of a layout tile as raw bits (4 registers; + the lo plane in 3xTF32):
// the memory kernels issue every load of a thread before decoding / storing, without the
// register cost of decoded floats (occupancy is what hides the HBM latency here).
template <int PREC>
struct Raw {
  uint4 h, l;
};
template <int PREC>
__device__ __forceinline__ Raw<PREC> load_raw(const void* base, const void* lo, long long idx, int n_valid, bool vec) {
  constexpr int ESZ = PREC == 0 ? 2 : 4, VE = 16 / ESZ;
  Raw<PREC> r;
  r.l = make_uint4(0, 0, 0, 0);
  const char* p = static_cast<const char*>(base) + idx * ESZ;
  const char* q = (PREC == 1 && lo) ? static_cast<const char*>(lo) + idx * ESZ : nullptr;
  if (vec) {
    r.h = __ldg(reinterpret_cast<const uint4*>(p));
    if (q) r.l = __ldg(reinterpret_cast<const uint4*>(q));
  } else {
    uint32_t w[4] = {0, 0, 0, 0}, wl[4] = {0, 0, 0, 0};
#pragma unroll
    for (int e = 0; e < VE; ++e) {
      if (e >= n_valid) continue;
      if (PREC == 0) {
        const uint32_t b = *reinterpret_cast<const unsigned short*>(p + 2 * e);
        w[e >> 1] |= b << (16 * (e & 1));
      } else {
        w[e] = *reinterpret_cast<const uint32_t*>(p + 4 * e);
        if (q) wl[e] = *reinterpret_cast<const uint32_t*>(q + 4 * e);
      }
    }
    r.h = make_uint4(w[0], w[1], w[2], w[3]);
    r.l = make_uint4(wl[0], wl[1], wl[2], wl[3]);
  }
  return r;
}

template <int PREC>   // 0 bf16, 1 fp32 hi+lo (3xTF32 split), 2 fp32
struct Vec {
  static constexpr int ESZ = PREC == 0 ? 2 : 4;
  static constexpr int VE = 16 / ESZ;
  float v[VE];
  __device__ __forceinline__ void from_raw(const Raw<PREC>& r) {
    if (PREC == 0) {
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r.h);
#pragma unroll
      for (int e = 0; e < 4; ++e) { const float2 f = __bfloat1622float2(h[e]); v[2 * e] = f.x; v[2 * e + 1] = f.y; }
    } else {
      v[0] = __uint_as_float(r.h.x); v[1] = __uint_as_float(r.h.y);
      v[2] = __uint_as_float(r.h.z); v[3] = __uint_as_float(r.h.w);
      if (PREC == 1) {
        v[0] += __uint_as_float(r.l.x); v[1] += __uint_as_float(r.l.y);
        v[2] += __uint_as_float(r.l.z); v[3] += __uint_as_float(r.l.w);
      }
    }
  }
  __device__ __forceinline__ void load(const void* base, const void* lo, long long idx, int n_valid, bool vec) {
    if (PREC == 0) {
      const __nv_bfloat16* p = static_cast<const __nv_bfloat16*>(base) + idx;
      if (vec) {
        const uint4 w = __ldg(reinterpret_cast<const uint4*>(p));
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
        for (int e = 0; e < 4; ++e) { const float2 f = __bfloat1622float2(h[e]); v[2 * e] = f.x; v[2 * e + 1] = f.y; }
      } else {
#pragma unroll
        for (int e = 0; e < VE; ++e) v[e] = e < n_valid ? __bfloat162float(p[e]) : 0.f;
      }
    } else {
      const float* p = static_cast<const float*>(base) + idx;
      const float* q = (PREC == 1 && lo) ? static_cast<const float*>(lo) + idx : nullptr;
      if (vec) {
        const float4 w = __ldg(reinterpret_cast<const float4*>(p));
        v[0] = w.x; v[1] = w.y; v[2] = w.z; v[3] = w.w;
        if (q) { const float4 l = __ldg(reinterpret_cast<const float4*>(q)); v[0] += l.x; v[1] += l.y; v[2] += l.z; v[3] += l.w; }
      } else {
#pragma unroll
        for (int e = 0; e < VE; ++e) v[e] = e < n_valid ? p[e] + (q ? q[e] : 0.f) : 0.f;
      }
    }
  }
  // store v * scale; split (PREC 1) writes tf32-truncated hi and the remainder to lo
  __device__ __forceinline__ void store(void* base, void* lo, long long idx, int n_valid, bool vec, float scale,
                                        bool split) const {
    if (PREC == 0) {
      __nv_bfloat16* p = static_cast<__nv_bfloat16*>(base) + idx;
      if (vec) {
        uint4 w;
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
        for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[2 * e] * scale, v[2 * e + 1] * scale);
        *reinterpret_cast<uint4*>(p) = w;
      } else {
#pragma unroll
        for (int e = 0; e < VE; ++e) if (e < n_valid) p[e] = __float2bfloat16_rn(v[e] * scale);
      }
    } else {
      float* p = static_cast<float*>(base) + idx;
      float* q = split ? static_cast<float*>(lo) + idx : nullptr;
      float o[VE], h[VE];
#pragma unroll
      for (int e = 0; e < VE; ++e) {
        o[e] = v[e] * scale;
        h[e] = split ? __uint_as_float(__float_as_uint(o[e]) & 0xFFFFE000u) : o[e];
      }
      if (vec) {
        *reinterpret_cast<float4*>(p) = make_float4(h[0], h[1], h[2], h[3]);
        if (q) *reinterpret_cast<float4*>(q) = make_float4(o[0] - h[0], o[1] - h[1], o[2] - h[2], o[3] - h[3]);
      } else {
#pragma unroll
        for (int e = 0; e < VE; ++e)
          if (e < n_valid) { p[e] = h[e]; if (q) q[e] = o[e] - h[e]; }
      }
    }
  }
};

// a1: X_0 = A / ||A||_F (same row-major layout), Y_0 = I (sqrt), state init.
// Inverse Newton: X_0 = I/c, M_0 = A/c^q (M in Y), c^q = 2||A||_F/(q+1).
template <int PREC>
__global__ void __launch_bounds__(256) k_normalize(SolveParams P) {
  griddep_wait();
  griddep_launch();
  using V = Vec<PREC>;
  const int t = blockIdx.x;
  const int b = __ldg(P.tile_mat + t);   // one load (a binary search over tile_off was ~6 dependent loads)
  const MatDesc& D = P.mats[b];
  if (D.fold) return;   // iteration 0 reads A itself (k_init_state did the rest)
  // the descriptor's fields in registers: read through the reference they would be reloaded
  // from global memory after every store (possible aliasing), a dependent load per vector
  const int Dm = D.m, Dn = D.n;
  const long long Dlda = D.lda, Dldx = D.ldx;
  const void* const DA = D.A;
  void* const X0 = D.X[0];
  void* const X0l = D.X_lo[0];
  void* const Y0 = D.Y[0];
  void* const Y0l = D.Y_lo[0];
  const double c = P.st[b].c;   // written by k_fro_final
  const float inv = c > 0.0 ? (float)(1.0 / c) : 0.f;
  const int TW = 32 * V::VE;
  const int tcn = (Dn + TW - 1) / TW;
  const int lt = t - P.tile_off[b];
  const int r0 = (lt / tcn) * 32, c0 = (lt % tcn) * TW;
  const bool src_vec = ((Dlda * V::ESZ) % 16 == 0) && ((reinterpret_cast<uintptr_t>(DA) & 15) == 0);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int slot = threadIdx.x + 256 * j;
    const int r = r0 + slot / 32, col = c0 + (slot % 32) * V::VE;
    if (r >= Dm || col >= Dn) continue;
    const int nv = min(V::VE, Dn - col);
    V x;
    x.load(DA, nullptr, (long long)r * Dlda + col, nv, src_vec && nv == V::VE);
    if (P.kind_db) {
      // DB Newton: X_0 = M_0 = A, Y_0 = I (no scaling, R28)
      x.store(X0, X0l, (long long)r * Dldx + col, nv, nv == V::VE, 1.f, PREC == 1);
#pragma unroll
      for (int e = 0; e < V::VE; ++e)
        if (e < nv) D.Mst[(long long)r * Dldx + col + e] = x.v[e];
#pragma unroll
      for (int e = 0; e < V::VE; ++e) x.v[e] = (col + e == r) ? 1.f : 0.f;
      x.store(Y0, Y0l, (long long)r * Dldx + col, nv, nv == V::VE, 1.f, PREC == 1);
      continue;
    }
    if (P.kind_cheb) {
      // A' = A/c (row-major, Y[0]) and X_0 = A'^T: transposed scalar stores
      x.store(Y0, Y0l, (long long)r * Dldx + col, nv, nv == V::VE, inv, PREC == 1);
#pragma unroll
      for (int e = 0; e < V::VE; ++e)
        if (e < nv) store_x(X0, X0l, (long long)(col + e) * Dldx + r, x.v[e] * inv, PREC);
      continue;
    }
    if (P.inv_q) {
      const double cq = 2.0 * c / (P.inv_q + 1);
      x.store(Y0, Y0l, (long long)r * Dldx + col, nv, nv == V::VE, c > 0.0 ? (float)(1.0 / cq) : 0.f,
              PREC == 1);
#pragma unroll
      for (int e = 0; e < V::VE; ++e) x.v[e] = (col + e == r) ? 1.f : 0.f;
      x.store(X0, X0l, (long long)r * Dldx + col, nv, nv == V::VE,
              c > 0.0 ? (float)pow(cq, -1.0 / P.inv_q) : 0.f, PREC == 1);
      continue;
    }
    x.store(X0, X0l, (long long)r * Dldx + col, nv, nv == V::VE, inv, PREC == 1);
    if (P.kind_sqrt) {
#pragma unroll
      for (int e = 0; e < V::VE; ++e) x.v[e] = (col + e == r) ? 1.f : 0.f;
      x.store(Y0, Y0l, (long long)r * Dldx + col, nv, nv == V::VE, 1.f, PREC == 1);
    }
  }

}

// Solver state of every matrix at the start of a solve (after ||A||_F): alpha, residual
// history bookkeeping, done / status (zero input), and the norm partials zeroed (the stop
// test sums every entry; unscheduled ones stay 0).  grid (batch).
__global__ void k_init_state(SolveParams P) {
  griddep_wait();
  griddep_launch();
  __shared__ int s_swap;
  const int b = blockIdx.x;
  const MatDesc& D = P.mats[b];
  for (int t = threadIdx.x; t < D.tiles_m * D.tiles_n; t += blockDim.x) D.norm_part[t] = 0.f;
  if (threadIdx.x == 0) {
    // folded polar: store the odd iterates in Q when the last solve ended after an odd
    // number of updates, so that a repeat needs no final copy (any choice is correct: it
    // only decides which buffer holds which iterate); the tables are flipped in place
    const int want = (D.flip_ok && P.parity) ? P.parity[b] : 0;
    s_swap = (P.flip_cur && want != P.flip_cur[b]) ? 1 : 0;
    if (s_swap) P.flip_cur[b] = want;
    P.st[b].flip = want;
    const double c = P.st[b].c;
    if (b == 0) *P.iter = 0;
    MatState& S = P.st[b];
    S.alpha = P.ataylor;
    S.r_prev = INFINITY;
    S.resid = 0.f;
    S.iters = 0;
    S.incr = 0;
    S.done = (c == 0.0) ? 1 : 0;
    S.stop_iter = (c == 0.0) ? -1 : 0x7fffffff;
    S.arrivals = 0;
    S.status = (c == 0.0) ? 4 : 1;
  }
  __syncthreads();
  if (s_swap) {
    constexpr int W = (int)(sizeof(GemmProblem) / 4);
    for (int j = 0; j < 3; ++j) {
      uint32_t* x = reinterpret_cast<uint32_t*>(P.flip_tab[2 * j] + b);
      uint32_t* y = reinterpret_cast<uint32_t*>(P.flip_tab[2 * j + 1] + b);
      for (int w = threadIdx.x; w < W; w += blockDim.x) {
        const uint32_t u = x[w];
        x[w] = y[w];
        y[w] = u;
      }
    }
  }
}

// Inverse Newton residual R_k = I - M_k, elementwise: R (compute dtype), fp32
// diag(M) (for Q = M S^T in the chain, as diag(G) for the other kinds) and per-tile
// sum of R^2 in the Gram epilogue's tile layout (128 x bn tiles, read by k_alpha).
// grid (tiles_n, tiles_m, batch) of the largest matrix; M_k is Y[k & 1].
template <int PREC>
__global__ void __launch_bounds__(256) k_resid_inv(SolveParams P, int bn) {
  griddep_wait();
  griddep_launch();
  __shared__ double scratch[8];
  using V = Vec<PREC>;
  const int b = blockIdx.z;
  const MatDesc& D = P.mats[b];
  if (P.st[b].done) return;
  const int tm = blockIdx.y, tn = blockIdx.x;
  if (tm >= D.tiles_m || tn >= D.tiles_n) return;
  const int n = D.s;
  const int par = *P.iter & 1;
  const int vpr = bn / V::VE;   // vectors per tile row
  double acc = 0.0;
  for (int e = threadIdx.x; e < 128 * vpr; e += 256) {
    const int i = tm * 128 + e / vpr, j = tn * bn + (e % vpr) * V::VE;
    if (i >= n || j >= n) continue;
    const int nv = min(V::VE, n - j);
    V x;
    x.load(D.Y[par], D.Y_lo[par], (long long)i * D.ldx + j, nv, nv == V::VE);
#pragma unroll
    for (int u = 0; u < V::VE; ++u) {
      const float mv = x.v[u];
      const float rv = (j + u == i ? 1.f : 0.f) - mv;
      if (j + u == i) D.gdiag[i] = mv;
      x.v[u] = u < nv ? rv : 0.f;
      acc += (double)x.v[u] * x.v[u];
    }
    x.store(D.R, D.R_lo, (long long)i * D.ldr + j, nv, nv == V::VE, 1.f, PREC == 1);
  }
  acc = block_sum<double, 256>(acc, scratch);
  if (threadIdx.x == 0) D.norm_part[tm * D.tiles_n + tn] = (float)acc;
}

// ----------------------------------------------------------------- DB Newton (f3)
// fp32 hi + lo (3xTF32 split) element access
__device__ __forceinline__ float ld_split(const void* hi, const void* lo, long long idx) {
  return static_cast<const float*>(hi)[idx] + static_cast<const float*>(lo)[idx];
}

// Iteration start: W = M_k (split, the matrix the sweep inverts in place) and the per-tile
// ||I - M_k||^2 (residual of P:505; M_k = X_k Y_k -> I) in the Gram tile layout.
// grid (tiles_n, tiles_m, batch), 128 x bn tiles.
__global__ void __launch_bounds__(256) k_db_begin(SolveParams P, int bn) {
  griddep_wait();
  griddep_launch();
  __shared__ double scratch[8];
  const int b = blockIdx.z;
  const MatDesc& D = P.mats[b];
  if (P.st[b].done) return;
  const int tm = blockIdx.y, tn = blockIdx.x;
  if (tm >= D.tiles_m || tn >= D.tiles_n) return;
  const int n = D.s;
  double acc = 0.0;
  for (int e = threadIdx.x; e < 128 * bn; e += 256) {
    const int i = tm * 128 + e / bn, j = tn * bn + e % bn;
    if (i >= n || j >= n) continue;
    const float m = D.Mst[(long long)i * D.ldx + j];
    store_x(D.R, D.R_lo, (long long)i * D.ldr + j, m, 1);
    const double r = (i == j ? 1.0 : 0.0) - (double)m;
    acc += r * r;
  }
  acc = block_sum<double, 256>(acc, scratch);
  residual_stage_end(P, b, tm * D.tiles_n + tn, acc);
}

constexpr int kGJ = 128;          // Gauss-Jordan block
constexpr int kGJCopy = 64;       // CTAs copying the row block per matrix

// Sweep step j, part 1: CTA 0 inverts the pivot block W_JJ (J = [128j, 128j + bj)) by
// Gauss-Jordan (SPD: no pivoting) into D; CTAs 1.. copy the row block E = W_J* (bj x n).
// grid (1 + kGJCopy, batch), 128 threads.
// Pivot CTA: thread c owns column c, all 128 rows in registers, kept in rotated order so
// that the pivot row of every step is register 0: step p reads column p (thread p's
// registers, broadcast through a double-buffered shared vector, one barrier per step),
// updates rows 1..127 into registers 0..126 and writes the new pivot row into register
// 127 — after bj steps row r sits in register (r - bj) mod 128.  Padding outside bj is
// the identity (untouched by steps p < bj).
__global__ void __launch_bounds__(kGJ) k_gj_pivot(SolveParams P, int j) {
  griddep_wait();
  griddep_launch();
  extern __shared__ float gsm[];
  const int b = blockIdx.y;
  const MatDesc& D = P.mats[b];
  if (P.st[b].done) return;
  const int n = D.s, J0 = kGJ * j;
  if (J0 >= n) return;
  const int bj = min(kGJ, n - J0);
  if (blockIdx.x == 0) {
    float* colf = gsm;   // [2][kGJ]
    float(*tile)[kGJ + 1] = reinterpret_cast<float(*)[kGJ + 1]>(gsm + 2 * kGJ);
    const int c = threadIdx.x;
    // the block through shared memory: coalesced 16-B loads (hi + lo), all in flight
    {
      const float* Rh = static_cast<const float*>(D.R);
      const float* Rl = static_cast<const float*>(D.R_lo);
#pragma unroll 8
      for (int q = c; q < kGJ * (kGJ / 4); q += kGJ) {
        const int r = q >> 5, c4 = (q & 31) * 4;
        float v[4];
        if (r < bj && c4 + 3 < bj) {
          const long long off = (long long)(J0 + r) * D.ldr + J0 + c4;
          const float4 h = __ldg(reinterpret_cast<const float4*>(Rh + off));
          const float4 l = __ldg(reinterpret_cast<const float4*>(Rl + off));
          v[0] = h.x + l.x; v[1] = h.y + l.y; v[2] = h.z + l.z; v[3] = h.w + l.w;
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int cc = c4 + e;
            v[e] = (r < bj && cc < bj) ? ld_split(D.R, D.R_lo, (long long)(J0 + r) * D.ldr + J0 + cc) : (r == cc ? 1.f : 0.f);
          }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) tile[r][c4 + e] = v[e];
      }
    }
    __syncthreads();
    float a[kGJ];
#pragma unroll
    for (int r = 0; r < kGJ; ++r) a[r] = tile[r][c];

#pragma unroll 1
    for (int p = 0; p < bj; ++p) {
      float* cf = colf + (p & 1) * kGJ;
      if (c == p) {
#pragma unroll
        for (int i = 0; i < kGJ; i += 4) *reinterpret_cast<float4*>(cf + i) = make_float4(a[i], a[i + 1], a[i + 2], a[i + 3]);
      }
      __syncthreads();
      const float inv = 1.f / cf[0];
      // new row r-1 = a[r] - colf[r] * (a[p] / pivot); the pivot column's owner (its old
      // registers already broadcast) zeroes them, so one FMA gives -colf[r] / pivot there
      const bool own = c == p;
      const float rr = own ? inv : a[0] * inv;
      if (own) {
#pragma unroll
        for (int i = 1; i < kGJ; ++i) a[i] = 0.f;
      }
#pragma unroll
      for (int i4 = 0; i4 < kGJ; i4 += 4) {
        const float4 f4 = *reinterpret_cast<const float4*>(cf + i4);
        const float f[4] = {f4.x, f4.y, f4.z, f4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i4 + u > 0) a[i4 + u - 1] = fmaf(-f[u], rr, a[i4 + u]);
      }
      a[kGJ - 1] = rr;   // the new pivot row: a[p] / pivot, and 1 / pivot on the diagonal
    }
    // row r is in register (r - bj) mod 128
#pragma unroll
    for (int i = 0; i < kGJ; ++i) {
      const int r = (i + bj) & (kGJ - 1);
      store_x(D.Dp, D.Dp_lo, (long long)r * kGJ + c, (r < bj && c < bj) ? a[i] : 0.f, 1);
    }
  } else {
    // rows blockIdx.x - 1, + kGJCopy, ... of E: 16-B vectors (ld and buffers are 64-element
    // aligned), scalar tail when n % 4 != 0
    const int n4 = n >> 2;
    for (int r = blockIdx.x - 1; r < bj; r += kGJCopy) {
      const float4* sh = reinterpret_cast<const float4*>(static_cast<const float*>(D.R) + (long long)(J0 + r) * D.ldr);
      const float4* sl = reinterpret_cast<const float4*>(static_cast<const float*>(D.R_lo) + (long long)(J0 + r) * D.ldr);
      float4* dh = reinterpret_cast<float4*>(static_cast<float*>(D.E) + (long long)r * D.ldx);
      float4* dl = reinterpret_cast<float4*>(static_cast<float*>(D.E_lo) + (long long)r * D.ldx);
      for (int q = threadIdx.x; q < n4; q += kGJ) {
        const float4 h = sh[q], l = sl[q];
        dh[q] = h;
        dl[q] = l;
      }
      for (int c = 4 * n4 + threadIdx.x; c < n; c += kGJ) {
        static_cast<float*>(D.E)[(long long)r * D.ldx + c] = static_cast<const float*>(D.R)[(long long)(J0 + r) * D.ldr + c];
        static_cast<float*>(D.E_lo)[(long long)r * D.ldx + c] = static_cast<const float*>(D.R_lo)[(long long)(J0 + r) * D.ldr + c];
      }
    }
  }
}

// Sweep step j, part 4 (after T = D E and W -= E^T T): row block J of W <- T, column block
// J <- T^T, W_JJ <- -D.  After every step, W = -M^{-1} (sweep convention).  grid
// (ceil(n_max / 128), batch) 128-column strips, 256 threads, dynamic smem 66 KB.
__global__ void __launch_bounds__(256) k_gj_fix(SolveParams P, int j) {
  griddep_wait();
  griddep_launch();
  extern __shared__ float gsm[];
  const int b = blockIdx.y;
  const MatDesc& D = P.mats[b];
  if (P.st[b].done) return;
  const int n = D.s, J0 = kGJ * j;
  if (J0 >= n) return;
  const int bj = min(kGJ, n - J0);
  const int c0 = kGJ * blockIdx.x;
  if (c0 >= n) return;
  const int w = min(kGJ, n - c0);
  if (c0 == J0) {
    for (int e = threadIdx.x; e < bj * bj; e += 256) {
      const int r = e / bj, c = e % bj;
      store_x(D.R, D.R_lo, (long long)(J0 + r) * D.ldr + J0 + c, -ld_split(D.Dp, D.Dp_lo, (long long)r * kGJ + c), 1);
    }
    return;
  }
  float(*t)[kGJ + 1] = reinterpret_cast<float(*)[kGJ + 1]>(gsm);
  if (bj == kGJ && w == kGJ) {
    // whole 128 x 128 tile: 16-B loads / stores (hi + lo planes), transpose through smem
    const float* Th = static_cast<const float*>(D.T);
    const float* Tl = static_cast<const float*>(D.T_lo);
    float* Rh = static_cast<float*>(D.R);
    float* Rl = static_cast<float*>(D.R_lo);
#pragma unroll 4
    for (int q = threadIdx.x; q < kGJ * kGJ / 4; q += 256) {
      const int r = q >> 5, c4 = (q & 31) * 4;
      const long long src = (long long)r * D.ldx + c0 + c4;
      const float4 h = __ldg(reinterpret_cast<const float4*>(Th + src));
      const float4 l = __ldg(reinterpret_cast<const float4*>(Tl + src));
      const float v[4] = {h.x + l.x, h.y + l.y, h.z + l.z, h.w + l.w};
      float hv[4], lv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        t[r][c4 + e] = v[e];
        hv[e] = __uint_as_float(__float_as_uint(v[e]) & 0xFFFFE000u);
        lv[e] = v[e] - hv[e];
      }
      const long long dst = (long long)(J0 + r) * D.ldr + c0 + c4;   // row block
      *reinterpret_cast<float4*>(Rh + dst) = make_float4(hv[0], hv[1], hv[2], hv[3]);
      *reinterpret_cast<float4*>(Rl + dst) = make_float4(lv[0], lv[1], lv[2], lv[3]);
    }
    __syncthreads();
#pragma unroll 4
    for (int q = threadIdx.x; q < kGJ * kGJ / 4; q += 256) {
      const int c = q >> 5, r4 = (q & 31) * 4;
      float hv[4], lv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float v = t[r4 + e][c];
        hv[e] = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
        lv[e] = v - hv[e];
      }
      const long long dst = (long long)(c0 + c) * D.ldr + J0 + r4;   // column block
      *reinterpret_cast<float4*>(Rh + dst) = make_float4(hv[0], hv[1], hv[2], hv[3]);
      *reinterpret_cast<float4*>(Rl + dst) = make_float4(lv[0], lv[1], lv[2], lv[3]);
    }
    return;
  }
  for (int e = threadIdx.x; e < bj * w; e += 256) {
    const int r = e / w, c = e % w;
    const float v = ld_split(D.T, D.T_lo, (long long)r * D.ldx + c0 + c);
    t[r][c] = v;
    store_x(D.R, D.R_lo, (long long)(J0 + r) * D.ldr + c0 + c, v, 1);   // row block
  }
  __syncthreads();
  for (int e = threadIdx.x; e < bj * w; e += 256) {
    const int c = e / bj, r = e % bj;
    store_x(D.R, D.R_lo, (long long)(c0 + c) * D.ldr + J0 + r, t[r][c], 1);   // column block
  }
}

// <E1,E1>, <E1,E2>, <E2,E2> per tile, E1 = I - M^{-1} = I + W, E2 = I - M (fp64; R27).
__global__ void __launch_bounds__(256) k_db_reduce(SolveParams P, int bn) {
  griddep_wait();
  griddep_launch();
  __shared__ double scratch[8];
  const int b = blockIdx.z;
  const MatDesc& D = P.mats[b];
  if (P.st[b].done) return;
  const int tm = blockIdx.y, tn = blockIdx.x;
  if (tm >= D.tiles_m || tn >= D.tiles_n) return;
  const int n = D.s;
  double s11 = 0.0, s12 = 0.0, s22 = 0.0;
  for (int e = threadIdx.x; e < 128 * bn; e += 256) {
    const int i = tm * 128 + e / bn, j = tn * bn + e % bn;
    if (i >= n || j >= n) continue;
    const double d = (i == j) ? 1.0 : 0.0;
    const double e2 = d - (double)D.Mst[(long long)i * D.ldx + j];
    const double e1 = d + (double)ld_split(D.R, D.R_lo, (long long)i * D.ldr + j);
    s11 += e1 * e1; s12 += e1 * e2; s22 += e2 * e2;
  }
  s11 = block_sum<double, 256>(s11, scratch);
  s12 = block_sum<double, 256>(s12, scratch);
  s22 = block_sum<double, 256>(s22, scratch);
  if (threadIdx.x == 0) {
    double* o = D.dbpart + 3 * (tm * D.tiles_n + tn);
    o[0] = s11; o[1] = s12; o[2] = s22;
  }
}

// M_{k+1} = 2a(1-a) I + (1-a)^2 M_k + a^2 M_k^{-1}  (W = -M_k^{-1})
__global__ void __launch_bounds__(256) k_db_update(SolveParams P, int bn) {
  griddep_wait();
  griddep_launch();
  const int b = blockIdx.z;
  const MatDesc& D = P.mats[b];
  if (P.st[b].done) return;
  const int tm = blockIdx.y, tn = blockIdx.x;
  if (tm >= D.tiles_m || tn >= D.tiles_n) return;
  const int n = D.s;
  const double a = P.st[b].alpha;
  const float c0 = (float)(2.0 * a * (1.0 - a)), c1 = (float)((1.0 - a) * (1.0 - a)), c2 = (float)(a * a);
  for (int e = threadIdx.x; e < 128 * bn; e += 256) {
    const int i = tm * 128 + e / bn, j = tn * bn + e % bn;
    if (i >= n || j >= n) continue;
    float* m = D.Mst + (long long)i * D.ldx + j;
    *m = (i == j ? c0 : 0.f) + c1 * *m - c2 * ld_split(D.R, D.R_lo, (long long)i * D.ldr + j);
  }
}

// ----------------------------------------------------------------- a4: Philox sketch
// Portable Box–Muller (R8): only IEEE-exact +,-,*,/,sqrt with explicit
// round-to-nearest intrinsics (no FMA contraction), so the bits equal the oracle's.
__device__ __forceinline__ void philox10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint32_t lo0 = 0xD2511F53u * c[0], hi0 = __umulhi(0xD2511F53u, c[0]);
    const uint32_t lo1 = 0xCD9E8D57u * c[2], hi1 = __umulhi(0xCD9E8D57u, c[2]);
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
  }
}

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

__device__ double portable_log(double u) {
  int e;
  double m = frexp(u, &e);                     // u = m 2^e, m in [0.5, 1)
  if (m < 0.70710678118654752440) { m = dmul(m, 2.0); e -= 1; }
  const double f = dadd(m, -1.0);
  const double t = __ddiv_rn(f, dadd(2.0, f));
  const double t2 = dmul(t, t);
  double acc = 1.0 / 21.0;
  acc = dadd(dmul(acc, t2), 1.0 / 19.0);
  acc = dadd(dmul(acc, t2), 1.0 / 17.0);
  acc = dadd(dmul(acc, t2), 1.0 / 15.0);
  acc = dadd(dmul(acc, t2), 1.0 / 13.0);
  acc = dadd(dmul(acc, t2), 1.0 / 11.0);
  acc = dadd(dmul(acc, t2), 1.0 / 9.0);
  acc = dadd(dmul(acc, t2), 1.0 / 7.0);
  acc = dadd(dmul(acc, t2), 1.0 / 5.0);
  acc = dadd(dmul(acc, t2), 1.0 / 3.0);
  acc = dadd(dmul(acc, t2), 1.0);
  const double lnm = dmul(dmul(2.0, t), acc);
  const double ed = (double)e;
  return dadd(dmul(ed, 6.93147180369123816490e-01), dadd(dmul(ed, 1.90821492927058770002e-10), lnm));
}

// sin and cos of 2*pi*K*2^-53
__device__ void portable_sincos_2pi(unsigned long long K, double* so, double* co) {
  const unsigned long long q = (K + (1ull << 50)) >> 51;
  const long long di = (long long)K - (long long)(q << 51);
  const double d = dmul((double)di, 0x1p-51);   // exact
  const double x = dmul(d, 1.5707963267948966);
  const double x2 = dmul(x, x);
  // sin: sum_{j=0..10} (-1)^j x^(2j+1)/(2j+1)!
  double s = 1.0 / 51090942171709440000.0;                    // +1/21!
  s = dadd(dmul(s, x2), -1.0 / 121645100408832000.0);         // -1/19!
  s = dadd(dmul(s, x2), 1.0 / 355687428096000.0);             // +1/17!
  s = dadd(dmul(s, x2), -1.0 / 1307674368000.0);              // -1/15!
  s = dadd(dmul(s, x2), 1.0 / 6227020800.0);                  // +1/13!
  s = dadd(dmul(s, x2), -1.0 / 39916800.0);                   // -1/11!
  s = dadd(dmul(s, x2), 1.0 / 362880.0);                      // +1/9!
  s = dadd(dmul(s, x2), -1.0 / 5040.0);                       // -1/7!
  s = dadd(dmul(s, x2), 1.0 / 120.0);                         // +1/5!
  s = dadd(dmul(s, x2), -1.0 / 6.0);                          // -1/3!
  s = dadd(dmul(s, x2), 1.0);
  s = dmul(x, s);
  // cos: sum_{j=0..11} (-1)^j x^(2j)/(2j)!
  double c = -1.0 / 1124000727777607680000.0;                 // -1/22!
  c = dadd(dmul(c, x2), 1.0 / 2432902008176640000.0);         //  1/20!
  c = dadd(dmul(c, x2), -1.0 / 6402373705728000.0);           // -1/18!
  c = dadd(dmul(c, x2), 1.0 / 20922789888000.0);              //  1/16!
  c = dadd(dmul(c, x2), -1.0 / 87178291200.0);                // -1/14!
  c = dadd(dmul(c, x2), 1.0 / 479001600.0);                   //  1/12!
  c = dadd(dmul(c, x2), -1.0 / 3628800.0);                    // -1/10!
  c = dadd(dmul(c, x2), 1.0 / 40320.0);                       //  1/8!
  c = dadd(dmul(c, x2), -1.0 / 720.0);                        // -1/6!
  c = dadd(dmul(c, x2), 1.0 / 24.0);                          //  1/4!
  c = dadd(dmul(c, x2), -1.0 / 2.0);                          // -1/2!
  c = dadd(dmul(c, x2), 1.0);
  switch ((int)(q & 3ull)) {
    case 0: *so = s; *co = c; break;
    case 1: *so = c; *co = -s; break;
    case 2: *so = -s; *co = -c; break;
    default: *so = -c; *co = s; break;
  }
}

__device__ __forceinline__ void sketch_pair(unsigned long long seed, uint32_t k, uint32_t b, uint32_t e, double* z0,
                                            double* z1) {
  uint32_t ctr[4] = {e, k, b, 0x534B4348u};
  philox10(ctr, (uint32_t)(seed & 0xFFFFFFFFull), (uint32_t)(seed >> 32));
  const unsigned long long K1 = ((unsigned long long)(ctr[0] >> 5) << 26) + (ctr[1] >> 6);
  const unsigned long long K2 = ((unsigned long long)(ctr[2] >> 5) << 26) + (ctr[3] >> 6);
  const double u1 = dmul((double)(K1 + 1ull), 0x1p-53);   // (0, 1], exact
  const double rad = __dsqrt_rn(dmul(-2.0, portable_log(u1)));
  double sn, cs;
  portable_sincos_2pi(K2, &sn, &cs);
  *z0 = dmul(rad, cs);   // even element: cos
  *z1 = dmul(rad, sn);   // odd element: sin
}

__device__ __forceinline__ void store_split(void* W, long long idx_hi, long long idx_lo, float v, int bf16) {
  if (bf16) {
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    static_cast<__nv_bfloat16*>(W)[idx_hi] = h;
    static_cast<__nv_bfloat16*>(W)[idx_lo] = __float2bfloat16_rn(v - __bfloat162float(h));
  } else {
    const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    static_cast<float*>(W)[idx_hi] = h;
    static_cast<float*>(W)[idx_lo] = v - h;
  }
}

// S_k (p x s, fp32) for every active matrix, and the first chain operand
// W[0] = [S_hi ; S_lo] (compute dtype).  grid (ceil(p*s/2/256), batch).
__device__ __forceinline__ bool fit_at(const SolveParams& P, int k) {
  return P.fit == 0 && k < P.max_iters && k >= P.warmup;
}

// Residual stage end + sketch, one launch after the residual product (GEMM epilogue or SIMT
// kernel wrote the per-tile sums of R^2): block x = 0 of matrix b runs the stop test of
// iteration k (R12) on ||R_k||_F from every norm partial (fixed order), so the chain, alpha,
// square and apply launches of iteration k all skip a matrix that stops here; blocks x >= 1
// draw S_k (and W = [S_hi; S_lo]) for the fit.  grid (1 + ceil(p s / 2 / 256), batch).
__global__ void __launch_bounds__(256) k_stop_sketch(SolveParams P) {
  griddep_wait();
  griddep_launch();
  const int b = blockIdx.y;
  const MatDesc& D = P.mats[b];
  const int k = *P.iter;
  if (blockIdx.x == 0) {
    __shared__ double scratch[8];
    MatState& S = P.st[b];
    if (S.done) return;
    double part = 0.0;
    const int nparts = D.tiles_m * D.tiles_n;   // unscheduled (lower-triangle) entries stay 0
    for (int t = threadIdx.x; t < nparts; t += 256) part += (double)D.norm_part[t];
    const double r2 = block_sum<double, 256>(part, scratch);
    if (threadIdx.x == 0) {
      const double r = sqrt(r2), s = (double)D.s;
      int stop = 0, status = 1, incr = 0;
      if (!isfinite(r)) { stop = 1; status = 3; }
      else if (r <= P.tol * sqrt(s)) { stop = 1; status = 0; }
      else {
        incr = (k >= 1 && r > S.r_prev) ? S.incr + 1 : 0;
        if (incr >= 5) { stop = 1; status = 2; }
        else if (k >= P.max_iters) { stop = 1; status = 1; }
      }
      P.resid_hist[(size_t)b * (P.max_iters + 1) + k] = (float)(r / sqrt(s));
      if (isfinite(r) && !(r <= P.tol * sqrt(s))) S.incr = incr;
      S.r_prev = r;
      S.resid = (float)(r / sqrt(s));
      S.iters = k;
      if (stop) {
        S.stop_iter = k;
        S.status = status;
        S.done = 1;
      }
    }
    return;
  }
  if (!fit_at(P, k) || P.st[b].done) return;
  const int s = D.s, p = P.p;
  const long long total = (long long)p * s;
  const long long e = (long long)(blockIdx.x - 1) * 256 + threadIdx.x;   // pair index
  if (2 * e >= total) return;
  double z[2];
  sketch_pair(P.seed, (uint32_t)k, (uint32_t)D.sketch_id, (uint32_t)e, &z[0], &z[1]);
  const int bf16 = P.precision == 0;
  for (int t = 0; t < 2; ++t) {
    const long long q = 2 * e + t;
    if (q >= total) break;
    const int row = (int)(q / s), col = (int)(q - (long long)row * s);
    const float v = __double2float_rn(z[t]);
    D.S[(long long)row * D.ldS + col] = v;
    // chain operand [S_hi; S_lo] of the row's chunk (prism.cu: chunks of 8 sketch rows)
    const int ch = D.nchunk > 1 ? row >> 3 : 0, r = D.nchunk > 1 ? row & 7 : row;
    const int pc = D.nchunk > 1 ? min(8, p - 8 * ch) : p, pw = D.nchunk > 1 ? 8 : p;
    const long long base = (long long)ch * 4 * pw * D.ldS;
    store_split(D.W[0], base + (long long)r * D.ldS + col, base + (long long)(pc + r) * D.ldS + col, v, bf16);
  }
}

// ----------------------------------------------------------------- a5: coefficient solve
// Real roots of a3 x^3 + a2 x^2 + a1 x + a0 (closed form; used by DB Newton's unconstrained
// argmin, R27, whose quartic has c4 = ||E1 + E2||^2 of the order of the other terms).
__device__ int real_roots_cubic(double a3, double a2, double a1, double a0, double* roots) {
  const double big = fmax(fabs(a2), fmax(fabs(a1), fabs(a0)));
  if (fabs(a3) <= 1e-12 * big) {
    if (fabs(a2) <= 1e-12 * fmax(fabs(a1), fabs(a0))) {
      if (a1 != 0.0) { roots[0] = -a0 / a1; return 1; }
      return 0;
    }
    const double disc = a1 * a1 - 4.0 * a2 * a0;
    if (disc < 0.0) return 0;
    const double sq = sqrt(disc);
    const double q = -0.5 * (a1 + (a1 >= 0.0 ? sq : -sq));
    roots[0] = q / a2;
    if (q != 0.0) { roots[1] = a0 / q; return 2; }
    return 1;
  }
  const double b = a2 / a3, c = a1 / a3, d = a0 / a3;
  const double p = c - b * b / 3.0;
  const double q = 2.0 * b * b * b / 27.0 - b * c / 3.0 + d;
  const double shift = -b / 3.0;
  const double disc = (q / 2.0) * (q / 2.0) + (p / 3.0) * (p / 3.0) * (p / 3.0);
  if (disc > 0.0) {
    const double sq = sqrt(disc);
    const double A = -copysign(1.0, q) * cbrt(fabs(q) / 2.0 + sq);
    const double t = (A != 0.0) ? A - p / (3.0 * A) : 0.0;
    roots[0] = t + shift;
    return 1;
  }
  if (p == 0.0) { roots[0] = shift; return 1; }
  const double r = 2.0 * sqrt(-p / 3.0);
  double arg = (3.0 * q / (2.0 * p)) * sqrt(-3.0 / p);
  arg = fmin(1.0, fmax(-1.0, arg));
  const double phi = acos(arg) / 3.0;
  for (int j = 0; j < 3; ++j) roots[j] = r * cos(phi - 2.0 * 3.14159265358979323846 * j / 3.0) + shift;
  return 3;
}


// Interval argmin of the quartic m(a) = sum c_i a^i on [lo, hi] (readings R15, R16):
// the roots of m'' (a quadratic: one sqrt) split [lo, hi] into at most three pieces on
// which m' is monotone; a piece whose ends have m' < 0 <= m' holds exactly one local
// minimum of m, bracketed to 1/32 of the piece by the warp's 32 samples of m', then located
// by Newton steps safeguarded by bisection (the bracket keeps m'(x0) < 0 <= m'(x1), so the
// limit is that minimum to the last bits).  Warp-collective: every lane passes the same c.  Candidates
// {lo, hi} U minima, the smallest m wins (ties -> smaller a); degenerate loss -> Taylor.
// (The closed-form Cardano roots this replaces lost the moderate roots when |c4| << |c3|
// and missed minima; its fp64 acos / cos / cbrt also cost 9-13 us inside k_alpha.)
__device__ double argmin_quartic(const double c[5], double lo, double hi, double aT) {
  const double scale = fmax(fmax(fabs(c[1]), fabs(c[2])), fmax(fabs(c[3]), fabs(c[4])));
  if (!isfinite(scale)) return aT;
  if (scale == 0.0 || scale <= 1e-14 * fabs(c[0])) return aT;
  const double d1 = c[1] / scale, d2 = c[2] / scale, d3 = c[3] / scale, d4 = c[4] / scale;
  auto m = [&](double a) { return (((d4 * a + d3) * a + d2) * a + d1) * a; };
  auto mp = [&](double a) { return ((4.0 * d4 * a + 3.0 * d3) * a + 2.0 * d2) * a + d1; };
  auto mpp = [&](double a) { return (12.0 * d4 * a + 6.0 * d3) * a + 2.0 * d2; };
  // breakpoints: lo, the roots of m'' inside (lo, hi), hi
  double br[4];
  int nb = 0;
  br[nb++] = lo;
  {
    const double A = 12.0 * d4, Bq = 6.0 * d3, Cq = 2.0 * d2;
    double r0 = NAN, r1 = NAN;
    if (A != 0.0) {
      const double disc = Bq * Bq - 4.0 * A * Cq;
      if (disc >= 0.0) {
        const double sq = sqrt(disc);
        const double q = -0.5 * (Bq + (Bq >= 0.0 ? sq : -sq));
        r0 = q / A;
        r1 = q != 0.0 ? Cq / q : r0;
      }
    } else if (Bq != 0.0) {
      r0 = -Cq / Bq;
    }
    if (r0 > r1) { const double t = r0; r0 = r1; r1 = t; }
    if (r0 > lo && r0 < hi) br[nb++] = r0;
    if (r1 > lo && r1 < hi && r1 != r0) br[nb++] = r1;
  }
  br[nb++] = hi;
  double best = lo, bm = m(lo);
  {
    const double mh = m(hi);
    if (mh < bm) { best = hi; bm = mh; }
  }
  const int lane = threadIdx.x & 31;
  for (int j = 0; j + 1 < nb; ++j) {
    double x0 = br[j], x1 = br[j + 1];
    if (!(mp(x0) < 0.0 && mp(x1) >= 0.0)) continue;
    {
      // m' increases through the piece: the warp samples it at 32 points and the first
      // lane with m' >= 0 narrows the bracket 32-fold, so Newton starts next to the root
      const double xl = lane == 31 ? x1 : x0 + (x1 - x0) * (double)(lane + 1) * (1.0 / 32.0);
      const unsigned pos = __ballot_sync(0xffffffffu, mp(xl) >= 0.0) | 0x80000000u;
      const int f = __ffs(pos) - 1;
      const double b1 = __shfl_sync(0xffffffffu, xl, f);
      const double b0 = __shfl_sync(0xffffffffu, xl, f > 0 ? f - 1 : 0);
      if (f > 0) x0 = b0;
      x1 = b1;
    }
    double x = 0.5 * (x0 + x1);
    for (int it = 0; it < 100; ++it) {
      const double f = mp(x);
      if (f < 0.0) x0 = x; else x1 = x;
      const double fp = mpp(x);
      double xn = (fp != 0.0) ? x - f / fp : 0.5 * (x0 + x1);
      if (!(xn > x0 && xn < x1)) xn = 0.5 * (x0 + x1);   // Newton left the bracket: bisect
      if (xn == x || xn <= x0 || xn >= x1) { x = (xn > x0 && xn < x1) ? xn : x; break; }
      x = xn;
    }
    // the bracket end on the non-negative side is the reported root (argmin_poly_warp rule)
    const double r = mp(x) >= 0.0 ? x : x1;
    const double mr = m(r);
    if (mr < bm || (mr == bm && r < best)) { best = r; bm = mr; }
  }
  return best;
}

// argmin_{a in [lo, hi]} of m(a) = sum_{i<=deg} c_i a^i for deg > 4 (inverse Newton q >= 3,
// R23), one warp: [lo, hi] cut into 32 cells; a cell whose ends have m' < 0 <= m' holds a
// local minimum, located by bisection of m'; candidates {lo, hi} U those minima, smallest m
// wins (ties -> smaller a); degenerate loss -> Taylor.  Every lane returns the result.
__device__ double argmin_poly_warp(const double* c, int deg, double lo, double hi, double aT) {
  const int lane = threadIdx.x & 31;
  double scale = 0.0;
  for (int i = 1; i <= deg; ++i) scale = fmax(scale, fabs(c[i]));
  if (!isfinite(scale)) return aT;
  if (scale == 0.0 || scale <= 1e-14 * fabs(c[0])) return aT;
  double d[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) d[i] = i <= deg ? c[i] / scale : 0.0;
  auto m = [&](double a) {   // c0 dropped: argmin-invariant
    double v = 0.0;
#pragma unroll
    for (int i = 8; i >= 1; --i) v = (v + d[i]) * a;
    return v;
  };
  auto mp = [&](double a) {
    double v = 0.0;
#pragma unroll
    for (int i = 8; i >= 1; --i) v = v * a + i * d[i];
    return v;
  };
  const double a0 = lo + (hi - lo) * lane / 32.0;
  const double a1 = lane == 31 ? hi : lo + (hi - lo) * (lane + 1) / 32.0;
  double best = lane == 0 ? lo : INFINITY, bm = lane == 0 ? m(lo) : INFINITY;
  if (lane == 31) {
    const double mh = m(hi);
    if (mh < bm) { best = hi; bm = mh; }
  }
  if (mp(a0) < 0.0 && mp(a1) >= 0.0) {
    double x0 = a0, x1 = a1;
    for (int it = 0; it < 64; ++it) {
      const double xm = 0.5 * (x0 + x1);
      if (xm <= x0 || xm >= x1) break;
      if (mp(xm) < 0.0) x0 = xm; else x1 = xm;
    }
    const double mr = m(x1);
    if (mr < bm || (mr == bm && x1 < best)) { best = x1; bm = mr; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o), om = __shfl_xor_sync(0xffffffffu, bm, o);
    if (om < bm || (om == bm && ob < best)) { best = ob; bm = om; }
  }
  return best;
}

// Unconstrained argmin of the quartic (DB Newton, R27): the real roots of m' (two Newton
// polishes), smallest m (ties -> smaller a); c4 <= 0 or degenerate -> a_default.
__device__ double argmin_quartic_free(const double c[5], double a_default) {
  const double scale = fmax(fmax(fabs(c[1]), fabs(c[2])), fmax(fabs(c[3]), fabs(c[4])));
  if (!isfinite(scale) || scale == 0.0 || scale <= 1e-14 * fabs(c[0]) || !(c[4] > 0.0)) return a_default;
  const double d1 = c[1] / scale, d2 = c[2] / scale, d3 = c[3] / scale, d4 = c[4] / scale;
  double roots[3];
  const int nr = real_roots_cubic(4.0 * d4, 3.0 * d3, 2.0 * d2, d1, roots);
  double best = a_default, bm = INFINITY;
  double cand[3];
  int nc = 0;
  for (int i = 0; i < nr; ++i) {
    double r = roots[i];
    for (int it = 0; it < 2; ++it) {
      const double m2 = (12.0 * d4 * r + 6.0 * d3) * r + 2.0 * d2;
      if (m2 != 0.0) {
        const double m1 = ((4.0 * d4 * r + 3.0 * d3) * r + 2.0 * d2) * r + d1;
        const double nr2 = r - m1 / m2;
        if (isfinite(nr2)) r = nr2;
      }
    }
    if (isfinite(r)) cand[nc++] = r;
  }
  for (int i = 1; i < nc; ++i)
    for (int j = i; j > 0 && cand[j] < cand[j - 1]; --j) { double t = cand[j]; cand[j] = cand[j - 1]; cand[j - 1] = t; }
  for (int i = 0; i < nc; ++i) {
    const double a = cand[i];
    const double ma = (((d4 * a + d3) * a + d2) * a + d1) * a;
    if (ma < bm) { best = a; bm = ma; }
  }
  return best;
}

// One block (256 threads) per matrix: residual norm, stop test (R12), and
// alpha_k from the factored sketched loss m(a) = ||V0 + a V1 + a^2 V2||^2.
// pre_wait = 1: the residual's norm partials were written at least two launches back (a
// sketch chain or the DB sweep runs in between), so the stop test is computed before
// waiting for the predecessor (its state writes still follow the wait: the predecessor
// reads the done flags); only the fit's inputs come from the predecessor.
// alpha_k of every active matrix: one warp per matrix, fp64.  Instantiated per kind so each
// launch carries only its own fit (a kernel holding every kind's argmin stalled on
// instruction fetch: ncu stall_no_inst 50 %): AK 0 polar / sqrt / sign (quartic of the
// factored loss), 1 Chebyshev (quadratic), 2 inverse Newton (degree 2q), 3 DB Newton (free quartic).
// One warp per matrix, kAlphaWarps matrices per block: the fit occupies ceil(B / 8) SMs,
// not B (a block on an SM keeps a GEMM CTA — which needs the whole register file — off it;
// the early square GEMM runs its mainloop on the others, prism.cu).
constexpr int kAlphaWarps = 8;

// k_alpha's extra blocks (kCompactBlocks, after the fit blocks): after this iteration's stop
// test (several launches back), the square and apply of this iteration and the next Gram
// need only the tiles of matrices still active; each list keeps its plan order with the runs
// of stopped matrices dropped, and the GEMMs stride over the active tiles alone (tail
// iterations: no pair holds several of the few remaining tiles while others idle).  Any
// order computes the same bits (per-element arithmetic never depends on the tile schedule).
// Every block derives the run prefix sums (runs in shared memory), then writes its share of
// the compacted lists, each element found by a binary search over the run prefixes.
constexpr int kCompactBlocks = 8;
__device__ void compact_tile_lists(const SolveParams& P, int cb) {
  __shared__ int s_pre[3][kMaxCompactRuns + 1];   // prefix of the active lengths (inactive: 0)
  __shared__ int s_src[3][kMaxCompactRuns];       // first source index of each run
  const int T = blockDim.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = T >> 5;
  const int nl = P.ncompact;
  int tot = 0;
  for (int l = 0; l < nl; ++l) tot += P.clist[l].nruns;
  // run lengths (0 for stopped matrices) and starts, all lists at once
  for (int x = threadIdx.x; x < tot; x += T) {
    int l = 0, r = x;
    while (r >= P.clist[l].nruns) r -= P.clist[l].nruns, ++l;
    const int* run = P.clist[l].runs + 3 * r;
    const int st = run[0], len = run[1], mat = run[2];
    s_src[l][r] = st;
    s_pre[l][r + 1] = P.st[mat].done ? 0 : len;
  }
  __syncthreads();
  for (int l = warp; l < nl; l += nw) {   // one warp per list: in-place inclusive scan
    const int n = P.clist[l].nruns;
    int carry = 0;
    if (lane == 0) s_pre[l][0] = 0;
    for (int r0 = 0; r0 < n; r0 += 32) {
      const int r = r0 + lane;
      int v = r < n ? s_pre[l][r + 1] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (r < n) s_pre[l][r + 1] = carry + v;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  for (int l = 0; l < nl; ++l) {
    const CompactList& C = P.clist[l];
    const int n = C.nruns, total = s_pre[l][n];
    const int per = (total + kCompactBlocks - 1) / kCompactBlocks;
    const int lo = cb * per, hi = min(total, lo + per);
    for (int d = lo + threadIdx.x; d < hi; d += T) {
      int a = 0, b = n;   // last run r with s_pre[r] <= d (zero-length runs precede their successor)
      while (b - a > 1) {
        const int m = (a + b) >> 1;
        if (s_pre[l][m] <= d) a = m; else b = m;
      }
      C.dst[d] = C.src[s_src[l][a] + d - s_pre[l][a]];
    }
    if (cb == 0 && threadIdx.x == 0) *C.count = total;
  }
}

template <int AK>
__global__ void __launch_bounds__(32 * kAlphaWarps) k_alpha(SolveParams P, int) {
  griddep_wait();
  griddep_launch();
  if constexpr (AK != 3) {
    const int cb = (int)blockIdx.x - (int)(gridDim.x - (P.ncompact ? kCompactBlocks : 0));
    if (cb >= 0) {
      compact_tile_lists(P, cb);
      return;
    }
  }
  const int k = *P.iter;
  const int do_fit = AK == 3 ? (P.fit != 1 && k < P.max_iters && k >= P.warmup) : (fit_at(P, k) ? 1 : 0);
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= P.batch) return;
  const MatDesc& D = P.mats[b];
  MatState& S = P.st[b];
  if (S.done) return;   // stopped in this iteration's residual stage (or earlier)
  double a;
  if (!do_fit) {
    a = (k < P.warmup) ? P.ahi : P.ataylor;
  } else if constexpr (AK == 3) {
    // <E1,E1>, <E1,E2>, <E2,E2> over the tiles (fixed order) -> the exact quartic
    // m(a) = a^4 <E1,E1> + 2 a^2 (1-a)^2 <E1,E2> + (1-a)^4 <E2,E2>  (R27)
    double s3[3] = {0.0, 0.0, 0.0};
    const int nt = D.tiles_m * D.tiles_n;
    for (int t = lane; t < nt; t += 32)
#pragma unroll
      for (int j = 0; j < 3; ++j) s3[j] += D.dbpart[3 * t + j];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s3[j] += __shfl_xor_sync(0xffffffffu, s3[j], o);
      s3[j] = __shfl_sync(0xffffffffu, s3[j], 0);   // lane 0's sums everywhere (no divergence)
    }
    const double A1 = s3[0], B1 = s3[1], C1 = s3[2];
    const double c[5] = {C1, -4.0 * C1, 2.0 * B1 + 6.0 * C1, -4.0 * B1 - 4.0 * C1, A1 + 2.0 * B1 + C1};
    a = argmin_quartic_free(c, P.ataylor);
  } else {
    // <Va, Vb> from the chain's per-32-row-group partials (R17): lane l
    // sums groups l, l+32, ... in order, then a fixed xor tree — reproducible bit for bit
    constexpr int NGMAX = AK == 0 ? 6 : AK == 1 ? 3 : kChainG;
    const int q = P.inv_q;
    const int ng = AK == 2 ? (q + 1) * (q + 2) / 2 : NGMAX;
    double g[NGMAX];
#pragma unroll
    for (int j = 0; j < NGMAX; ++j) g[j] = 0.0;
    const double* __restrict__ cpart = D.chain_part;
    const int ctiles = D.chain_tiles;
#pragma unroll 4
    for (int t = lane; t < ctiles; t += 32) {   // four groups' loads in flight per lane
      const double* cp = cpart + kChainG * t;
#pragma unroll
      for (int j = 0; j < NGMAX; ++j)
        if (j < ng) g[j] += cp[j];
    }
#pragma unroll
    for (int j = 0; j < NGMAX; ++j) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) g[j] += __shfl_xor_sync(0xffffffffu, g[j], o);
    }
    // every lane takes lane 0's sums: the xor tree adds in a lane-dependent order, and
    // lanes whose last bits differed took different branches of the argmin (a divergent
    // warp ran it ~8x slower); lane 0's values are the ones whose alpha is stored
#pragma unroll
    for (int j = 0; j < NGMAX; ++j) g[j] = __shfl_sync(0xffffffffu, g[j], 0);
    if constexpr (AK == 1) {
      // Chebyshev: m(a) = ||U - a V||^2 (R26), closed form on [1/2, 2]
      double c[5] = {g[0], -2.0 * g[1], g[2], 0.0, 0.0};
      a = (k < P.warmup) ? P.ahi : argmin_quartic(c, P.alo, P.ahi, P.ataylor);
    } else if constexpr (AK == 2) {
      // inverse Newton: m(a) = ||sum_i a^i V_i||^2 -> c_{i+j} += (2 - [i == j]) <V_i, V_j>
      double c[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      int idx = 0;
      for (int i = 0; i <= q; ++i)
        for (int j = i; j <= q; ++j) c[i + j] += (i == j ? 1.0 : 2.0) * g[idx++];
      if (k < P.warmup) a = P.ahi;
      else if (q <= 2) a = argmin_quartic(c, P.alo, P.ahi, P.ataylor);   // degree <= 4
      else a = argmin_poly_warp(c, 2 * q, P.alo, P.ahi, P.ataylor);
    } else {
      double c[5] = {g[0], 2.0 * g[1], g[3] + 2.0 * g[2], 2.0 * g[4], g[5]};
      a = (k < P.warmup) ? P.ahi : argmin_quartic(c, P.alo, P.ahi, P.ataylor);
    }
  }
  if (lane == 0) {
    S.alpha = a;
    P.alpha_hist[(size_t)b * P.max_iters + k] = a;
  }
}

// ----------------------------------------------------------------- a7: outputs
// a7: polar Q = X_final; sqrt A^{1/2} = sqrt(c) X, A^{-1/2} = Y / sqrt(c) (cast to the user dtype).
template <int PREC>
__global__ void __launch_bounds__(256) k_finalize(SolveParams P) {
  griddep_wait();
  griddep_launch();
  using V = Vec<PREC>;
  using VO = Vec<PREC == 0 ? 0 : 2>;   // user output: bf16 or plain fp32
  const int t = blockIdx.x;
  const int b = __ldg(P.tile_mat + t);
  const MatDesc& D = P.mats[b];
  const int Dm = D.m, Dn = D.n;
  const long long Dldx = D.ldx, Dldq = D.ldq;
  void* const DQ = D.Q;
  void* const DQ2 = D.Q2;
  const MatState& S = P.st[b];
  const int par = S.iters & 1;
  const bool zero = S.status == 4;   // ZERO_INPUT: output 0 (X may be an unwritten buffer)
  if (D.fold && P.parity && t == P.out_tile_off[b] && threadIdx.x == 0) P.parity[b] = par;   // next solve's flip
  // folded plans: X[0] is the caller's output itself, holding the even iterates (odd ones with
  // S.flip): nothing to copy when the last one landed there; X[1] (workspace) holds the
  // others.  X_0 = A/||A||_F was never written (a solve that stops at k = 0 writes it here).
  const bool from_a = D.fold && S.iters == 0 && !zero;
  if (D.fold && (par ^ S.flip) == 0 && !zero && !from_a) return;
  const int src = D.fold ? 1 : par;
  const void* const Xp = D.X[src];
  const void* const Xpl = D.X_lo[src];
  const void* const Yp = D.Y[par];
  const void* const Ypl = D.Y_lo[par];
  const int TW = 32 * V::VE;
  const int tcn = (Dn + TW - 1) / TW;
  const int lt = t - P.out_tile_off[b];
  const int r0 = (lt / tcn) * 32, c0 = (lt % tcn) * TW;
  const float fs = P.kind_sqrt ? (float)sqrt(S.c) : 1.f;
  const float fi = (P.kind_sqrt && S.c > 0.0) ? (float)(1.0 / sqrt(S.c)) : 0.f;
  const bool q_vec = ((Dldq * V::ESZ) % 16 == 0);
  const bool two = (P.kind_sqrt || P.kind_db) && DQ2;
  const float sq = P.kind_db ? 1.f : P.kind_cheb ? (S.c > 0.0 ? (float)(1.0 / S.c) : 0.f)
                               : (P.kind_sqrt && S.c > 0.0) ? fs : (P.kind_sqrt ? 0.f : 1.f);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int slot = threadIdx.x + 256 * j;
    const int r = r0 + slot / 32, col = c0 + (slot % 32) * V::VE;
    if (r >= Dm || col >= Dn) continue;
    const int nv = min(V::VE, Dn - col);
    const long long xi = (long long)r * (src ? Dldx : D.ldx0) + col, qi = (long long)r * Dldq + col;
    const long long yi = (long long)r * Dldx + col;
    if (DQ) {
      V x;
      if (zero) {
#pragma unroll
        for (int e = 0; e < V::VE; ++e) x.v[e] = 0.f;
      } else if (from_a) {
        x.load(D.A, nullptr, (long long)r * D.lda + col, nv, false);
#pragma unroll
        for (int e = 0; e < V::VE; ++e) x.v[e] *= (float)S.inv_c;
      } else {
        x.load(Xp, Xpl, xi, nv, nv == V::VE);
      }
      VO o;
#pragma unroll
      for (int e = 0; e < V::VE; ++e) o.v[e] = x.v[e];
      const bool vq = q_vec && nv == V::VE && ((reinterpret_cast<uintptr_t>(DQ) & 15) == 0);
      o.store(DQ, nullptr, qi, nv, vq, sq, false);
    }
    if (two) {
      V y;
      y.load(Yp, Ypl, yi, nv, nv == V::VE);
      VO o;
#pragma unroll
      for (int e = 0; e < V::VE; ++e) o.v[e] = y.v[e];
      const bool vq = q_vec && nv == V::VE && ((reinterpret_cast<uintptr_t>(DQ2) & 15) == 0);
      o.store(DQ2, nullptr, qi, nv, vq, P.kind_db ? 1.f : fi, false);
    }
  }
}

// End of one loop iteration: k <- k + 1; keep looping while any matrix is active.
// (In the CUDA-graph path this sets the WHILE node's condition on the device.)
__global__ void k_advance(SolveParams P, cudaGraphConditionalHandle handle, int use_handle, int* all_done_out) {
  griddep_wait();
  griddep_launch();
  __shared__ int active;
  if (threadIdx.x == 0) active = 0;
  __syncthreads();
  int a = 0;
  for (int b = threadIdx.x; b < P.batch; b += blockDim.x) a |= !P.st[b].done;
  if (a) atomicOr(&active, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    *P.iter = *P.iter + 1;
    if (all_done_out) *all_done_out = active ? 0 : 1;
    if (use_handle) cudaGraphSetConditional(handle, active ? 1u : 0u);
  }
}

// Copy the solve's report (state + histories kept in the workspace) to the caller's buffers.
__global__ void k_report(SolveParams P) {
  griddep_wait();
  griddep_launch();
  const int nh = P.max_iters, nr = P.max_iters + 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.batch * nr; i += gridDim.x * blockDim.x) {
    const int b = i / nr, k = i - b * nr;
    const int it = P.st[b].iters;
    if (P.rep_resid_hist) P.rep_resid_hist[i] = (k <= it) ? P.resid_hist[i] : __int_as_float(0x7fc00000);
    if (P.rep_alphas && k < nh) P.rep_alphas[(size_t)b * nh + k] = (k < it) ? P.alpha_hist[(size_t)b * nh + k] : __longlong_as_double(0x7ff8000000000000ll);
    if (k == 0) {
      if (P.rep_iters) P.rep_iters[b] = it;
      if (P.rep_resid) P.rep_resid[b] = P.st[b].resid;
      if (P.rep_status) P.rep_status[b] = P.st[b].status;
    }
  }
}

}  // namespace prism
