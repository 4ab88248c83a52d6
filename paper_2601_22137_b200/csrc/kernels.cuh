// SIMT kernels of the PRISM iteration (everything that is not a dense
// contraction): Frobenius pre-scaling, layout/cast, the Philox sketch, the
// thin sketch chain, the single-CTA fp64 coefficient solve, and the output
// write-back.  All reductions are fixed-order (no float atomics), so results
// are bit-reproducible run to run.
#pragma once
#include "ptx.cuh"

namespace prism {

// Per-matrix solver state (device memory, one per matrix of the batch).
struct MatState {
  double c;          // ||A||_F
  double alpha;      // current alpha_k (read by GEMM epilogues)
  double r_prev;     // ||R_{k-1}||_F
  float resid;       // ||R_final||_F / sqrt(s)
  int done;          // 1 once the matrix stopped (skip all further work)
  int iters;         // updates applied
  int status;        // PRISM_CONVERGED ...
  int incr;          // consecutive residual increases
  int pad_;
};

// Per-matrix static description (device memory).
struct MatDesc {
  const void* A;       // user input (row-major, lda)
  void* Q;             // polar output / sqrt output
  void* Q2;            // inv-sqrt output (sqrt path) or null
  long long lda, ldq;
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
  float* S;            // [p x s] sketch
  float* chain;        // chain buffers: 5 blocks of [s x 2p]
};

struct SolveParams {
  MatDesc* mats;
  MatState* st;
  double* alpha_hist;   // [batch * max_iters] or null (user)
  float* resid_hist;    // [batch * (max_iters+1)] or null (user)
  int32_t* rep_iters;   // user report (device) or null
  float* rep_resid;
  int32_t* rep_status;
  double* fro_part;     // [batch * kFroParts]
  int batch, p, d, max_iters, warmup, fit, precision, kind_sqrt;
  double tol, alo, ahi, ataylor;
  unsigned long long seed;
};

constexpr int kFroParts = 32;

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

// ----------------------------------------------------------------- a1: ||A||_F partials
// grid (kFroParts, batch), 256 threads; block j handles rows r = j, j+kFroParts, ...
__global__ void __launch_bounds__(256) k_fro_partials(SolveParams P) {
  __shared__ double scratch[8];
  const MatDesc& D = P.mats[blockIdx.y];
  const int bf16 = P.precision == 0;
  double acc = 0.0;
  for (int r = blockIdx.x; r < D.m; r += kFroParts) {
    for (int c = threadIdx.x; c < D.n; c += 256) {
      double x = (double)load_val(D.A, (long long)r * D.lda + c, bf16);
      acc += x * x;
    }
  }
  acc = block_sum<double, 256>(acc, scratch);
  if (threadIdx.x == 0) P.fro_part[blockIdx.y * kFroParts + blockIdx.x] = acc;
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

// a1: X_0 = A / ||A||_F in the compute layout (polar: Xt = s x L), Y_0 = I (sqrt),
// state init.  grid (ceil(cols/32), ceil(rows/32), batch) over the *output* Xt,
// 32x8 threads with a smem transpose for the tall case.
__global__ void __launch_bounds__(256) k_normalize(SolveParams P) {
  __shared__ float tile[32][33];
  const int b = blockIdx.z;
  const MatDesc& D = P.mats[b];
  // every block recomputes c from the fixed-order partials (deterministic)
  double ss = 0.0;
  for (int j = 0; j < kFroParts; ++j) ss += P.fro_part[b * kFroParts + j];
  const double c = sqrt(ss);
  const float inv = c > 0.0 ? (float)(1.0 / c) : 0.f;
  const int bf16 = P.precision == 0;
  const int rows = P.kind_sqrt ? D.n : D.s;   // rows of Xt
  const int cols = P.kind_sqrt ? D.n : D.L;
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  if (r0 >= rows || c0 >= cols) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  if (D.trans) {
    // Xt[r][c] = A[c][r]: read A rows c0.. (coalesced over r), transpose through smem
    for (int k = ty; k < 32; k += 8) {
      const int ar = c0 + k, ac = r0 + tx;
      tile[k][tx] = (ar < D.m && ac < D.n) ? load_val(D.A, (long long)ar * D.lda + ac, bf16) : 0.f;
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
      const int xr = r0 + k, xc = c0 + tx;
      if (xr < rows && xc < cols) store_x(D.X[0], D.X_lo[0], (long long)xr * D.ldx + xc, tile[tx][k] * inv, P.precision);
    }
  } else {
    for (int k = ty; k < 32; k += 8) {
      const int xr = r0 + k, xc = c0 + tx;
      if (xr < rows && xc < cols) {
        float v = load_val(D.A, (long long)xr * D.lda + xc, bf16) * inv;
        store_x(D.X[0], D.X_lo[0], (long long)xr * D.ldx + xc, v, P.precision);
        if (P.kind_sqrt) store_x(D.Y[0], D.Y_lo[0], (long long)xr * D.ldx + xc, xr == xc ? 1.f : 0.f, P.precision);
      }
    }
  }
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    MatState& S = P.st[b];
    S.c = c;
    S.alpha = P.ataylor;
    S.r_prev = INFINITY;
    S.resid = 0.f;
    S.iters = 0;
    S.incr = 0;
    S.done = (c == 0.0) ? 1 : 0;
    S.status = (c == 0.0) ? 4 : 1;   // ZERO_INPUT / MAX_ITERS until decided
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

// S_k (p x s, fp32) for every active matrix.  grid (ceil(p*s/2/256), batch).
__global__ void __launch_bounds__(256) k_sketch(SolveParams P, int k) {
  const int b = blockIdx.y;
  const MatDesc& D = P.mats[b];
  if (P.st[b].done) return;
  const int s = D.s;
  const long long total = (long long)P.p * s;
  const long long e = (long long)blockIdx.x * 256 + threadIdx.x;   // pair index
  if (2 * e >= total) return;
  uint32_t ctr[4] = {(uint32_t)e, (uint32_t)k, (uint32_t)D.sketch_id, 0x534B4348u};
  philox10(ctr, (uint32_t)(P.seed & 0xFFFFFFFFull), (uint32_t)(P.seed >> 32));
  const unsigned long long K1 = ((unsigned long long)(ctr[0] >> 5) << 26) + (ctr[1] >> 6);
  const unsigned long long K2 = ((unsigned long long)(ctr[2] >> 5) << 26) + (ctr[3] >> 6);
  const double u1 = dmul((double)(K1 + 1ull), 0x1p-53);   // (0, 1], exact
  const double rad = __dsqrt_rn(dmul(-2.0, portable_log(u1)));
  double sn, cs;
  portable_sincos_2pi(K2, &sn, &cs);
  D.S[2 * e] = __double2float_rn(dmul(rad, cs));
  if (2 * e + 1 < total) D.S[2 * e + 1] = __double2float_rn(dmul(rad, sn));
}

// ----------------------------------------------------------------- a4: sketch chain
// OUT[i][c] = sum_j R[i][j] * IN[j][c], c < w (<= 16), fp32 accumulate.
// IN is staged per j-chunk into smem as [c][j] from one of the sources:
enum ChainSrc : int { SRC_S = 0, SRC_K1Q = 1, SRC_Q = 2, SRC_BUF = 3 };
struct ChainPass {
  int src, w, in_off, in_ld;   // SRC_BUF: IN[j][c] = in[j*in_ld + in_off + c]
  int in_blk, out_blk;         // chain block indices (each [s x 2p] floats)
};
constexpr int kChainRows = 32;     // rows per block (4 per warp)
constexpr int kChainJC = 256;      // j-chunk

template <int BF16>
__global__ void __launch_bounds__(256) k_chain(SolveParams P, ChainPass C) {
  __shared__ float sIn[16][kChainJC + 2];
  const int b = blockIdx.y;
  const MatDesc& D = P.mats[b];
  if (P.st[b].done) return;
  const int s = D.s, p = P.p, w = C.w;
  const int row0 = blockIdx.x * kChainRows;
  if (row0 >= s) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t blk = (size_t)s * 2 * p;
  const float* in = D.chain + C.in_blk * blk;
  float* out = D.chain + C.out_blk * blk;
  float acc[4][16];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 16; ++c) acc[r][c] = 0.f;

  for (int j0 = 0; j0 < s; j0 += kChainJC) {
    __syncthreads();
    // stage IN[j0 .. j0+JC) into sIn[c][jj]
    for (int idx = threadIdx.x; idx < w * kChainJC; idx += 256) {
      const int c = idx / kChainJC, jj = idx - c * kChainJC, j = j0 + jj;
      float v = 0.f;
      if (j < s) {
        if (C.src == SRC_S) {
          v = D.S[(size_t)c * s + j];
        } else if (C.src == SRC_BUF) {
          v = in[(size_t)j * C.in_ld + C.in_off + c];
        } else {
          // K1 = R S^T (chain block in_blk, [s][p]); Q = G S^T with G_jj exact in fp32:
          // Q_j = G_jj S_j - (K1_j - R_jj S_j)   (off-diagonal part of -R S^T)
          const int cc = (C.src == SRC_K1Q && c < p) ? c : (C.src == SRC_K1Q ? c - p : c);
          const float k1 = in[(size_t)j * p + cc];
          if (C.src == SRC_K1Q && c < p) {
            v = k1;
          } else {
            const float sj = D.S[(size_t)cc * s + j];
            float rjj;
            if (BF16) rjj = __bfloat162float(static_cast<const __nv_bfloat16*>(D.R)[(size_t)j * D.ldr + j]);
            else rjj = static_cast<const float*>(D.R)[(size_t)j * D.ldr + j] +
                       (D.R_lo ? static_cast<const float*>(D.R_lo)[(size_t)j * D.ldr + j] : 0.f);
            v = D.gdiag[j] * sj - (k1 - rjj * sj);
          }
        }
      }
      sIn[c][jj] = v;
    }
    __syncthreads();
    // each warp: 4 rows; lanes over j pairs
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = row0 + warp * 4 + r;
      if (i >= s) break;
      for (int jj = 2 * lane; jj < kChainJC; jj += 64) {
        const int j = j0 + jj;
        if (j >= s) break;
        float r0, r1;
        if (BF16) {
          const __nv_bfloat16* rp = static_cast<const __nv_bfloat16*>(D.R) + (size_t)i * D.ldr + j;
          if (j + 1 < s) {
            float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(rp));
            r0 = f.x; r1 = f.y;
          } else {
            r0 = __bfloat162float(rp[0]); r1 = 0.f;
          }
        } else {
          const float* rp = static_cast<const float*>(D.R) + (size_t)i * D.ldr + j;
          const float* rl = D.R_lo ? static_cast<const float*>(D.R_lo) + (size_t)i * D.ldr + j : nullptr;
          r0 = rp[0] + (rl ? rl[0] : 0.f);
          r1 = (j + 1 < s) ? rp[1] + (rl ? rl[1] : 0.f) : 0.f;
        }
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          if (c < w) {
            const float2 x = *reinterpret_cast<const float2*>(&sIn[c][jj]);
            acc[r][c] = fmaf(r0, x.x, acc[r][c]);
            acc[r][c] = fmaf(r1, x.y, acc[r][c]);
          }
        }
      }
    }
  }
  // reduce over lanes (fixed tree) and store
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int i = row0 + warp * 4 + r;
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      float v = acc[r][c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && c < w && i < s) out[(size_t)i * w + c] = v;
    }
  }
}

// ----------------------------------------------------------------- a5: coefficient solve
// Robust interval argmin of the quartic (R15/R16): same written
// procedure as the oracle, implemented independently here.
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

__device__ double argmin_quartic(const double c[5], double lo, double hi, double aT) {
  const double scale = fmax(fmax(fabs(c[1]), fabs(c[2])), fmax(fabs(c[3]), fabs(c[4])));
  if (!isfinite(scale)) return aT;
  if (scale == 0.0 || scale <= 1e-14 * fabs(c[0])) return aT;
  const double d1 = c[1] / scale, d2 = c[2] / scale, d3 = c[3] / scale, d4 = c[4] / scale;
  double roots[3];
  const int nr = real_roots_cubic(4.0 * d4, 3.0 * d3, 2.0 * d2, d1, roots);
  double cand[5];
  int nc = 0;
  cand[nc++] = lo;
  cand[nc++] = hi;
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
    if (isfinite(r) && r >= lo && r <= hi) cand[nc++] = r;
  }
  // sort ascending (insertion), pick the first strict minimum
  for (int i = 1; i < nc; ++i)
    for (int j = i; j > 0 && cand[j] < cand[j - 1]; --j) { double t = cand[j]; cand[j] = cand[j - 1]; cand[j - 1] = t; }
  double best = cand[0];
  double bm = (((d4 * best + d3) * best + d2) * best + d1) * best;
  for (int i = 1; i < nc; ++i) {
    const double a = cand[i];
    const double ma = (((d4 * a + d3) * a + d2) * a + d1) * a;
    if (ma < bm) { best = a; bm = ma; }
  }
  return best;
}

// One block (256 threads) per matrix: residual norm, stop test (R12), and
// alpha_k from the factored sketched loss m(a) = ||V0 + a V1 + a^2 V2||^2.
__global__ void __launch_bounds__(256) k_alpha(SolveParams P, int k, int do_fit) {
  __shared__ double scratch[8];
  __shared__ int s_stop;
  const int b = blockIdx.x;
  const MatDesc& D = P.mats[b];
  MatState& S = P.st[b];
  if (S.done) return;
  const int s = D.s;
  // ||R_k||_F^2 from the Gram per-tile partials (fixed order, scheduled tiles only)
  double part = 0.0;
  const int ntile = D.tiles_m * D.tiles_n;
  for (int t = threadIdx.x; t < ntile; t += 256) {
    const int tm = t / D.tiles_n, tn = t - tm * D.tiles_n;
    const bool sched = !D.sym || (tn * 256 + 255 >= tm * 128);   // bf16 tiles (BM=128, BN=256)
    const bool sched_tf = !D.sym || (tn * 128 + 127 >= tm * 128);
    if (P.precision == 0 ? sched : sched_tf) part += (double)D.norm_part[t];
  }
  const double r2 = block_sum<double, 256>(part, scratch);
  const double r = sqrt(r2);
  if (threadIdx.x == 0) {
    if (P.resid_hist) P.resid_hist[(size_t)b * (P.max_iters + 1) + k] = (float)(r / sqrt((double)s));
    int stop = 0, status = 1;
    if (!isfinite(r)) { stop = 1; status = 3; }
    else if (r <= P.tol * sqrt((double)s)) { stop = 1; status = 0; }
    else {
      S.incr = (k >= 1 && r > S.r_prev) ? S.incr + 1 : 0;
      if (S.incr >= 5) { stop = 1; status = 2; }
      else if (k >= P.max_iters) { stop = 1; status = 1; }
    }
    S.r_prev = r;
    S.resid = (float)(r / sqrt((double)s));
    if (stop) {
      S.done = 1;
      S.status = status;
      S.iters = k;
    } else {
      S.iters = k;
    }
    s_stop = stop;
  }
  __syncthreads();
  if (s_stop) return;
  double a;
  if (!do_fit) {
    a = (k < P.warmup) ? P.ahi : P.ataylor;
  } else {
    // V vectors from the chain blocks (factored form R17)
    const int p = P.p;
    const size_t blk = (size_t)s * 2 * p;
    const float* ch = D.chain;
    double g00 = 0, g01 = 0, g02 = 0, g11 = 0, g12 = 0, g22 = 0;
    for (int e = threadIdx.x; e < s * p; e += 256) {
      const int i = e / p, c = e - i * p;
      double v0, v1, v2;
      if (P.d == 1) {
        // blk0 = K1 [s][p]; blk1 = L1 [s][p]; blk2 = L2 [s][p]
        v0 = (double)ch[0 * blk + (size_t)i * p + c];
        v1 = -2.0 * (double)ch[1 * blk + (size_t)i * p + c];
        v2 = -(double)ch[2 * blk + (size_t)i * p + c];
      } else {
        // blk1 = [K2 | L1] [s][2p]; blk2 = [K3 | L2] [s][2p]; blk3 = L3 [s][p]; blk4 = L4 [s][p]
        const double K2 = ch[1 * blk + (size_t)i * 2 * p + c];
        const double K3 = ch[2 * blk + (size_t)i * 2 * p + c];
        const double L2 = ch[2 * blk + (size_t)i * 2 * p + p + c];
        const double L3 = ch[3 * blk + (size_t)i * p + c];
        const double L4 = ch[4 * blk + (size_t)i * p + c];
        v0 = 0.25 * (3.0 * K2 + K3);
        v1 = -(L3 + 2.0 * L2);
        v2 = -L4;
      }
      g00 += v0 * v0; g01 += v0 * v1; g02 += v0 * v2;
      g11 += v1 * v1; g12 += v1 * v2; g22 += v2 * v2;
    }
    g00 = block_sum<double, 256>(g00, scratch);
    g01 = block_sum<double, 256>(g01, scratch);
    g02 = block_sum<double, 256>(g02, scratch);
    g11 = block_sum<double, 256>(g11, scratch);
    g12 = block_sum<double, 256>(g12, scratch);
    g22 = block_sum<double, 256>(g22, scratch);
    double c[5] = {g00, 2.0 * g01, g11 + 2.0 * g02, 2.0 * g12, g22};
    a = (k < P.warmup) ? P.ahi : argmin_quartic(c, P.alo, P.ahi, P.ataylor);
  }
  if (threadIdx.x == 0) {
    S.alpha = a;
    if (P.alpha_hist) P.alpha_hist[(size_t)b * P.max_iters + k] = a;
  }
}

// ----------------------------------------------------------------- a7: outputs
// Polar: Q = Xt^T (tall) or Xt (wide); sqrt: A^{1/2} = sqrt(c) X, A^{-1/2} = Y/sqrt(c).
__global__ void __launch_bounds__(256) k_finalize(SolveParams P) {
  __shared__ float tile[32][33];
  const int b = blockIdx.z;
  const MatDesc& D = P.mats[b];
  const MatState& S = P.st[b];
  const int par = S.iters & 1;
  const int bf16 = P.precision == 0;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;   // over the *output* (m x n)
  auto ld = [&](const void* hi, const void* lo, long long idx) -> float {
    float v = load_val(hi, idx, bf16);
    if (P.precision == 1 && lo) v += static_cast<const float*>(lo)[idx];
    return v;
  };
  auto st = [&](void* q, long long idx, float v) {
    if (bf16) static_cast<__nv_bfloat16*>(q)[idx] = __float2bfloat16_rn(v);
    else static_cast<float*>(q)[idx] = v;
  };
  if (r0 >= D.m || c0 >= D.n) return;
  if (P.kind_sqrt) {
    const float fs = (float)sqrt(S.c);
    const float fi = S.c > 0.0 ? (float)(1.0 / sqrt(S.c)) : 0.f;
    for (int k = ty; k < 32; k += 8) {
      const int r = r0 + k, c = c0 + tx;
      if (r < D.m && c < D.n) {
        const long long xi = (long long)r * D.ldx + c;
        if (D.Q) st(D.Q, (long long)r * D.ldq + c, S.c > 0.0 ? fs * ld(D.X[par], D.X_lo[par], xi) : 0.f);
        if (D.Q2) st(D.Q2, (long long)r * D.ldq + c, fi * ld(D.Y[par], D.Y_lo[par], xi));
      }
    }
  } else if (D.trans) {
    // Q[r][c] = Xt[c][r]
    for (int k = ty; k < 32; k += 8) {
      const int xr = c0 + k, xc = r0 + tx;
      tile[k][tx] = (xr < D.n && xc < D.m) ? ld(D.X[par], D.X_lo[par], (long long)xr * D.ldx + xc) : 0.f;
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
      const int r = r0 + k, c = c0 + tx;
      if (r < D.m && c < D.n) st(D.Q, (long long)r * D.ldq + c, tile[tx][k]);
    }
  } else {
    for (int k = ty; k < 32; k += 8) {
      const int r = r0 + k, c = c0 + tx;
      if (r < D.m && c < D.n) st(D.Q, (long long)r * D.ldq + c, ld(D.X[par], D.X_lo[par], (long long)r * D.ldx + c));
    }
  }
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    if (P.rep_iters) P.rep_iters[b] = S.iters;
    if (P.rep_resid) P.rep_resid[b] = S.resid;
    if (P.rep_status) P.rep_status[b] = S.status;
  }
}

}  // namespace prism
