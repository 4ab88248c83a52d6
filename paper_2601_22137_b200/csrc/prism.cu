// Host side of libprism.so: argument validation, planning (workspace layout,
// TMA tensor maps, grouped tile lists), and the device-side iteration loop
// (no host synchronisation anywhere on the solve path).  See include/prism.h
// for the contract and DESIGN.md for the data layout.
#include "../../include/prism.h"
#include "gemm.cuh"
#include "kernels.cuh"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <list>
#include <memory>
#include <string>
#include <vector>

using namespace prism;

namespace {

thread_local std::string g_err;

prism_status fail(prism_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define PRISM_CK(x)                                                                        \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) return fail(PRISM_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ------------------------------------------------------------------ TMA maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

enum OpKind { OP_A = 0, OP_BK = 1, OP_BMN = 2 };

struct MapSpec {
  const void* ptr;
  int rows, cols;
  long long ld;
  int esz;
  OpKind kind;
  int BN, BK;
};

bool encode_map(CUtensorMap* out, const MapSpec& s) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)s.cols, (cuuint64_t)s.rows};
  cuuint64_t strides[1] = {(cuuint64_t)(s.ld * s.esz)};
  cuuint32_t box[2];
  if (s.kind == OP_A) { box[0] = s.BK; box[1] = 128; }
  else if (s.kind == OP_BK) { box[0] = s.BK; box[1] = s.BN; }
  else { box[0] = 128 / s.esz; box[1] = s.BK; }
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(out, s.esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                  const_cast<void*>(s.ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  (s.kind == OP_BMN && s.esz == 4) ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// ------------------------------------------------------------------ kernel dispatch
int g_num_sms = 0;

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

template <class Cfg>
cudaError_t launch_gemm_cfg(const GemmLaunch& L, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(prism_gemm_kernel<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (L.ntiles <= 0) return cudaSuccess;
  const int grid = std::min(L.ntiles, num_sms());
  prism_gemm_kernel<Cfg><<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(L);
  return cudaGetLastError();
}

cudaError_t launch_gemm(int precision, bool bmn, const GemmLaunch& L, cudaStream_t st) {
  if (precision == PRISM_BF16)
    return bmn ? launch_gemm_cfg<GemmCfg<0, false, true>>(L, st) : launch_gemm_cfg<GemmCfg<0, false, false>>(L, st);
  if (precision == PRISM_FP32)
    return bmn ? launch_gemm_cfg<GemmCfg<1, true, true>>(L, st) : launch_gemm_cfg<GemmCfg<1, true, false>>(L, st);
  return bmn ? launch_gemm_cfg<GemmCfg<1, false, true>>(L, st) : launch_gemm_cfg<GemmCfg<1, false, false>>(L, st);
}

int tile_bn(int precision) { return precision == PRISM_BF16 ? 256 : 128; }
int tile_bk(int precision) { return precision == PRISM_BF16 ? 64 : 32; }
int elem_size(int precision) { return precision == PRISM_BF16 ? 2 : 4; }

// ------------------------------------------------------------------ planning
struct HostProblem {
  GemmProblem p;      // tm* fields hold map indices (+1; 0 = none) until serialised
  int mapA, mapB, mapA_lo, mapB_lo;
};

struct LaunchDesc {
  std::vector<HostProblem> probs;
  std::vector<uint32_t> tiles;
  bool bmn = false;
  // filled at serialisation
  size_t probs_off = 0, tiles_off = 0;
};

struct PinnedDeleter {
  void operator()(uint8_t* p) const { if (p) cudaFreeHost(p); }
};

struct Plan {
  std::vector<long long> key;
  size_t ws_need = 0;
  size_t meta_off = 0, meta_bytes = 0;
  std::unique_ptr<uint8_t, PinnedDeleter> blob;
  SolveParams params{};
  LaunchDesc gram[2], square, apply[2];
  bool has_square = false;
  int max_s = 0, max_rows = 0, max_cols = 0, max_m = 0, max_n = 0;
};

struct Request {
  bool sqrt_kind;
  int batch;
  const int64_t* m;
  const int64_t* n;
  const void* const* A;
  const int64_t* lda;
  void* const* Q;
  void* const* Q2;
  const int64_t* ldq;
  const int64_t* ids;
  prism_options o;
  char* ws;   // null: size query only
};

void resolve_interval(prism_options& o, double& lo, double& hi, double& aT, int& d) {
  d = (o.degree == 3) ? 1 : 2;
  const double dlo = d == 1 ? 0.5 : 0.375, dhi = d == 1 ? 1.0 : 1.45;
  aT = d == 1 ? 0.5 : 0.375;   // Taylor coefficient of xi^d in (1-xi)^{-1/2}
  lo = std::isnan(o.alpha_lo) ? dlo : o.alpha_lo;
  hi = std::isnan(o.alpha_hi) ? dhi : o.alpha_hi;
}

struct Bump {
  char* base;
  size_t off = 0;
  char* take(size_t bytes, size_t align = 256) {
    off = align_up(off, align);
    char* p = base + off;
    off += bytes;
    return p;
  }
};

void add_tiles(LaunchDesc& L, int prob, int M, int N, int BN, bool sym) {
  const int tm_n = (M + 127) / 128, tn_n = (N + BN - 1) / BN;
  for (int tm = 0; tm < tm_n; ++tm)
    for (int tn = 0; tn < tn_n; ++tn) {
      if (sym && tn * BN + BN - 1 < tm * 128) continue;
      L.tiles.push_back(((uint32_t)prob << 20) | ((uint32_t)tm << 10) | (uint32_t)tn);
    }
}

void sort_tiles_by_cost(LaunchDesc& L) {
  std::stable_sort(L.tiles.begin(), L.tiles.end(), [&](uint32_t a, uint32_t b) {
    return L.probs[a >> 20].p.K > L.probs[b >> 20].p.K;
  });
}

// Build the full plan.  When r.ws == nullptr only sizes are computed.
prism_status build_plan(const Request& r, Plan& P) {
  prism_options o = r.o;
  double lo, hi, aT;
  int d;
  resolve_interval(o, lo, hi, aT, d);
  const int prec = o.precision;
  const int esz = elem_size(prec);
  const bool split = prec == PRISM_FP32;
  const int BN = tile_bn(prec), BK = tile_bk(prec);
  const int p = o.sketch_size;
  const int B = r.batch;
  Bump bump{r.ws};

  // state region
  MatState* d_st = reinterpret_cast<MatState*>(bump.take(sizeof(MatState) * B));
  double* d_fro = reinterpret_cast<double*>(bump.take(sizeof(double) * B * kFroParts));

  std::vector<MatDesc> mats(B);
  std::vector<MapSpec> maps;
  auto add_map = [&](const void* ptr, int rows, int cols, long long ld, OpKind k) -> int {
    maps.push_back(MapSpec{ptr, rows, cols, ld, esz, k, BN, BK});
    return (int)maps.size();   // 1-based index
  };

  P.max_s = P.max_rows = P.max_cols = P.max_m = P.max_n = 0;
  for (int i = 0; i < B; ++i) {
    MatDesc& D = mats[i];
    std::memset(&D, 0, sizeof(D));
    const int m = (int)r.m[i];
    const int n = r.sqrt_kind ? (int)r.m[i] : (int)r.n[i];
    D.A = r.A[i];
    D.Q = r.Q ? r.Q[i] : nullptr;
    D.Q2 = r.Q2 ? r.Q2[i] : nullptr;
    D.lda = r.lda[i];
    D.ldq = r.ldq[i];
    D.m = m;
    D.n = n;
    if (r.sqrt_kind) { D.s = n; D.L = n; D.trans = 0; }
    else { D.s = std::min(m, n); D.L = std::max(m, n); D.trans = (m >= n) ? 1 : 0; }
    D.sketch_id = r.ids ? (int)r.ids[i] : i;
    const int s = D.s, L = D.L;
    const long long ldx = (long long)align_up(L, 64), ldr = (long long)align_up(s, 64);
    D.ldx = ldx;
    D.ldr = ldr;
    const size_t xbytes = (size_t)s * ldx * esz, rbytes = (size_t)s * ldr * esz;
    for (int t = 0; t < 2; ++t) {
      D.X[t] = bump.take(xbytes);
      D.X_lo[t] = split ? bump.take(xbytes) : nullptr;
      if (r.sqrt_kind) {
        D.Y[t] = bump.take(xbytes);
        D.Y_lo[t] = split ? bump.take(xbytes) : nullptr;
      }
    }
    D.R = bump.take(rbytes);
    D.R_lo = split ? bump.take(rbytes) : nullptr;
    void* Pm = (d == 2) ? bump.take(rbytes) : nullptr;
    void* Pm_lo = (d == 2 && split) ? bump.take(rbytes) : nullptr;
    D.gdiag = reinterpret_cast<float*>(bump.take(sizeof(float) * s));
    D.tiles_m = (s + 127) / 128;
    D.tiles_n = (s + BN - 1) / BN;
    D.sym = r.sqrt_kind ? 0 : 1;
    D.norm_part = reinterpret_cast<float*>(bump.take(sizeof(float) * D.tiles_m * D.tiles_n));
    D.S = reinterpret_cast<float*>(bump.take(sizeof(float) * p * s));
    D.chain = reinterpret_cast<float*>(bump.take(sizeof(float) * 5 * (size_t)s * 2 * p));
    P.max_s = std::max(P.max_s, s);
    P.max_rows = std::max(P.max_rows, s);
    P.max_cols = std::max(P.max_cols, L);
    P.max_m = std::max(P.max_m, m);
    P.max_n = std::max(P.max_n, n);
    if (L / BN >= 1023 || s / 128 >= 1023)
      return fail(PRISM_ERR_UNSUPPORTED, "matrix too large for the tile encoding");

    const double* alpha_ptr = &d_st[i].alpha;
    auto mk = [&](int M, int N, int K, int mode, int sym, void* out, void* out_lo, long long ldo, const void* C,
                  const void* C_lo, long long ldc) {
      HostProblem h;
      std::memset(&h, 0, sizeof(h));
      h.p.M = M; h.p.N = N; h.p.K = K; h.p.mode = mode; h.p.sym = sym; h.p.matrix = i;
      h.p.out = out; h.p.out_lo = out_lo; h.p.ldo = ldo; h.p.C = C; h.p.C_lo = C_lo; h.p.ldc = ldc;
      h.p.alpha = alpha_ptr;
      h.p.tiles_n = (N + BN - 1) / BN;
      return h;
    };
    if (!r.sqrt_kind) {
      // polar, compute layout Xt (s x L): G = Xt Xt^T, P = R/2 + a R^2, Xt' = Xt + P Xt
      for (int t = 0; t < 2; ++t) {
        HostProblem g = mk(s, s, L, EPI_RESID, 1, D.R, D.R_lo, ldr, nullptr, nullptr, 0);
        g.p.norm_part = D.norm_part;
        g.p.gdiag = D.gdiag;
        g.mapA = add_map(D.X[t], s, L, ldx, OP_A);
        g.mapB = add_map(D.X[t], s, L, ldx, OP_BK);
        if (split) { g.mapA_lo = add_map(D.X_lo[t], s, L, ldx, OP_A); g.mapB_lo = add_map(D.X_lo[t], s, L, ldx, OP_BK); }
        P.gram[t].probs.push_back(g);
        const void* Pa = d == 2 ? Pm : D.R;
        const void* Pa_lo = d == 2 ? Pm_lo : D.R_lo;
        HostProblem a = mk(s, L, s, EPI_APPLY, 0, D.X[1 - t], D.X_lo[1 - t], ldx, D.X[t], D.X_lo[t], ldx);
        a.p.scale_by_alpha = d == 1;
        a.mapA = add_map(Pa, s, s, ldr, OP_A);
        a.mapB = add_map(D.X[t], s, L, ldx, OP_BMN);
        if (split) { a.mapA_lo = add_map(Pa_lo, s, s, ldr, OP_A); a.mapB_lo = add_map(D.X_lo[t], s, L, ldx, OP_BMN); }
        P.apply[t].probs.push_back(a);
      }
      if (d == 2) {
        HostProblem q = mk(s, s, s, EPI_POLY, 1, Pm, Pm_lo, ldr, D.R, D.R_lo, ldr);
        q.p.c1 = 0.5f;
        q.mapA = add_map(D.R, s, s, ldr, OP_A);
        q.mapB = add_map(D.R, s, s, ldr, OP_BK);
        if (split) { q.mapA_lo = add_map(D.R_lo, s, s, ldr, OP_A); q.mapB_lo = add_map(D.R_lo, s, s, ldr, OP_BK); }
        P.square.probs.push_back(q);
      }
    } else {
      // sqrt: G = Y X, P = R/2 + a R^2, X' = X + X P, Y' = Y + P Y (Theorem-3 ordering, R11)
      const int nn = s;
      for (int t = 0; t < 2; ++t) {
        HostProblem g = mk(nn, nn, nn, EPI_RESID, 0, D.R, D.R_lo, ldr, nullptr, nullptr, 0);
        g.p.norm_part = D.norm_part;
        g.p.gdiag = D.gdiag;
        g.mapA = add_map(D.Y[t], nn, nn, ldx, OP_A);
        g.mapB = add_map(D.X[t], nn, nn, ldx, OP_BMN);
        if (split) { g.mapA_lo = add_map(D.Y_lo[t], nn, nn, ldx, OP_A); g.mapB_lo = add_map(D.X_lo[t], nn, nn, ldx, OP_BMN); }
        P.gram[t].probs.push_back(g);
        const void* Pa = d == 2 ? Pm : D.R;
        const void* Pa_lo = d == 2 ? Pm_lo : D.R_lo;
        HostProblem ax = mk(nn, nn, nn, EPI_APPLY, 0, D.X[1 - t], D.X_lo[1 - t], ldx, D.X[t], D.X_lo[t], ldx);
        ax.p.scale_by_alpha = d == 1;
        ax.mapA = add_map(D.X[t], nn, nn, ldx, OP_A);
        ax.mapB = add_map(Pa, nn, nn, ldr, OP_BMN);
        if (split) { ax.mapA_lo = add_map(D.X_lo[t], nn, nn, ldx, OP_A); ax.mapB_lo = add_map(Pa_lo, nn, nn, ldr, OP_BMN); }
        P.apply[t].probs.push_back(ax);
        HostProblem ay = mk(nn, nn, nn, EPI_APPLY, 0, D.Y[1 - t], D.Y_lo[1 - t], ldx, D.Y[t], D.Y_lo[t], ldx);
        ay.p.scale_by_alpha = d == 1;
        ay.mapA = add_map(Pa, nn, nn, ldr, OP_A);
        ay.mapB = add_map(D.Y[t], nn, nn, ldx, OP_BMN);
        if (split) { ay.mapA_lo = add_map(Pa_lo, nn, nn, ldr, OP_A); ay.mapB_lo = add_map(D.Y_lo[t], nn, nn, ldx, OP_BMN); }
        P.apply[t].probs.push_back(ay);
      }
      if (d == 2) {
        HostProblem q = mk(nn, nn, nn, EPI_POLY, 0, Pm, Pm_lo, ldr, D.R, D.R_lo, ldr);
        q.p.c1 = 0.5f;
        q.mapA = add_map(D.R, nn, nn, ldr, OP_A);
        q.mapB = add_map(D.R, nn, nn, ldr, OP_BMN);
        if (split) { q.mapA_lo = add_map(D.R_lo, nn, nn, ldr, OP_A); q.mapB_lo = add_map(D.R_lo, nn, nn, ldr, OP_BMN); }
        P.square.probs.push_back(q);
      }
    }
  }
  P.has_square = (d == 2);
  // tile lists (problem index within its launch)
  auto finish = [&](LaunchDesc& L, bool bmn) {
    L.bmn = bmn;
    L.tiles.clear();
    for (int j = 0; j < (int)L.probs.size(); ++j)
      add_tiles(L, j, L.probs[j].p.M, L.probs[j].p.N, BN, L.probs[j].p.sym != 0);
    sort_tiles_by_cost(L);
  };
  const bool polar_k = !r.sqrt_kind;
  for (int t = 0; t < 2; ++t) {
    finish(P.gram[t], !polar_k);
    finish(P.apply[t], true);
  }
  if (P.has_square) finish(P.square, !polar_k);
  if ((int)P.apply[0].probs.size() >= 4096) return fail(PRISM_ERR_UNSUPPORTED, "batch too large (max 2047 sqrt / 4095 polar)");

  // meta region (serialised blob): [mats][problems...][tiles...][maps]
  P.meta_off = align_up(bump.off, 1024);
  size_t off = 0;
  const size_t mats_off = off;
  off += sizeof(MatDesc) * B;
  LaunchDesc* all[5] = {&P.gram[0], &P.gram[1], &P.apply[0], &P.apply[1], &P.square};
  for (LaunchDesc* L : all) {
    off = align_up(off, 128);
    L->probs_off = off;
    off += sizeof(GemmProblem) * L->probs.size();
  }
  for (LaunchDesc* L : all) {
    off = align_up(off, 128);
    L->tiles_off = off;
    off += sizeof(uint32_t) * L->tiles.size();
  }
  off = align_up(off, 128);
  const size_t maps_off = off;
  off += sizeof(CUtensorMap) * maps.size();
  P.meta_bytes = align_up(off, 256);
  P.ws_need = P.meta_off + P.meta_bytes;
  if (!r.ws) return PRISM_OK;

  char* meta_dev = r.ws + P.meta_off;
  uint8_t* blob = nullptr;
  if (cudaMallocHost(&blob, P.meta_bytes) != cudaSuccess) return fail(PRISM_ERR_CUDA, "cudaMallocHost(plan blob)");
  P.blob.reset(blob);
  std::memset(blob, 0, P.meta_bytes);
  std::memcpy(blob + mats_off, mats.data(), sizeof(MatDesc) * B);
  CUtensorMap* hmaps = reinterpret_cast<CUtensorMap*>(blob + maps_off);
  for (size_t j = 0; j < maps.size(); ++j)
    if (!encode_map(&hmaps[j], maps[j])) return fail(PRISM_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  auto mapptr = [&](int idx) -> const CUtensorMap* {
    return idx ? reinterpret_cast<const CUtensorMap*>(meta_dev + maps_off + (size_t)(idx - 1) * sizeof(CUtensorMap))
               : nullptr;
  };
  for (LaunchDesc* L : all) {
    GemmProblem* gp = reinterpret_cast<GemmProblem*>(blob + L->probs_off);
    for (size_t j = 0; j < L->probs.size(); ++j) {
      GemmProblem q = L->probs[j].p;
      q.tmA = mapptr(L->probs[j].mapA);
      q.tmB = mapptr(L->probs[j].mapB);
      q.tmA_lo = mapptr(L->probs[j].mapA_lo);
      q.tmB_lo = mapptr(L->probs[j].mapB_lo);
      gp[j] = q;
    }
    std::memcpy(blob + L->tiles_off, L->tiles.data(), sizeof(uint32_t) * L->tiles.size());
  }

  SolveParams& S = P.params;
  std::memset(&S, 0, sizeof(S));
  S.mats = reinterpret_cast<MatDesc*>(meta_dev + mats_off);
  S.st = d_st;
  S.fro_part = d_fro;
  S.batch = B;
  S.p = p;
  S.d = d;
  S.max_iters = o.max_iters;
  S.warmup = o.warmup_iters;
  S.fit = o.fit;
  S.precision = prec;
  S.kind_sqrt = r.sqrt_kind ? 1 : 0;
  S.tol = o.tol;
  S.alo = lo;
  S.ahi = hi;
  S.ataylor = aT;
  S.seed = o.seed;
  return PRISM_OK;
}

GemmLaunch make_launch(const Plan& P, const LaunchDesc& L, char* ws) {
  GemmLaunch g;
  char* meta = ws + P.meta_off;
  g.probs = reinterpret_cast<const GemmProblem*>(meta + L.probs_off);
  g.tiles = reinterpret_cast<const uint32_t*>(meta + L.tiles_off);
  g.done = &P.params.st[0].done;
  g.done_stride = sizeof(MatState) / sizeof(int);
  g.ntiles = (int)L.tiles.size();
  return g;
}

prism_status validate(const Request& r) {
  const prism_options& o = r.o;
  if (r.batch < 1) return fail(PRISM_ERR_INVALID_ARG, "batch must be >= 1");
  if (!r.m || !r.lda || !r.A || (!r.sqrt_kind && (!r.n || !r.Q || !r.ldq)))
    return fail(PRISM_ERR_INVALID_ARG, "null size/pointer array");
  if (o.degree != 3 && o.degree != 5) return fail(PRISM_ERR_INVALID_ARG, "degree must be 3 or 5");
  if (o.max_iters < 1 || o.max_iters > 10000) return fail(PRISM_ERR_INVALID_ARG, "max_iters out of range");
  if (!(o.tol > 0.0)) return fail(PRISM_ERR_INVALID_ARG, "tol must be > 0");
  if (o.precision < 0 || o.precision > 2) return fail(PRISM_ERR_INVALID_ARG, "bad precision");
  if (o.fit != PRISM_FIT_SKETCHED && o.fit != PRISM_FIT_TAYLOR)
    return fail(PRISM_ERR_UNSUPPORTED, "fit must be SKETCHED or TAYLOR on the device");
  if (o.sketch_size < 1) return fail(PRISM_ERR_INVALID_ARG, "sketch_size must be >= 1");
  if (o.sketch_size > 8) return fail(PRISM_ERR_UNSUPPORTED, "sketch_size > 8 not supported");
  if (o.warmup_iters < 0) return fail(PRISM_ERR_INVALID_ARG, "warmup_iters must be >= 0");
  const int esz = elem_size(o.precision);
  for (int i = 0; i < r.batch; ++i) {
    const int64_t m = r.m[i], n = r.sqrt_kind ? r.m[i] : r.n[i];
    if (m < 1 || n < 1 || m > (1 << 20) || n > (1 << 20)) return fail(PRISM_ERR_INVALID_ARG, "bad matrix size");
    if (!r.A[i]) return fail(PRISM_ERR_INVALID_ARG, "null input matrix");
    if (r.lda[i] < n) return fail(PRISM_ERR_INVALID_ARG, "lda < n");
    if (!r.sqrt_kind && !r.Q[i]) return fail(PRISM_ERR_INVALID_ARG, "null output matrix");
    if ((r.Q || r.Q2) && r.ldq[i] < n) return fail(PRISM_ERR_INVALID_ARG, "ldq < n");
    if (std::min(m, n) < o.sketch_size) return fail(PRISM_ERR_INVALID_ARG, "sketch_size > min(m, n)");
    if (reinterpret_cast<uintptr_t>(r.A[i]) % esz) return fail(PRISM_ERR_INVALID_ARG, "misaligned input");
  }
  return PRISM_OK;
}

}  // namespace

// ====================================================================== handle
struct prism_handle_s {
  std::list<std::unique_ptr<Plan>> plans;   // most recent first
};

static std::vector<long long> make_key(const Request& r) {
  std::vector<long long> k;
  k.push_back(r.sqrt_kind);
  k.push_back(r.batch);
  const prism_options& o = r.o;
  long long tolbits, alo, ahi;
  std::memcpy(&tolbits, &o.tol, 8);
  std::memcpy(&alo, &o.alpha_lo, 8);
  std::memcpy(&ahi, &o.alpha_hi, 8);
  for (long long v : {(long long)o.degree, (long long)o.max_iters, (long long)o.sketch_size, tolbits,
                      (long long)o.seed, (long long)o.precision, (long long)o.fit, (long long)o.warmup_iters, alo, ahi})
    k.push_back(v);
  k.push_back((long long)(uintptr_t)r.ws);
  for (int i = 0; i < r.batch; ++i) {
    k.push_back(r.m[i]);
    k.push_back(r.sqrt_kind ? r.m[i] : r.n[i]);
    k.push_back(r.lda[i]);
    k.push_back(r.ldq ? r.ldq[i] : 0);
    k.push_back((long long)(uintptr_t)r.A[i]);
    k.push_back(r.Q ? (long long)(uintptr_t)r.Q[i] : 0);
    k.push_back(r.Q2 ? (long long)(uintptr_t)r.Q2[i] : 0);
    k.push_back(r.ids ? r.ids[i] : i);
  }
  return k;
}

static prism_status run_solve(prism_handle h, const Request& r0, const prism_report* rep, size_t ws_bytes,
                              cudaStream_t st) {
  Request r = r0;
  if (!h) return fail(PRISM_ERR_INVALID_ARG, "null handle");
  prism_status v = validate(r);
  if (v) return v;
  if (!r.ws) return fail(PRISM_ERR_INVALID_ARG, "null workspace");
  if (reinterpret_cast<uintptr_t>(r.ws) % 256) return fail(PRISM_ERR_INVALID_ARG, "workspace must be 256-B aligned");
  std::vector<long long> key = make_key(r);
  Plan* P = nullptr;
  for (auto it = h->plans.begin(); it != h->plans.end(); ++it) {
    if ((*it)->key == key) {
      h->plans.splice(h->plans.begin(), h->plans, it);
      P = h->plans.front().get();
      break;
    }
  }
  if (!P) {
    std::unique_ptr<Plan> np(new Plan());
    Request q = r;
    q.ws = nullptr;
    prism_status s0 = build_plan(q, *np);
    if (s0) return s0;
    if (ws_bytes < np->ws_need) return fail(PRISM_ERR_INVALID_ARG, "workspace too small");
    np.reset(new Plan());
    prism_status s1 = build_plan(r, *np);
    if (s1) return s1;
    np->key = key;
    h->plans.push_front(std::move(np));
    while (h->plans.size() > 16) h->plans.pop_back();
    P = h->plans.front().get();
  }
  if (ws_bytes < P->ws_need) return fail(PRISM_ERR_INVALID_ARG, "workspace too small");

  PRISM_CK(cudaMemcpyAsync(r.ws + P->meta_off, P->blob.get(), P->meta_bytes, cudaMemcpyHostToDevice, st));
  SolveParams S = P->params;
  S.alpha_hist = rep ? rep->alphas : nullptr;
  S.resid_hist = rep ? rep->resid_hist : nullptr;
  S.rep_iters = rep ? rep->iters : nullptr;
  S.rep_resid = rep ? rep->resid : nullptr;
  S.rep_status = rep ? rep->status : nullptr;
  const int B = r.batch;
  const int prec = r.o.precision;

  k_fro_partials<<<dim3(kFroParts, B), 256, 0, st>>>(S);
  k_normalize<<<dim3((P->max_cols + 31) / 32, (P->max_rows + 31) / 32, B), 256, 0, st>>>(S);
  PRISM_CK(cudaGetLastError());
  const GemmLaunch g_gram[2] = {make_launch(*P, P->gram[0], r.ws), make_launch(*P, P->gram[1], r.ws)};
  const GemmLaunch g_apply[2] = {make_launch(*P, P->apply[0], r.ws), make_launch(*P, P->apply[1], r.ws)};
  const GemmLaunch g_sq = make_launch(*P, P->square, r.ws);
  const int p = S.p;
  const dim3 chain_grid((P->max_s + kChainRows - 1) / kChainRows, B);
  for (int k = 0; k <= r.o.max_iters; ++k) {
    const int par = k & 1;
    PRISM_CK(launch_gemm(prec, P->gram[par].bmn, g_gram[par], st));
    const bool fit = r.o.fit == PRISM_FIT_SKETCHED && k < r.o.max_iters && k >= r.o.warmup_iters;
    if (fit) {
      k_sketch<<<dim3((p * P->max_s / 2 + 256) / 256, B), 256, 0, st>>>(S, k);
      auto chain = [&](int src, int w, int in_blk, int in_ld, int in_off, int out_blk) {
        ChainPass c{src, w, in_off, in_ld, in_blk, out_blk};
        if (prec == PRISM_BF16) k_chain<1><<<chain_grid, 256, 0, st>>>(S, c);
        else k_chain<0><<<chain_grid, 256, 0, st>>>(S, c);
      };
      if (S.d == 2) {
        chain(SRC_S, p, 0, 0, 0, 0);             // K1 = R S^T
        chain(SRC_K1Q, 2 * p, 0, p, 0, 1);       // [K2 | L1] = R [K1 | Q]
        chain(SRC_BUF, 2 * p, 1, 2 * p, 0, 2);   // [K3 | L2] = R [K2 | L1]
        chain(SRC_BUF, p, 2, 2 * p, p, 3);       // L3 = R L2
        chain(SRC_BUF, p, 3, p, 0, 4);           // L4 = R L3
      } else {
        chain(SRC_S, p, 0, 0, 0, 0);             // K1 = R S^T
        chain(SRC_Q, p, 0, p, 0, 1);             // L1 = R Q
        chain(SRC_BUF, p, 1, p, 0, 2);           // L2 = R L1
      }
    }
    k_alpha<<<B, 256, 0, st>>>(S, k, fit ? 1 : 0);
    PRISM_CK(cudaGetLastError());
    if (k < r.o.max_iters) {
      if (P->has_square) PRISM_CK(launch_gemm(prec, P->square.bmn, g_sq, st));
      PRISM_CK(launch_gemm(prec, P->apply[par].bmn, g_apply[par], st));
    }
  }
  k_finalize<<<dim3((P->max_n + 31) / 32, (P->max_m + 31) / 32, B), 256, 0, st>>>(S);
  PRISM_CK(cudaGetLastError());
  return PRISM_OK;
}

// ====================================================================== debug kernels
namespace prism {
__global__ void k_sketch_debug(unsigned long long seed, int b, int k, int p, int s, float* S) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)p * s;
  if (2 * e >= total) return;
  uint32_t ctr[4] = {(uint32_t)e, (uint32_t)k, (uint32_t)b, 0x534B4348u};
  philox10(ctr, (uint32_t)(seed & 0xFFFFFFFFull), (uint32_t)(seed >> 32));
  const unsigned long long K1 = ((unsigned long long)(ctr[0] >> 5) << 26) + (ctr[1] >> 6);
  const unsigned long long K2 = ((unsigned long long)(ctr[2] >> 5) << 26) + (ctr[3] >> 6);
  const double u1 = dmul((double)(K1 + 1ull), 0x1p-53);
  const double rad = __dsqrt_rn(dmul(-2.0, portable_log(u1)));
  double sn, cs;
  portable_sincos_2pi(K2, &sn, &cs);
  S[2 * e] = __double2float_rn(dmul(rad, cs));
  if (2 * e + 1 < total) S[2 * e + 1] = __double2float_rn(dmul(rad, sn));
}
__global__ void k_argmin_debug(int n, const double* c, double lo, double hi, double aT, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = argmin_quartic(c + 5 * i, lo, hi, aT);
}
}  // namespace prism

// ====================================================================== C ABI
extern "C" {

void prism_default_options(prism_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->degree = 5;
  o->max_iters = 30;
  o->sketch_size = 8;
  o->tol = 1e-6;
  o->seed = 42;
  o->precision = PRISM_BF16;
  o->fit = PRISM_FIT_SKETCHED;
  o->warmup_iters = 0;
  o->alpha_lo = NAN;
  o->alpha_hi = NAN;
}

prism_status prism_create(prism_handle* h) {
  if (!h) return fail(PRISM_ERR_INVALID_ARG, "null handle pointer");
  try {
    *h = new prism_handle_s();
  } catch (...) {
    return fail(PRISM_ERR_INTERNAL, "allocation failed");
  }
  return PRISM_OK;
}

prism_status prism_destroy(prism_handle h) {
  delete h;
  return PRISM_OK;
}

const char* prism_last_error(void) { return g_err.c_str(); }

int prism_abi_version(void) { return PRISM_VERSION_MAJOR * 100 + PRISM_VERSION_MINOR; }

size_t prism_polar_workspace(prism_handle h, int batch, const int64_t* m, const int64_t* n, const prism_options* o) {
  if (!h || !o || !m || !n || batch < 1) return 0;
  std::vector<const void*> fakeA(batch, reinterpret_cast<const void*>(256));
  std::vector<void*> fakeQ(batch, reinterpret_cast<void*>(256));
  std::vector<int64_t> ld(batch);
  for (int i = 0; i < batch; ++i) ld[i] = std::max(m[i], n[i]);
  Request r{false, batch, m, n, fakeA.data(), ld.data(), fakeQ.data(), nullptr, ld.data(), nullptr, *o, nullptr};
  if (validate(r)) return 0;
  Plan P;
  if (build_plan(r, P)) return 0;
  return P.ws_need;
}

prism_status prism_polar(prism_handle h, int batch, const int64_t* m, const int64_t* n, const void* const* A,
                         const int64_t* lda, void* const* Q, const int64_t* ldq, const int64_t* matrix_ids,
                         const prism_options* o, const prism_report* rep, void* workspace, size_t ws_bytes,
                         void* stream) {
  try {
    if (!o) return fail(PRISM_ERR_INVALID_ARG, "null options");
    Request r{false, batch, m, n, A, lda, Q, nullptr, ldq, matrix_ids, *o, static_cast<char*>(workspace)};
    return run_solve(h, r, rep, ws_bytes, static_cast<cudaStream_t>(stream));
  } catch (...) {
    return fail(PRISM_ERR_INTERNAL, "exception in prism_polar");
  }
}

size_t prism_sqrt_workspace(prism_handle h, int batch, const int64_t* n, const prism_options* o) {
  if (!h || !o || !n || batch < 1) return 0;
  std::vector<const void*> fakeA(batch, reinterpret_cast<const void*>(256));
  std::vector<int64_t> ld(n, n + batch);
  Request r{true, batch, n, n, fakeA.data(), ld.data(), nullptr, nullptr, ld.data(), nullptr, *o, nullptr};
  if (validate(r)) return 0;
  Plan P;
  if (build_plan(r, P)) return 0;
  return P.ws_need;
}

prism_status prism_sqrt_invsqrt(prism_handle h, int batch, const int64_t* n, const void* const* A,
                                const int64_t* lda, void* const* Asqrt, void* const* Ainvsqrt,
                                const int64_t* ld_out, const int64_t* matrix_ids, const prism_options* o,
                                const prism_report* rep, void* workspace, size_t ws_bytes, void* stream) {
  try {
    if (!o) return fail(PRISM_ERR_INVALID_ARG, "null options");
    if ((Asqrt || Ainvsqrt) && !ld_out) return fail(PRISM_ERR_INVALID_ARG, "null ld_out");
    Request r{true, batch, n, n, A, lda, Asqrt, Ainvsqrt, ld_out, matrix_ids, *o, static_cast<char*>(workspace)};
    return run_solve(h, r, rep, ws_bytes, static_cast<cudaStream_t>(stream));
  } catch (...) {
    return fail(PRISM_ERR_INTERNAL, "exception in prism_sqrt_invsqrt");
  }
}

prism_status prism_lpt_partition(int batch, const double* cost, int ranks, int32_t* owner) {
  if (batch < 0 || ranks < 1 || (batch > 0 && (!cost || !owner))) return fail(PRISM_ERR_INVALID_ARG, "bad LPT args");
  std::vector<int> order(batch);
  for (int i = 0; i < batch; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
  std::vector<double> load(ranks, 0.0);
  for (int i : order) {
    int best = 0;
    for (int q = 1; q < ranks; ++q)
      if (load[q] < load[best]) best = q;
    owner[i] = best;
    load[best] += cost[i];
  }
  return PRISM_OK;
}

double prism_polar_flops_per_iter(int64_t m, int64_t n, int degree, int sketch_size) {
  const double L = (double)std::max(m, n), s = (double)std::min(m, n), p = sketch_size;
  double f = L * s * (s + 1) + 2.0 * L * s * s;               // symmetric Gram + apply
  if (degree == 5) f += s * s * (s + 1) + 14.0 * s * s * p;   // symmetric square + 7p chain columns
  else f += 6.0 * s * s * p;                                  // 3p chain columns
  return f;
}

double prism_sqrt_flops_per_iter(int64_t n, int degree, int sketch_size) {
  const double x = (double)n, p = sketch_size;
  double f = 2.0 * x * x * x + 4.0 * x * x * x;                // Y X, X P, P Y
  if (degree == 5) f += 2.0 * x * x * x + 14.0 * x * x * p;
  else f += 6.0 * x * x * p;
  return f;
}

prism_status prism_debug_gemm(prism_handle h, int precision, int b_mn, int mode, int sym, int M, int N, int K,
                              const void* A, const void* A_lo, int64_t lda, const void* B, const void* B_lo,
                              int64_t ldb, const void* C, const void* C_lo, int64_t ldc, void* out, void* out_lo,
                              int64_t ldo, const double* alpha_dev, float c1, int scale_by_alpha, float* norm_part,
                              float* gdiag, void* workspace, size_t ws_bytes, void* stream) {
  if (!h || !A || !B || !out || !workspace) return fail(PRISM_ERR_INVALID_ARG, "null pointer");
  if (precision < 0 || precision > 2 || mode < 0 || mode > 3 || M < 1 || N < 1 || K < 1)
    return fail(PRISM_ERR_INVALID_ARG, "bad debug_gemm args");
  if (sym && M != N) return fail(PRISM_ERR_INVALID_ARG, "sym needs M == N");
  const bool split = precision == PRISM_FP32;
  if (split && (!A_lo || !B_lo || !out_lo)) return fail(PRISM_ERR_INVALID_ARG, "FP32 needs lo planes");
  const int esz = elem_size(precision), BN = tile_bn(precision), BK = tile_bk(precision);
  if ((lda * esz) % 16 || (ldb * esz) % 16 || (ldo * esz) % 16 || (C && (ldc * esz) % 16))
    return fail(PRISM_ERR_INVALID_ARG, "leading dimensions must be 16-B multiples");
  const size_t need = 4096 + 4 * sizeof(CUtensorMap) + sizeof(GemmProblem) + 4 * ((M + 127) / 128) * ((N + BN - 1) / BN);
  if (ws_bytes < need) return fail(PRISM_ERR_INVALID_ARG, "workspace too small");
  static thread_local std::unique_ptr<uint8_t, PinnedDeleter> blob;
  static thread_local size_t blob_size = 0;
  if (blob_size < need) {
    uint8_t* b = nullptr;
    if (cudaMallocHost(&b, need) != cudaSuccess) return fail(PRISM_ERR_CUDA, "cudaMallocHost");
    blob.reset(b);
    blob_size = need;
  }
  PRISM_CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));   // debug path: reuse of the pinned blob
  uint8_t* hb = blob.get();
  std::memset(hb, 0, need);
  char* wsd = static_cast<char*>(workspace);
  CUtensorMap* hm = reinterpret_cast<CUtensorMap*>(hb);
  const OpKind bk = b_mn ? OP_BMN : OP_BK;
  const int brows = b_mn ? K : N, bcols = b_mn ? N : K;
  if (!encode_map(&hm[0], MapSpec{A, M, K, lda, esz, OP_A, BN, BK}) ||
      !encode_map(&hm[1], MapSpec{B, brows, bcols, ldb, esz, bk, BN, BK}))
    return fail(PRISM_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  if (split) {
    if (!encode_map(&hm[2], MapSpec{A_lo, M, K, lda, esz, OP_A, BN, BK}) ||
        !encode_map(&hm[3], MapSpec{B_lo, brows, bcols, ldb, esz, bk, BN, BK}))
      return fail(PRISM_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  }
  GemmProblem* gp = reinterpret_cast<GemmProblem*>(hb + 4 * sizeof(CUtensorMap));
  const CUtensorMap* dm = reinterpret_cast<const CUtensorMap*>(wsd);
  gp->tmA = dm; gp->tmB = dm + 1;
  gp->tmA_lo = split ? dm + 2 : nullptr; gp->tmB_lo = split ? dm + 3 : nullptr;
  gp->out = out; gp->out_lo = out_lo; gp->C = C; gp->C_lo = C_lo;
  gp->norm_part = norm_part; gp->gdiag = gdiag; gp->alpha = alpha_dev;
  gp->ldo = ldo; gp->ldc = ldc; gp->M = M; gp->N = N; gp->K = K;
  gp->mode = mode; gp->sym = sym; gp->matrix = 0; gp->scale_by_alpha = scale_by_alpha;
  gp->tiles_n = (N + BN - 1) / BN; gp->c1 = c1;
  LaunchDesc L;
  HostProblem hp;
  hp.p = *gp;
  L.probs.push_back(hp);
  add_tiles(L, 0, M, N, BN, sym != 0);
  const size_t tiles_off = 4 * sizeof(CUtensorMap) + align_up(sizeof(GemmProblem), 128);
  std::memcpy(hb + tiles_off, L.tiles.data(), 4 * L.tiles.size());
  PRISM_CK(cudaMemcpyAsync(wsd, hb, need, cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)));
  GemmLaunch g;
  g.probs = reinterpret_cast<const GemmProblem*>(wsd + 4 * sizeof(CUtensorMap));
  g.tiles = reinterpret_cast<const uint32_t*>(wsd + tiles_off);
  g.done = nullptr;
  g.done_stride = 0;
  g.ntiles = (int)L.tiles.size();
  PRISM_CK(launch_gemm(precision, b_mn != 0, g, static_cast<cudaStream_t>(stream)));
  PRISM_CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  return PRISM_OK;
}

prism_status prism_debug_sketch(uint64_t seed, int64_t b, int k, int p, int s, float* S_dev, void* stream) {
  if (!S_dev || p < 1 || s < 1) return fail(PRISM_ERR_INVALID_ARG, "bad sketch args");
  const long long pairs = ((long long)p * s + 1) / 2;
  k_sketch_debug<<<(unsigned)((pairs + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      seed, (int)b, k, p, s, S_dev);
  PRISM_CK(cudaGetLastError());
  return PRISM_OK;
}

prism_status prism_debug_argmin(int n, const double* c_dev, double lo, double hi, double a_taylor,
                                double* alpha_dev, void* stream) {
  if (n < 1 || !c_dev || !alpha_dev) return fail(PRISM_ERR_INVALID_ARG, "bad argmin args");
  k_argmin_debug<<<(n + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(n, c_dev, lo, hi, a_taylor,
                                                                                 alpha_dev);
  PRISM_CK(cudaGetLastError());
  return PRISM_OK;
}

}  // extern "C"
