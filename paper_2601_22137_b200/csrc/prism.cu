// Host side of libprism.so: argument validation, planning (workspace layout,
// TMA tensor maps, grouped tile lists), and the device-side iteration loop
// (no host synchronisation anywhere on the solve path).  See include/prism.h
// for the contract and DESIGN.md for the data layout.
#include "../../include/prism.h"
#include "launch.h"
#include "kernels.cuh"
#include "internal.h"

#include <algorithm>
#include <atomic>
#include <array>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <list>
#include <map>
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
  static const EncodeTiledFn fn = [] {   // thread-safe one-time lookup
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeTiledFn>(p);
    return (EncodeTiledFn) nullptr;
  }();
  return fn;
}

// OP_A: K-major A tile (box BK x 128); OP_BK: K-major B tile (box BK x BN);
// OP_MN: MN-major operand (box 128-B x BK), A or B.
enum OpKind { OP_A = 0, OP_BK = 1, OP_MN = 2, OP_EPI = 3 };   // OP_EPI: 32 x 32 epilogue block

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
  if (s.kind == OP_EPI) { box[0] = 32; box[1] = 32; }
  else if (s.kind == OP_A) { box[0] = s.BK; box[1] = 128; }
  else if (s.kind == OP_BK) { box[0] = s.BK; box[1] = s.BN; }   // BN = rows of B per CTA
  else { box[0] = 128 / s.esz; box[1] = s.BK; }
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(out, s.esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                  const_cast<void*>(s.ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  s.kind == OP_EPI                  ? CU_TENSOR_MAP_SWIZZLE_64B
                  : (s.kind == OP_MN && s.esz == 4) ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                                                    : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// ------------------------------------------------------------------ kernel dispatch
constexpr int kTileM = 256;   // main GEMMs run on CTA pairs: tiles of 256 rows x BN columns
constexpr int kChunkP = 8;    // sketch columns per chain problem (chaint.cuh: 4 x 8 W rows per MMA)
constexpr int kMaxSketch = 64;

int tile_bn(int precision) { return precision == PRISM_BF16 ? 256 : 128; }
int tile_bk(int precision) { return precision == PRISM_BF16 ? 64 : 32; }
int elem_size(int precision) { return precision == PRISM_BF16 ? 2 : 4; }

// ------------------------------------------------------------------ planning
struct HostProblem {
  GemmProblem p;      // tm* fields hold map indices (+1; 0 = none) until serialised
  int mapA, mapB, mapA_lo, mapB_lo;
  int mapC, mapO;     // bf16 epilogue blocks (TMA load of C, TMA store of the output)
  int mapO2;          // bf16 APPLY2 second output
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
  ~Plan() {
    if (exec) cudaGraphExecDestroy(exec);
    if (meta_dev) cudaFree(meta_dev);
  }
  // plan constants (matrix descriptors, tile lists, problem tables, tensor maps) in a
  // device allocation owned by the plan, uploaded once when the plan is built: a per-solve
  // upload would queue behind unrelated host->device copies on the copy engine
  char* meta_dev = nullptr;
  cudaGraphExec_t exec = nullptr;   // CUDA graph: WHILE(any matrix active) { one iteration }
  int* d_iter = nullptr;            // device iteration counter
  int* d_all_done = nullptr;
  int per_iter_launches = 0;
  std::vector<long long> key;
  size_t ws_need = 0;
  size_t meta_off = 0, meta_bytes = 0;
  std::unique_ptr<uint8_t, PinnedDeleter> blob;
  SolveParams params{};
  LaunchDesc gram[2], square, square2, apply[2], chaint[5];
  LaunchDesc gram0, apply0;   // folded normalisation: iteration 0 reads A (scaled by 1/c) instead of X_0
  LaunchDesc apply0f;         // ... and writes X_1 into Q (matrices whose Q holds the odd iterates)
  bool square_early = false;  // the square GEMM's mainloop runs under k_alpha (run_solve)
  // per-iteration compacted tile lists (k_alpha's compaction blocks): 0 Gram, 1 square, 2 apply
  struct Compact {
    bool on = false;
    int c_from = 0;
    std::vector<int> runs;   // (start, length, matrix) per run of one matrix's tiles
    size_t runs_off = 0, dst_off = 0, count_off = 0;
  } compact[3];
  bool fold = false;          // some matrix folds (iteration-0 tables present)
  bool unfolded = true;       // some matrix needs k_normalize
  // row-block split: packed partial-Gram launches per panel group, the
  // APPLY2 launch (Y = X R, X + Y/2) of d = 2, the packed fp32 Gram, its layout
  std::vector<LaunchDesc> rbgram[2];
  LaunchDesc rb1[2];
  float* Gp = nullptr;
  double* rb_fro2 = nullptr;
  std::vector<long long> panel_off;   // float offset of panel t, [ceil(n/256) + 1]
  std::vector<int> group_end;         // first panel after group g
  std::vector<LaunchDesc> gjT, gjS;   // DB Newton sweep steps: T = D E, W -= E^T T
  bool db = false;
  int db_steps = 0;
  int n_chain = 0;
  std::vector<std::pair<size_t, size_t>> guards;   // workspace guard bands (diagnostics)
  int chain_ksplit = 1;   // cluster size of the chain launches (split-K; 1, 2 or 4)
  int chain_bn = 256;     // rows of R per chain tile (128 when the 128-row tiles still fit the SMs)
  bool has_square = false, has_square2 = false;
  int inv_q = 0;                    // inverse Newton root order (0: other kinds)
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
  bool rowblock = false;   // row-block member of a split tall matrix: force the tall form, s = n
  int rb_groups = 1;       // row-block: panel groups of the packed Gram (all-reduced one by one)
  bool sign_kind = false;  // matrix sign: square path, R = I - X^2, X only (output in Q)
  int inv_q = 0;           // coupled inverse Newton A^{-1/q}: X in X[], M in Y[], R = I - M (output in Q)
  bool cheb_kind = false;  // Chebyshev inverse: A' = A/c in Y[0], R stored transposed, output X / c in Q
  bool db_kind = false;    // DB Newton product form (sqrt path shapes; FP32 only; outputs in Q, Q2)
};

void resolve_interval(prism_options& o, double& lo, double& hi, double& aT, int& d, int inv_q = 0,
                      bool cheb = false, bool db = false) {
  d = (o.degree == 3) ? 1 : 2;
  double dlo = d == 1 ? 0.5 : 0.375, dhi = d == 1 ? 1.0 : 1.45;
  aT = d == 1 ? 0.5 : 0.375;   // Taylor coefficient of xi^d in (1-xi)^{-1/2}
  if (inv_q) {                 // inverse Newton (first order): [1/(2q), 2/q], Taylor 1/q (R22)
    d = 1;
    dlo = 0.5 / inv_q;
    dhi = 2.0 / inv_q;
    aT = 1.0 / inv_q;
  }
  if (cheb) {                  // Chebyshev: [1/2, 2], Taylor 1 (f_2 = 1 + xi + xi^2)
    d = 2;
    dlo = 0.5;
    dhi = 2.0;
    aT = 1.0;
  }
  if (db) {                    // DB Newton: unconstrained; classical step 1/2
    d = 1;
    dlo = dhi = aT = 0.5;
  }
  lo = std::isnan(o.alpha_lo) ? dlo : o.alpha_lo;
  hi = std::isnan(o.alpha_hi) ? dhi : o.alpha_hi;
}

// Workspace guard bands (diagnostics, prism_debug_workspace_guards): with the switch on,
// every workspace sub-buffer is followed by kGuardBytes that no kernel may touch; the
// plan records them and prism_debug_guards_fill / _check test them around a solve (the
// pool refuses compute-sanitizer).
constexpr size_t kGuardBytes = 256;
static std::atomic<int> g_guard_ws{0};

struct Bump {
  char* base;
  std::vector<std::pair<size_t, size_t>>* guards = nullptr;   // (offset, bytes) when guarded
  size_t off = 0;
  char* take(size_t bytes, size_t align = 256) {
    off = align_up(off, align);
    char* p = base + off;
    off += bytes;
    if (guards) {
      off = align_up(off, 16);
      guards->push_back({off, kGuardBytes});
      off += kGuardBytes;
    }
    return p;
  }
};

void add_tiles(LaunchDesc& L, int prob, int M, int N, int BN, bool sym) {
  const int tm_n = (M + kTileM - 1) / kTileM, tn_n = (N + BN - 1) / BN;
  for (int tm = 0; tm < tm_n; ++tm)
    for (int tn = 0; tn < tn_n; ++tn) {
      if (sym && tn * BN + BN - 1 < tm * kTileM) continue;
      L.tiles.push_back(((uint32_t)prob << 20) | ((uint32_t)tm << 10) | (uint32_t)tn);
    }
}

// Chain split-K factor of one matrix (cluster of CTAs sharing a 256-row tile of R): a
// function of its size s alone (never of the batch), so a matrix's bits do not depend on
// what it is batched with (or on the rank it lands on).  Each slice keeps >= 8 k-blocks.
int chain_ks(int s) {   // clusters of 8 do not all co-schedule
  return s < 1024 ? 1 : s < 2048 ? 2 : 4;
}

// GEMM tile order within a matrix: groups of 8 tile rows walked column by column, so that a
// wave of 74 pair tiles reads ~8 A and ~9 B panels instead of ~2 and all of them: matrices
// larger than L2 re-read fewer operand panels from HBM (8192^2 polar 23.6-25.3 -> 22.7-23.0 ms;
// smaller ones unchanged; scripts/probe_raster.py).  prism_debug_raster_rows overrides it.
static uint32_t g_raster_rows = 8;
void sort_tiles_by_cost(LaunchDesc& L, bool raster = false) {
  std::stable_sort(L.tiles.begin(), L.tiles.end(), [&](uint32_t a, uint32_t b) {
    return L.probs[a >> 20].p.K > L.probs[b >> 20].p.K;
  });
  if (!raster || g_raster_rows <= 1) return;
  size_t i = 0;
  while (i < L.tiles.size()) {
    size_t j = i;
    while (j < L.tiles.size() && (L.tiles[j] >> 20) == (L.tiles[i] >> 20)) ++j;
    std::stable_sort(L.tiles.begin() + i, L.tiles.begin() + j, [&](uint32_t a, uint32_t b) {
      const uint32_t ga = ((a >> 10) & 1023) / g_raster_rows, gb = ((b >> 10) & 1023) / g_raster_rows;
      if (ga != gb) return ga < gb;
      if ((a & 1023) != (b & 1023)) return (a & 1023) < (b & 1023);
      return ((a >> 10) & 1023) < ((b >> 10) & 1023);
    });
    i = j;
  }
}

// Packed upper-triangle layout of the row-block Gram (gemm.cuh epi_gram32): panel t = rows
// [256t, 256t + 256) x columns [256t, n), ld n - 256t; groups of panels with about equal
// upper-triangle tile counts (each group is all-reduced as soon as its launch completes).
void rowblock_layout(long long n, int ngroups, std::vector<long long>& off, std::vector<int>& gend) {
  const int T = (int)((n + kTileM - 1) / kTileM);
  off.assign(T + 1, 0);
  std::vector<double> tiles(T);
  double tot = 0.0;
  for (int t = 0; t < T; ++t) {
    const long long h = std::min<long long>(kTileM, n - (long long)kTileM * t), w = n - (long long)kTileM * t;
    off[t + 1] = off[t] + h * w;
    tiles[t] = (double)w;
    tot += tiles[t];
  }
  ngroups = std::max(1, std::min(ngroups, T));
  gend.assign(ngroups, T);
  double acc = 0.0;
  int g = 0;
  for (int t = 0; t < T && g < ngroups - 1; ++t) {
    acc += tiles[t];
    if (acc >= tot * (g + 1) / ngroups) gend[g++] = t + 1;
  }
  for (; g < ngroups - 1; ++g) gend[g] = T;
  for (int x = 1; x < ngroups; ++x) gend[x] = std::max(gend[x], gend[x - 1]);
}

// Build the full plan.  When r.ws == nullptr only sizes are computed.
prism_status build_plan(const Request& r, Plan& P) {
  prism_options o = r.o;
  double lo, hi, aT;
  int d;
  resolve_interval(o, lo, hi, aT, d, r.inv_q, r.cheb_kind, r.db_kind);
  const bool cheb = r.cheb_kind;
  const bool db = r.db_kind;
  int db_steps = 0;
  const int prec = o.precision;
  const int iq = r.inv_q;
  const int esz = elem_size(prec);
  const bool split = prec == PRISM_FP32;
  const int BN = tile_bn(prec), BK = tile_bk(prec);
  const int p = o.sketch_size;
  const int B = r.batch;
  Bump bump{r.ws};
  P.guards.clear();
  if (g_guard_ws.load()) bump.guards = &P.guards;

  // state region
  MatState* d_st = reinterpret_cast<MatState*>(bump.take(sizeof(MatState) * B));
  double* d_fro = reinterpret_cast<double*>(bump.take(sizeof(double) * B * kFroParts));
  int* d_iter = reinterpret_cast<int*>(bump.take(2 * sizeof(int)));
  double* d_ahist = reinterpret_cast<double*>(bump.take(sizeof(double) * B * o.max_iters));
  float* d_rhist = reinterpret_cast<float*>(bump.take(sizeof(float) * B * (o.max_iters + 1)));

  std::vector<MatDesc> mats(B);
  std::vector<MapSpec> maps;
  auto add_map = [&](const void* ptr, int rows, int cols, long long ld, OpKind k) -> int {
    maps.push_back(MapSpec{ptr, rows, cols, ld, esz, k, BN / 2, BK});   // CTA pairs: half of B per CTA
    return (int)maps.size();   // 1-based index
  };

  P.max_s = P.max_rows = P.max_cols = P.max_m = P.max_n = 0;
  // Folded normalisation (BF16 / TF32 polar): iteration 0's Gram and apply read A itself with
  // 1/c^2 and 1/c in their epilogues, and X[0] is the caller's output Q, so no pass writes
  // X_0 = A/||A||_F and a solve ending on an even iteration needs no final copy.  Needs
  // TMA-legal A and Q (16-B aligned base and leading dimension); 3xTF32 needs split operands.
  // Per matrix (a matrix's bits never depend on what it is batched with); the plan carries
  // iteration-0 tables whenever any matrix folds (the others read their X_0 there).
  const bool fold_kind = !r.sqrt_kind && !r.sign_kind && !iq && !cheb && !db && !r.rowblock && prec != PRISM_FP32 &&
                         d == 2 && r.Q;
  auto fold_ok = [&](int i) {
    return fold_kind && ((uintptr_t)r.A[i] % 16 == 0) && ((r.lda[i] * esz) % 16 == 0) && r.Q[i] &&
           ((uintptr_t)r.Q[i] % 16 == 0) && ((r.ldq[i] * esz) % 16 == 0);
  };
  bool fold = false, unfolded = false;
  for (int i = 0; i < B; ++i) {
    fold = fold || fold_ok(i);
    unfolded = unfolded || !fold_ok(i);
  }
  P.fold = fold;
  P.unfolded = unfolded;
  // Q may take the odd iterates (iteration 0's apply writes X_1 there while the same launch
  // still reads the inputs) only when it overlaps no input of the batch
  auto span = [&](const void* p, long long ld, int i) {
    const uintptr_t b = (uintptr_t)p;
    return std::make_pair(b, b + (uintptr_t)(((long long)(r.m[i] - 1) * ld + r.n[i]) * esz));
  };
  auto flip_ok = [&](int i) {
    if (!fold_ok(i)) return false;
    const auto q = span(r.Q[i], r.ldq[i], i);
    for (int j = 0; j < B; ++j) {
      const auto a = span(r.A[j], r.lda[j], j);
      if (a.first < q.second && q.first < a.second) return false;
    }
    return true;
  };
  for (int i = 0; i < B; ++i) {
    MatDesc& D = mats[i];
    std::memset(&D, 0, sizeof(D));
    const int m = (int)r.m[i];
    const int n = (r.sqrt_kind || db) ? (int)r.m[i] : (int)r.n[i];
    D.A = r.A[i];
    D.Q = r.Q ? r.Q[i] : nullptr;
    D.Q2 = r.Q2 ? r.Q2[i] : nullptr;
    D.lda = r.lda[i];
    D.ldq = r.ldq[i];
    D.m = m;
    D.n = n;
    if (r.sqrt_kind || db) { D.s = n; D.L = n; }
    else if (r.rowblock) { D.s = n; D.L = m; }
    else { D.s = std::min(m, n); D.L = std::max(m, n); }
    D.trans = 0;   // X keeps A's row-major layout (no transposes; MN-major operands instead)
    D.sketch_id = r.ids ? (int)r.ids[i] : i;
    const int s = D.s, L = D.L;
    const long long ldx = (long long)align_up(n, 64), ldr = (long long)align_up(s, 64);
    D.ldx = ldx;
    D.ldr = ldr;
    const size_t xbytes = (size_t)m * ldx * esz, rbytes = (size_t)s * ldr * esz;
    D.ldx0 = ldx;
    for (int t = 0; t < 2; ++t) {
      D.X[t] = bump.take(xbytes);   // (taken even when X[0] is Q: the size must not depend on pointers)
      D.X_lo[t] = split ? bump.take(xbytes) : nullptr;
      if (r.sqrt_kind || iq || db || (cheb && t == 0) || (r.rowblock && d == 2)) {   // row-block: Y, X + Y/2
        D.Y[t] = bump.take(xbytes);
        D.Y_lo[t] = split ? bump.take(xbytes) : nullptr;
      }
    }
    D.fold = fold_ok(i) ? 1 : 0;
    D.flip_ok = flip_ok(i) ? 1 : 0;
    if (D.fold) {
      D.X[0] = r.Q[i];
      D.ldx0 = r.ldq[i];
    }
    const long long ldxs[2] = {D.ldx0, ldx};
    D.R = bump.take(rbytes);
    D.R_lo = split ? bump.take(rbytes) : nullptr;
    void* Pm = (iq ? iq >= 2 : (d == 2 && !db && !r.rowblock)) ? bump.take(rbytes) : nullptr;   // Chebyshev: d = 2 (P^T)
    void* Pm_lo = (Pm && split) ? bump.take(rbytes) : nullptr;
    void* Pm2 = iq >= 3 ? bump.take(rbytes) : nullptr;
    void* Pm2_lo = (Pm2 && split) ? bump.take(rbytes) : nullptr;
    D.gdiag = reinterpret_cast<float*>(bump.take(sizeof(float) * s));
    D.tiles_m = (s + 127) / 128;
    D.tiles_n = (s + BN - 1) / BN;
    if (r.rowblock) D.tiles_m = D.tiles_n = (s + 63) / 64;   // k_resid_packed's 64 x 64 norm tiles
    D.sym = (r.sqrt_kind || r.sign_kind || iq || cheb || db || r.rowblock) ? 0 : 1;
    D.norm_part = reinterpret_cast<float*>(bump.take(sizeof(float) * D.tiles_m * D.tiles_n));
    const long long ldS = (long long)align_up(s, 64);
    D.ldS = ldS;
    // Sketch columns are processed in chunks of <= kChunkP (the products R^i S^T are column-
    // separable; each chunk is its own chain problem with its own W / keep / partials, and
    // k_alpha sums the <Va,Vb> partials of every chunk): p up to kMaxSketch.
    const int nch = (p + kChunkP - 1) / kChunkP;
    const int pw = nch == 1 ? p : kChunkP;   // width of a chunk region
    D.nchunk = nch;
    D.S = reinterpret_cast<float*>(bump.take(sizeof(float) * p * ldS));
    D.W[0] = bump.take((size_t)esz * 4 * pw * ldS * nch);
    D.W[1] = bump.take((size_t)esz * 4 * pw * ldS * nch);
    D.keep = reinterpret_cast<float*>(bump.take(sizeof(float) * 4 * (size_t)s * pw * nch));
    // <Va,Vb> partials of the chain: one per 32-row group of R and chunk (chaint.cuh, epi_chain)
    D.chain_tiles = nch * ((s + 31) / 32);
    D.chain_part = reinterpret_cast<double*>(bump.take(sizeof(double) * kChainG * D.chain_tiles));
    P.max_s = std::max(P.max_s, s);
    P.max_rows = std::max(P.max_rows, s);
    P.max_cols = std::max(P.max_cols, L);
    P.max_m = std::max(P.max_m, m);
    P.max_n = std::max(P.max_n, n);
    if (L / BN >= 1023 || L / 128 >= 1023)
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
      h.p.c1 = 1.f;                          // out = c1 a^eC C + kA a^eA D
      h.p.kA = 1.f;
      h.p.eA = mode == EPI_POLY ? 1 : 0;
      if (esz == 2 && (mode == EPI_RESID || mode == EPI_POLY || mode == EPI_APPLY || mode == EPI_STORE ||
                       mode == EPI_APPLY2)) {
        maps.push_back(MapSpec{out, M, N, ldo, esz, OP_EPI, 32, 32});
        h.mapO = (int)maps.size();
        if (C) {
          maps.push_back(MapSpec{C, M, N, ldc, esz, OP_EPI, 32, 32});
          h.mapC = (int)maps.size();
        }
      }
      return h;
    };
    if (db) {
      // DB Newton: W (= R) is swept in place into -M^{-1} by blocked
      // Gauss-Jordan (R28), then X' = (1-a) X - a X W, Y' = (1-a) Y - a Y W
      const int nn = s;
      const size_t ebytes = (size_t)kGJ * ldx * esz;
      D.Mst = reinterpret_cast<float*>(bump.take((size_t)nn * ldx * sizeof(float)));
      D.E = bump.take(ebytes);
      D.E_lo = bump.take(ebytes);
      D.T = bump.take(ebytes);
      D.T_lo = bump.take(ebytes);
      D.Dp = bump.take((size_t)kGJ * kGJ * esz);
      D.Dp_lo = bump.take((size_t)kGJ * kGJ * esz);
      D.dbpart = reinterpret_cast<double*>(bump.take(sizeof(double) * 3 * D.tiles_m * D.tiles_n));
      const int nb = (nn + kGJ - 1) / kGJ;
      db_steps = std::max(db_steps, nb);
      if ((int)P.gjT.size() < nb) { P.gjT.resize(nb); P.gjS.resize(nb); }
      for (int j = 0; j < nb; ++j) {
        const int bj = std::min(kGJ, nn - kGJ * j);
        HostProblem tp = mk(bj, nn, bj, EPI_STORE, 0, D.T, D.T_lo, ldx, nullptr, nullptr, 0);   // T = D E
        tp.p.b_mn = 1;
        tp.mapA = add_map(D.Dp, bj, bj, kGJ, OP_A);
        tp.mapA_lo = add_map(D.Dp_lo, bj, bj, kGJ, OP_A);
        tp.mapB = add_map(D.E, bj, nn, ldx, OP_MN);
        tp.mapB_lo = add_map(D.E_lo, bj, nn, ldx, OP_MN);
        P.gjT[j].probs.push_back(tp);
        HostProblem sp = mk(nn, nn, bj, EPI_POLY, 1, D.R, D.R_lo, ldr, D.R, D.R_lo, ldr);       // W -= E^T T
        sp.p.c1 = 1.f; sp.p.eC = 0; sp.p.kA = -1.f; sp.p.eA = 0;
        sp.p.a_mn = sp.p.b_mn = 1;
        sp.mapA = add_map(D.E, bj, nn, ldx, OP_MN);
        sp.mapA_lo = add_map(D.E_lo, bj, nn, ldx, OP_MN);
        sp.mapB = add_map(D.T, bj, nn, ldx, OP_MN);
        sp.mapB_lo = add_map(D.T_lo, bj, nn, ldx, OP_MN);
        P.gjS[j].probs.push_back(sp);
      }
      for (int t = 0; t < 2; ++t) {
        for (int y = 0; y < 2; ++y) {
          void* const* Z = y ? D.Y : D.X;
          void* const* Zl = y ? D.Y_lo : D.X_lo;
          HostProblem u = mk(nn, nn, nn, EPI_APPLY, 0, Z[1 - t], Zl[1 - t], ldx, Z[t], Zl[t], ldx);
          u.p.c1 = -1.f; u.p.eC = 1; u.p.lC = 1.f;    // (1 - a) Z
          u.p.kA = -1.f; u.p.eA = 1;                   // - a Z W = a Z M^{-1}
          u.mapA = add_map(Z[t], nn, nn, ldx, OP_A);
          u.mapB = add_map(D.R, nn, nn, ldr, OP_BK);   // W symmetric: rows of W
          u.mapA_lo = add_map(Zl[t], nn, nn, ldx, OP_A);
          u.mapB_lo = add_map(D.R_lo, nn, nn, ldr, OP_BK);
          P.apply[t].probs.push_back(u);
        }
      }
    } else if (cheb) {
      // Chebyshev with R^T stored: R^T = I - X^T A'^T (A = X MN-major, B = A'
      // K-major), P^T = R^T + a R^T R^T, X' = X + X P (B = P^T K-major)
      const int nn = s;
      for (int t = 0; t < 2; ++t) {
        HostProblem g = mk(nn, nn, nn, EPI_RESID, 0, D.R, D.R_lo, ldr, nullptr, nullptr, 0);
        g.p.norm_part = D.norm_part;
        g.p.gdiag = D.gdiag;
        g.p.a_mn = 1;
        g.mapA = add_map(D.X[t], nn, nn, ldx, OP_MN);
        g.mapB = add_map(D.Y[0], nn, nn, ldx, OP_BK);
        if (split) { g.mapA_lo = add_map(D.X_lo[t], nn, nn, ldx, OP_MN); g.mapB_lo = add_map(D.Y_lo[0], nn, nn, ldx, OP_BK); }
        P.gram[t].probs.push_back(g);
        HostProblem ax = mk(nn, nn, nn, EPI_APPLY, 0, D.X[1 - t], D.X_lo[1 - t], ldx, D.X[t], D.X_lo[t], ldx);
        ax.mapA = add_map(D.X[t], nn, nn, ldx, OP_A);
        ax.mapB = add_map(Pm, nn, nn, ldr, OP_BK);
        if (split) { ax.mapA_lo = add_map(D.X_lo[t], nn, nn, ldx, OP_A); ax.mapB_lo = add_map(Pm_lo, nn, nn, ldr, OP_BK); }
        P.apply[t].probs.push_back(ax);
      }
      HostProblem q = mk(nn, nn, nn, EPI_POLY, 0, Pm, Pm_lo, ldr, D.R, D.R_lo, ldr);   // c1 = 1, a^1
      q.p.b_mn = 1;
      q.mapA = add_map(D.R, nn, nn, ldr, OP_A);
      q.mapB = add_map(D.R, nn, nn, ldr, OP_MN);
      if (split) { q.mapA_lo = add_map(D.R_lo, nn, nn, ldr, OP_A); q.mapB_lo = add_map(D.R_lo, nn, nn, ldr, OP_MN); }
      P.square.probs.push_back(q);
    } else if (iq) {
      // coupled inverse Newton: R = I - M (elementwise, k_resid_inv),
      // X' = X + a X R, M' = (I + a R)^q M = M + P_q M with P_q = (I + a R)^q - I:
      //   q = 1: P_1 = a R (in the apply epilogue)
      //   q = 2: P_2 = 2a R + a^2 R.R
      //   q = 3: T = 3a R + a^2 R.R, P_3 = 3a R + a R.T   (Horner)
      //   q = 4: P_2 as above, P_4 = 2 P_2 + P_2.P_2      (squaring)
      const int nn = s;
      auto poly = [&](void* out, void* out_lo, const void* C, const void* C_lo, const void* Aop, const void* Aop_lo,
                      const void* Bop, const void* Bop_lo, float kC, int eC, float kA, int eA) {
        HostProblem q = mk(nn, nn, nn, EPI_POLY, 0, out, out_lo, ldr, C, C_lo, ldr);
        q.p.c1 = kC; q.p.eC = eC; q.p.kA = kA; q.p.eA = eA;
        q.p.b_mn = 1;
        q.mapA = add_map(Aop, nn, nn, ldr, OP_A);
        q.mapB = add_map(Bop, nn, nn, ldr, OP_MN);
        if (split) { q.mapA_lo = add_map(Aop_lo, nn, nn, ldr, OP_A); q.mapB_lo = add_map(Bop_lo, nn, nn, ldr, OP_MN); }
        return q;
      };
      const void* Pq = D.R;
      const void* Pq_lo = D.R_lo;
      if (iq == 2) {
        P.square.probs.push_back(poly(Pm, Pm_lo, D.R, D.R_lo, D.R, D.R_lo, D.R, D.R_lo, 2.f, 1, 1.f, 2));
        Pq = Pm; Pq_lo = Pm_lo;
      } else if (iq == 3) {
        P.square.probs.push_back(poly(Pm, Pm_lo, D.R, D.R_lo, D.R, D.R_lo, D.R, D.R_lo, 3.f, 1, 1.f, 2));
        P.square2.probs.push_back(poly(Pm2, Pm2_lo, D.R, D.R_lo, D.R, D.R_lo, Pm, Pm_lo, 3.f, 1, 1.f, 1));
        Pq = Pm2; Pq_lo = Pm2_lo;
      } else if (iq == 4) {
        P.square.probs.push_back(poly(Pm, Pm_lo, D.R, D.R_lo, D.R, D.R_lo, D.R, D.R_lo, 2.f, 1, 1.f, 2));
        P.square2.probs.push_back(poly(Pm2, Pm2_lo, Pm, Pm_lo, Pm, Pm_lo, Pm, Pm_lo, 2.f, 0, 1.f, 0));
        Pq = Pm2; Pq_lo = Pm2_lo;
      }
      for (int t = 0; t < 2; ++t) {
        HostProblem ax = mk(nn, nn, nn, EPI_APPLY, 0, D.X[1 - t], D.X_lo[1 - t], ldx, D.X[t], D.X_lo[t], ldx);
        ax.p.scale_by_alpha = ax.p.eA = 1;                     // X + a X R
        ax.p.b_mn = 1;
        ax.mapA = add_map(D.X[t], nn, nn, ldx, OP_A);
        ax.mapB = add_map(D.R, nn, nn, ldr, OP_MN);
        if (split) { ax.mapA_lo = add_map(D.X_lo[t], nn, nn, ldx, OP_A); ax.mapB_lo = add_map(D.R_lo, nn, nn, ldr, OP_MN); }
        P.apply[t].probs.push_back(ax);
        HostProblem am = mk(nn, nn, nn, EPI_APPLY, 0, D.Y[1 - t], D.Y_lo[1 - t], ldx, D.Y[t], D.Y_lo[t], ldx);
        am.p.scale_by_alpha = am.p.eA = iq == 1;               // M + P_q M
        am.p.b_mn = 1;
        am.mapA = add_map(Pq, nn, nn, ldr, OP_A);
        am.mapB = add_map(D.Y[t], nn, nn, ldx, OP_MN);
        if (split) { am.mapA_lo = add_map(Pq_lo, nn, nn, ldr, OP_A); am.mapB_lo = add_map(D.Y_lo[t], nn, nn, ldx, OP_MN); }
        P.apply[t].probs.push_back(am);
      }
    } else if (r.rowblock) {
      // row-block member (rows x n of one tall polar problem): packed partial
      // Gram X_r^T X_r (fp32 panels, one launch per panel group), then d = 2:
      //   Y = X_r R and Xh = X_r + Y/2 (APPLY2), X_r' = Xh + a Y R (APPLY)   [= X_r g_2(R; a)]
      // d = 1: X_r' = X_r + a X_r R.  R is stored whole (both triangles) by k_resid_packed.
      rowblock_layout(n, r.rb_groups, P.panel_off, P.group_end);
      P.Gp = reinterpret_cast<float*>(bump.take(sizeof(float) * (size_t)P.panel_off.back()));
      P.rb_fro2 = reinterpret_cast<double*>(bump.take(sizeof(double)));
      for (int t = 0; t < 2; ++t) {
        P.rbgram[t].assign(r.rb_groups, LaunchDesc{});
        for (int g = 0; g < r.rb_groups; ++g) {
          HostProblem gp = mk(s, s, m, EPI_GRAM32, 1, P.Gp, nullptr, 0, nullptr, nullptr, 0);
          gp.p.a_mn = gp.p.b_mn = 1;
          gp.mapA = gp.mapB = add_map(D.X[t], m, n, ldx, OP_MN);
          if (split) gp.mapA_lo = gp.mapB_lo = add_map(D.X_lo[t], m, n, ldx, OP_MN);
          P.rbgram[t][g].probs.push_back(gp);
        }
        if (d == 2) {
          HostProblem a1 = mk(m, n, s, EPI_APPLY2, 0, D.Y[1], D.Y_lo[1], ldx, D.X[t], D.X_lo[t], ldx);
          a1.p.kA = 0.5f;   // X + D/2 (no alpha)
          a1.p.eA = 0;
          a1.p.out2 = D.Y[0];
          a1.p.out2_lo = D.Y_lo[0];
          if (esz == 2) {
            maps.push_back(MapSpec{D.Y[0], m, n, ldx, esz, OP_EPI, 32, 32});
            a1.mapO2 = (int)maps.size();
          }
          a1.mapA = add_map(D.X[t], m, n, ldx, OP_A);
          a1.mapB = add_map(D.R, s, s, ldr, OP_BK);   // R symmetric: its rows are its columns
          if (split) { a1.mapA_lo = add_map(D.X_lo[t], m, n, ldx, OP_A); a1.mapB_lo = add_map(D.R_lo, s, s, ldr, OP_BK); }
          P.rb1[t].probs.push_back(a1);
          HostProblem a2 = mk(m, n, s, EPI_APPLY, 0, D.X[1 - t], D.X_lo[1 - t], ldx, D.Y[1], D.Y_lo[1], ldx);
          a2.p.scale_by_alpha = a2.p.eA = 1;
          a2.mapA = add_map(D.Y[0], m, n, ldx, OP_A);
          a2.mapB = add_map(D.R, s, s, ldr, OP_BK);
          if (split) { a2.mapA_lo = add_map(D.Y_lo[0], m, n, ldx, OP_A); a2.mapB_lo = add_map(D.R_lo, s, s, ldr, OP_BK); }
          P.apply[t].probs.push_back(a2);
        } else {
          HostProblem a = mk(m, n, s, EPI_APPLY, 0, D.X[1 - t], D.X_lo[1 - t], ldx, D.X[t], D.X_lo[t], ldx);
          a.p.scale_by_alpha = a.p.eA = 1;
          a.mapA = add_map(D.X[t], m, n, ldx, OP_A);
          a.mapB = add_map(D.R, s, s, ldr, OP_BK);
          if (split) { a.mapA_lo = add_map(D.X_lo[t], m, n, ldx, OP_A); a.mapB_lo = add_map(D.R_lo, s, s, ldr, OP_BK); }
          P.apply[t].probs.push_back(a);
        }
      }
    } else if (!r.sqrt_kind && !r.sign_kind) {
      // polar: X keeps A's row-major layout (m x n).  Tall (m >= n): G = X^T X with both
      // operands MN-major, X' = X + X P (A = X K-major, B = P K-major by symmetry).
      // Wide (m < n): G = X X^T (both K-major), X' = X + P X (B = X MN-major).
      const bool tall = m >= n;
      // t = 0, 1: X[t] -> X[1-t]; t = 2 (folded plans): iteration 0, A (lda) -> X[1] with 1/c;
      // t = 3: iteration 0's apply writing X_1 into Q = X[0] (flipped parity, MatState.flip)
      for (int t = 0; t < (fold ? 4 : 2); ++t) {
        const bool from_a = t >= 2 && D.fold;   // iteration 0 of a folded matrix: A, scaled by 1/c
        const int src = t == 1 ? 1 : 0;
        const void* Xi = from_a ? r.A[i] : D.X[src];
        const void* Xil = from_a ? nullptr : D.X_lo[src];
        const long long ldi = from_a ? r.lda[i] : ldxs[src];
        const int to = t < 2 ? 1 - t : (t == 3 && D.flip_ok) ? 0 : 1;
        if (t < 3) {
        HostProblem g = mk(s, s, L, EPI_RESID, 1, D.R, D.R_lo, ldr, nullptr, nullptr, 0);
        g.p.norm_part = D.norm_part;
        g.p.gdiag = D.gdiag;
        if (tall) {
          g.p.a_mn = g.p.b_mn = 1;
          g.mapA = g.mapB = add_map(Xi, m, n, ldi, OP_MN);
          if (split) g.mapA_lo = g.mapB_lo = add_map(Xil, m, n, ldi, OP_MN);
        } else {
          g.mapA = add_map(Xi, m, n, ldi, OP_A);
          g.mapB = add_map(Xi, m, n, ldi, OP_BK);
          if (split) { g.mapA_lo = add_map(Xil, m, n, ldi, OP_A); g.mapB_lo = add_map(Xil, m, n, ldi, OP_BK); }
        }
        if (from_a) {   // R_0 = I - A^T A / c^2: the scale through the alpha operand of the epilogue
          g.p.alpha = &d_st[i].inv_c2;
          g.p.eA = 1;
        }
        (t < 2 ? P.gram[t] : P.gram0).probs.push_back(g);
        }
        const void* Pa = d == 2 ? Pm : D.R;
        const void* Pa_lo = d == 2 ? Pm_lo : D.R_lo;
        HostProblem a = mk(m, n, s, EPI_APPLY, 0, D.X[to], D.X_lo[to], ldxs[to], Xi, Xil, ldi);
        a.p.scale_by_alpha = a.p.eA = d == 1;
        if (tall) {
          a.mapA = add_map(Xi, m, n, ldi, OP_A);
          a.mapB = add_map(Pa, s, s, ldr, OP_BK);
          if (split) { a.mapA_lo = add_map(Xil, m, n, ldi, OP_A); a.mapB_lo = add_map(Pa_lo, s, s, ldr, OP_BK); }
        } else {
          a.p.b_mn = 1;
          a.mapA = add_map(Pa, s, s, ldr, OP_A);
          a.mapB = add_map(Xi, m, n, ldi, OP_MN);
          if (split) { a.mapA_lo = add_map(Pa_lo, s, s, ldr, OP_A); a.mapB_lo = add_map(Xil, m, n, ldi, OP_MN); }
        }
        if (from_a) {   // X_1 = A/c + (A/c) P: both epilogue coefficients scaled by 1/c (d = 2: P fixed)
          a.p.alpha = &d_st[i].inv_c;
          a.p.eA = a.p.eC = 1;
        }
        (t < 2 ? P.apply[t] : t == 2 ? P.apply0 : P.apply0f).probs.push_back(a);
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
      // sign: G = X X, X' = X + X P (R general: no symmetric kernels)
      const int nn = s;
      for (int t = 0; t < 2; ++t) {
        HostProblem g = mk(nn, nn, nn, EPI_RESID, 0, D.R, D.R_lo, ldr, nullptr, nullptr, 0);
        g.p.norm_part = D.norm_part;
        g.p.gdiag = D.gdiag;
        g.p.b_mn = 1;
        void* const GA = r.sign_kind ? D.X[t] : D.Y[t];
        void* const GA_lo = r.sign_kind ? D.X_lo[t] : D.Y_lo[t];
        g.mapA = add_map(GA, nn, nn, ldx, OP_A);
        g.mapB = add_map(D.X[t], nn, nn, ldx, OP_MN);
        if (split) { g.mapA_lo = add_map(GA_lo, nn, nn, ldx, OP_A); g.mapB_lo = add_map(D.X_lo[t], nn, nn, ldx, OP_MN); }
        P.gram[t].probs.push_back(g);
        const void* Pa = d == 2 ? Pm : D.R;
        const void* Pa_lo = d == 2 ? Pm_lo : D.R_lo;
        HostProblem ax = mk(nn, nn, nn, EPI_APPLY, 0, D.X[1 - t], D.X_lo[1 - t], ldx, D.X[t], D.X_lo[t], ldx);
        ax.p.scale_by_alpha = ax.p.eA = d == 1;
        ax.p.b_mn = 1;
        ax.mapA = add_map(D.X[t], nn, nn, ldx, OP_A);
        ax.mapB = add_map(Pa, nn, nn, ldr, OP_MN);
        if (split) { ax.mapA_lo = add_map(D.X_lo[t], nn, nn, ldx, OP_A); ax.mapB_lo = add_map(Pa_lo, nn, nn, ldr, OP_MN); }
        P.apply[t].probs.push_back(ax);
        if (r.sign_kind) continue;
        HostProblem ay = mk(nn, nn, nn, EPI_APPLY, 0, D.Y[1 - t], D.Y_lo[1 - t], ldx, D.Y[t], D.Y_lo[t], ldx);
        ay.p.scale_by_alpha = ay.p.eA = d == 1;
        ay.p.b_mn = 1;
        ay.mapA = add_map(Pa, nn, nn, ldr, OP_A);
        ay.mapB = add_map(D.Y[t], nn, nn, ldx, OP_MN);
        if (split) { ay.mapA_lo = add_map(Pa_lo, nn, nn, ldr, OP_A); ay.mapB_lo = add_map(D.Y_lo[t], nn, nn, ldx, OP_MN); }
        P.apply[t].probs.push_back(ay);
      }
      if (d == 2) {
        HostProblem q = mk(nn, nn, nn, EPI_POLY, 0, Pm, Pm_lo, ldr, D.R, D.R_lo, ldr);
        q.p.c1 = 0.5f;
        q.p.b_mn = 1;
        q.mapA = add_map(D.R, nn, nn, ldr, OP_A);
        q.mapB = add_map(D.R, nn, nn, ldr, OP_MN);
        if (split) { q.mapA_lo = add_map(D.R_lo, nn, nn, ldr, OP_A); q.mapB_lo = add_map(D.R_lo, nn, nn, ldr, OP_MN); }
        P.square.probs.push_back(q);
      }
    }
    // sketch chain (thin tcgen05 GEMMs): pass j reads W[j%2], writes W[(j+1)%2]
    if (!db) {
      static const int codes2[5] = {CH2_P1, CH2_P2, CH2_P3, CH2_P4, CH2_P5};
      static const int codes1[3] = {CH1_P1, CH1_P2, CH1_P3};
      static const int nin2[5] = {2, 4, 4, 2, 2};   // rows of B (= 2 x input width) in units of p
      static const int nin1[3] = {2, 2, 2};
      static const int codesi[4][5] = {{CH1_P1, CHI_L1}, {CH1_P1, CH1_P2, CHI_L2}, {CH1_P1, CH1_P2, CHI_K2, CHI_L3},
                                       {CH1_P1, CH1_P2, CHI_K2, CH2_P4, CHI_L4}};
      static const int codesc[3] = {CHC_P1, CHC_P2, CHC_P3};
      const int npass = cheb ? 3 : iq ? iq + 1 : d == 2 ? 5 : 3;
      for (int ch = 0; ch < nch; ++ch) {
      const int pc = std::min(pw, p - ch * pw);    // sketch rows of this chunk
      const size_t wch = (size_t)esz * 4 * pw * ldS * ch;   // byte offset of the chunk's W region
      for (int j = 0; j < npass; ++j) {
        const int N = ((iq || cheb) ? 2 : d == 2 ? nin2[j] : nin1[j]) * pc;
        HostProblem c = mk(s, N, s, EPI_CHAIN, 0, nullptr, nullptr, 0, nullptr, nullptr, 0);
        c.p.pass = cheb ? codesc[j] : iq ? codesi[iq - 1][j] : d == 2 ? codes2[j] : codes1[j];
        c.p.S = D.S + (size_t)ch * pw * ldS;
        c.p.Rg = D.R;
        c.p.Rg_lo = D.R_lo;
        c.p.gdiag = D.gdiag;
        c.p.Wn = static_cast<char*>(D.W[(j + 1) % 2]) + wch;
        c.p.Wi = static_cast<char*>(D.W[j % 2]) + wch;
        c.p.keep = D.keep + (size_t)4 * s * pw * ch;
        c.p.chain_part = D.chain_part + (size_t)kChainG * ((s + 31) / 32) * ch;
        c.p.ldS = D.ldS;
        c.p.ldr = ldr;
        c.p.p = pc;
        c.p.tiles_n = 1;
        c.p.ksplit = chain_ks(s);
        // A = W (rows c, K-major [c][ldS]; box 32 rows, OOB rows zero), B = R (256-row box)
        maps.push_back(MapSpec{static_cast<char*>(D.W[j % 2]) + wch, N, s, D.ldS, esz, OP_BK, 32, BK});
        c.mapA = (int)maps.size();
        maps.push_back(MapSpec{D.R, s, s, ldr, esz, OP_BK, 256, BK});
        c.mapB = (int)maps.size();
        if (split) {
          maps.push_back(MapSpec{D.R_lo, s, s, ldr, esz, OP_BK, 256, BK});
          c.mapB_lo = (int)maps.size();
        }
        P.chaint[j].probs.push_back(c);
      }
      }
    }
  }
  P.inv_q = iq;
  P.has_square = r.rowblock ? false : iq ? iq >= 2 : d == 2;
  P.has_square2 = iq >= 3;
  P.n_chain = db ? 0 : cheb ? 3 : iq ? iq + 1 : (d == 2) ? 5 : 3;
  if (db) P.has_square = false;
  P.db = db;
  P.db_steps = db_steps;
  // tile lists (problem index within its launch)
  auto finish = [&](LaunchDesc& L, bool apply) {
    L.tiles.clear();
    for (int j = 0; j < (int)L.probs.size(); ++j)
      add_tiles(L, j, L.probs[j].p.M, L.probs[j].p.N, BN, L.probs[j].p.sym != 0);
    sort_tiles_by_cost(L, true);
    // bf16 applies: the last, partial wave of the persistent launch (tiles t >= R - R % pairs
    // run one per CTA pair while the other pairs idle) is split in N into BN/2-column tiles,
    // so it takes about half a tile time (4096^2: 34 of 256 tiles -> 68 half tiles on 74 pairs).
    // The per-element accumulation is the same for any N, so a matrix's bits do not depend on
    // the split (GPU test: batch vs single solves).
    bool all_apply = apply && prec == PRISM_BF16 && !L.probs.empty();
    for (const HostProblem& hp : L.probs) all_apply = all_apply && hp.p.mode == EPI_APPLY && hp.p.sym == 0;
    const int pairs = device_sms() / 2, nt = (int)L.tiles.size(), rem = nt % pairs;
    if (all_apply && rem > 0 && 2 * rem <= pairs) {
      std::vector<uint32_t> last(L.tiles.end() - rem, L.tiles.end());
      L.tiles.resize(nt - rem);
      for (uint32_t code : last) {
        const uint32_t q = code >> 20, tm = (code >> 10) & 1023, tn = code & 1023;
        const int N = L.probs[q].p.N;
        for (uint32_t hh = 0; hh < 2; ++hh)
          if ((int)((2 * tn + hh) * (BN / 2)) < N)
            L.tiles.push_back((q << 20) | (tm << 10) | kHalfTile | (2 * tn + hh));
      }
    }
  };
  const bool polar_k = !r.sqrt_kind;
  if (P.fold) {
    finish(P.gram0, false);
    finish(P.apply0, true);
  }
  for (int t = 0; t < 2; ++t) {
    finish(P.gram[t], !polar_k);
    finish(P.apply[t], true);
    if (r.rowblock) {
      finish(P.rb1[t], true);
      // packed Gram: group g holds the upper-triangle tiles of tile rows [group_end[g-1], group_end[g])
      for (int g = 0; g < (int)P.rbgram[t].size(); ++g) {
        LaunchDesc& L = P.rbgram[t][g];
        L.tiles.clear();
        const int t0 = g ? P.group_end[g - 1] : 0, t1 = P.group_end[g];
        const int M = L.probs[0].p.M;
        for (int tm = t0; tm < t1; ++tm)
          for (int tn = 0; tn < (M + BN - 1) / BN; ++tn)
            if (tn * BN + BN - 1 >= tm * kTileM) L.tiles.push_back(((uint32_t)tm << 10) | (uint32_t)tn);
      }
    }
  }
  if (P.has_square) finish(P.square, !polar_k);
  if (P.has_square2) finish(P.square2, !polar_k);
  for (LaunchDesc& L : P.gjT) finish(L, false);
  for (LaunchDesc& L : P.gjS) finish(L, false);
  // chain tiles (chaint.cuh): 256- (or 128-) row tiles of R, each split over a cluster of C CTAs,
  // C = the largest factor of the launch's matrices (smaller factors: empty slices).
  // Tiles of one row tile are contiguous and C-aligned, so slice == cluster rank.
  // A launch whose unsplit row tiles already fill the SMs runs every matrix's slices
  // in one CTA, in order (same bits, no exchange); otherwise each slice gets a CTA.
  P.chain_ksplit = 1;
  P.chain_bn = 256;
  if (P.n_chain) {
    long long rows = 0, rows128 = 0;
    int kmax = 1;
    for (const HostProblem& hp : P.chaint[0].probs) {
      rows += (hp.p.M + 255) / 256;
      rows128 += (hp.p.M + 127) / 128;
      kmax = std::max(kmax, hp.p.ksplit);
    }
    P.chain_ksplit = rows >= device_sms() ? 1 : kmax;
    // 3xTF32: 128-row tiles when they still give one CTA per SM.  Its stages carry R_hi and
    // R_lo (68 KB with 256-row tiles: two stages, latency-bound); 128-row tiles give five
    // (4096^2 fp32 chain 3.65 -> 2.4-2.8 ms per step).  bf16 / tf32 keep 256 rows: their
    // 128-row tiles stayed TMA-bound at the same k-block rate and the larger grid started
    // more CTAs late (4096^2 bf16 chain 0.84 -> 0.90 ms).
    if (prec == PRISM_FP32 && rows128 * P.chain_ksplit <= device_sms()) P.chain_bn = 128;
    // the chain's R maps were made with 256-row boxes: match the tile height
    for (int j = 0; j < P.n_chain; ++j)
      for (const HostProblem& hp : P.chaint[j].probs) {
        if (hp.mapB) maps[hp.mapB - 1].BN = P.chain_bn;
        if (hp.mapB_lo) maps[hp.mapB_lo - 1].BN = P.chain_bn;
      }
  }
  for (int j = 0; j < P.n_chain; ++j) {
    LaunchDesc& T = P.chaint[j];
    T.tiles.clear();
    for (int q = 0; q < (int)T.probs.size(); ++q)
      for (int tn = 0; tn < (T.probs[q].p.M + P.chain_bn - 1) / P.chain_bn; ++tn)
        for (int ks = 0; ks < P.chain_ksplit; ++ks)
          T.tiles.push_back(((uint32_t)q << 20) | ((uint32_t)tn << 10) | (uint32_t)ks);
    sort_tiles_by_cost(T);
  }
  if ((int)P.apply[0].probs.size() >= 4096) return fail(PRISM_ERR_UNSUPPORTED, "batch too large (max 2047 sqrt / 4095 polar)");
  // the square GEMM of bf16 polar batches <= 16 runs its mainloop under k_alpha (it reads
  // its tile list before the wait, so it keeps the full list); see run_solve
  P.square_early = !r.sqrt_kind && !r.sign_kind && !cheb && !iq && !db && !r.rowblock && prec == PRISM_BF16 && B <= 16;
  {
    const LaunchDesc* cl[3] = {&P.gram[0], &P.square, &P.apply[0]};
    const bool want[3] = {!r.rowblock && !db && !iq, P.has_square && !P.square_early && !r.rowblock && !db,
                          !r.rowblock && !db};
    for (int l = 0; l < 3; ++l) {
      Plan::Compact& C = P.compact[l];
      C = Plan::Compact{};
      // bf16 only (the tf32 GEMMs would spill); batches of >= 8 matrices (a lone matrix gains
      // nothing and k_alpha's extra blocks cost ~1.5 us per iteration: sign / Chebyshev 4096^2)
      if (!want[l] || prec != PRISM_BF16 || B < 8 || cl[l]->tiles.empty()) continue;
      const std::vector<uint32_t>& T = cl[l]->tiles;
      for (size_t t = 0; t < T.size();) {
        size_t u = t;
        while (u < T.size() && (T[u] >> 20) == (T[t] >> 20)) ++u;
        C.runs.push_back((int)t);
        C.runs.push_back((int)(u - t));
        C.runs.push_back(cl[l]->probs[T[t] >> 20].p.matrix);
        t = u;
      }
      C.on = (int)C.runs.size() / 3 <= kMaxCompactRuns;
      C.c_from = l == 0 ? 1 : 0;   // iteration 0's Gram runs before any stop test
    }
  }

  // flat 64x64 tile prefixes for the layout kernels (normalise over Xt, finalise over the output)
  std::vector<int> toff(B + 1, 0), ooff(B + 1, 0), foff(B + 1, 0);
  for (int i = 0; i < B; ++i) {
    const MatDesc& D = mats[i];
    foff[i + 1] = foff[i] + fro_parts(D.m, D.n);
    const int tw = 32 * (16 / esz);   // layout tile: 32 rows x 32 16-byte vectors
    toff[i + 1] = toff[i] + ((D.m + 31) / 32) * ((D.n + tw - 1) / tw);
    ooff[i + 1] = toff[i + 1];
  }
  // meta region (serialised blob): [mats][tile prefixes][problems...][tiles...][maps]
  P.meta_off = align_up(bump.off, 1024);
  size_t off = 0;
  const size_t mats_off = off;
  off += sizeof(MatDesc) * B;
  off = align_up(off, 128);
  const size_t toff_off = off;
  off += sizeof(int) * (B + 1);
  const size_t ooff_off = off;
  off += sizeof(int) * (B + 1);
  const size_t foff_off = off;
  off += sizeof(int) * (B + 1);
  off = align_up(off, 128);
  const size_t tmat_off = off;   // layout tile -> matrix (normalise / finalise: no search)
  off += sizeof(int) * (size_t)toff[B];
  off = align_up(off, 128);
  const size_t parity_off = off;   // [B] final parity of each matrix's last solve (k_finalize),
  off += 2 * sizeof(int) * (size_t)B;   // [B] the parity the ping-pong tables currently hold
  const LaunchDesc* clists[3] = {&P.gram[0], &P.square, &P.apply[0]};
  for (int l = 0; l < 3; ++l) {
    Plan::Compact& C = P.compact[l];
    if (!C.on) continue;
    off = align_up(off, 128);
    C.runs_off = off;
    off += sizeof(int) * C.runs.size();
    off = align_up(off, 128);
    C.dst_off = off;
    off += sizeof(uint32_t) * clists[l]->tiles.size();
    off = align_up(off, 128);
    C.count_off = off;
    off += sizeof(int);
  }
  std::vector<LaunchDesc*> all = {&P.gram[0],   &P.gram[1],   &P.apply[0],  &P.apply[1],  &P.square,
                                  &P.chaint[0], &P.chaint[1], &P.chaint[2], &P.chaint[3], &P.chaint[4],
                                  &P.square2, &P.rb1[0], &P.rb1[1], &P.gram0, &P.apply0,
                                  &P.apply0f};
  for (int t = 0; t < 2; ++t)
    for (LaunchDesc& L : P.rbgram[t]) all.push_back(&L);
  for (LaunchDesc& L : P.gjT) all.push_back(&L);
  for (LaunchDesc& L : P.gjS) all.push_back(&L);
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
  P.ws_need = P.meta_off;
  if (!r.ws) return PRISM_OK;

  if (cudaMalloc(&P.meta_dev, P.meta_bytes) != cudaSuccess) return fail(PRISM_ERR_CUDA, "cudaMalloc(plan constants)");
  char* meta_dev = P.meta_dev;
  uint8_t* blob = nullptr;
  if (cudaMallocHost(&blob, P.meta_bytes) != cudaSuccess) return fail(PRISM_ERR_CUDA, "cudaMallocHost(plan blob)");
  P.blob.reset(blob);
  std::memset(blob, 0, P.meta_bytes);
  std::memcpy(blob + mats_off, mats.data(), sizeof(MatDesc) * B);
  std::memcpy(blob + toff_off, toff.data(), sizeof(int) * (B + 1));
  std::memcpy(blob + ooff_off, ooff.data(), sizeof(int) * (B + 1));
  std::memcpy(blob + foff_off, foff.data(), sizeof(int) * (B + 1));
  for (int l = 0; l < 3; ++l)
    if (P.compact[l].on)
      std::memcpy(blob + P.compact[l].runs_off, P.compact[l].runs.data(), sizeof(int) * P.compact[l].runs.size());
  {
    int* par = reinterpret_cast<int*>(blob + parity_off);   // first solve: Q takes the odd iterates
    for (int i = 0; i < B; ++i) par[i] = 1, par[B + i] = 0;
  }
  {
    int* tm = reinterpret_cast<int*>(blob + tmat_off);
    for (int i = 0; i < B; ++i)
      for (int t = toff[i]; t < toff[i + 1]; ++t) tm[t] = i;
  }
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
      q.tmC = mapptr(L->probs[j].mapC);
      q.tmO = mapptr(L->probs[j].mapO);
      q.tmO2 = mapptr(L->probs[j].mapO2);
      gp[j] = q;
    }
    std::memcpy(blob + L->tiles_off, L->tiles.data(), sizeof(uint32_t) * L->tiles.size());
  }

  if (cudaMemcpy(P.meta_dev, blob, P.meta_bytes, cudaMemcpyHostToDevice) != cudaSuccess)
    return fail(PRISM_ERR_CUDA, "upload of plan constants");

  SolveParams& S = P.params;
  std::memset(&S, 0, sizeof(S));
  S.mats = reinterpret_cast<MatDesc*>(meta_dev + mats_off);
  S.tile_off = reinterpret_cast<const int*>(meta_dev + toff_off);
  S.tile_mat = reinterpret_cast<const int*>(meta_dev + tmat_off);
  S.out_tile_off = reinterpret_cast<const int*>(meta_dev + ooff_off);
  // folded polar: k_init_state swaps a matrix's entries of the ping-pong tables (entry b of
  // each is matrix b) when the parity it predicts for Q differs from the tables' current one
  S.parity = P.fold ? reinterpret_cast<int*>(meta_dev + parity_off) : nullptr;
  S.flip_cur = P.fold ? reinterpret_cast<int*>(meta_dev + parity_off) + B : nullptr;
  if (P.fold) {
    const LaunchDesc* tabs[6] = {&P.gram[0], &P.gram[1], &P.apply[0], &P.apply[1], &P.apply0, &P.apply0f};
    for (int j = 0; j < 6; ++j) {
      if ((int)tabs[j]->probs.size() != B) return fail(PRISM_ERR_INTERNAL, "parity tables: one entry per matrix");
      S.flip_tab[j] = reinterpret_cast<GemmProblem*>(meta_dev + tabs[j]->probs_off);
    }
  }
  S.ncompact = 0;
  for (int l = 0; l < 3; ++l) {
    const Plan::Compact& C = P.compact[l];
    if (!C.on) continue;
    CompactList& D = S.clist[S.ncompact++];
    D.runs = reinterpret_cast<const int*>(meta_dev + C.runs_off);
    D.nruns = (int)C.runs.size() / 3;
    D.src = reinterpret_cast<const uint32_t*>(meta_dev + clists[l]->tiles_off);
    D.dst = reinterpret_cast<uint32_t*>(meta_dev + C.dst_off);
    D.count = reinterpret_cast<int*>(meta_dev + C.count_off);
  }
  S.fro_off = reinterpret_cast<const int*>(meta_dev + foff_off);
  S.n_fro_blocks = foff[B];
  S.n_tiles = toff[B];
  S.n_out_tiles = ooff[B];
  S.st = d_st;
  S.iter = d_iter;
  S.alpha_hist = d_ahist;
  S.resid_hist = d_rhist;
  P.d_iter = d_iter;
  P.d_all_done = d_iter + 1;
  S.fro_part = d_fro;
  S.batch = B;
  S.p = p;
  S.d = d;
  S.max_iters = o.max_iters;
  S.warmup = o.warmup_iters;
  S.fit = o.fit;
  S.precision = prec;
  S.kind_sqrt = r.sqrt_kind ? 1 : 0;
  S.inv_q = iq;
  S.kind_cheb = cheb ? 1 : 0;
  S.kind_db = db ? 1 : 0;
  S.tol = o.tol;
  S.alo = lo;
  S.ahi = hi;
  S.ataylor = aT;
  S.seed = o.seed;
  return PRISM_OK;
}

// pass code of chain launch j (all problems of one chain launch share it)
int chain_pass(const Plan& P, int j) {
  return P.chaint[j].probs.empty() ? CH2_P1 : P.chaint[j].probs[0].p.pass;
}

static int g_debug_gemm_max_ctas = 0;   // prism_debug_gemm_max_ctas: persistent GEMM grids capped

GemmLaunch make_launch(const Plan& P, const LaunchDesc& L, const LaunchDesc* odd, char* ws, int lo, int hi,
                       const LaunchDesc* k0 = nullptr) {
  GemmLaunch g{};
  const bool chain = !L.probs.empty() && L.probs[0].p.mode == EPI_CHAIN;
  g.ksplit = chain ? P.chain_ksplit : 1;
  // chain problems are matrix-major, one per sketch chunk (build_plan)
  g.probs_per_matrix = chain ? (int)L.probs.size() / P.params.batch : 0;
  g.chain_bn = P.chain_bn;
  if (chain)
    for (int b = 0; b < kFirstCodes && b < (int)L.tiles.size(); ++b) g.first_code[b] = L.tiles[b];
  (void)ws;
  char* meta = P.meta_dev;
  g.probs = reinterpret_cast<const GemmProblem*>(meta + L.probs_off);
  g.probs_odd = odd ? reinterpret_cast<const GemmProblem*>(meta + odd->probs_off) : nullptr;
  g.probs_k0 = k0 ? reinterpret_cast<const GemmProblem*>(meta + k0->probs_off) : nullptr;
  g.tiles = reinterpret_cast<const uint32_t*>(meta + L.tiles_off);
  g.done = &P.params.st[0].done;
  g.done_stride = sizeof(MatState) / sizeof(int);
  g.ntiles = (int)L.tiles.size();
  g.iter = P.params.iter;
  g.iter_lo = lo;
  g.iter_hi = hi;
  if (!chain) g.max_ctas = g_debug_gemm_max_ctas;
  return g;
}

constexpr int kGJSmem = (kGJ * (kGJ + 1) + 2 * kGJ) * 4;   // Gauss-Jordan pivot / fix-up tiles

// Make every kernel's large-smem attribute current (on this device) before any graph capture.
void ensure_attrs() {
  static std::array<char, kMaxDevices> done{};
  const int dev = current_device();
  if (done[dev]) return;
  done[dev] = 1;
  cudaFuncSetAttribute(k_gj_pivot, cudaFuncAttributeMaxDynamicSharedMemorySize, kGJSmem);
  cudaFuncSetAttribute(k_gj_fix, cudaFuncAttributeMaxDynamicSharedMemorySize, kGJSmem);
  GemmLaunch z{};
  z.ntiles = 0;
  for (int prec = 0; prec < 3; ++prec) {
    for (int role = ROLE_GRAM; role <= ROLE_OTHER; ++role) launch_gemm(prec, role, z, 0);
    for (int pass = CH2_P1; pass < CH_NCODES; ++pass) launch_chain(prec, pass, z, 0);
  }
}

prism_status validate(const Request& r) {
  const prism_options& o = r.o;
  if (r.batch < 1) return fail(PRISM_ERR_INVALID_ARG, "batch must be >= 1");
  if (!r.m || !r.lda || !r.A || (!r.sqrt_kind && !r.db_kind && (!r.n || !r.Q || !r.ldq)))
    return fail(PRISM_ERR_INVALID_ARG, "null size/pointer array");
  if (o.degree != 3 && o.degree != 5) return fail(PRISM_ERR_INVALID_ARG, "degree must be 3 or 5");
  if (r.inv_q < 0 || r.inv_q > 4) return fail(PRISM_ERR_UNSUPPORTED, "inverse root order q must be 1..4");
  if (r.db_kind && o.precision != PRISM_FP32)
    return fail(PRISM_ERR_UNSUPPORTED, "DB Newton needs precision FP32 (its M^{-1} sweep is not run in bf16/tf32)");
  if (o.max_iters < 1 || o.max_iters > 10000) return fail(PRISM_ERR_INVALID_ARG, "max_iters out of range");
  if (!(o.tol > 0.0)) return fail(PRISM_ERR_INVALID_ARG, "tol must be > 0");
  if (o.precision < 0 || o.precision > 2) return fail(PRISM_ERR_INVALID_ARG, "bad precision");
  if (o.fit != PRISM_FIT_SKETCHED && o.fit != PRISM_FIT_TAYLOR)
    return fail(PRISM_ERR_UNSUPPORTED, "fit must be SKETCHED or TAYLOR on the device");
  if (o.sketch_size < 1) return fail(PRISM_ERR_INVALID_ARG, "sketch_size must be >= 1");
  if (o.sketch_size > kMaxSketch) return fail(PRISM_ERR_UNSUPPORTED, "sketch_size > 64 not supported");
  if (o.warmup_iters < 0) return fail(PRISM_ERR_INVALID_ARG, "warmup_iters must be >= 0");
  const int esz = elem_size(o.precision);
  for (int i = 0; i < r.batch; ++i) {
    const int64_t m = r.m[i], n = (r.sqrt_kind || r.db_kind) ? r.m[i] : r.n[i];
    if (m < 1 || n < 1 || m > (1 << 20) || n > (1 << 20)) return fail(PRISM_ERR_INVALID_ARG, "bad matrix size");
    if (!r.A[i]) return fail(PRISM_ERR_INVALID_ARG, "null input matrix");
    if (r.lda[i] < n) return fail(PRISM_ERR_INVALID_ARG, "lda < n");
    if (!r.sqrt_kind && !r.db_kind && !r.Q[i]) return fail(PRISM_ERR_INVALID_ARG, "null output matrix");
    if ((r.Q || r.Q2) && r.ldq[i] < n) return fail(PRISM_ERR_INVALID_ARG, "ldq < n");
    if ((r.rowblock ? n : std::min(m, n)) < o.sketch_size) return fail(PRISM_ERR_INVALID_ARG, "sketch_size > min(m, n)");
    if (reinterpret_cast<uintptr_t>(r.A[i]) % esz) return fail(PRISM_ERR_INVALID_ARG, "misaligned input");
  }
  return PRISM_OK;
}

}  // namespace

// ====================================================================== handle
constexpr int kKinds = 6;
struct prism_handle_s {
  std::list<std::unique_ptr<Plan>> plans;   // most recent first
  std::vector<std::pair<size_t, size_t>> last_guards;   // guard bands of the last plan (diagnostics)
  char* last_ws = nullptr;
  std::map<std::vector<long long>, size_t> ws_cache;   // workspace size per argument key
  long long launches = 0;                   // launches of the last solve
  bool profiling = false;
  std::vector<cudaEvent_t> pool;            // reusable events
  size_t pool_used = 0;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> marks;   // (kind, (start, stop))
  std::vector<long long> mark_launches;
  double acc_ms[kKinds] = {0};
  long long acc_launches[kKinds] = {0};
  cudaStream_t cap = nullptr;               // private stream for graph capture
  // launch ledger since the last prism_launch_count: per solve (device iteration counter of its
  // plan, launches outside the loop, launches per iteration); direct-launch loops record their
  // host-counted total with a null counter
  struct LedgerEntry {
    const int* iter;
    long long fixed, per_iter;
  };
  std::vector<LedgerEntry> ledger;
  int* h_flag = nullptr;                    // pinned host flag (profiling path)
  // host-buffer path (prism_polar_host / prism_sqrt_invsqrt_host): device staging
  // slots, upload / solve / download on three internal streams, ordered by events, so
  // call k+1's upload and call k's download overlap the solves
  struct HostSlot {
    char* in = nullptr;
    char* out = nullptr;
    char* out2 = nullptr;
    size_t in_bytes = 0, out_bytes = 0;
    cudaEvent_t ev_h2d = nullptr, ev_comp = nullptr, ev_d2h = nullptr;
    bool used = false;
  };
  static constexpr int kMaxSlots = 4;
  HostSlot slots[kMaxSlots];
  int slot_next = 0;
  cudaStream_t s_in = nullptr, s_comp = nullptr, s_out = nullptr;
  // multi-GPU: per-device auxiliary (communication) stream and reusable ordering events
  std::map<int, cudaStream_t> aux;
  std::map<int, std::array<cudaEvent_t, 16>> aux_ev;
  char* hws = nullptr;   // workspace of the host-path solves (they run in order on s_comp)
  size_t hws_bytes = 0;
  ~prism_handle_s() {
    plans.clear();
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
    if (cap) cudaStreamDestroy(cap);
    if (h_flag) cudaFreeHost(h_flag);
    if (s_in || s_comp || s_out) cudaDeviceSynchronize();
    for (HostSlot& sl : slots) {
      if (sl.in) cudaFree(sl.in);
      if (sl.out) cudaFree(sl.out);
      if (sl.out2) cudaFree(sl.out2);
      for (cudaEvent_t e : {sl.ev_h2d, sl.ev_comp, sl.ev_d2h})
        if (e) cudaEventDestroy(e);
    }
    if (hws) cudaFree(hws);
    for (auto& kv : aux) cudaStreamDestroy(kv.second);
    for (auto& kv : aux_ev)
      for (cudaEvent_t e : kv.second)
        if (e) cudaEventDestroy(e);
    for (cudaStream_t x : {s_in, s_comp, s_out})
      if (x) cudaStreamDestroy(x);
  }
  cudaEvent_t next_event() {
    if (pool_used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[pool_used++];
  }
};

// Scoped timing of one launch group (no-op unless profiling is enabled).
struct KindTimer {
  prism_handle_s* h;
  cudaStream_t st;
  int kind;
  long long nl;
  cudaEvent_t a = nullptr;
  KindTimer(prism_handle_s* h_, cudaStream_t st_, int kind_, long long nl_) : h(h_), st(st_), kind(kind_), nl(nl_) {
    h->launches += nl;
    if (h->profiling) {
      a = h->next_event();
      cudaEventRecord(a, st);
    }
  }
  ~KindTimer() {
    if (h->profiling) {
      cudaEvent_t b = h->next_event();
      cudaEventRecord(b, st);
      h->marks.push_back({kind, {a, b}});
      h->mark_launches.push_back(nl);
    }
  }
};

namespace prism {
prism_status fail_ext(prism_status s, const std::string& msg) { return fail(s, msg); }
cudaStream_t handle_aux_stream(prism_handle h) {
  const int d = current_device();
  auto it = h->aux.find(d);
  if (it != h->aux.end()) return it->second;
  cudaStream_t s = nullptr;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
  h->aux[d] = s;
  return s;
}
cudaEvent_t handle_event(prism_handle h, int idx) {
  auto& a = h->aux_ev[current_device()];
  cudaEvent_t& e = a[idx & 15];
  if (!e) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  return e;
}
}  // namespace prism

static std::vector<long long> make_key(const Request& r) {
  std::vector<long long> k;
  k.push_back(current_device());   // plans hold device allocations and per-device graphs
  k.push_back(g_guard_ws.load());  // guarded workspaces lay the buffers out differently
  k.push_back(r.sqrt_kind);
  k.push_back(r.sign_kind);
  k.push_back(r.inv_q);
  k.push_back(r.cheb_kind);
  k.push_back(r.db_kind);
  k.push_back(r.rowblock);
  k.push_back(r.rb_groups);
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
    k.push_back((r.sqrt_kind || r.db_kind) ? r.m[i] : r.n[i]);
    k.push_back(r.lda[i]);
    k.push_back(r.ldq ? r.ldq[i] : 0);
    k.push_back((long long)(uintptr_t)r.A[i]);
    k.push_back(r.Q ? (long long)(uintptr_t)r.Q[i] : 0);
    k.push_back(r.Q2 ? (long long)(uintptr_t)r.Q2[i] : 0);
    k.push_back(r.ids ? r.ids[i] : i);
  }
  return k;
}

// Workspace size of a request (size-only plan), cached per argument key on the handle:
// the bindings query it before every call.
static size_t ws_query(prism_handle h, const Request& r) {
  if (validate(r)) return 0;
  std::vector<long long> key = make_key(r);
  auto it = h->ws_cache.find(key);
  if (it != h->ws_cache.end()) return it->second;
  Plan P;
  if (build_plan(r, P)) return 0;
  if (h->ws_cache.size() > 1024) h->ws_cache.clear();
  h->ws_cache[key] = P.ws_need;
  return P.ws_need;
}

// Plan lookup (LRU keyed by every argument that shapes the tables) or build.
static prism_status get_plan(prism_handle h, const Request& r, size_t ws_bytes, Plan** out) {
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
  h->last_guards = P->guards;   // diagnostics: the guard bands of the last plan used
  h->last_ws = static_cast<char*>(r.ws);
  *out = P;
  return PRISM_OK;
}

static prism_status run_solve(prism_handle h, const Request& r0, const prism_report* rep, size_t ws_bytes,
                              cudaStream_t st) {
  NvtxRange nv_call(r0.rowblock ? "prism:rowblock" : r0.sqrt_kind ? "prism:sqrt_invsqrt" : r0.sign_kind ? "prism:sign"
                     : r0.inv_q ? "prism:inv_root" : r0.cheb_kind ? "prism:chebyshev_inverse"
                     : r0.db_kind ? "prism:db_newton" : "prism:polar");
  Request r = r0;
  Plan* P = nullptr;
  prism_status gs;
  {
    NvtxRange nv("prism:plan");
    gs = get_plan(h, r, ws_bytes, &P);
  }
  if (gs) return gs;

  SolveParams S = P->params;   // report pointers are only read by k_report (outside the graph)
  S.rep_iters = rep ? rep->iters : nullptr;
  S.rep_resid = rep ? rep->resid : nullptr;
  S.rep_status = rep ? rep->status : nullptr;
  S.rep_alphas = rep ? rep->alphas : nullptr;
  S.rep_resid_hist = rep ? rep->resid_hist : nullptr;
  const int B = r.batch;
  const int prec = r.o.precision;

  h->launches = 0;
  {
    KindTimer t(h, st, 5, P->unfolded ? 4 : 3);
    PRISM_CK(launch_k(k_fro_partials, dim3(S.n_fro_blocks), dim3(256), 0, st, 1, S));
    PRISM_CK(launch_k(k_fro_final, dim3(B), dim3(256), 0, st, 1, S));
    PRISM_CK(launch_k(k_init_state, dim3(B), dim3(256), 0, st, 1, S));
    if (!P->unfolded) {
    } else if (prec == PRISM_BF16) PRISM_CK(launch_k(k_normalize<0>, dim3(S.n_tiles), dim3(256), 0, st, 1, S));
    else if (prec == PRISM_FP32) PRISM_CK(launch_k(k_normalize<1>, dim3(S.n_tiles), dim3(256), 0, st, 1, S));
    else PRISM_CK(launch_k(k_normalize<2>, dim3(S.n_tiles), dim3(256), 0, st, 1, S));
  }
  PRISM_CK(cudaGetLastError());
  const int M = r.o.max_iters;
  GemmLaunch g_gram = make_launch(*P, P->gram[0], &P->gram[1], r.ws, 0, M + 1, P->fold ? &P->gram0 : nullptr);
  GemmLaunch g_apply = make_launch(*P, P->apply[0], &P->apply[1], r.ws, 0, M, P->fold ? &P->apply0 : nullptr);
  GemmLaunch g_sq = make_launch(*P, P->square, nullptr, r.ws, 0, M);
  // the square GEMM reads R (written by the residual step, several launches back): its
  // mainloop can run while k_alpha finishes, only its epilogue waiting for alpha.
  // Used where it was measured to pay (scripts/ab_early.sh, alternating runs on one box):
  // bf16 polar with few matrices — k_alpha then holds few SMs and the square GEMM fills
  // the rest (4096^2: 3.69 -> 3.54 ms per step).  Not for 3xTF32 (its epilogue consumes
  // the accumulator in K chunks during the mainloop, so a waiting epilogue stalls the
  // MMAs: shampoo 4 % slower), large batches (k_alpha holds B SMs: GPT-2 unchanged, 1B
  // batch 1 % slower) or the general square products of sign / Chebyshev (1-2 % slower).
  const bool polar_kind = !r.sqrt_kind && !r.sign_kind && !r.cheb_kind && !r.inv_q && !r.db_kind;
  // k_alpha: one warp per matrix, kAlphaWarps per block (it holds ceil(B / 8) SMs)
  const dim3 alpha_grid((B + kAlphaWarps - 1) / kAlphaWarps + (S.ncompact ? kCompactBlocks : 0)),
      alpha_block(32 * std::min(B, kAlphaWarps));
  // (with k_alpha packed on ceil(B / 8) SMs and the square grid capped to leave them, the
  // GPT-2 batch measured the same step time: the early square stays at B <= 16)
  if (P->square_early) g_sq.early = 1;
  (void)polar_kind;
  // per-iteration compacted tile lists (written by k_alpha's compaction blocks)
  {
    GemmLaunch* gl[3] = {&g_gram, &g_sq, &g_apply};
    for (int l = 0; l < 3; ++l) {
      const Plan::Compact& C = P->compact[l];
      if (!C.on) continue;
      gl[l]->ctiles = reinterpret_cast<const uint32_t*>(P->meta_dev + C.dst_off);
      gl[l]->ccount = reinterpret_cast<const int*>(P->meta_dev + C.count_off);
      gl[l]->c_from = C.c_from;
    }
  }
  const GemmLaunch g_sq2 = make_launch(*P, P->square2, nullptr, r.ws, 0, M);
  std::vector<GemmLaunch> g_gjT, g_gjS;
  for (int j = 0; j < P->db_steps; ++j) {
    g_gjT.push_back(make_launch(*P, P->gjT[j], nullptr, r.ws, 0, M));
    g_gjS.push_back(make_launch(*P, P->gjS[j], nullptr, r.ws, 0, M));
  }
  int rtm = 1, rtn = 1;   // inverse Newton / DB Newton: tile grid of the elementwise kernels (largest matrix)
  if (P->inv_q || P->db) {
    rtm = (P->max_s + 127) / 128;
    rtn = (P->max_s + tile_bn(prec) - 1) / tile_bn(prec);
  }
  GemmLaunch g_chaint[5];
  for (int j = 0; j < P->n_chain; ++j) g_chaint[j] = make_launch(*P, P->chaint[j], nullptr, r.ws, r.o.warmup_iters, M);
  const int n_chain_launches = P->n_chain;
  const bool sketched = r.o.fit == PRISM_FIT_SKETCHED;
  const int p = S.p;
  // one iteration k (k read on the device): R_k, stop test, S_k, chain, alpha_k, P, X_{k+1}
  auto body = [&](cudaStream_t s2, cudaGraphConditionalHandle ch, int use_handle, bool timed) -> prism_status {
    if (P->db) {
      // DB Newton: W = M_k, sweep W -> -M_k^{-1}, fit a, X/Y GEMMs, M update
      const dim3 eg(rtn, rtm, B);
      const int bn = tile_bn(prec);
      {
        KindTimer t(h, s2, 0, timed ? 1 : 0);
        PRISM_CK(launch_k(k_db_begin, eg, dim3(256), 0, s2, 1, S, bn));
      }
      {
        KindTimer t(h, s2, 1, timed ? 4 * P->db_steps : 0);
        const int strips = (P->max_s + kGJ - 1) / kGJ;
        for (int j = 0; j < P->db_steps; ++j) {
          PRISM_CK(launch_k(k_gj_pivot, dim3(1 + kGJCopy, B), dim3(kGJ), kGJSmem, s2, 1, S, j));
          PRISM_CK(launch_gemm(prec, ROLE_OTHER, g_gjT[j], s2));
          PRISM_CK(launch_gemm(prec, ROLE_OTHER, g_gjS[j], s2));
          PRISM_CK(launch_k(k_gj_fix, dim3(strips, B), dim3(256), kGJSmem, s2, 1, S, j));
        }
      }
      {
        KindTimer t(h, s2, 3, timed ? 1 : 0);
        PRISM_CK(launch_k(k_db_reduce, eg, dim3(256), 0, s2, 1, S, bn));
      }
      {
        KindTimer t(h, s2, 4, timed ? 1 : 0);
        PRISM_CK(launch_k(k_alpha<3>, alpha_grid, alpha_block, 0, s2, 1, S, 1));
      }
      {
        KindTimer t(h, s2, 2, timed ? 2 : 0);
        PRISM_CK(launch_gemm(prec, ROLE_APPLY, g_apply, s2));
        PRISM_CK(launch_k(k_db_update, eg, dim3(256), 0, s2, 1, S, bn));
      }
      PRISM_CK(launch_k(k_advance, dim3(1), dim3(256), 0, s2, 1, S, ch, use_handle, P->d_all_done));
      PRISM_CK(cudaGetLastError());
      return PRISM_OK;
    }
    {
      KindTimer t(h, s2, 0, timed ? 1 : 0);
      if (P->inv_q) {
        const dim3 grid(rtn, rtm, B);
        if (prec == PRISM_BF16) PRISM_CK(launch_k(k_resid_inv<0>, grid, dim3(256), 0, s2, 1, S, tile_bn(prec)));
        else if (prec == PRISM_FP32) PRISM_CK(launch_k(k_resid_inv<1>, grid, dim3(256), 0, s2, 1, S, tile_bn(prec)));
        else PRISM_CK(launch_k(k_resid_inv<2>, grid, dim3(256), 0, s2, 1, S, tile_bn(prec)));
      } else {
        PRISM_CK(launch_gemm(prec, ROLE_GRAM, g_gram, s2));
      }
    }
    {
      // residual-stage stop test (block 0 per matrix) + S_k: every later launch of the
      // iteration skips the matrices that stop here
      KindTimer t(h, s2, 3, timed ? 1 + (sketched ? n_chain_launches : 0) : 0);
      const int nsk = sketched ? (p * P->max_s / 2 + 255) / 256 : 0;
      PRISM_CK(launch_k(k_stop_sketch, dim3(1 + nsk, B), dim3(256), 0, s2, 1, S));
      if (sketched)
        for (int j = 0; j < P->n_chain; ++j) PRISM_CK(launch_chain(prec, chain_pass(*P, j), g_chaint[j], s2));
    }
    {
      // norm partials from the residual step; a sketch chain in between makes them final
      // before k_alpha's wait
      KindTimer t(h, s2, 4, timed ? 1 : 0);
      if (P->inv_q) PRISM_CK(launch_k(k_alpha<2>, alpha_grid, alpha_block, 0, s2, 1, S, 0));
      else if (r.cheb_kind) PRISM_CK(launch_k(k_alpha<1>, alpha_grid, alpha_block, 0, s2, 1, S, 0));
      else PRISM_CK(launch_k(k_alpha<0>, alpha_grid, alpha_block, 0, s2, 1, S, 0));
    }
    if (P->has_square) {
      KindTimer t(h, s2, 1, timed ? (P->has_square2 ? 2 : 1) : 0);
      PRISM_CK(launch_gemm(prec, ROLE_SQUARE, g_sq, s2));
      if (P->has_square2) PRISM_CK(launch_gemm(prec, ROLE_SQUARE, g_sq2, s2));
    }
    {
      KindTimer t(h, s2, 2, timed ? 1 : 0);
      PRISM_CK(launch_gemm(prec, ROLE_APPLY, g_apply, s2));
    }
    PRISM_CK(launch_k(k_advance, dim3(1), dim3(256), 0, s2, 1, S, ch, use_handle, P->d_all_done));
    PRISM_CK(cudaGetLastError());
    return PRISM_OK;
  };
  P->per_iter_launches = P->db ? 6 + 4 * P->db_steps
                                : 3 + 1 + (sketched ? n_chain_launches : 0) + (P->has_square ? 1 : 0) +
                                      (P->has_square2 ? 1 : 0) + 1;
  ensure_attrs();   // large-smem attributes: before the graph capture and the direct launches
  if (!h->profiling) {
    if (!P->exec) {
      // build the device-driven loop once per plan: WHILE(any active) { body }
      if (!h->cap) PRISM_CK(cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking));
      cudaGraph_t g;
      PRISM_CK(cudaGraphCreate(&g, 0));
      cudaGraphConditionalHandle ch;
      PRISM_CK(cudaGraphConditionalHandleCreate(&ch, g, 1, cudaGraphCondAssignDefault));
      alignas(cudaGraphNodeParams) unsigned char cp_buf[sizeof(cudaGraphNodeParams)] = {};
      cudaGraphNodeParams& cp = *reinterpret_cast<cudaGraphNodeParams*>(cp_buf);
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = ch;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t cn;
      PRISM_CK(cudaGraphAddNode(&cn, g, nullptr, 0, &cp));
      cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
      PRISM_CK(cudaStreamBeginCaptureToGraph(h->cap, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
      const long long saved = h->launches;
      prism_status bs = body(h->cap, ch, 1, false);
      h->launches = saved;
      cudaGraph_t got;
      cudaError_t ec = cudaStreamEndCapture(h->cap, &got);
      if (bs) { cudaGraphDestroy(g); return bs; }
      if (ec != cudaSuccess) { cudaGraphDestroy(g); return fail(PRISM_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ec)); }
      cudaError_t ei = cudaGraphInstantiate(&P->exec, g, 0);
      cudaGraphDestroy(g);
      if (ei != cudaSuccess) { P->exec = nullptr; return fail(PRISM_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ei)); }
    }
    NvtxRange nv("prism:iterate (CUDA-graph WHILE loop)");
    PRISM_CK(cudaGraphLaunch(P->exec, st));
  } else {
    // profiling: direct launches bracketed by events, host-side exit once all matrices stopped
    if (!h->h_flag) PRISM_CK(cudaMallocHost(&h->h_flag, sizeof(int)));
    for (int k = 0; k <= M; ++k) {
      NvtxRange nv("prism:iteration (direct launches)");
      prism_status bs = body(st, 0, 0, true);
      if (bs) return bs;
      PRISM_CK(cudaMemcpyAsync(h->h_flag, P->d_all_done, sizeof(int), cudaMemcpyDeviceToHost, st));
      PRISM_CK(cudaStreamSynchronize(st));
      if (*h->h_flag) break;
    }
  }
  {
    KindTimer t(h, st, 5, 1);
    if (prec == PRISM_BF16) PRISM_CK(launch_k(k_finalize<0>, dim3(S.n_out_tiles), dim3(256), 0, st, 1, S));
    else if (prec == PRISM_FP32) PRISM_CK(launch_k(k_finalize<1>, dim3(S.n_out_tiles), dim3(256), 0, st, 1, S));
    else PRISM_CK(launch_k(k_finalize<2>, dim3(S.n_out_tiles), dim3(256), 0, st, 1, S));
  }
  if (rep) PRISM_CK(launch_k(k_report, dim3(std::max(1, std::min(64, (B * (M + 1) + 255) / 256))), dim3(256), 0, st, 1, S));
  if (h->ledger.size() < (1u << 16))
    h->ledger.push_back({P->d_iter, 4 + (P->unfolded ? 1 : 0) + (rep ? 1 : 0), P->per_iter_launches});
  PRISM_CK(cudaGetLastError());
  return PRISM_OK;
}

// ====================================================================== debug kernels
namespace prism {
__global__ void k_sketch_debug(unsigned long long seed, int b, int k, int p, int s, float* S) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)p * s;
  if (2 * e >= total) return;
  double z0, z1;
  sketch_pair(seed, (uint32_t)k, (uint32_t)b, (uint32_t)e, &z0, &z1);
  S[2 * e] = __double2float_rn(z0);
  if (2 * e + 1 < total) S[2 * e + 1] = __double2float_rn(z1);
}
__global__ void k_argmin_debug(int n, const double* c, double lo, double hi, double aT, double* out) {
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);   // one warp per quartic
  if (i >= n) return;
  const double a = argmin_quartic(c + 5 * i, lo, hi, aT);
  if ((threadIdx.x & 31) == 0) out[i] = a;
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
  return ws_query(h, r);
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

// Host <-> device copy of an m x w block (element size esz): one linear copy when both
// sides are compact (cudaMemcpy2DAsync would move it row by row), else a 2-D copy.
static cudaError_t copy_block(void* dst, size_t dld, const void* src, size_t sld, size_t w, size_t m, size_t esz,
                              cudaMemcpyKind kind, cudaStream_t st) {
  if (dld == w && sld == w) return cudaMemcpyAsync(dst, src, m * w * esz, kind, st);
  return cudaMemcpy2DAsync(dst, dld * esz, src, sld * esz, w * esz, m, kind, st);
}

// End-to-end path on host buffers (see prism.h): stage, solve, return, pipelined.
// kind: 0 polar, 1 sqrt / inverse sqrt, 2 sign, 3 inverse q-th root, 4 Chebyshev inverse,
// 5 DB Newton sqrt / inverse sqrt (square inputs for 1-5)
static prism_status host_solve(prism_handle h, int kind, int inv_q, int batch, const int64_t* m, const int64_t* n,
                               const void* const* A_host, const int64_t* lda, void* const* O1, void* const* O2,
                               const int64_t* ldo, const int64_t* ids, const prism_options* o,
                               const prism_report* rep, cudaStream_t caller) {
  if (!h || !o) return fail(PRISM_ERR_INVALID_ARG, "null handle / options");
  NvtxRange nv_call("prism:host path (upload / solve / download)");
  const bool sqrt_kind = kind == 1 || kind == 5, square = kind != 0;
  if (batch < 1 || !m || !A_host || !lda || !ldo || (kind == 0 && !n) || (!sqrt_kind && !O1))
    return fail(PRISM_ERR_INVALID_ARG, "bad host-path arguments");
  const size_t esz = (size_t)elem_size(o->precision);
  // compact device staging (ld = n)
  std::vector<size_t> off(batch + 1, 0);
  for (int i = 0; i < batch; ++i) {
    const int64_t mm = m[i], nn = square ? m[i] : n[i];
    if (mm < 1 || nn < 1 || lda[i] < nn || ldo[i] < nn) return fail(PRISM_ERR_INVALID_ARG, "bad host-path shape");
    off[i + 1] = off[i] + align_up((size_t)(mm * nn) * esz, 256);
  }
  const size_t bytes = off[batch];
  if (!h->s_in) {
    for (cudaStream_t* x : {&h->s_in, &h->s_comp, &h->s_out})
      PRISM_CK(cudaStreamCreateWithFlags(x, cudaStreamNonBlocking));
    for (auto& sl : h->slots)
      for (cudaEvent_t* e : {&sl.ev_h2d, &sl.ev_comp, &sl.ev_d2h})
        PRISM_CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  std::vector<int64_t> ldc(batch);
  std::vector<const void*> din(batch);
  std::vector<void*> dout(batch), dout2(batch);
  constexpr int nslots = 3;   // upload / solve / download of three consecutive calls in flight
  auto& sl = h->slots[h->slot_next];
  h->slot_next = (h->slot_next + 1) % nslots;
  const bool two = sqrt_kind && O2;   // second output (A^{-1/2}) requested, with or without the first
  const size_t ws_need = kind == 5 ? prism_db_newton_workspace(h, batch, m, o)
                         : sqrt_kind ? prism_sqrt_workspace(h, batch, m, o)
                         : kind == 2 ? prism_sign_workspace(h, batch, m, o)
                         : kind == 3 ? prism_inv_root_workspace(h, batch, m, inv_q, o)
                         : kind == 4 ? prism_chebyshev_inverse_workspace(h, batch, m, o)
                                     : prism_polar_workspace(h, batch, m, n, o);
  if (!ws_need) return fail(PRISM_ERR_INVALID_ARG, "workspace query failed");
  if (sl.in_bytes < bytes || sl.out_bytes < bytes || (two && !sl.out2) || h->hws_bytes < ws_need) {
    PRISM_CK(cudaDeviceSynchronize());   // growing: nothing of the old buffers may be in flight
    if (sl.in_bytes < bytes || sl.out_bytes < bytes) {
      if (sl.in) cudaFree(sl.in);
      if (sl.out) cudaFree(sl.out);
      if (sl.out2) cudaFree(sl.out2);
      sl.in = sl.out = sl.out2 = nullptr;
      PRISM_CK(cudaMalloc(&sl.in, bytes));
      PRISM_CK(cudaMalloc(&sl.out, bytes));
      sl.in_bytes = sl.out_bytes = bytes;
    }
    if (two && !sl.out2) PRISM_CK(cudaMalloc(&sl.out2, sl.out_bytes));
    if (h->hws_bytes < ws_need) {
      if (h->hws) cudaFree(h->hws);
      h->hws = nullptr;
      PRISM_CK(cudaMalloc(&h->hws, ws_need));
      h->hws_bytes = ws_need;
    }
  }
  for (int i = 0; i < batch; ++i) {
    ldc[i] = square ? m[i] : n[i];
    din[i] = sl.in + off[i];
    dout[i] = sl.out + off[i];
    dout2[i] = sl.out2 ? sl.out2 + off[i] : nullptr;
  }
  // upload: as soon as this slot's previous solve has consumed its inputs.  Not ordered
  // after work queued earlier on the caller's stream: that stream waits for every previous
  // call's download, so such an order would serialise call k+1's upload behind call k's
  // download (measured: GPT-2 batch 11.7 k -> 5.3 k solves/s end to end).  The inputs must
  // hold their values when the call is made (include/prism.h).
  if (sl.used) PRISM_CK(cudaStreamWaitEvent(h->s_in, sl.ev_comp, 0));
  for (int i = 0; i < batch; ++i)
    PRISM_CK(copy_block(sl.in + off[i], ldc[i], A_host[i], lda[i], ldc[i], m[i], esz, cudaMemcpyHostToDevice,
                        h->s_in));
  PRISM_CK(cudaEventRecord(sl.ev_h2d, h->s_in));
  // solve (after the upload, and after this slot's previous download has read its outputs)
  PRISM_CK(cudaStreamWaitEvent(h->s_comp, sl.ev_h2d, 0));
  if (sl.used) PRISM_CK(cudaStreamWaitEvent(h->s_comp, sl.ev_d2h, 0));
  prism_status st;
  if (kind == 5)
    st = prism_db_newton(h, batch, m, din.data(), ldc.data(), O1 ? dout.data() : nullptr, O2 ? dout2.data() : nullptr,
                         ldc.data(), ids, o, rep, h->hws, h->hws_bytes, h->s_comp);
  else if (sqrt_kind)
    st = prism_sqrt_invsqrt(h, batch, m, din.data(), ldc.data(), O1 ? dout.data() : nullptr,
                            O2 ? dout2.data() : nullptr, ldc.data(), ids, o, rep, h->hws, h->hws_bytes, h->s_comp);
  else if (kind == 4)
    st = prism_chebyshev_inverse(h, batch, m, din.data(), ldc.data(), dout.data(), ldc.data(), ids, o, rep, h->hws,
                                 h->hws_bytes, h->s_comp);
  else if (kind == 3)
    st = prism_inv_root(h, batch, m, inv_q, din.data(), ldc.data(), dout.data(), ldc.data(), ids, o, rep, h->hws,
                        h->hws_bytes, h->s_comp);
  else if (kind == 2)
    st = prism_sign(h, batch, m, din.data(), ldc.data(), dout.data(), ldc.data(), ids, o, rep, h->hws, h->hws_bytes,
                    h->s_comp);
  else
    st = prism_polar(h, batch, m, n, din.data(), ldc.data(), dout.data(), ldc.data(), ids, o, rep, h->hws,
                     h->hws_bytes, h->s_comp);
  if (st) return st;
  PRISM_CK(cudaEventRecord(sl.ev_comp, h->s_comp));
  // download
  PRISM_CK(cudaStreamWaitEvent(h->s_out, sl.ev_comp, 0));
  for (int i = 0; i < batch; ++i) {
    if (O1 && O1[i])
      PRISM_CK(copy_block(O1[i], ldo[i], sl.out + off[i], ldc[i], ldc[i], m[i], esz, cudaMemcpyDeviceToHost,
                          h->s_out));
    if (two && O2[i])
      PRISM_CK(copy_block(O2[i], ldo[i], sl.out2 + off[i], ldc[i], ldc[i], m[i], esz, cudaMemcpyDeviceToHost,
                          h->s_out));
  }
  PRISM_CK(cudaEventRecord(sl.ev_d2h, h->s_out));
  PRISM_CK(cudaStreamWaitEvent(caller, sl.ev_d2h, 0));
  sl.used = true;
  return PRISM_OK;
}

prism_status prism_polar_host(prism_handle h, int batch, const int64_t* m, const int64_t* n, const void* const* A,
                              const int64_t* lda, void* const* Q, const int64_t* ldq, const int64_t* matrix_ids,
                              const prism_options* o, const prism_report* rep, void* stream) {
  try {
    return host_solve(h, 0, 0, batch, m, n, A, lda, Q, nullptr, ldq, matrix_ids, o, rep,
                      static_cast<cudaStream_t>(stream));
  } catch (...) {
    return fail(PRISM_ERR_INTERNAL, "exception in prism_polar_host");
  }
}

prism_status prism_sqrt_invsqrt_host(prism_handle h, int batch, const int64_t* n, const void* const* A,
                                     const int64_t* lda, void* const* Asqrt, void* const* Ainvsqrt,
                                     const int64_t* ld_out, const int64_t* matrix_ids, const prism_options* o,
                                     const prism_report* rep, void* stream) {
  try {
    return host_solve(h, 1, 0, batch, n, n, A, lda, Asqrt, Ainvsqrt, ld_out, matrix_ids, o, rep,
                      static_cast<cudaStream_t>(stream));
  } catch (...) {
    return fail(PRISM_ERR_INTERNAL, "exception in prism_sqrt_invsqrt_host");
  }
}

prism_status prism_sign_host(prism_handle h, int batch, const int64_t* n, const void* const* A, const int64_t* lda,
                             void* const* S, const int64_t* lds, const int64_t* matrix_ids, const prism_options* o,
                             const prism_report* rep, void* stream) {
  try {
    return host_solve(h, 2, 0, batch, n, n, A, lda, S, nullptr, lds, matrix_ids, o, rep,
                      static_cast<cudaStream_t>(stream));
  } catch (...) {
    return fail(PRISM_ERR_INTERNAL, "exception in prism_sign_host");
  }
}

size_t prism_inv_root_workspace(prism_handle h, int batch, const int64_t* n, int q, const prism_options* o) {
  if (!h || !o || !n || batch < 1) return 0;
  std::vector<const void*> fakeA(batch, reinterpret_cast<const void*>(256));
  std::vector<void*> fakeQ(batch, reinterpret_cast<void*>(256));
  std::vector<int64_t> ld(n, n + batch);
  Request r{false, batch, n, n, fakeA.data(), ld.data(), fakeQ.data(), nullptr, ld.data(), nullptr, *o, nullptr};
  r.inv_q = q;
  if (q < 1) return 0;
  return ws_query(h, r);
}

prism_status prism_inv_root(prism_handle h, int batch, const int64_t* n, int q, const void* const* A,
                            const int64_t* lda, void* const* X, const int64_t* ldx, const int64_t* matrix_ids,
                            const prism_options* o, const prism_report* rep, void* workspace, size_t ws_bytes,
                            void* stream) {
  try {
    if (!o) return fail(PRISM_ERR_INVALID_ARG, "null options");
    if (q < 1) return fail(PRISM_ERR_INVALID_ARG, "q must be >= 1");
    Request r{false, batch, n, n, A, lda, X, nullptr, ldx, matrix_ids, *o, static_cast<char*>(workspace)};
    r.inv_q = q;
    return run_solve(h, r, rep, ws_bytes, static_cast<cudaStream_t>(stream));
  } catch (...) {
    return fail(PRISM_ERR_INTERNAL, "exception in prism_inv_root");
  }
}

prism_status prism_inv_root_host(prism_handle h, int batch, const int64_t* n, int q, const void* const* A,
                                 const int64_t* lda, void* const* X, const int64_t* ldx, const int64_t* matrix_ids,
                                 const prism_options* o, const prism_report* rep, void* stream) {
  try {
    if (q < 1) return fail(PRISM_ERR_INVALID_ARG, "q must be >= 1");
    return host_solve(h, 3, q, batch, n, n, A, lda, X, nullptr, ldx, matrix_ids, o, rep,
                      static_cast<cudaStream_t>(stream));
  } catch (...) {
    return fail(PRISM_ERR_INTERNAL, "exception in prism_inv_root_host");
  }
}

size_t prism_chebyshev_inverse_workspace(prism_handle h, int batch, const int64_t* n, const prism_options* o) {
  if (!h || !o || !n || batch < 1) return 0;
  std::vector<const void*> fakeA(batch, reinterpret_cast<const void*>(256));
  std::vector<void*> fakeQ(batch, reinterpret_cast<void*>(256));
  std::vector<int64_t> ld(n, n + batch);
  Request r{false, batch, n, n, fakeA.data(), ld.data(), fakeQ.data(), nullptr, ld.data(), nullptr, *o, nullptr};
  r.cheb_kind = true;
  return ws_query(h, r);
}

prism_status prism_chebyshev_inverse(prism_handle h, int batch, const int64_t* n, const void* const* A,
                                     const int64_t* lda, void* const* X, const int64_t* ldx,
                                     const int64_t* matrix_ids, const prism_options* o, const prism_report* rep,
                                     void* workspace, size_t ws_bytes, void* stream) {
  try {
    if (!o) return fail(PRISM_ERR_INVALID_ARG, "null options");
    Request r{false, batch, n, n, A, lda, X, nullptr, ldx, matrix_ids, *o, static_cast<char*>(workspace)};
    r.cheb_kind = true;
    return run_solve(h, r, rep, ws_bytes, static_cast<cudaStream_t>(stream));
  } catch (...) {
    return fail(PRISM_ERR_INTERNAL, "exception in prism_chebyshev_inverse");
  }
}

prism_status prism_chebyshev_inverse_host(prism_handle h, int batch, const int64_t* n, const void* const* A,
                                          const int64_t* lda, void* const* X, const int64_t* ldx,
                                          const int64_t* matrix_ids, const prism_options* o,
                                          const prism_report* rep, void* stream) {
  try {
    return host_solve(h, 4, 0, batch, n, n, A, lda, X, nullptr, ldx, matrix_ids, o, rep,
                      static_cast<cudaStream_t>(stream));
  } catch (...) {
    return fail(PRISM_ERR_INTERNAL, "exception in prism_chebyshev_inverse_host");
  }
}

size_t prism_db_newton_workspace(prism_handle h, int batch, const int64_t* n, const prism_options* o) {
  if (!h || !o || !n || batch < 1) return 0;
  std::vector<const void*> fakeA(batch, reinterpret_cast<const void*>(256));
  std::vector<int64_t> ld(n, n + batch);
  Request r{false, batch, n, n, fakeA.data(), ld.data(), nullptr, nullptr, ld.data(), nullptr, *o, nullptr};
  r.db_kind = true;
  return ws_query(h, r);
}

prism_status prism_db_newton(prism_handle h, int batch, const int64_t* n, const void* const* A, const int64_t* lda,
                             void* const* Asqrt, void* const* Ainvsqrt, const int64_t* ld_out,
                             const int64_t* matrix_ids, const prism_options* o, const prism_report* rep,
                             void* workspace, size_t ws_bytes, void* stream) {
  try {
    if (!o) return fail(PRISM_ERR_INVALID_ARG, "null options");
    Request r{false, batch, n, n, A, lda, Asqrt, Ainvsqrt, ld_out, matrix_ids, *o, static_cast<char*>(workspace)};
    r.db_kind = true;
    return run_solve(h, r, rep, ws_bytes, static_cast<cudaStream_t>(stream));
  } catch (...) {
    return fail(PRISM_ERR_INTERNAL, "exception in prism_db_newton");
  }
}

prism_status prism_db_newton_host(prism_handle h, int batch, const int64_t* n, const void* const* A,
                                  const int64_t* lda, void* const* Asqrt, void* const* Ainvsqrt,
                                  const int64_t* ld_out, const int64_t* matrix_ids, const prism_options* o,
                                  const prism_report* rep, void* stream) {
  try {
    return host_solve(h, 5, 0, batch, n, n, A, lda, Asqrt, Ainvsqrt, ld_out, matrix_ids, o, rep,
                      static_cast<cudaStream_t>(stream));
  } catch (...) {
    return fail(PRISM_ERR_INTERNAL, "exception in prism_db_newton_host");
  }
}

size_t prism_sqrt_workspace(prism_handle h, int batch, const int64_t* n, const prism_options* o) {
  if (!h || !o || !n || batch < 1) return 0;
  std::vector<const void*> fakeA(batch, reinterpret_cast<const void*>(256));
  std::vector<int64_t> ld(n, n + batch);
  Request r{true, batch, n, n, fakeA.data(), ld.data(), nullptr, nullptr, ld.data(), nullptr, *o, nullptr};
  return ws_query(h, r);
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

size_t prism_sign_workspace(prism_handle h, int batch, const int64_t* n, const prism_options* o) {
  if (!h || !o || !n || batch < 1) return 0;
  std::vector<const void*> fakeA(batch, reinterpret_cast<const void*>(256));
  std::vector<void*> fakeQ(batch, reinterpret_cast<void*>(256));
  std::vector<int64_t> ld(n, n + batch);
  Request r{false, batch, n, n, fakeA.data(), ld.data(), fakeQ.data(), nullptr, ld.data(), nullptr, *o, nullptr};
  r.sign_kind = true;
  return ws_query(h, r);
}

prism_status prism_sign(prism_handle h, int batch, const int64_t* n, const void* const* A, const int64_t* lda,
                        void* const* S, const int64_t* lds, const int64_t* matrix_ids, const prism_options* o,
                        const prism_report* rep, void* workspace, size_t ws_bytes, void* stream) {
  try {
    if (!o) return fail(PRISM_ERR_INVALID_ARG, "null options");
    Request r{false, batch, n, n, A, lda, S, nullptr, lds, matrix_ids, *o, static_cast<char*>(workspace)};
    r.sign_kind = true;
    return run_solve(h, r, rep, ws_bytes, static_cast<cudaStream_t>(stream));
  } catch (...) {
    return fail(PRISM_ERR_INTERNAL, "exception in prism_sign");
  }
}

int64_t prism_launch_count(prism_handle h) {
  // per ledger entry: fixed launches + per-iteration launches x iterations executed (the
  // device counter of that plan's most recent solve: synchronises the device)
  if (!h) return -1;
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  std::map<const int*, int> iters;
  int64_t total = 0;
  for (const auto& e : h->ledger) {
    int k = 0;
    if (e.iter) {
      auto it = iters.find(e.iter);
      if (it == iters.end()) {
        if (cudaMemcpy(&k, e.iter, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
        iters[e.iter] = k;
      } else {
        k = it->second;
      }
    }
    total += e.fixed + e.per_iter * (int64_t)k;
  }
  h->ledger.clear();
  return total;
}

prism_status prism_profile_enable(prism_handle h, int enable) {
  if (!h) return fail(PRISM_ERR_INVALID_ARG, "null handle");
  h->profiling = enable != 0;
  return PRISM_OK;
}

prism_status prism_profile_read(prism_handle h, double* ms, int64_t* launches, int reset) {
  if (!h) return fail(PRISM_ERR_INVALID_ARG, "null handle");
  for (size_t j = 0; j < h->marks.size(); ++j) {
    const auto& m = h->marks[j];
    PRISM_CK(cudaEventSynchronize(m.second.second));
    float t = 0.f;
    PRISM_CK(cudaEventElapsedTime(&t, m.second.first, m.second.second));
    h->acc_ms[m.first] += t;
    h->acc_launches[m.first] += h->mark_launches[j];
  }
  h->marks.clear();
  h->mark_launches.clear();
  h->pool_used = 0;
  for (int k = 0; k < kKinds; ++k) {
    if (ms) ms[k] = h->acc_ms[k];
    if (launches) launches[k] = h->acc_launches[k];
    if (reset) { h->acc_ms[k] = 0; h->acc_launches[k] = 0; }
  }
  return PRISM_OK;
}

// ---------------------------------------------------------------- row-block split
static Request rowblock_request(int64_t* rows, int64_t* n, const void** A, int64_t* lda, void** Q, int64_t* ldq,
                                const prism_options* o, char* ws, int nranks) {
  Request r{false, 1, rows, n, A, lda, Q, nullptr, ldq, nullptr, *o, ws};
  r.rowblock = true;
  r.rb_groups = nranks > 1 ? 4 : 1;   // pipelined all-reduce of the packed Gram by panel group
  return r;
}

size_t prism_polar_rowblock_workspace(prism_handle h, int64_t rows, int64_t n, const prism_options* o) {
  if (!h || !o || rows < 1 || n < 1) return 0;
  const void* fakeA = reinterpret_cast<const void*>(256);
  void* fakeQ = reinterpret_cast<void*>(256);
  int64_t ld = n;
  // the 4-group layout needs the same bytes as the 1-group one (one packed buffer)
  Request r = rowblock_request(&rows, &n, &fakeA, &ld, &fakeQ, &ld, o, nullptr, 2);
  return ws_query(h, r);
}

prism_status prism_polar_rowblock_tr(prism_handle h, const prism_transport* tr, int64_t m_global, int64_t n,
                                     const void* A_rows, int64_t row0, int64_t rows, int64_t lda, void* Q_rows,
                                     int64_t ldq, const prism_options* o, const prism_report* rep, void* workspace,
                                     size_t ws_bytes, void* stream) {
  try {
    if (!h || !tr || !o || !tr->allreduce_sum) return fail(PRISM_ERR_INVALID_ARG, "null handle / transport / options");
    if (rows < 1 || n < 1 || row0 < 0 || row0 + rows > m_global)
      return fail(PRISM_ERR_INVALID_ARG, "row block outside the global matrix");
    const void* A = A_rows;
    void* Q = Q_rows;
    Request r = rowblock_request(&rows, &n, &A, &lda, &Q, &ldq, o, static_cast<char*>(workspace), tr->nranks);
    Plan* P = nullptr;
    prism_status gs = get_plan(h, r, ws_bytes, &P);
    if (gs) return gs;
    ensure_attrs();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaStream_t cs = prism::handle_aux_stream(h);
    if (!cs) return fail(PRISM_ERR_CUDA, "aux stream");
    if (!h->h_flag) PRISM_CK(cudaMallocHost(&h->h_flag, sizeof(int)));
    SolveParams S = P->params;
    S.rep_iters = rep ? rep->iters : nullptr;
    S.rep_resid = rep ? rep->resid : nullptr;
    S.rep_status = rep ? rep->status : nullptr;
    S.rep_alphas = rep ? rep->alphas : nullptr;
    S.rep_resid_hist = rep ? rep->resid_hist : nullptr;
    const int prec = o->precision, M = o->max_iters, ng = (int)P->group_end.size();
    const bool pipelined = tr->nranks > 1 && ng > 1;
    auto allreduce = [&](void* buf, size_t count, int dtype, cudaStream_t s2) -> prism_status {
      if (tr->allreduce_sum(tr->ctx, buf, buf, count, dtype, s2)) return fail(PRISM_ERR_NCCL, "all-reduce failed");
      return PRISM_OK;
    };
    // c = ||A||_F over all ranks: local sum of squares, all-reduced, then X_0 = A_r / c
    S.fro2_out = P->rb_fro2;
    PRISM_CK(cudaMemsetAsync(P->Gp, 0, sizeof(float) * (size_t)P->panel_off.back(), st));
    PRISM_CK(launch_k(k_fro_partials, dim3(S.n_fro_blocks), dim3(256), 0, st, 1, S));
    PRISM_CK(launch_k(k_fro_final, dim3(1), dim3(256), 0, st, 1, S));
    if (prism_status e = allreduce(P->rb_fro2, 1, PRISM_DT_F64, st)) return e;
    S.fro2_out = nullptr;
    S.fro2_in = P->rb_fro2;
    PRISM_CK(launch_k(k_set_c, dim3(1), dim3(32), 0, st, 1, S));
    PRISM_CK(launch_k(k_init_state, dim3(1), dim3(256), 0, st, 1, S));
    if (prec == PRISM_BF16) PRISM_CK(launch_k(k_normalize<0>, dim3(S.n_tiles), dim3(256), 0, st, 1, S));
    else if (prec == PRISM_FP32) PRISM_CK(launch_k(k_normalize<1>, dim3(S.n_tiles), dim3(256), 0, st, 1, S));
    else PRISM_CK(launch_k(k_normalize<2>, dim3(S.n_tiles), dim3(256), 0, st, 1, S));
    const bool sketched = o->fit == PRISM_FIT_SKETCHED;
    const int nt = (int)((n + 63) / 64);
    cudaEvent_t ev_stop = prism::handle_event(h, 8);
    long long nl = 5;   // launches of this call (the launch ledger, prism_launch_count)
    for (int k = 0; k <= M; ++k) {
      NvtxRange nv("prism:rowblock iteration");
      nl += ng + 5 + (sketched ? P->n_chain : 0) + (P->rb1[0].probs.size() ? 1 : 0);
      const int t = k & 1;
      // 1. packed partial Gram, all-reduced panel group by panel group (on the aux stream,
      //    overlapping the next group's launch; the Gram grid leaves SMs to the collective)
      for (int g = 0; g < ng; ++g) {
        GemmLaunch gl = make_launch(*P, P->rbgram[t][g], nullptr, r.ws, 0, M + 1);
        if (pipelined) gl.max_ctas = device_sms() - 16;
        PRISM_CK(launch_gemm(prec, ROLE_GRAM, gl, st));
        const size_t beg = (size_t)(g ? P->panel_off[P->group_end[g - 1]] : 0);
        const size_t end = (size_t)P->panel_off[P->group_end[g]];
        if (end == beg) continue;
        if (pipelined) {
          cudaEvent_t e = prism::handle_event(h, 9 + (g & 3));
          PRISM_CK(cudaEventRecord(e, st));
          PRISM_CK(cudaStreamWaitEvent(cs, e, 0));
          if (prism_status x = allreduce(P->Gp + beg, end - beg, PRISM_DT_F32, cs)) return x;
        } else {
          if (prism_status x = allreduce(P->Gp + beg, end - beg, PRISM_DT_F32, st)) return x;
        }
      }
      if (pipelined) {
        cudaEvent_t e = prism::handle_event(h, 13);
        PRISM_CK(cudaEventRecord(e, cs));
        PRISM_CK(cudaStreamWaitEvent(st, e, 0));
      }
      // 2. R = I - G, sketch, chain, stop test and alpha (identical on every rank)
      if (prec == PRISM_BF16) PRISM_CK(launch_k(k_resid_packed<0>, dim3(nt, nt), dim3(256), 0, st, 1, S, (const float*)P->Gp));
      else if (prec == PRISM_FP32) PRISM_CK(launch_k(k_resid_packed<1>, dim3(nt, nt), dim3(256), 0, st, 1, S, (const float*)P->Gp));
      else PRISM_CK(launch_k(k_resid_packed<2>, dim3(nt, nt), dim3(256), 0, st, 1, S, (const float*)P->Gp));
      PRISM_CK(launch_k(k_stop_sketch, dim3(1 + (sketched ? (S.p * P->max_s / 2 + 255) / 256 : 0), 1), dim3(256), 0,
                        st, 1, S));
      if (sketched) {
        for (int j = 0; j < P->n_chain; ++j)
          PRISM_CK(launch_chain(prec, chain_pass(*P, j), make_launch(*P, P->chaint[j], nullptr, r.ws, o->warmup_iters, M), st));
      }
      PRISM_CK(launch_k(k_alpha<0>, dim3(1), dim3(32), 0, st, 1, S, 0));   // one matrix: one warp
      PRISM_CK(cudaMemcpyAsync(h->h_flag, &P->params.st[0].done, sizeof(int), cudaMemcpyDeviceToHost, st));
      PRISM_CK(cudaEventRecord(ev_stop, st));
      // 3. this rank's rows: X_r g_d(R; alpha) without R^2 (skipped on the device once stopped)
      if (P->rb1[0].probs.size()) PRISM_CK(launch_gemm(prec, ROLE_APPLY, make_launch(*P, P->rb1[0], &P->rb1[1], r.ws, 0, M), st));
      PRISM_CK(launch_gemm(prec, ROLE_APPLY, make_launch(*P, P->apply[0], &P->apply[1], r.ws, 0, M), st));
      PRISM_CK(launch_k(k_advance, dim3(1), dim3(256), 0, st, 1, S, (cudaGraphConditionalHandle)0, 0, P->d_all_done));
      PRISM_CK(cudaGetLastError());
      if (tr->async_error && tr->async_error(tr->ctx)) return fail(PRISM_ERR_NCCL, "communicator error");
      // the device keeps the updates of iteration k while the host reads its stop flag
      PRISM_CK(cudaEventSynchronize(ev_stop));
      if (*h->h_flag) break;
    }
    if (prec == PRISM_BF16) PRISM_CK(launch_k(k_finalize<0>, dim3(S.n_out_tiles), dim3(256), 0, st, 1, S));
    else if (prec == PRISM_FP32) PRISM_CK(launch_k(k_finalize<1>, dim3(S.n_out_tiles), dim3(256), 0, st, 1, S));
    else PRISM_CK(launch_k(k_finalize<2>, dim3(S.n_out_tiles), dim3(256), 0, st, 1, S));
    if (rep) PRISM_CK(launch_k(k_report, dim3(1), dim3(256), 0, st, 1, S));
    PRISM_CK(cudaGetLastError());
    nl += 1 + (rep ? 1 : 0);
    if (h->ledger.size() < (1u << 16)) h->ledger.push_back({nullptr, nl, 0});
    return PRISM_OK;
  } catch (...) {
    return fail(PRISM_ERR_INTERNAL, "exception in prism_polar_rowblock");
  }
}

prism_status prism_polar_rowblock(prism_handle h, void* comm, int64_t m_global, int64_t n, const void* A_rows,
                                  int64_t row0, int64_t rows, int64_t lda, void* Q_rows, int64_t ldq,
                                  const prism_options* o, const prism_report* rep, void* workspace, size_t ws_bytes,
                                  void* stream) {
  prism_transport tr;
  prism_status s = prism_nccl_transport(comm, &tr);
  if (s) return s;
  return prism_polar_rowblock_tr(h, &tr, m_global, n, A_rows, row0, rows, lda, Q_rows, ldq, o, rep, workspace,
                                 ws_bytes, stream);
}

prism_status prism_rowblock_layout(int64_t n, int ngroups, int64_t* panel_off, int32_t* group_end) {
  if (n < 1 || ngroups < 1 || !panel_off || !group_end) return fail(PRISM_ERR_INVALID_ARG, "bad layout args");
  std::vector<long long> off;
  std::vector<int> ge;
  rowblock_layout(n, ngroups, off, ge);
  for (size_t t = 0; t < off.size(); ++t) panel_off[t] = off[t];
  for (int g = 0; g < ngroups; ++g) group_end[g] = g < (int)ge.size() ? ge[g] : ge.back();
  return PRISM_OK;
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

prism_status prism_debug_raster_rows(int rows) {
  g_raster_rows = rows < 1 ? 1u : (uint32_t)rows;
  return PRISM_OK;
}

prism_status prism_debug_gemm_max_ctas(int max_ctas) {
  g_debug_gemm_max_ctas = max_ctas < 0 ? 0 : max_ctas;
  return PRISM_OK;
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
  const size_t need = 4096 + 6 * sizeof(CUtensorMap) + sizeof(GemmProblem) + 4 * ((M + 127) / 128) * ((N + BN - 1) / BN);
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
  const OpKind bk = b_mn ? OP_MN : OP_BK;
  const int brows = b_mn ? K : N, bcols = b_mn ? N : K;
  if (!encode_map(&hm[0], MapSpec{A, M, K, lda, esz, OP_A, BN, BK}) ||
      !encode_map(&hm[1], MapSpec{B, brows, bcols, ldb, esz, bk, BN / 2, BK}))
    return fail(PRISM_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  if (split) {
    if (!encode_map(&hm[2], MapSpec{A_lo, M, K, lda, esz, OP_A, BN, BK}) ||
        !encode_map(&hm[3], MapSpec{B_lo, brows, bcols, ldb, esz, bk, BN / 2, BK}))
      return fail(PRISM_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  }
  // bf16 epilogue blocks: TMA store of the output, TMA load of C (maps 4 and 5)
  if (esz == 2) {
    if (!encode_map(&hm[4], MapSpec{out, M, N, ldo, esz, OP_EPI, 32, 32}) ||
        (C && !encode_map(&hm[5], MapSpec{C, M, N, ldc, esz, OP_EPI, 32, 32})))
      return fail(PRISM_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  }
  GemmProblem* gp = reinterpret_cast<GemmProblem*>(hb + 6 * sizeof(CUtensorMap));
  const CUtensorMap* dm = reinterpret_cast<const CUtensorMap*>(wsd);
  gp->tmA = dm; gp->tmB = dm + 1;
  gp->tmA_lo = split ? dm + 2 : nullptr; gp->tmB_lo = split ? dm + 3 : nullptr;
  gp->tmO = esz == 2 ? dm + 4 : nullptr; gp->tmC = (esz == 2 && C) ? dm + 5 : nullptr;
  gp->out = out; gp->out_lo = out_lo; gp->C = C; gp->C_lo = C_lo;
  gp->norm_part = norm_part; gp->gdiag = gdiag; gp->alpha = alpha_dev;
  gp->ldo = ldo; gp->ldc = ldc; gp->M = M; gp->N = N; gp->K = K;
  gp->mode = mode; gp->sym = sym; gp->matrix = 0; gp->scale_by_alpha = scale_by_alpha;
  gp->tiles_n = (N + BN - 1) / BN;
  gp->c1 = mode == EPI_POLY ? c1 : 1.f;
  gp->kA = 1.f;
  gp->eA = (mode == EPI_POLY || (mode == EPI_APPLY && scale_by_alpha)) ? 1 : 0;
  gp->eC = 0;
  gp->lA = gp->lC = 0.f;
  gp->a_mn = 0; gp->b_mn = b_mn ? 1 : 0;
  LaunchDesc L;
  HostProblem hp;
  hp.p = *gp;
  L.probs.push_back(hp);
  add_tiles(L, 0, M, N, BN, sym != 0);
  const size_t tiles_off = 6 * sizeof(CUtensorMap) + align_up(sizeof(GemmProblem), 128);
  std::memcpy(hb + tiles_off, L.tiles.data(), 4 * L.tiles.size());
  PRISM_CK(cudaMemcpyAsync(wsd, hb, need, cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)));
  GemmLaunch g{};
  g.probs = reinterpret_cast<const GemmProblem*>(wsd + 6 * sizeof(CUtensorMap));
  g.tiles = reinterpret_cast<const uint32_t*>(wsd + tiles_off);
  g.done = nullptr;
  g.done_stride = 0;
  g.ntiles = (int)L.tiles.size();
  g.max_ctas = g_debug_gemm_max_ctas;
  PRISM_CK(launch_gemm(precision, ROLE_OTHER, g, static_cast<cudaStream_t>(stream)));
  PRISM_CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  return PRISM_OK;
}


prism_status prism_debug_trace_gemm(unsigned long long* buf_dev, int mode) {
  const int m = mode < 0 ? -1 : (mode & 0xFF);
  if (set_gemm_trace_bf16(buf_dev, m) != cudaSuccess || set_gemm_trace_f32x3(buf_dev, m) != cudaSuccess ||
      set_gemm_trace_tf32(buf_dev, m) != cudaSuccess)
    return fail(PRISM_ERR_CUDA, "trace hook");
  return PRISM_OK;
}

prism_status prism_debug_workspace_guards(int enable) {
  g_guard_ws.store(enable ? 1 : 0);
  return PRISM_OK;
}

prism_status prism_debug_guards_fill(prism_handle h, void* stream) {
  if (!h || !h->last_ws) return fail(PRISM_ERR_INVALID_ARG, "no guarded solve on this handle");
  for (const auto& g : h->last_guards)
    PRISM_CK(cudaMemsetAsync(h->last_ws + g.first, 0xA5, g.second, static_cast<cudaStream_t>(stream)));
  return PRISM_OK;
}

prism_status prism_debug_guards_poke(prism_handle h, int64_t idx, void* stream) {
  if (!h || !h->last_ws || idx < 0 || idx >= (int64_t)h->last_guards.size())
    return fail(PRISM_ERR_INVALID_ARG, "no such guard band");
  PRISM_CK(cudaMemsetAsync(h->last_ws + h->last_guards[idx].first, 0, 1, static_cast<cudaStream_t>(stream)));
  return PRISM_OK;
}

prism_status prism_debug_guards_check(prism_handle h, int64_t* bad_bytes, int64_t* guards, void* stream) {
  if (!h || !bad_bytes || !guards) return fail(PRISM_ERR_INVALID_ARG, "null argument");
  std::vector<unsigned char> buf;
  int64_t bad = 0;
  PRISM_CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  for (const auto& g : h->last_guards) {
    buf.resize(g.second);
    PRISM_CK(cudaMemcpy(buf.data(), h->last_ws + g.first, g.second, cudaMemcpyDeviceToHost));
    for (unsigned char c : buf) bad += c != 0xA5;
  }
  *bad_bytes = bad;
  *guards = (int64_t)h->last_guards.size();
  return PRISM_OK;
}

prism_status prism_debug_trace_chain(unsigned long long* buf_dev) {
  if (set_chain_trace_bf16(buf_dev) != cudaSuccess || set_chain_trace_f32x3(buf_dev) != cudaSuccess ||
      set_chain_trace_tf32(buf_dev) != cudaSuccess)
    return fail(PRISM_ERR_CUDA, "trace hook");
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
  k_argmin_debug<<<(n + 3) / 4, 128, 0, static_cast<cudaStream_t>(stream)>>>(n, c_dev, lo, hi, a_taylor,
                                                                                 alpha_dev);
  PRISM_CK(cudaGetLastError());
  return PRISM_OK;
}

}  // extern "C"
