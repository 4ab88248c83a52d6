// Multi-GPU layer of libprism.so (include/prism.h "multi-GPU"):
//   * NCCL resolved at run time (dlopen of the libnccl.so.2 the process already loaded, so
//     the caller's and the library's communicators are the same NCCL) and the NCCL transport;
//   * the sharded batch: LPT plan, per-rank bucketed solves through prism_polar with global
//     sketch ids, owners' broadcasts of each bucket overlapping the next bucket's solve,
//     and the report all-reduce.
// The row-block split lives in prism.cu (it needs the solver's plan internals).
#include "../../include/prism.h"
#include "internal.h"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

namespace {

using prism::fail_ext;

// ------------------------------------------------------------------ NCCL at run time
struct NcclApi {
  bool ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclBroadcast) Broadcast = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclCommGetAsyncError) CommGetAsyncError = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  decltype(&ncclCommCount) CommCount = nullptr;
  decltype(&ncclCommUserRank) CommUserRank = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // an NCCL already in the process first (torch's bundled libnccl.so.2), else the system one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("libnccl.so.2 not found: ") + dlerror();
      return a;
    }
#define PRISM_SYM(f)                                                  \
  a.f = reinterpret_cast<decltype(a.f)>(dlsym(h, "nccl" #f));           \
  if (!a.f) {                                                           \
    a.why = "NCCL symbol nccl" #f " missing";                           \
    return a;                                                           \
  }
    PRISM_SYM(GetUniqueId)
    PRISM_SYM(CommInitRank)
    PRISM_SYM(CommDestroy)
    PRISM_SYM(AllReduce)
    PRISM_SYM(Broadcast)
    PRISM_SYM(GroupStart)
    PRISM_SYM(GroupEnd)
    PRISM_SYM(CommGetAsyncError)
    PRISM_SYM(GetErrorString)
    PRISM_SYM(CommCount)
    PRISM_SYM(CommUserRank)
#undef PRISM_SYM
    a.ok = true;
    return a;
  }();
  return api;
}

prism_status nccl_fail(const char* what, ncclResult_t r) {
  return fail_ext(PRISM_ERR_NCCL, std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?"));
}

ncclDataType_t nccl_type(int dtype) {
  return dtype == PRISM_DT_F32 ? ncclFloat32 : dtype == PRISM_DT_F64 ? ncclFloat64 : dtype == PRISM_DT_I32 ? ncclInt32
                                                                                                           : ncclUint8;
}

int tr_allreduce(void* ctx, const void* send, void* recv, size_t count, int dtype, void* stream) {
  return (int)nccl().AllReduce(send, recv, count, nccl_type(dtype), ncclSum, static_cast<ncclComm_t>(ctx),
                               static_cast<cudaStream_t>(stream));
}
int tr_broadcast(void* ctx, void* buf, size_t bytes, int root, void* stream) {
  return (int)nccl().Broadcast(buf, buf, bytes, ncclUint8, root, static_cast<ncclComm_t>(ctx),
                               static_cast<cudaStream_t>(stream));
}
int tr_group_start(void*) { return (int)nccl().GroupStart(); }
int tr_group_end(void*) { return (int)nccl().GroupEnd(); }
int tr_async_error(void* ctx) {
  ncclResult_t e = ncclSuccess;
  if (nccl().CommGetAsyncError(static_cast<ncclComm_t>(ctx), &e) != ncclSuccess) return 1;
  return (e == ncclSuccess || e == ncclInProgress) ? 0 : (int)e;
}

// ------------------------------------------------------------------ sharded batch
// Report entries of one bucket's local solve -> global (batch-indexed) arrays.
struct ScatterIdx {
  int n;
  int idx[1000];   // global matrix index of local entry b (kernel parameter: <= 4 KB)
};
constexpr int kMaxBucket = 1000;

__global__ void k_rep_scatter(ScatterIdx ix, int max_iters, const int32_t* li, const float* lr, const int32_t* ls,
                              const double* la, const float* lh, int32_t* gi, float* gr, int32_t* gs, double* ga,
                              float* gh) {
  const int nr = max_iters + 1;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ix.n * nr; t += gridDim.x * blockDim.x) {
    const int b = t / nr, k = t - b * nr, g = ix.idx[b];
    gh[(size_t)g * nr + k] = lh[(size_t)b * nr + k];
    if (k < max_iters) ga[(size_t)g * max_iters + k] = la[(size_t)b * max_iters + k];
    if (k == 0) {
      gi[g] = li[b];
      gr[g] = lr[b];
      gs[g] = ls[b];
    }
  }
}

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

struct ShardLayout {
  std::vector<int> owner, bucket;
  std::vector<std::vector<int>> mine;   // [bucket] -> global indices owned by this rank
  size_t local_rep = 0, global_rep = 0, solve_ws = 0, total = 0;
  int max_nb = 0;
};

// Report arrays of `cnt` matrices laid out from `base`: iters, status (i32), resid (f32),
// alphas (f64, cnt x M), hist (f32, cnt x (M + 1)).
struct RepView {
  int32_t* iters;
  int32_t* status;
  float* resid;
  double* alphas;
  float* hist;
};
size_t rep_bytes(int cnt, int M) {
  return align256(4ull * cnt) * 3 + align256(8ull * cnt * M) + align256(4ull * cnt * (M + 1));
}
RepView rep_view(char* base, int cnt, int M) {
  RepView v;
  v.iters = reinterpret_cast<int32_t*>(base);
  base += align256(4ull * cnt);
  v.status = reinterpret_cast<int32_t*>(base);
  base += align256(4ull * cnt);
  v.resid = reinterpret_cast<float*>(base);
  base += align256(4ull * cnt);
  v.alphas = reinterpret_cast<double*>(base);
  base += align256(8ull * cnt * M);
  v.hist = reinterpret_cast<float*>(base);
  return v;
}

// kind 0: polar (m x n), 1: coupled sqrt / inverse sqrt (n x n, m == n)
prism_status shard_layout(prism_handle h, int kind, int nranks, int rank, int batch, const int64_t* m, const int64_t* n,
                          const prism_options* o, int nbuckets, ShardLayout& L) {
  if (!o || !m || !n || batch < 1 || nranks < 1 || rank < 0 || rank >= nranks || nbuckets < 1)
    return fail_ext(PRISM_ERR_INVALID_ARG, "bad sharded-batch arguments");
  L.owner.assign(batch, 0);
  L.bucket.assign(batch, 0);
  prism_status s = prism_shard_plan(batch, m, n, o->degree, o->sketch_size, nranks, nbuckets, L.owner.data(),
                                    L.bucket.data());
  if (s) return s;
  L.mine.assign(nbuckets, {});
  for (int i = 0; i < batch; ++i)
    if (L.owner[i] == rank) L.mine[L.bucket[i]].push_back(i);
  L.max_nb = 0;
  L.solve_ws = 0;
  for (const auto& b : L.mine) {
    if (b.empty()) continue;
    if ((int)b.size() > kMaxBucket) return fail_ext(PRISM_ERR_UNSUPPORTED, "more than 1000 matrices in a bucket");
    L.max_nb = std::max(L.max_nb, (int)b.size());
    std::vector<int64_t> mm, nn;
    for (int i : b) {
      mm.push_back(m[i]);
      nn.push_back(n[i]);
    }
    const size_t w = kind == 0 ? prism_polar_workspace(h, (int)b.size(), mm.data(), nn.data(), o)
                               : prism_sqrt_workspace(h, (int)b.size(), nn.data(), o);
    if (!w) return fail_ext(PRISM_ERR_INVALID_ARG, std::string("bucket workspace query failed: ") + prism_last_error());
    L.solve_ws = std::max(L.solve_ws, w);
  }
  L.local_rep = align256(rep_bytes(std::max(1, L.max_nb), o->max_iters));
  L.global_rep = align256(rep_bytes(batch, o->max_iters));
  L.total = L.local_rep + L.global_rep + align256(L.solve_ws);
  return PRISM_OK;
}

}  // namespace

extern "C" {

prism_status prism_nccl_get_unique_id(void* id) {
  if (!id) return fail_ext(PRISM_ERR_INVALID_ARG, "null id");
  if (!nccl().ok) return fail_ext(PRISM_ERR_NCCL, nccl().why);
  ncclUniqueId u;
  ncclResult_t r = nccl().GetUniqueId(&u);
  if (r != ncclSuccess) return nccl_fail("ncclGetUniqueId", r);
  std::memcpy(id, &u, sizeof(u));
  return PRISM_OK;
}

prism_status prism_nccl_comm_init(void** comm, int nranks, const void* id, int rank) {
  if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks) return fail_ext(PRISM_ERR_INVALID_ARG, "bad comm args");
  if (!nccl().ok) return fail_ext(PRISM_ERR_NCCL, nccl().why);
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclComm_t c = nullptr;
  ncclResult_t r = nccl().CommInitRank(&c, nranks, u, rank);
  if (r != ncclSuccess) return nccl_fail("ncclCommInitRank", r);
  *comm = c;
  return PRISM_OK;
}

prism_status prism_nccl_comm_destroy(void* comm) {
  if (!comm) return PRISM_OK;
  if (!nccl().ok) return fail_ext(PRISM_ERR_NCCL, nccl().why);
  ncclResult_t r = nccl().CommDestroy(static_cast<ncclComm_t>(comm));
  return r == ncclSuccess ? PRISM_OK : nccl_fail("ncclCommDestroy", r);
}

prism_status prism_nccl_transport(void* comm, prism_transport* tr) {
  if (!comm || !tr) return fail_ext(PRISM_ERR_INVALID_ARG, "null comm / transport");
  if (!nccl().ok) return fail_ext(PRISM_ERR_NCCL, nccl().why);
  int n = 0, r = 0;
  ncclResult_t e = nccl().CommCount(static_cast<ncclComm_t>(comm), &n);
  if (e != ncclSuccess) return nccl_fail("ncclCommCount", e);
  e = nccl().CommUserRank(static_cast<ncclComm_t>(comm), &r);
  if (e != ncclSuccess) return nccl_fail("ncclCommUserRank", e);
  tr->ctx = comm;
  tr->nranks = n;
  tr->rank = r;
  tr->allreduce_sum = tr_allreduce;
  tr->broadcast = tr_broadcast;
  tr->group_start = tr_group_start;
  tr->group_end = tr_group_end;
  tr->async_error = tr_async_error;
  return PRISM_OK;
}

prism_status prism_shard_plan(int batch, const int64_t* m, const int64_t* n, int degree, int sketch_size, int nranks,
                              int nbuckets, int32_t* owner, int32_t* bucket) {
  if (batch < 1 || !m || !n || nranks < 1 || nbuckets < 1 || !owner || !bucket)
    return fail_ext(PRISM_ERR_INVALID_ARG, "bad shard-plan arguments");
  // LPT on F_min per iteration (iteration counts are not known before the solve)
  std::vector<double> cost(batch);
  for (int i = 0; i < batch; ++i) cost[i] = prism_polar_flops_per_iter(m[i], n[i], degree, sketch_size);
  prism_status s = prism_lpt_partition(batch, cost.data(), nranks, owner);
  if (s) return s;
  // buckets: each rank's matrices in index order, cut into nbuckets runs of about equal cost
  std::vector<double> tot(nranks, 0.0), acc(nranks, 0.0);
  for (int i = 0; i < batch; ++i) tot[owner[i]] += cost[i];
  for (int i = 0; i < batch; ++i) {
    const int r = owner[i];
    const double mid = acc[r] + 0.5 * cost[i];
    int b = tot[r] > 0.0 ? (int)(nbuckets * mid / tot[r]) : 0;
    bucket[i] = std::min(nbuckets - 1, std::max(0, b));
    acc[r] += cost[i];
  }
  return PRISM_OK;
}

size_t prism_polar_sharded_workspace(prism_handle h, int nranks, int rank, int batch, const int64_t* m,
                                     const int64_t* n, const prism_options* o, int nbuckets) {
  if (!h) return 0;
  ShardLayout L;
  if (shard_layout(h, 0, nranks, rank, batch, m, n, o, nbuckets, L)) return 0;
  return L.total;
}

}  // extern "C"

namespace {
// The sharded batch of either kind (include/prism.h): plan, bucketed solves with global sketch
// ids straight into the outputs, owners' broadcasts of each bucket (Q and, for sqrt, Q2) on the
// aux stream, report all-reduce.
prism_status sharded_impl(prism_handle h, const prism_transport* tr, int kind, int batch, const int64_t* m,
                          const int64_t* n, const void* const* A, const int64_t* lda, void* const* Q, void* const* Q2,
                          const int64_t* ldq, const prism_options* o, int nbuckets, const prism_report* rep,
                          void* workspace, size_t ws_bytes, void* stream) {
  try {
    if (!h || !tr || !tr->broadcast || !tr->allreduce_sum) return fail_ext(PRISM_ERR_INVALID_ARG, "bad transport");
    if (!A || !lda || (!Q && !Q2) || !ldq) return fail_ext(PRISM_ERR_INVALID_ARG, "null matrix arrays");
    ShardLayout L;
    prism_status s = shard_layout(h, kind, tr->nranks, tr->rank, batch, m, n, o, nbuckets, L);
    if (s) return s;
    if (!workspace || ws_bytes < L.total) return fail_ext(PRISM_ERR_INVALID_ARG, "workspace too small");
    for (int i = 0; i < batch; ++i)
      if (!A[i] || (Q && !Q[i]) || (Q2 && !Q2[i]) || ldq[i] < n[i])
        return fail_ext(PRISM_ERR_INVALID_ARG, "bad output / input matrix");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaStream_t cs = prism::handle_aux_stream(h);
    if (!cs) return fail_ext(PRISM_ERR_CUDA, "aux stream");
    const int M = o->max_iters;
    char* ws = static_cast<char*>(workspace);
    RepView lv = rep_view(ws, std::max(1, L.max_nb), M);
    RepView gv = rep_view(ws + L.local_rep, batch, M);
    char* sws = ws + L.local_rep + L.global_rep;
    const size_t esz = o->precision == PRISM_BF16 ? 2 : 4;
    if (rep && cudaMemsetAsync(ws + L.local_rep, 0, L.global_rep, st) != cudaSuccess)
      return fail_ext(PRISM_ERR_CUDA, "report scratch memset");
    // the comm stream starts after everything the caller queued before this call
    cudaEvent_t e0 = prism::handle_event(h, 0);
    if (cudaEventRecord(e0, st) != cudaSuccess || cudaStreamWaitEvent(cs, e0, 0) != cudaSuccess)
      return fail_ext(PRISM_ERR_CUDA, "stream ordering");
    const int nb = (int)L.mine.size();
    prism::NvtxRange nv_call(kind == 0 ? "prism:polar_sharded" : "prism:sqrt_invsqrt_sharded");
    for (int j = 0; j < nb; ++j) {
      prism::NvtxRange nv("prism:sharded bucket (solve + owners' broadcasts)");
      const std::vector<int>& b = L.mine[j];
      if (!b.empty()) {
        std::vector<int64_t> mm, nn, la, lq, ids;
        std::vector<const void*> a;
        std::vector<void*> q, q2;
        for (int i : b) {
          mm.push_back(m[i]);
          nn.push_back(n[i]);
          la.push_back(lda[i]);
          lq.push_back(ldq[i]);
          ids.push_back(i);
          a.push_back(A[i]);
          if (Q) q.push_back(Q[i]);
          if (Q2) q2.push_back(Q2[i]);
        }
        prism_report lr{lv.iters, lv.resid, lv.status, lv.alphas, lv.hist};
        if (kind == 0)
          s = prism_polar(h, (int)b.size(), mm.data(), nn.data(), a.data(), la.data(), q.data(), lq.data(),
                          ids.data(), o, rep ? &lr : nullptr, sws, L.solve_ws, stream);
        else
          s = prism_sqrt_invsqrt(h, (int)b.size(), nn.data(), a.data(), la.data(), Q ? q.data() : nullptr,
                                 Q2 ? q2.data() : nullptr, lq.data(), ids.data(), o, rep ? &lr : nullptr, sws,
                                 L.solve_ws, stream);
        if (s) return s;
        if (rep) {
          ScatterIdx ix;
          ix.n = (int)b.size();
          for (int t = 0; t < ix.n; ++t) ix.idx[t] = b[t];
          k_rep_scatter<<<std::max(1, std::min(64, (ix.n * (M + 1) + 255) / 256)), 256, 0, st>>>(
              ix, M, lv.iters, lv.resid, lv.status, lv.alphas, lv.hist, gv.iters, gv.resid, gv.status, gv.alphas,
              gv.hist);
          if (cudaGetLastError() != cudaSuccess) return fail_ext(PRISM_ERR_CUDA, "report scatter launch");
        }
      }
      // bucket j of every rank: owners broadcast their outputs (in place) once solved
      cudaEvent_t ej = prism::handle_event(h, 1 + (j & 1));
      if (cudaEventRecord(ej, st) != cudaSuccess || cudaStreamWaitEvent(cs, ej, 0) != cudaSuccess)
        return fail_ext(PRISM_ERR_CUDA, "stream ordering");
      if (tr->group_start && tr->group_start(tr->ctx)) return fail_ext(PRISM_ERR_NCCL, "group start");
      for (int i = 0; i < batch; ++i) {
        if (L.bucket[i] != j) continue;
        const size_t bytes = ((size_t)(m[i] - 1) * ldq[i] + n[i]) * esz;
        if (Q && tr->broadcast(tr->ctx, Q[i], bytes, L.owner[i], cs)) return fail_ext(PRISM_ERR_NCCL, "broadcast");
        if (Q2 && tr->broadcast(tr->ctx, Q2[i], bytes, L.owner[i], cs)) return fail_ext(PRISM_ERR_NCCL, "broadcast");
      }
      if (tr->group_end && tr->group_end(tr->ctx)) return fail_ext(PRISM_ERR_NCCL, "group end");
    }
    if (rep) {
      // every matrix's report on every rank: non-owners contribute zeros
      cudaEvent_t ej = prism::handle_event(h, 3);
      if (cudaEventRecord(ej, st) != cudaSuccess || cudaStreamWaitEvent(cs, ej, 0) != cudaSuccess)
        return fail_ext(PRISM_ERR_CUDA, "stream ordering");
      if (tr->group_start && tr->group_start(tr->ctx)) return fail_ext(PRISM_ERR_NCCL, "group start");
      int e = 0;
      if (rep->iters) e |= tr->allreduce_sum(tr->ctx, gv.iters, rep->iters, batch, PRISM_DT_I32, cs);
      if (rep->status) e |= tr->allreduce_sum(tr->ctx, gv.status, rep->status, batch, PRISM_DT_I32, cs);
      if (rep->resid) e |= tr->allreduce_sum(tr->ctx, gv.resid, rep->resid, batch, PRISM_DT_F32, cs);
      if (rep->alphas) e |= tr->allreduce_sum(tr->ctx, gv.alphas, rep->alphas, (size_t)batch * M, PRISM_DT_F64, cs);
      if (rep->resid_hist)
        e |= tr->allreduce_sum(tr->ctx, gv.hist, rep->resid_hist, (size_t)batch * (M + 1), PRISM_DT_F32, cs);
      if (tr->group_end && tr->group_end(tr->ctx)) return fail_ext(PRISM_ERR_NCCL, "group end");
      if (e) return fail_ext(PRISM_ERR_NCCL, "report all-reduce");
    }
    cudaEvent_t ef = prism::handle_event(h, 4);
    if (cudaEventRecord(ef, cs) != cudaSuccess || cudaStreamWaitEvent(st, ef, 0) != cudaSuccess)
      return fail_ext(PRISM_ERR_CUDA, "stream ordering");
    if (tr->async_error && tr->async_error(tr->ctx)) return fail_ext(PRISM_ERR_NCCL, "communicator error");
    return PRISM_OK;
  } catch (...) {
    return fail_ext(PRISM_ERR_INTERNAL, "exception in the sharded batch");
  }
}
}  // namespace

extern "C" {

prism_status prism_polar_sharded_tr(prism_handle h, const prism_transport* tr, int batch, const int64_t* m,
                                    const int64_t* n, const void* const* A, const int64_t* lda, void* const* Q,
                                    const int64_t* ldq, const prism_options* o, int nbuckets,
                                    const prism_report* rep, void* workspace, size_t ws_bytes, void* stream) {
  if (!Q) return fail_ext(PRISM_ERR_INVALID_ARG, "null outputs");
  return sharded_impl(h, tr, 0, batch, m, n, A, lda, Q, nullptr, ldq, o, nbuckets, rep, workspace, ws_bytes, stream);
}

prism_status prism_sqrt_invsqrt_sharded_tr(prism_handle h, const prism_transport* tr, int batch, const int64_t* n,
                                           const void* const* A, const int64_t* lda, void* const* Asqrt,
                                           void* const* Ainvsqrt, const int64_t* ld_out, const prism_options* o,
                                           int nbuckets, const prism_report* rep, void* workspace, size_t ws_bytes,
                                           void* stream) {
  return sharded_impl(h, tr, 1, batch, n, n, A, lda, Asqrt, Ainvsqrt, ld_out, o, nbuckets, rep, workspace, ws_bytes,
                      stream);
}

size_t prism_sqrt_invsqrt_sharded_workspace(prism_handle h, int nranks, int rank, int batch, const int64_t* n,
                                            const prism_options* o, int nbuckets) {
  if (!h) return 0;
  ShardLayout L;
  if (shard_layout(h, 1, nranks, rank, batch, n, n, o, nbuckets, L)) return 0;
  return L.total;
}

prism_status prism_sqrt_invsqrt_sharded(prism_handle h, void* comm, int batch, const int64_t* n, const void* const* A,
                                        const int64_t* lda, void* const* Asqrt, void* const* Ainvsqrt,
                                        const int64_t* ld_out, const prism_options* o, int nbuckets,
                                        const prism_report* rep, void* workspace, size_t ws_bytes, void* stream) {
  prism_transport tr;
  prism_status s = prism_nccl_transport(comm, &tr);
  if (s) return s;
  return prism_sqrt_invsqrt_sharded_tr(h, &tr, batch, n, A, lda, Asqrt, Ainvsqrt, ld_out, o, nbuckets, rep, workspace,
                                       ws_bytes, stream);
}

prism_status prism_polar_sharded(prism_handle h, void* comm, int batch, const int64_t* m, const int64_t* n,
                                 const void* const* A, const int64_t* lda, void* const* Q, const int64_t* ldq,
                                 const prism_options* o, int nbuckets, const prism_report* rep, void* workspace,
                                 size_t ws_bytes, void* stream) {
  prism_transport tr;
  prism_status s = prism_nccl_transport(comm, &tr);
  if (s) return s;
  return prism_polar_sharded_tr(h, &tr, batch, m, n, A, lda, Q, ldq, o, nbuckets, rep, workspace, ws_bytes, stream);
}

}  // extern "C"
