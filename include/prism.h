/*
 * prism.h — C ABI of the B200-native PRISM Newton–Schulz library (libprism.so).
 *
 * PRISM (arXiv 2601.22137, /root/reference/PAPER.md = "P:<line>") computes
 * matrix functions by a Newton–Schulz iteration whose top polynomial
 * coefficient alpha_k is refitted every step from a Gaussian-sketched residual
 * (eq. (4); Appendix A.1).  This library runs that
 * iteration for batches of matrices on one sm_100a GPU:
 *   prism_polar          polar factor U V^T of A = U S V^T (Table 1
 *                        rows P:252-254) — Muon orthogonalisation;
 *   prism_sqrt_invsqrt   A^{1/2} and A^{-1/2} of SPD A (Theorem 3
 *                        P:273-275) — Shampoo preconditioners.
 *
 * Conventions (all entry points):
 *   - Matrices are dense, row-major, addressed by a device pointer and a
 *     leading dimension in ELEMENTS.  Element type follows the precision:
 *     PRISM_BF16 -> __nv_bfloat16 (2 bytes); PRISM_FP32 / PRISM_TF32 -> float.
 *   - Arrays of per-matrix pointers / sizes (A, lda, m, n, ...) are HOST arrays
 *     of length `batch`; the pointers they hold are DEVICE pointers.
 *   - Ownership: the caller owns every device buffer (inputs, outputs, report,
 *     workspace).  The library never allocates device memory; the handle owns
 *     only host-side pinned staging and cached plans.
 *   - Asynchrony: work is enqueued on `stream` (a cudaStream_t, may be NULL for
 *     the legacy default stream) and the call returns without synchronising.
 *     Outputs and the report are valid after the caller synchronises the stream.
 *   - The workspace must not be used by anything else until the stream has
 *     finished the call; it holds the solver state and the per-call tables.
 *   - Errors: argument errors are detected on the host before any launch and
 *     return a non-zero prism_status; prism_last_error() describes the last
 *     failure of the calling thread.  No C++ exception crosses the ABI.
 *     Numerical outcomes are per-matrix report status values, not call errors.
 *   - Thread safety: a handle may be used by one host thread at a time.
 */
#ifndef PRISM_H_
#define PRISM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PRISM_VERSION_MAJOR 0
#define PRISM_VERSION_MINOR 1

typedef struct prism_handle_s* prism_handle;

typedef enum {
  PRISM_OK = 0,
  PRISM_ERR_INVALID_ARG = 1, /* null pointer, bad size/option, workspace too small */
  PRISM_ERR_UNSUPPORTED = 2, /* valid but not supported (e.g. sketch_size > 64, DB Newton outside FP32) */
  PRISM_ERR_CUDA = 3,        /* a CUDA runtime/driver call failed */
  PRISM_ERR_INTERNAL = 4,
  PRISM_ERR_NCCL = 5         /* NCCL unavailable, or a collective / communicator failed */
} prism_status;

typedef enum {
  PRISM_BF16 = 0, /* bf16 storage, bf16 tcgen05 MMA (kind::f16), fp32 accumulate */
  PRISM_FP32 = 1, /* fp32 storage, 3xTF32 tcgen05 MMA (hi*hi + hi*lo + lo*hi), fp32 accumulate */
  PRISM_TF32 = 2  /* fp32 storage, 1xTF32 tcgen05 MMA */
} prism_precision;

typedef enum {
  PRISM_FIT_SKETCHED = 0, /* alpha_k from the sketched quartic, eq. (4) */
  PRISM_FIT_TAYLOR = 1    /* alpha_k = Taylor coefficient: classical Newton–Schulz */
} prism_fit;

typedef enum {
  PRISM_CONVERGED = 0,  /* ||I - G_k||_F <= tol * sqrt(s) before an update */
  PRISM_MAX_ITERS = 1,  /* max_iters updates applied without converging */
  PRISM_DIVERGED = 2,   /* ||R_k||_F increased 5 times in a row (R12) */
  PRISM_NONFINITE = 3,  /* NaN / Inf residual */
  PRISM_ZERO_INPUT = 4  /* ||A||_F = 0: output is zero */
} prism_solve_status;

typedef struct {
  int degree;          /* 3 ("PRISM-3", d=1: g = I + aR) or 5 ("PRISM-5", d=2: g = I + R/2 + aR^2) */
  int max_iters;       /* >= 1: maximum number of updates */
  int sketch_size;     /* p, rows of the Gaussian sketch S_k; default 8; limits above */
  double tol;          /* > 0: stop before the update when ||R_k||_F <= tol * sqrt(s) (R12) */
  uint64_t seed;       /* Philox key; S_k depends only on (seed, matrix id, k) (R8) */
  int precision;       /* prism_precision */
  int fit;             /* prism_fit */
  int warmup_iters;    /* alpha_k = u for k < warmup_iters; 0 for the paper's eq. (4) everywhere */
  double alpha_lo;     /* interval [l, u] for alpha; NaN -> paper default */
  double alpha_hi;     /*   [1/2, 1] for degree 3, [3/8, 29/20] for degree 5 */
} prism_options;

/* Per-matrix results, DEVICE pointers (any may be NULL), written on `stream`. */
typedef struct {
  int32_t* iters;      /* [batch] updates applied */
  float* resid;        /* [batch] final ||R||_F / sqrt(s) */
  int32_t* status;     /* [batch] prism_solve_status */
  double* alphas;      /* [batch * max_iters] alpha_k history (row b, column k), or NULL */
  float* resid_hist;   /* [batch * (max_iters + 1)] ||R_k||_F / sqrt(s), or NULL */
} prism_report;

/* Fill `o` with defaults: degree 5, max_iters 30, p 8, tol 1e-6, seed 42, BF16, sketched, no warmup.
 * sketch_size p: 1 <= p <= min(s, 32) for polar / sqrt / sign ("as small as 5"; Theorem 2,
 * P:229, asks for more); 1 <= p <= min(s, 8) for the inverse root and Chebyshev kinds. */
void prism_default_options(prism_options* o);

prism_status prism_create(prism_handle* h);
prism_status prism_destroy(prism_handle h);
/* Message for the last failing call made by this thread (never NULL). */
const char* prism_last_error(void);
/* Number of exported entry points and their names (for ABI checks). */
int prism_abi_version(void);

/*
 * Polar factor.  For matrix i of the batch: A_i is m[i] x n[i] (row-major, lda[i]),
 * Q_i receives U V^T with the same shape (ldq[i]; Q_i may alias A_i exactly; no other
 * overlap of an output with an input of the batch is allowed).  BF16 / TF32 solves use Q_i
 * as one of the two iterate buffers, so it holds intermediate values
 * until the call's work on `stream` completes.  Wide inputs (m < n) are handled as A^T
 * (P:456 assumes m >= n; R14).
 * matrix_ids: optional HOST array of global matrix indices used as the sketch
 * stream id (so a batch split across GPUs draws the same S_k); NULL -> 0..batch-1.
 * Workspace: at least prism_polar_workspace(...) bytes of device memory, 256-B aligned.
 */
size_t prism_polar_workspace(prism_handle h, int batch, const int64_t* m, const int64_t* n,
                             const prism_options* o);
prism_status prism_polar(prism_handle h, int batch, const int64_t* m, const int64_t* n,
                         const void* const* A, const int64_t* lda, void* const* Q, const int64_t* ldq,
                         const int64_t* matrix_ids, const prism_options* o, const prism_report* rep,
                         void* workspace, size_t ws_bytes, void* stream);

/*
 * End-to-end path on HOST buffers.  A[i] / Q[i] are page-locked host memory
 * (cudaHostAlloc / cudaHostRegister / torch pin_memory), shapes and leading dimensions as
 * prism_polar.  The call enqueues, on handle-internal streams, the upload into one of three
 * handle-owned device staging slots, the solve, and the download into Q, then returns;
 * `stream` is made to wait for the download, so a sync of `stream` (or later work on it)
 * observes Q.  Successive calls on one handle pipeline: the upload of call k+1 and the
 * download of call k overlap the solves.  The upload starts when the call is made (it is
 * not ordered after work queued earlier on `stream`): A must hold its values at the call.  Staging and workspace are device memory owned by
 * the handle (grown on demand, which synchronises the device).  rep: optional DEVICE
 * report, written in call order (read it once no later call is in flight).
 */
prism_status prism_polar_host(prism_handle h, int batch, const int64_t* m, const int64_t* n, const void* const* A,
                              const int64_t* lda, void* const* Q, const int64_t* ldq, const int64_t* matrix_ids,
                              const prism_options* o, const prism_report* rep, void* stream);

/*
 * Coupled square root / inverse square root of SPD n[i] x n[i] matrices
 * (symmetry is the caller's contract; a non-SPD input shows up as a
 * DIVERGED / NONFINITE / MAX_ITERS status).  Asqrt / Ainvsqrt: either array,
 * or any entry, may be NULL.  Output leading dimension ld_out[i].
 */
size_t prism_sqrt_workspace(prism_handle h, int batch, const int64_t* n, const prism_options* o);
prism_status prism_sqrt_invsqrt(prism_handle h, int batch, const int64_t* n, const void* const* A,
                                const int64_t* lda, void* const* Asqrt, void* const* Ainvsqrt,
                                const int64_t* ld_out, const int64_t* matrix_ids, const prism_options* o,
                                const prism_report* rep, void* workspace, size_t ws_bytes, void* stream);
/*
 * Matrix sign sign(A) = A (A^2)^{-1/2} of square n[i] x n[i] matrices (the paper's case
 * study): X_0 = A/||A||_F, R_k = I - X_k^2, X_{k+1} = X_k g_d(R_k; a_k) with
 * the same sketched fit.  A^2 symmetric is the paper's standing assumption;
 * otherwise convergence is not guaranteed (status).  S[i] receives sign(A_i) (ld lds[i];
 * may alias A).  Other arguments as prism_polar.
 */
size_t prism_sign_workspace(prism_handle h, int batch, const int64_t* n, const prism_options* o);
prism_status prism_sign(prism_handle h, int batch, const int64_t* n, const void* const* A, const int64_t* lda,
                        void* const* S, const int64_t* lds, const int64_t* matrix_ids, const prism_options* o,
                        const prism_report* rep, void* workspace, size_t ws_bytes, void* stream);

/*
 * Inverse q-th root A^{-1/q} of SPD n[i] x n[i] matrices by the PRISM-accelerated
 * coupled inverse Newton iteration (Appendix A.3; the paper's p is q here):
 *   c = (2||A||_F/(q+1))^{1/q},  X_0 = I/c,  M_0 = A/c^q,  R_k = I - M_k,
 *   X_{k+1} = X_k (I + a_k R_k),  M_{k+1} = (I + a_k R_k)^q M_k,
 *   a_k = argmin over [1/(2q), 2/q] (overridable by alpha_lo/hi) of the sketched
 *   degree-2q loss ||S_k (R_k + sum_i C(q,i) a^i (R_k^{i+1} - R_k^i))||_F^2.
 * q in 1..4 (PRISM_ERR_UNSUPPORTED otherwise); options.degree is ignored (the method is
 * first order); fit SKETCHED or TAYLOR (a = 1/q: the classical coupled inverse Newton).
 * X[i] receives A_i^{-1/q} (ld ldx[i]; may alias A).  Other arguments as prism_polar.
 */
size_t prism_inv_root_workspace(prism_handle h, int batch, const int64_t* n, int q, const prism_options* o);
prism_status prism_inv_root(prism_handle h, int batch, const int64_t* n, int q, const void* const* A,
                            const int64_t* lda, void* const* X, const int64_t* ldx, const int64_t* matrix_ids,
                            const prism_options* o, const prism_report* rep, void* workspace, size_t ws_bytes,
                            void* stream);
/* prism_inv_root on page-locked HOST buffers, pipelined as prism_polar_host. */
prism_status prism_inv_root_host(prism_handle h, int batch, const int64_t* n, int q, const void* const* A,
                                 const int64_t* lda, void* const* X, const int64_t* ldx, const int64_t* matrix_ids,
                                 const prism_options* o, const prism_report* rep, void* stream);

/*
 * Inverse A^{-1} of square full-rank n[i] x n[i] matrices (general, not necessarily
 * symmetric) by the PRISM-accelerated Chebyshev iteration (Appendix A.4):
 *   A' = A/||A||_F,  X_0 = A'^T,  R_k = I - A' X_k,  X_{k+1} = X_k (I + R_k + a_k R_k^2),
 *   a_k = argmin over [1/2, 2] (overridable) of ||S_k (R_k^2 - a (R_k^2 - R_k^3))||_F^2
 *   (closed form), A^{-1} = X / ||A||_F.  options.degree is ignored; fit SKETCHED or
 * TAYLOR (a = 1: the classical Chebyshev iteration).  X[i] receives A_i^{-1} (ld ldx[i];
 * may alias A: the iteration reads its own copy of A' in the workspace).  Other
 * arguments as prism_polar.
 */
size_t prism_chebyshev_inverse_workspace(prism_handle h, int batch, const int64_t* n, const prism_options* o);
prism_status prism_chebyshev_inverse(prism_handle h, int batch, const int64_t* n, const void* const* A,
                                     const int64_t* lda, void* const* X, const int64_t* ldx,
                                     const int64_t* matrix_ids, const prism_options* o, const prism_report* rep,
                                     void* workspace, size_t ws_bytes, void* stream);
/* prism_chebyshev_inverse on page-locked HOST buffers, pipelined as prism_polar_host. */
prism_status prism_chebyshev_inverse_host(prism_handle h, int batch, const int64_t* n, const void* const* A,
                                          const int64_t* lda, void* const* X, const int64_t* ldx,
                                          const int64_t* matrix_ids, const prism_options* o,
                                          const prism_report* rep, void* stream);

/*
 * A^{1/2} and A^{-1/2} of SPD n[i] x n[i] matrices by PRISM-accelerated DB Newton in
 * product form (Appendix A.2):
 *   M_0 = X_0 = A, Y_0 = I,  M_{k+1} = 2a(1-a) I + (1-a)^2 M_k + a^2 M_k^{-1},
 *   X_{k+1} = (1-a) X_k + a X_k M_k^{-1},  Y_{k+1} = (1-a) Y_k + a Y_k M_k^{-1},
 *   a_k = argmin over the reals of the exact quartic ||I - M_{k+1}||_F^2 (no sketch,
 *   no interval); fit TAYLOR keeps a = 1/2 (the classical product form).
 * Stops when ||I - M_k||_F <= tol sqrt(n).  M_k^{-1} is computed on the device by a
 * blocked Gauss-Jordan sweep (128-blocks, tcgen05 GEMMs).  precision must be
 * PRISM_FP32 (PRISM_ERR_UNSUPPORTED otherwise); options.degree / sketch_size unused.
 * Asqrt / Ainvsqrt as prism_sqrt_invsqrt (either may be NULL; unscaled).
 */
size_t prism_db_newton_workspace(prism_handle h, int batch, const int64_t* n, const prism_options* o);
prism_status prism_db_newton(prism_handle h, int batch, const int64_t* n, const void* const* A, const int64_t* lda,
                             void* const* Asqrt, void* const* Ainvsqrt, const int64_t* ld_out,
                             const int64_t* matrix_ids, const prism_options* o, const prism_report* rep,
                             void* workspace, size_t ws_bytes, void* stream);
/* prism_db_newton on page-locked HOST buffers, pipelined as prism_polar_host. */
prism_status prism_db_newton_host(prism_handle h, int batch, const int64_t* n, const void* const* A,
                                  const int64_t* lda, void* const* Asqrt, void* const* Ainvsqrt,
                                  const int64_t* ld_out, const int64_t* matrix_ids, const prism_options* o,
                                  const prism_report* rep, void* stream);

/* prism_sign on page-locked HOST buffers, pipelined as prism_polar_host. */
prism_status prism_sign_host(prism_handle h, int batch, const int64_t* n, const void* const* A, const int64_t* lda,
                             void* const* S, const int64_t* lds, const int64_t* matrix_ids, const prism_options* o,
                             const prism_report* rep, void* stream);

/* prism_sqrt_invsqrt on page-locked HOST buffers, pipelined as prism_polar_host. */
prism_status prism_sqrt_invsqrt_host(prism_handle h, int batch, const int64_t* n, const void* const* A,
                                     const int64_t* lda, void* const* Asqrt, void* const* Ainvsqrt,
                                     const int64_t* ld_out, const int64_t* matrix_ids, const prism_options* o,
                                     const prism_report* rep, void* stream);

/*
 * LPT partition: assign `batch` matrices with costs cost[i]
 * (e.g. F_min x expected iterations) to `ranks` ranks, largest first to the
 * least-loaded rank, ties by lower index / lower rank.  Writes owner[i] in
 * [0, ranks).  Deterministic: every rank computes the same plan.  Host only.
 */
prism_status prism_lpt_partition(int batch, const double* cost, int ranks, int32_t* owner);

/* ---- multi-GPU: one process per GPU ----------------------------------
 *
 * Exchange layer.  The multi-GPU entry points move data only through a transport: the
 * library's NCCL transport (prism_nccl_transport) or any caller-supplied one (a test
 * harness).  Every function returns 0 on success; the operation is enqueued on `stream`
 * (a cudaStream_t) or completed before returning.  Buffers are DEVICE memory.
 */
typedef enum { PRISM_DT_F32 = 0, PRISM_DT_F64 = 1, PRISM_DT_I32 = 2, PRISM_DT_BYTES = 3 } prism_dtype;
typedef struct {
  void* ctx;
  int nranks;
  int rank;
  /* recv[i] = sum over ranks of send[i], i < count (send may equal recv) */
  int (*allreduce_sum)(void* ctx, const void* send, void* recv, size_t count, int dtype, void* stream);
  /* buf (bytes) of rank `root` copied into buf on every rank */
  int (*broadcast)(void* ctx, void* buf, size_t bytes, int root, void* stream);
  int (*group_start)(void* ctx);   /* bracket several collectives (may be NULL) */
  int (*group_end)(void* ctx);
  int (*async_error)(void* ctx);   /* non-zero once the communicator has failed (may be NULL) */
} prism_transport;

/*
 * NCCL, resolved at run time from the libnccl.so.2 the process has loaded (torch's bundled
 * NCCL after `import torch`; else the system one): the library does not link NCCL, so one
 * NCCL serves the caller and the library.  `comm` is an ncclComm_t of that NCCL — from
 * prism_nccl_comm_init, or the caller's own.  id: 128-byte ncclUniqueId (rank 0 creates it,
 * the caller distributes it).  Errors: PRISM_ERR_NCCL (library not found, call failed).
 */
prism_status prism_nccl_get_unique_id(void* id);
prism_status prism_nccl_comm_init(void** comm, int nranks, const void* id, int rank);
prism_status prism_nccl_comm_destroy(void* comm);
prism_status prism_nccl_transport(void* comm, prism_transport* tr);

/*
 * Sharded batch (BASELINE configs[4]; problem statement P:18): every
 * rank passes the SAME full batch (a data-parallel step's reduced gradients).  Matrices are
 * assigned to ranks by prism_shard_plan (LPT on F_min, deterministic), each rank solves its
 * share with prism_polar in `nbuckets` sub-batches with the GLOBAL matrix index as sketch id
 * (so every result is bit-identical to the single-GPU solve of the whole batch), writing
 * straight into Q[i]; after each sub-batch the owners broadcast its outputs, so the exchange
 * of bucket j overlaps the solve of bucket j+1.  On return every rank's Q holds all outputs
 * once `stream` completes.  Q[i] must not alias A[i] on a non-owner (it is overwritten by the
 * broadcast of rows m x ldq, including the padding between rows).  rep (device, [batch]
 * layout as prism_polar, optional) receives every matrix's report on every rank.
 * Workspace: prism_polar_sharded_workspace bytes (depends on nranks / rank).
 */
size_t prism_polar_sharded_workspace(prism_handle h, int nranks, int rank, int batch, const int64_t* m,
                                     const int64_t* n, const prism_options* o, int nbuckets);
prism_status prism_polar_sharded(prism_handle h, void* comm, int batch, const int64_t* m, const int64_t* n,
                                 const void* const* A, const int64_t* lda, void* const* Q, const int64_t* ldq,
                                 const prism_options* o, int nbuckets, const prism_report* rep, void* workspace,
                                 size_t ws_bytes, void* stream);
prism_status prism_polar_sharded_tr(prism_handle h, const prism_transport* tr, int batch, const int64_t* m,
                                    const int64_t* n, const void* const* A, const int64_t* lda, void* const* Q,
                                    const int64_t* ldq, const prism_options* o, int nbuckets,
                                    const prism_report* rep, void* workspace, size_t ws_bytes, void* stream);
/*
 * Sharded coupled A^{1/2}, A^{-1/2} (Shampoo blocks shard like the Muon batch):
 * the same protocol as prism_polar_sharded over prism_sqrt_invsqrt, both outputs broadcast
 * from their owners (either output array may be NULL; ld_out as prism_sqrt_invsqrt).
 */
size_t prism_sqrt_invsqrt_sharded_workspace(prism_handle h, int nranks, int rank, int batch, const int64_t* n,
                                            const prism_options* o, int nbuckets);
prism_status prism_sqrt_invsqrt_sharded(prism_handle h, void* comm, int batch, const int64_t* n, const void* const* A,
                                        const int64_t* lda, void* const* Asqrt, void* const* Ainvsqrt,
                                        const int64_t* ld_out, const prism_options* o, int nbuckets,
                                        const prism_report* rep, void* workspace, size_t ws_bytes, void* stream);
prism_status prism_sqrt_invsqrt_sharded_tr(prism_handle h, const prism_transport* tr, int batch, const int64_t* n,
                                           const void* const* A, const int64_t* lda, void* const* Asqrt,
                                           void* const* Ainvsqrt, const int64_t* ld_out, const prism_options* o,
                                           int nbuckets, const prism_report* rep, void* workspace, size_t ws_bytes,
                                           void* stream);
/* The plan (host only): owner[i] in [0, nranks) and bucket[i] in [0, nbuckets) of matrix i. */
prism_status prism_shard_plan(int batch, const int64_t* m, const int64_t* n, int degree, int sketch_size, int nranks,
                              int nbuckets, int32_t* owner, int32_t* bucket);

/*
 * Row-block split of ONE polar problem too large for one GPU (BASELINE
 * configs[3], 8192^2 over 2/4/8 GPUs; the iteration is Table 1).  Rank r holds
 * rows [row0, row0 + rows) of the global m_global x n matrix A (rows summed over ranks =
 * m_global).  Per iteration k every rank
 *   1. forms its partial Gram X_r^T X_r (symmetric: upper-triangle tiles only) as fp32
 *      panels of 256 rows, packed (panel t: rows [256t, 256t+256) x columns [256t, n)),
 *      and all-reduces (sums) each panel group as soon as it is computed, overlapping the
 *      rest of the Gram;
 *   2. unpacks R = I - G, runs the sketch (matrix id 0), chain and alpha fit — identical
 *      inputs on every rank, so alpha_k and the stop decision are identical;
 *   3. updates its rows with no R^2 and no second collective: d = 2: Y_r = X_r R and
 *      X_r' = (X_r + Y_r / 2) + alpha Y_r R; d = 1: X_r' = X_r + alpha X_r R
 *      (= X_r g_d(R_k; alpha_k): 5 (rows) n^2 FLOP per rank per iteration for d = 2).
 * The host loop stays ahead of the device: after enqueuing iteration k it waits only for
 * iteration k's stop test (its updates still queued) before deciding to enqueue k + 1, so
 * the call returns once the iteration count is known, with the tail enqueued on `stream`.
 * Q_rows receives rows [row0, row0 + rows) of U V^T (may alias A_rows).  rep: [1] (device).
 */
size_t prism_polar_rowblock_workspace(prism_handle h, int64_t rows, int64_t n, const prism_options* o);
prism_status prism_polar_rowblock(prism_handle h, void* comm, int64_t m_global, int64_t n, const void* A_rows,
                                  int64_t row0, int64_t rows, int64_t lda, void* Q_rows, int64_t ldq,
                                  const prism_options* o, const prism_report* rep, void* workspace, size_t ws_bytes,
                                  void* stream);
prism_status prism_polar_rowblock_tr(prism_handle h, const prism_transport* tr, int64_t m_global, int64_t n,
                                     const void* A_rows, int64_t row0, int64_t rows, int64_t lda, void* Q_rows,
                                     int64_t ldq, const prism_options* o, const prism_report* rep, void* workspace,
                                     size_t ws_bytes, void* stream);
/* Packed Gram layout (host only): panel_off[t] = float offset of panel t (t = 0..ceil(n/256)),
 * panel_off[ceil(n/256)] = total floats; group_end[g] = first panel after group g (groups
 * of about equal tile counts, g < ngroups). */
prism_status prism_rowblock_layout(int64_t n, int ngroups, int64_t* panel_off, int32_t* group_end);

/* Per-iteration F_min (symmetric products counted once) of a polar solve. */
double prism_polar_flops_per_iter(int64_t m, int64_t n, int degree, int sketch_size);
/* Dense-GEMM flop count per sqrt iteration (general products). */
double prism_sqrt_flops_per_iter(int64_t n, int degree, int sketch_size);

/* ---- measurement (bench.py) ---------------------------------------------------- */

/* Kernel launches of the library issued by the calls on h since the previous
 * prism_launch_count (which it resets): per graph solve, the launches outside its loop plus
 * the launches per iteration times the iterations of that plan's most recent solve; per
 * row-block call, the launches it issued.  Synchronises the device. */
int64_t prism_launch_count(prism_handle h);
/*
 * Per-kernel-kind device timing.  When enabled, every launch group is bracketed
 * with CUDA events on the caller's stream (kinds: 0 residual GEMM, 1 square GEMM,
 * 2 apply GEMM, 3 sketch + chain, 4 alpha solve, 5 normalise/finalise).
 * prism_profile_read synchronises those events and returns the accumulated
 * milliseconds and launch counts per kind since the last reset (arrays of 6).
 */
prism_status prism_profile_enable(prism_handle h, int enable);
prism_status prism_profile_read(prism_handle h, double* ms, int64_t* launches, int reset);

/* ---- test hooks (exercised by tests/test_gpu_*.py) ---------------------------- */

/*
 * One grouped tcgen05 GEMM problem: out = epilogue(A * B) with A (M x K, row-major,
 * lda) and B either K-major (b_mn = 0: B stored N x K, ldb, i.e. out = A B^T) or
 * MN-major (b_mn = 1: B stored K x N).  mode: 0 RESID (I - D, with per-tile
 * sum of squares into norm_part[tiles_m*tiles_n] and diag(D) into gdiag),
 * 1 POLY (c1*C + alpha*D), 2 APPLY (C + (scale_by_alpha ? alpha : 1)*D), 3 STORE.
 * sym: triangle schedule + mirrored stores (requires M == N).  FP32 precision
 * (3xTF32) takes the lo planes A_lo, B_lo, C_lo, out_lo (hi planes pre-truncated).
 * alpha_dev: device double.  Leading dimensions must be multiples of 16 bytes.
 */
prism_status prism_debug_gemm(prism_handle h, int precision, int b_mn, int mode, int sym, int M, int N, int K,
                              const void* A, const void* A_lo, int64_t lda, const void* B, const void* B_lo,
                              int64_t ldb, const void* C, const void* C_lo, int64_t ldc, void* out,
                              void* out_lo, int64_t ldo, const double* alpha_dev, float c1, int scale_by_alpha,
                              float* norm_part, float* gdiag, void* workspace, size_t ws_bytes, void* stream);
/* S_k for (seed, matrix id b, iteration k): p x s floats into S_dev (R8). */
prism_status prism_debug_sketch(uint64_t seed, int64_t b, int k, int p, int s, float* S_dev, void* stream);
/* Device quartic argmin on [lo, hi] (R15/R16): n problems, c_dev[5*n] -> alpha_dev[n]. */
prism_status prism_debug_argmin(int n, const double* c_dev, double lo, double hi, double a_taylor,
                                double* alpha_dev, void* stream);
/* Main-GEMM k-block timeline (diagnostics only): buf_dev = device u64[148 * 376]; launches
 * whose epilogue mode is `mode` (0 residual, 1 poly, 2 apply; < 0 off) record per-CTA
 * globaltimer stamps (gemm.cuh).  NULL disables. */
prism_status prism_debug_trace_gemm(unsigned long long* buf_dev, int mode);
/* Diagnostics (the pool refuses compute-sanitizer): with guards enabled, plans built from then
 * on follow every workspace sub-buffer with a 256-B band no kernel may touch (plans are keyed
 * by the switch; the workspace query grows accordingly).  _fill sets the bands of the last plan
 * used on `h` to 0xA5 (on `stream`); _check synchronises `stream` and counts the changed bytes
 * over all bands (bad_bytes) and the bands (guards). */
prism_status prism_debug_workspace_guards(int enable);
prism_status prism_debug_guards_fill(prism_handle h, void* stream);
prism_status prism_debug_guards_check(prism_handle h, int64_t* bad_bytes, int64_t* guards, void* stream);
/* Positive control of the checker: clears the first byte of guard band idx of the last plan. */
prism_status prism_debug_guards_poke(prism_handle h, int64_t idx, void* stream);
/* Diagnostics: persistent-grid cap (CTAs) of prism_debug_gemm launches and of the GEMMs of
 * solve plans built afterwards (0: all SMs; the row-block pipelined Gram keeps its own cap). */
prism_status prism_debug_gemm_max_ctas(int max_ctas);
/* Diagnostics: GEMM tile order of plans built afterwards — within a matrix, groups of `rows`
 * tile rows walked column by column (default 8; 1: row-major).  Never changes results. */
prism_status prism_debug_raster_rows(int rows);
/* Sketch-chain timeline hook: buf_dev (16 iterations x 32 pass codes x 160 CTAs x 32 u64,
 * zeroed by the caller) receives per CTA globaltimer ns at entry, after the PDL wait, when the
 * first tile's accumulator is ready, when its epilogue ends, and the epilogue's inner marks
 * (staged, barrier, reduced, row epilogue done), [8, 24) the MMA's full-barrier arrival of the
 * first tile's first 16 k-blocks and [24, 32) the producer's W issue of its first 8; NULL
 * turns it off. */
prism_status prism_debug_trace_chain(unsigned long long* buf_dev);

#ifdef __cplusplus
}
#endif
#endif /* PRISM_H_ */
