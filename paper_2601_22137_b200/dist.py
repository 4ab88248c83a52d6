"""Multi-GPU PRISM: marshalling of the library's multi-GPU C ABI.

One process per GPU.  Every exchange happens inside libprism through a prism_transport:

* ``Comm``          an NCCL communicator created by the library (prism_nccl_comm_init;
                    NCCL resolved at run time from the libnccl the process loaded, i.e.
                    torch's) over the ranks of a torch.distributed group — the unique id
                    travels through torch.distributed, the collectives through NCCL.
* ``polar_sharded`` a Muon/Shampoo step's batch, LPT-sharded by matrix over the ranks
                    (prism_polar_sharded): every rank passes the full batch, solves its
                    share in buckets with global sketch ids (bit-identical to the
                    single-GPU solve), and the owners broadcast each bucket's outputs while
                    the next bucket solves; every rank returns every output.
* ``sqrt_invsqrt_sharded`` the same for Shampoo's A^{1/2}, A^{-1/2} batch
                    (prism_sqrt_invsqrt_sharded).
* ``polar_rowblock`` one matrix too large for one GPU, split by rows
                    (prism_polar_rowblock): per iteration a packed upper-triangle fp32
                    Gram all-reduce pipelined by panel group, then Y_r = X_r R and
                    X_r + Y_r/2 + a Y_r R locally (no R^2, no second collective).
* ``HostGroup`` / ``HostTransport``  a transport whose collectives run on the host
                    (stream synchronised, device <-> host copies, a fixed-order sum):
                    lets a test run several ranks as threads on one GPU through the real
                    library code, with no kernel ever waiting on another rank's kernel.
"""

from __future__ import annotations

import ctypes
import threading
from typing import List, Sequence

from . import binding as B

_cudart = None


def _rt():
    """cudart of the process (torch's), for the host transport's copies."""
    global _cudart
    if _cudart is None:
        import os
        import torch  # noqa: F401  (loads cudart)
        for name in ("libcudart.so.12", "libcudart.so.13", "libcudart.so"):
            try:
                _cudart = ctypes.CDLL(name, mode=getattr(os, "RTLD_NOLOAD", 0) | os.RTLD_NOW)
                break
            except OSError:
                continue
        if _cudart is None:
            raise B.PrismError("cudart not loaded")
        _cudart.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
        _cudart.cudaStreamSynchronize.argtypes = [ctypes.c_void_p]
    return _cudart


# ---------------------------------------------------------------- transports
class Comm:
    """NCCL communicator (ncclComm_t) over the ranks of a torch.distributed group, created
    by prism_nccl_comm_init on the current CUDA device; `transport` is its prism_transport."""

    def __init__(self, group=None):
        import torch.distributed as dist
        single = not (dist.is_available() and dist.is_initialized())
        self.rank = 0 if single else dist.get_rank(group)
        self.world = 1 if single else dist.get_world_size(group)
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            B.check(B.lib().prism_nccl_get_unique_id(uid), "prism_nccl_get_unique_id")
        if not single:   # rank 0's id to every rank of the group
            obj = [uid.raw if self.rank == 0 else None]
            src = dist.get_global_rank(group, 0) if group is not None else 0
            dist.broadcast_object_list(obj, src=src, group=group)
            uid = ctypes.create_string_buffer(obj[0], 128)
        self.comm = ctypes.c_void_p()
        B.check(B.lib().prism_nccl_comm_init(ctypes.byref(self.comm), self.world, uid, self.rank),
                "prism_nccl_comm_init")
        self.transport = B.Transport()
        B.check(B.lib().prism_nccl_transport(self.comm, ctypes.byref(self.transport)), "prism_nccl_transport")

    def close(self):
        if self.comm:
            B.check(B.lib().prism_nccl_comm_destroy(self.comm), "prism_nccl_comm_destroy")
            self.comm = ctypes.c_void_p()


class HostGroup:
    """Shared state of `world` thread-ranks exchanging through the host."""

    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world


class HostTransport:
    """prism_transport whose collectives synchronise the stream, copy the buffer to the host,
    exchange through a HostGroup (sum in rank order: identical bits on every rank) and copy
    back.  Test infrastructure for emulating ranks on one GPU."""

    _NP = {0: "float32", 1: "float64", 2: "int32", 3: "uint8"}

    def __init__(self, group: HostGroup, rank: int):
        self.g = group
        self.rank = rank
        self.calls = {"allreduce": 0, "broadcast": 0}
        self._ar = B.ALLREDUCE_FN(self._allreduce)
        self._bc = B.BROADCAST_FN(self._broadcast)
        self._none = B.GROUP_FN(lambda ctx: 0)
        self.transport = B.Transport(None, group.world, rank, self._ar, self._bc, self._none, self._none, self._none)

    def _fetch(self, ptr, nbytes, dtype, stream):
        import numpy as np
        rt = _rt()
        rt.cudaStreamSynchronize(ctypes.c_void_p(stream))
        a = np.empty(nbytes // np.dtype(dtype).itemsize, dtype=dtype)
        rt.cudaMemcpy(a.ctypes.data, ctypes.c_void_p(ptr), nbytes, 4)
        return a

    def _allreduce(self, ctx, send, recv, count, dtype, stream):
        try:
            import numpy as np
            dt = np.dtype(self._NP[dtype])
            self.calls["allreduce"] += 1
            self.g.slots[self.rank] = self._fetch(send, count * dt.itemsize, dt, stream)
            self.g.barrier.wait()
            tot = self.g.slots[0].copy()
            for r in range(1, self.g.world):
                tot += self.g.slots[r]
            self.g.barrier.wait()
            _rt().cudaMemcpy(ctypes.c_void_p(recv), tot.ctypes.data, count * dt.itemsize, 4)
            return 0
        except Exception:   # pragma: no cover - surfaced as PRISM_ERR_NCCL
            return 1

    def _broadcast(self, ctx, buf, nbytes, root, stream):
        try:
            self.calls["broadcast"] += 1
            if self.rank == root:
                self.g.slots[root] = self._fetch(buf, nbytes, "uint8", stream)
            else:
                _rt().cudaStreamSynchronize(ctypes.c_void_p(stream))
            self.g.barrier.wait()
            if self.rank != root:
                src = self.g.slots[root]
                _rt().cudaMemcpy(ctypes.c_void_p(buf), src.ctypes.data, nbytes, 4)
            self.g.barrier.wait()
            return 0
        except Exception:   # pragma: no cover
            return 1


def _transport_of(t):
    return t.transport if hasattr(t, "transport") else t


# ---------------------------------------------------------------- plans (host only)
def shard_plan(shapes: Sequence[tuple], nranks: int, nbuckets: int = 2, degree: int = 5, sketch_size: int = 8):
    """(owner, bucket) per matrix (prism_shard_plan; deterministic, identical on every rank)."""
    n = len(shapes)
    own = (ctypes.c_int32 * n)()
    bk = (ctypes.c_int32 * n)()
    B.check(B.lib().prism_shard_plan(n, B._i64([s[0] for s in shapes]), B._i64([s[1] for s in shapes]), degree,
                                     sketch_size, nranks, nbuckets, own, bk), "prism_shard_plan")
    return list(own), list(bk)


def lpt_plan(shapes: Sequence[tuple], world: int, degree: int = 5, iters_est: Sequence[int] | None = None) -> List[int]:
    """Owner rank of each matrix by LPT on F_min x expected iterations (prism_lpt_partition)."""
    costs = []
    for i, (m, n) in enumerate(shapes):
        f = B.polar_flops_per_iter(m, n, degree, 8)
        costs.append(f * (iters_est[i] if iters_est is not None else 1))
    return B.lpt_partition(costs, world)


def rowblock_layout(n: int, ngroups: int):
    """(panel_off, group_end) of the packed row-block Gram (prism_rowblock_layout)."""
    T = (n + 255) // 256
    off = (ctypes.c_int64 * (T + 1))()
    ge = (ctypes.c_int32 * ngroups)()
    B.check(B.lib().prism_rowblock_layout(n, ngroups, off, ge), "prism_rowblock_layout")
    return list(off), list(ge)


# ---------------------------------------------------------------- solves
def polar_sharded(mats, comm, out=None, nbuckets: int = 2, report: bool = True, handle=None, stream=None,
                  degree=5, max_iters=30, sketch_size=8, tol=1e-6, seed=42, precision=None, fit="sketched",
                  warmup_iters=0, alpha_lo=None, alpha_hi=None):
    """Polar factors of the whole batch on every rank (prism_polar_sharded_tr); `mats` is the
    full batch, identical on every rank.  Returns (outputs, report of every matrix)."""
    import torch
    mats = list(mats)
    tr = _transport_of(comm)
    precision = B._precision_of(mats[0], precision)
    B._check_dtype(mats, precision)
    dev = mats[0].device
    h = handle or B.default_handle()
    o = B.make_options(degree, max_iters, sketch_size, tol, seed, precision, fit, warmup_iters, alpha_lo, alpha_hi)
    n_ = len(mats)
    m = B._i64([t.shape[0] for t in mats])
    n = B._i64([t.shape[1] for t in mats])
    out = B._outputs(mats, True, out, "polar_sharded", False)
    L = B.lib()
    with torch.cuda.device(dev):
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        need = L.prism_polar_sharded_workspace(h.h, tr.nranks, tr.rank, n_, m, n, ctypes.byref(o), nbuckets)
        if need == 0:
            raise B.PrismError("prism_polar_sharded_workspace rejected the arguments: " + L.prism_last_error().decode())
        ws = h.workspace(need, dev, st)
        rb = B._report_buffers(n_, max_iters, dev) if report else None
        rep = B._report_struct(rb) if report else None
        B.check(L.prism_polar_sharded_tr(h.h, ctypes.byref(tr), n_, m, n, B._ptrs(mats),
                                         B._i64([t.stride(0) for t in mats]), B._ptrs(out),
                                         B._i64([t.stride(0) for t in out]), ctypes.byref(o), int(nbuckets),
                                         ctypes.byref(rep) if report else None, ws.data_ptr(), ws.numel(),
                                         ctypes.c_void_p(st.cuda_stream)), "prism_polar_sharded")
    return out, rb


def sqrt_invsqrt_sharded(mats, comm, want_sqrt=True, want_invsqrt=True, out_sqrt=None, out_invsqrt=None,
                         nbuckets: int = 2, report: bool = True, handle=None, stream=None, degree=5, max_iters=30,
                         sketch_size=8, tol=1e-6, seed=42, precision=None, fit="sketched", warmup_iters=0,
                         alpha_lo=None, alpha_hi=None):
    """A^{1/2}, A^{-1/2} of the whole SPD batch on every rank (prism_sqrt_invsqrt_sharded_tr):
    the Shampoo-preconditioner form of polar_sharded.  Returns (sqrt, invsqrt, report)."""
    import torch
    mats = list(mats)
    if any(t.shape[0] != t.shape[1] for t in mats):
        raise B.PrismError("sqrt_invsqrt_sharded: matrices must be square")
    tr = _transport_of(comm)
    precision = B._precision_of(mats[0], precision)
    B._check_dtype(mats, precision)
    dev = mats[0].device
    h = handle or B.default_handle()
    o = B.make_options(degree, max_iters, sketch_size, tol, seed, precision, fit, warmup_iters, alpha_lo, alpha_hi)
    n_ = len(mats)
    n = B._i64([t.shape[1] for t in mats])
    o1 = B._outputs(mats, want_sqrt, out_sqrt, "sqrt_invsqrt_sharded", False)
    o2 = B._outputs(mats, want_invsqrt, out_invsqrt, "sqrt_invsqrt_sharded", False)
    L = B.lib()
    with torch.cuda.device(dev):
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        need = L.prism_sqrt_invsqrt_sharded_workspace(h.h, tr.nranks, tr.rank, n_, n, ctypes.byref(o), nbuckets)
        if need == 0:
            raise B.PrismError("prism_sqrt_invsqrt_sharded_workspace rejected the arguments: " +
                               L.prism_last_error().decode())
        ws = h.workspace(need, dev, st)
        rb = B._report_buffers(n_, max_iters, dev) if report else None
        rep = B._report_struct(rb) if report else None
        B.check(L.prism_sqrt_invsqrt_sharded_tr(h.h, ctypes.byref(tr), n_, n, B._ptrs(mats),
                                                B._i64([t.stride(0) for t in mats]),
                                                B._ptrs(o1) if o1 else None, B._ptrs(o2) if o2 else None,
                                                B._ld_out(o1, o2, mats, "sqrt_invsqrt_sharded"), ctypes.byref(o),
                                                int(nbuckets), ctypes.byref(rep) if report else None, ws.data_ptr(),
                                                ws.numel(), ctypes.c_void_p(st.cuda_stream)),
                "prism_sqrt_invsqrt_sharded")
    return o1, o2, rb


def polar_rowblock(A_rows, comm, m_global: int, row0: int, out=None, handle=None, stream=None, degree=5,
                   max_iters=30, sketch_size=8, tol=1e-6, seed=42, precision=None, fit="sketched", warmup_iters=0,
                   alpha_lo=None, alpha_hi=None):
    """Rows [row0, row0 + rows) of the polar factor of the m_global x n matrix whose row block
    A_rows this rank holds (prism_polar_rowblock_tr).  Returns (Q_rows, report).  The call
    returns once the iteration count is decided (the host follows the device's stop flag)."""
    import torch
    tr = _transport_of(comm)
    precision = B._precision_of(A_rows, precision)
    B._check_dtype([A_rows], precision)
    dev = A_rows.device
    h = handle or B.Handle()
    o = B.make_options(degree, max_iters, sketch_size, tol, seed, precision, fit, warmup_iters, alpha_lo, alpha_hi)
    rows, n = A_rows.shape
    Q = B._outputs([A_rows], True, [out] if out is not None else None, "polar_rowblock", False)[0]
    L = B.lib()
    with torch.cuda.device(dev):
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        need = L.prism_polar_rowblock_workspace(h.h, rows, n, ctypes.byref(o))
        if need == 0:
            raise B.PrismError("prism_polar_rowblock_workspace rejected the arguments: " +
                               L.prism_last_error().decode())
        ws = h.workspace(need, dev, st)
        rb = B._report_buffers(1, max_iters, dev)
        rep = B._report_struct(rb)
        B.check(L.prism_polar_rowblock_tr(h.h, ctypes.byref(tr), int(m_global), n, A_rows.data_ptr(), int(row0), rows,
                                          A_rows.stride(0), Q.data_ptr(), Q.stride(0), ctypes.byref(o),
                                          ctypes.byref(rep), ws.data_ptr(), ws.numel(),
                                          ctypes.c_void_p(st.cuda_stream)), "prism_polar_rowblock")
    return Q, rb
