"""ctypes binding of libprism.so (include/prism.h).

Argument marshalling only: torch is used for device memory (outputs, workspace,
report buffers), streams and the current device; every step of the PRISM
iteration runs in the library's CUDA kernels.  If the library is missing the
calls raise — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import math
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libprism.so")

PRECISION = {"bf16": 0, "fp32": 1, "tf32": 2}
FIT = {"sketched": 0, "taylor": 1}
STATUS = {0: "converged", 1: "max_iters", 2: "diverged", 3: "nonfinite", 4: "zero_input"}


class PrismError(RuntimeError):
    pass


class Options(ctypes.Structure):
    _fields_ = [
        ("degree", ctypes.c_int),
        ("max_iters", ctypes.c_int),
        ("sketch_size", ctypes.c_int),
        ("tol", ctypes.c_double),
        ("seed", ctypes.c_uint64),
        ("precision", ctypes.c_int),
        ("fit", ctypes.c_int),
        ("warmup_iters", ctypes.c_int),
        ("alpha_lo", ctypes.c_double),
        ("alpha_hi", ctypes.c_double),
    ]


class Report(ctypes.Structure):
    _fields_ = [
        ("iters", ctypes.c_void_p),
        ("resid", ctypes.c_void_p),
        ("status", ctypes.c_void_p),
        ("alphas", ctypes.c_void_p),
        ("resid_hist", ctypes.c_void_p),
    ]


# prism_transport (include/prism.h): exchange callbacks of the multi-GPU entry points
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                ctypes.c_int, ctypes.c_void_p)
BROADCAST_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                ctypes.c_void_p)
GROUP_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p)


class Transport(ctypes.Structure):
    _fields_ = [
        ("ctx", ctypes.c_void_p),
        ("nranks", ctypes.c_int),
        ("rank", ctypes.c_int),
        ("allreduce_sum", ALLREDUCE_FN),
        ("broadcast", BROADCAST_FN),
        ("group_start", GROUP_FN),
        ("group_end", GROUP_FN),
        ("async_error", GROUP_FN),
    ]


DT = {"f32": 0, "f64": 1, "i32": 2, "bytes": 3}

# ---------------------------------------------------------------- signatures
_vp, _i32, _i64, _dbl, _u64, _sz = (ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double,
                                    ctypes.c_uint64, ctypes.c_size_t)
_i64p = ctypes.POINTER(ctypes.c_int64)
_vpp = ctypes.POINTER(ctypes.c_void_p)
_opt = ctypes.POINTER(Options)
_rep = ctypes.POINTER(Report)
_trp = ctypes.POINTER(Transport)
_i32p = ctypes.POINTER(ctypes.c_int32)
_ST = ctypes.c_int   # prism_status

# name -> (restype, argtypes); EXPORTS is exactly the symbol set include/prism.h declares
_SIGS = {
    "prism_default_options": (None, [_opt]),
    "prism_create": (_ST, [ctypes.POINTER(_vp)]),
    "prism_destroy": (_ST, [_vp]),
    "prism_last_error": (ctypes.c_char_p, []),
    "prism_abi_version": (_i32, []),
    # device-buffer solves and their workspace queries
    "prism_polar_workspace": (_sz, [_vp, _i32, _i64p, _i64p, _opt]),
    "prism_polar": (_ST, [_vp, _i32, _i64p, _i64p, _vpp, _i64p, _vpp, _i64p, _i64p, _opt, _rep, _vp, _sz, _vp]),
    "prism_sqrt_workspace": (_sz, [_vp, _i32, _i64p, _opt]),
    "prism_sqrt_invsqrt": (_ST, [_vp, _i32, _i64p, _vpp, _i64p, _vpp, _vpp, _i64p, _i64p, _opt, _rep, _vp, _sz,
                                 _vp]),
    "prism_sign_workspace": (_sz, [_vp, _i32, _i64p, _opt]),
    "prism_sign": (_ST, [_vp, _i32, _i64p, _vpp, _i64p, _vpp, _i64p, _i64p, _opt, _rep, _vp, _sz, _vp]),
    "prism_inv_root_workspace": (_sz, [_vp, _i32, _i64p, _i32, _opt]),
    "prism_inv_root": (_ST, [_vp, _i32, _i64p, _i32, _vpp, _i64p, _vpp, _i64p, _i64p, _opt, _rep, _vp, _sz, _vp]),
    "prism_chebyshev_inverse_workspace": (_sz, [_vp, _i32, _i64p, _opt]),
    "prism_chebyshev_inverse": (_ST, [_vp, _i32, _i64p, _vpp, _i64p, _vpp, _i64p, _i64p, _opt, _rep, _vp, _sz,
                                      _vp]),
    "prism_db_newton_workspace": (_sz, [_vp, _i32, _i64p, _opt]),
    "prism_db_newton": (_ST, [_vp, _i32, _i64p, _vpp, _i64p, _vpp, _vpp, _i64p, _i64p, _opt, _rep, _vp, _sz, _vp]),
    # host-buffer (end-to-end) forms
    "prism_polar_host": (_ST, [_vp, _i32, _i64p, _i64p, _vpp, _i64p, _vpp, _i64p, _i64p, _opt, _rep, _vp]),
    "prism_sqrt_invsqrt_host": (_ST, [_vp, _i32, _i64p, _vpp, _i64p, _vpp, _vpp, _i64p, _i64p, _opt, _rep, _vp]),
    "prism_sign_host": (_ST, [_vp, _i32, _i64p, _vpp, _i64p, _vpp, _i64p, _i64p, _opt, _rep, _vp]),
    "prism_inv_root_host": (_ST, [_vp, _i32, _i64p, _i32, _vpp, _i64p, _vpp, _i64p, _i64p, _opt, _rep, _vp]),
    "prism_chebyshev_inverse_host": (_ST, [_vp, _i32, _i64p, _vpp, _i64p, _vpp, _i64p, _i64p, _opt, _rep, _vp]),
    "prism_db_newton_host": (_ST, [_vp, _i32, _i64p, _vpp, _i64p, _vpp, _vpp, _i64p, _i64p, _opt, _rep, _vp]),
    # multi-GPU
    "prism_lpt_partition": (_ST, [_i32, ctypes.POINTER(_dbl), _i32, ctypes.POINTER(ctypes.c_int32)]),
    "prism_nccl_get_unique_id": (_ST, [_vp]),
    "prism_nccl_comm_init": (_ST, [ctypes.POINTER(_vp), _i32, _vp, _i32]),
    "prism_nccl_comm_destroy": (_ST, [_vp]),
    "prism_nccl_transport": (_ST, [_vp, _trp]),
    "prism_shard_plan": (_ST, [_i32, _i64p, _i64p, _i32, _i32, _i32, _i32, _i32p, _i32p]),
    "prism_polar_sharded_workspace": (_sz, [_vp, _i32, _i32, _i32, _i64p, _i64p, _opt, _i32]),
    "prism_polar_sharded": (_ST, [_vp, _vp, _i32, _i64p, _i64p, _vpp, _i64p, _vpp, _i64p, _opt, _i32, _rep, _vp, _sz,
                                  _vp]),
    "prism_polar_sharded_tr": (_ST, [_vp, _trp, _i32, _i64p, _i64p, _vpp, _i64p, _vpp, _i64p, _opt, _i32, _rep, _vp,
                                     _sz, _vp]),
    "prism_sqrt_invsqrt_sharded_workspace": (_sz, [_vp, _i32, _i32, _i32, _i64p, _opt, _i32]),
    "prism_sqrt_invsqrt_sharded": (_ST, [_vp, _vp, _i32, _i64p, _vpp, _i64p, _vpp, _vpp, _i64p, _opt, _i32, _rep, _vp,
                                         _sz, _vp]),
    "prism_sqrt_invsqrt_sharded_tr": (_ST, [_vp, _trp, _i32, _i64p, _vpp, _i64p, _vpp, _vpp, _i64p, _opt, _i32, _rep,
                                            _vp, _sz, _vp]),
    "prism_polar_rowblock_workspace": (_sz, [_vp, _i64, _i64, _opt]),
    "prism_polar_rowblock": (_ST, [_vp, _vp, _i64, _i64, _vp, _i64, _i64, _i64, _vp, _i64, _opt, _rep, _vp, _sz, _vp]),
    "prism_polar_rowblock_tr": (_ST, [_vp, _trp, _i64, _i64, _vp, _i64, _i64, _i64, _vp, _i64, _opt, _rep, _vp, _sz,
                                      _vp]),
    "prism_rowblock_layout": (_ST, [_i64, _i32, _i64p, _i32p]),
    # measurement
    "prism_polar_flops_per_iter": (_dbl, [_i64, _i64, _i32, _i32]),
    "prism_sqrt_flops_per_iter": (_dbl, [_i64, _i32, _i32]),
    "prism_launch_count": (_i64, [_vp]),
    "prism_profile_enable": (_ST, [_vp, _i32]),
    "prism_profile_read": (_ST, [_vp, ctypes.POINTER(_dbl), ctypes.POINTER(_i64), _i32]),
    # test hooks
    "prism_debug_gemm": (_ST, [_vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _i64, _vp, _vp, _i64, _vp,
                               _vp, _i64, _vp, _vp, _i64, _vp, ctypes.c_float, _i32, _vp, _vp, _vp, _sz, _vp]),
    "prism_debug_sketch": (_ST, [_u64, _i64, _i32, _i32, _i32, _vp, _vp]),
    "prism_debug_argmin": (_ST, [_i32, _vp, _dbl, _dbl, _dbl, _vp, _vp]),
    "prism_debug_trace_gemm": (_ST, [_vp, _i32]),
    "prism_debug_trace_chain": (_ST, [_vp]),
    "prism_debug_gemm_max_ctas": (_ST, [_i32]),
    "prism_debug_raster_rows": (_ST, [_i32]),
    "prism_debug_workspace_guards": (_ST, [_i32]),
    "prism_debug_guards_fill": (_ST, [_vp, _vp]),
    "prism_debug_guards_check": (_ST, [_vp, _i64p, _i64p, _vp]),
    "prism_debug_guards_poke": (_ST, [_vp, _i64, _vp]),
}
EXPORTS = sorted(_SIGS)

_lib = None
_lock = threading.Lock()


def lib():
    """Load libprism.so once and declare the C signatures."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise PrismError(f"{LIB_PATH} not built (run `python build.py`); no CPU fallback exists")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
        return L


def check(status: int, what: str):
    if status != 0:
        msg = lib().prism_last_error().decode(errors="replace")
        raise PrismError(f"{what} failed (status {status}): {msg}")


def _i64(vals):
    return (ctypes.c_int64 * len(vals))(*[int(v) for v in vals])


def _ptrs(ts):
    return (ctypes.c_void_p * len(ts))(*[(t.data_ptr() if t is not None else None) for t in ts])


class Handle:
    """A prism_handle plus reusable device workspaces, one per (device, stream): solves
    queued on different streams never share a workspace.  A handle is used by one host
    thread at a time (include/prism.h)."""

    KINDS = ("gram", "square", "apply", "sketch_chain", "alpha", "norm_final")

    def __init__(self):
        h = ctypes.c_void_p()
        check(lib().prism_create(ctypes.byref(h)), "prism_create")
        self.h = h
        self._ws = {}
        self._marshal = {}   # ctypes argument arrays per batch signature (binding._solve)

    def __del__(self):
        try:
            if self.h and _lib is not None:
                _lib.prism_destroy(self.h)
        except Exception:
            pass

    def launch_count(self) -> int:
        """Kernel launches issued by the last solve on this handle."""
        return int(lib().prism_launch_count(self.h))

    def profile(self, enable: bool):
        check(lib().prism_profile_enable(self.h, 1 if enable else 0), "prism_profile_enable")

    def profile_read(self, reset: bool = True) -> dict:
        ms = (ctypes.c_double * 6)()
        nl = (ctypes.c_int64 * 6)()
        check(lib().prism_profile_read(self.h, ms, nl, 1 if reset else 0), "prism_profile_read")
        return {k: {"ms": ms[i], "launches": nl[i]} for i, k in enumerate(self.KINDS)}

    def workspace(self, nbytes: int, device, stream=None):
        import torch
        key = (str(device), int(stream.cuda_stream) if stream is not None else 0)
        ws = self._ws.get(key)
        if ws is None or ws.numel() < nbytes:
            ws = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
            self._ws[key] = ws
        return ws


_default = None


def default_handle() -> Handle:
    global _default
    if _default is None:
        _default = Handle()
    return _default


def make_options(degree=5, max_iters=30, sketch_size=8, tol=1e-6, seed=42, precision="bf16", fit="sketched",
                 warmup_iters=0, alpha_lo=None, alpha_hi=None) -> Options:
    o = Options()
    lib().prism_default_options(ctypes.byref(o))
    o.degree = int(degree)
    o.max_iters = int(max_iters)
    o.sketch_size = int(sketch_size)
    o.tol = float(tol)
    o.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    o.precision = PRECISION[precision] if isinstance(precision, str) else int(precision)
    o.fit = FIT[fit] if isinstance(fit, str) else int(fit)
    o.warmup_iters = int(warmup_iters)
    o.alpha_lo = math.nan if alpha_lo is None else float(alpha_lo)
    o.alpha_hi = math.nan if alpha_hi is None else float(alpha_hi)
    return o


def _precision_of(t, precision):
    import torch
    if precision is not None:
        return precision
    return "bf16" if t.dtype == torch.bfloat16 else "fp32"


def _check_dtype(ts, precision, on_host=False):
    import torch
    want = torch.bfloat16 if precision == "bf16" else torch.float32
    where = "pinned host" if on_host else "CUDA"
    # set comprehensions: one attribute read per tensor and property (a per-tensor chain of
    # checks cost ~20 us on a 48-matrix batch)
    T = torch.Tensor
    if ({t.dtype for t in ts} != {want} or {t.is_cuda for t in ts} != {not on_host}
            or set(map(T.dim, ts)) != {2} or {st[1] for st in map(T.stride, ts)} != {1}):
        raise PrismError(f"inputs must be 2-D {where} {want} tensors with unit column stride")
    if on_host and not all(t.is_pinned() for t in ts):
        raise PrismError("host-path tensors must be pinned CPU tensors (tensor.pin_memory())")


def _report_buffers(batch, max_iters, device):
    """The report tensors of one call, views of one allocation (k_report writes every entry:
    NaN past a matrix's last iteration).  Fresh per call: a report may outlive the next call."""
    import torch
    M = max_iters
    a4 = (4 * batch + 255) // 256 * 256
    a8 = (8 * batch * M + 255) // 256 * 256
    buf = torch.empty(3 * a4 + a8 + 4 * batch * (M + 1), dtype=torch.uint8, device=device)
    return {
        "iters": buf[0:4 * batch].view(torch.int32),
        "resid": buf[a4:a4 + 4 * batch].view(torch.float32),
        "status": buf[2 * a4:2 * a4 + 4 * batch].view(torch.int32),
        "alphas": buf[3 * a4:3 * a4 + 8 * batch * M].view(torch.float64).view(batch, M),
        "resid_hist": buf[3 * a4 + a8:].view(torch.float32).view(batch, M + 1),
    }


def _report_struct(rb):
    r = Report()
    for k in ("iters", "resid", "status", "alphas", "resid_hist"):
        setattr(r, k, rb[k].data_ptr())
    return r


def _outputs(mats, want, given, what, host):
    """Output matrices: the caller's (same shape / dtype / device as the inputs, unit column
    stride) or fresh ones.  Reusing the same output buffers across calls keeps the handle's
    plan (keyed by every pointer it bakes into its tables) and its CUDA graph warm."""
    import torch
    if not want:
        return None
    if given is None:
        return [torch.empty_like(t).pin_memory() if host else torch.empty_like(t) for t in mats]
    given = list(given)
    if len(given) != len(mats):
        raise PrismError(f"{what}: {len(given)} outputs for {len(mats)} matrices")
    T = torch.Tensor
    if (list(map(T.size, given)) != list(map(T.size, mats)) or {g.dtype for g in given} != {mats[0].dtype}
            or set(map(T.get_device, given)) != {mats[0].get_device()}
            or {st[1] for st in map(T.stride, given)} != {1}):
        raise PrismError(f"{what}: each output must match its input's shape, dtype and device, rows contiguous")
    if host and not all(g.is_pinned() for g in given):
        raise PrismError(f"{what}: host-path outputs must be pinned")
    return given


def _ld_out(o1, o2, mats, what):
    a = o1 if o1 is not None else o2
    if a is None:
        return _i64([t.shape[1] for t in mats])
    if o1 is not None and o2 is not None and any(x.stride(0) != y.stride(0) for x, y in zip(o1, o2)):
        raise PrismError(f"{what}: the two outputs of a matrix must share one row stride")
    return _i64([t.stride(0) for t in a])


# kind -> (C entry point, workspace query, shape args: "mn" (m, n arrays), "n" or "nq")
_KINDS = {
    "polar": ("prism_polar", "prism_polar_workspace", "mn", 1),
    "sign": ("prism_sign", "prism_sign_workspace", "n", 1),
    "inv_root": ("prism_inv_root", "prism_inv_root_workspace", "nq", 1),
    "chebyshev": ("prism_chebyshev_inverse", "prism_chebyshev_inverse_workspace", "n", 1),
    "sqrt": ("prism_sqrt_invsqrt", "prism_sqrt_workspace", "n", 2),
    "db_newton": ("prism_db_newton", "prism_db_newton_workspace", "n", 2),
}


def _solve(kind, mats, *, host=False, q=0, degree=5, max_iters=30, sketch_size=8, tol=1e-6, seed=42,
           precision=None, fit="sketched", warmup_iters=0, alpha_lo=None, alpha_hi=None, out=None, out2=None,
           want1=True, want2=True, matrix_ids=None, stream=None, handle=None, device=None):
    """One library call: marshal the batch, outputs, options, report and workspace, call the
    C entry point of `kind` on the right device and stream, return (out, out2, report)."""
    import torch
    fn, fn_ws, shape, nout = _KINDS[kind]
    mats = list(mats)
    if not mats:
        return [], ([] if nout == 2 else None), {}
    precision = _precision_of(mats[0], precision)
    _check_dtype(mats, precision, on_host=host)
    if shape != "mn" and any(t.shape[0] != t.shape[1] for t in mats):
        raise PrismError(f"{kind}: matrices must be square")
    if host:
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    else:
        dev = mats[0].device
        if any(t.device != dev for t in mats):
            raise PrismError(f"{kind}: all matrices must be on one device")
    h = handle or default_handle()
    o = make_options(degree, max_iters, sketch_size, tol, seed, precision, fit, warmup_iters, alpha_lo, alpha_hi)
    B = len(mats)
    o1 = _outputs(mats, want1, out, kind, host)
    o2 = _outputs(mats, want2, out2, kind, host) if nout == 2 else None
    # the ctypes argument arrays of this batch (sizes, pointers, leading dimensions, ids),
    # cached on the handle by everything they encode: building them for a 48-matrix batch
    # cost ~100 us per call, more than the whole host side of the library call
    T = torch.Tensor
    key = (kind, tuple(map(T.data_ptr, mats)), tuple(map(T.size, mats)), tuple(map(T.stride, mats)),
           tuple(map(T.data_ptr, o1)) if o1 else None, tuple(map(T.stride, o1)) if o1 else None,
           tuple(map(T.data_ptr, o2)) if o2 else None, tuple(map(T.stride, o2)) if o2 else None,
           tuple(matrix_ids) if matrix_ids is not None else None)
    arrs = h._marshal.get(key)
    if arrs is None:
        m = _i64([t.shape[0] for t in mats])
        n = _i64([t.shape[1] for t in mats])
        ids = _i64(matrix_ids) if matrix_ids is not None else None
        base = [m] + ([n] if shape == "mn" else [])
        io = [_ptrs(mats), _i64([t.stride(0) for t in mats])]
        if nout == 1:
            io += [_ptrs(o1), _i64([t.stride(0) for t in o1])]
        else:
            io += [_ptrs(o1) if o1 else None, _ptrs(o2) if o2 else None, _ld_out(o1, o2, mats, kind)]
        arrs = (base, io, ids)
        if len(h._marshal) > 64:
            h._marshal.clear()
        h._marshal[key] = arrs
    base, io, ids = arrs
    m = base[0]
    n = base[1] if shape == "mn" else None
    L = lib()
    with torch.cuda.device(dev):
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        rb = _report_buffers(B, max_iters, dev)
        rep = _report_struct(rb)
        args = [h.h, B] + base + ([int(q)] if shape == "nq" else [])
        args += io
        args += [ids, ctypes.byref(o), ctypes.byref(rep)]
        if host:
            check(getattr(L, fn + "_host")(*args, ctypes.c_void_p(st.cuda_stream)), fn + "_host")
        else:
            wargs = [h.h, B, m] + ([n] if shape == "mn" else []) + ([int(q)] if shape == "nq" else [])
            need = getattr(L, fn_ws)(*wargs, ctypes.byref(o))
            if need == 0:
                raise PrismError(f"{fn_ws} rejected the arguments: " + L.prism_last_error().decode())
            ws = h.workspace(need, dev, st)
            check(getattr(L, fn)(*args, ws.data_ptr(), ws.numel(), ctypes.c_void_p(st.cuda_stream)), fn)
    return o1, o2, rb


# ---------------------------------------------------------------- public API
# Device forms take CUDA tensors and return device outputs plus a device report (iters,
# resid, status, alphas [batch, max_iters], resid_hist [batch, max_iters + 1]); they are
# asynchronous on `stream` (default: the current stream of the inputs' device).  Host forms
# (*_host) take pinned CPU tensors and run the library's pipelined upload / solve / download
# path (prism_*_host); their outputs are valid once `stream` reaches the call.

def polar(mats, out=None, **kw):
    """Polar factors U V^T via prism_polar -> (outputs, report)."""
    o1, _, rb = _solve("polar", mats, out=out, **kw)
    return o1, rb


def polar_host(mats, out=None, **kw):
    o1, _, rb = _solve("polar", mats, host=True, out=out, **kw)
    return o1, rb


def sign(mats, out=None, **kw):
    """Matrix signs of square matrices via prism_sign -> (outputs, report)."""
    o1, _, rb = _solve("sign", mats, out=out, **kw)
    return o1, rb


def sign_host(mats, out=None, **kw):
    o1, _, rb = _solve("sign", mats, host=True, out=out, **kw)
    return o1, rb


def inv_root(mats, q=4, out=None, **kw):
    """A^{-1/q} of SPD matrices by the coupled inverse Newton iteration."""
    kw.pop("degree", None)
    o1, _, rb = _solve("inv_root", mats, q=q, out=out, **kw)
    return o1, rb


def inv_root_host(mats, q=4, out=None, **kw):
    kw.pop("degree", None)
    o1, _, rb = _solve("inv_root", mats, host=True, q=q, out=out, **kw)
    return o1, rb


def chebyshev_inverse(mats, max_iters=40, out=None, **kw):
    """A^{-1} of square matrices by the Chebyshev iteration."""
    kw.pop("degree", None)
    o1, _, rb = _solve("chebyshev", mats, max_iters=max_iters, out=out, **kw)
    return o1, rb


def chebyshev_inverse_host(mats, max_iters=40, out=None, **kw):
    kw.pop("degree", None)
    o1, _, rb = _solve("chebyshev", mats, host=True, max_iters=max_iters, out=out, **kw)
    return o1, rb


def sqrt_invsqrt(mats, want_sqrt=True, want_invsqrt=True, out_sqrt=None, out_invsqrt=None, **kw):
    """A^{1/2}, A^{-1/2} of SPD matrices (Theorem 3) -> (sqrt, invsqrt, report)."""
    return _solve("sqrt", mats, want1=want_sqrt, want2=want_invsqrt, out=out_sqrt, out2=out_invsqrt, **kw)


def sqrt_invsqrt_host(mats, want_sqrt=True, want_invsqrt=True, out_sqrt=None, out_invsqrt=None, **kw):
    return _solve("sqrt", mats, host=True, want1=want_sqrt, want2=want_invsqrt, out=out_sqrt, out2=out_invsqrt,
                  **kw)


def db_newton(mats, want_sqrt=True, want_invsqrt=True, out_sqrt=None, out_invsqrt=None, precision="fp32", **kw):
    """A^{1/2}, A^{-1/2} by PRISM DB Newton, product form, FP32 only."""
    kw.pop("sketch_size", None)
    return _solve("db_newton", mats, want1=want_sqrt, want2=want_invsqrt, out=out_sqrt, out2=out_invsqrt,
                  precision=precision, **kw)


def db_newton_host(mats, want_sqrt=True, want_invsqrt=True, out_sqrt=None, out_invsqrt=None, precision="fp32",
                   **kw):
    kw.pop("sketch_size", None)
    return _solve("db_newton", mats, host=True, want1=want_sqrt, want2=want_invsqrt, out=out_sqrt,
                  out2=out_invsqrt, precision=precision, **kw)


def lpt_partition(costs, ranks: int):
    """Deterministic LPT assignment (prism_lpt_partition): owner rank per matrix."""
    B = len(costs)
    c = (ctypes.c_double * B)(*[float(x) for x in costs])
    own = (ctypes.c_int32 * B)()
    check(lib().prism_lpt_partition(B, c, int(ranks), own), "prism_lpt_partition")
    return list(own)


def polar_flops_per_iter(m, n, degree=5, sketch_size=8) -> float:
    return float(lib().prism_polar_flops_per_iter(int(m), int(n), int(degree), int(sketch_size)))


def sqrt_flops_per_iter(n, degree=5, sketch_size=8) -> float:
    return float(lib().prism_sqrt_flops_per_iter(int(n), int(degree), int(sketch_size)))

