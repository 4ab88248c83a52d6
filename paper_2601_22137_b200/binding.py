"""ctypes binding of libprism.so (include/prism.h).

Argument marshalling only: torch is used for device memory (outputs,
workspace, report buffers) and streams; every step of the PRISM iteration
runs in the library's CUDA kernels.  If the library is missing the calls
raise — there is no CPU fallback.
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

c_i64p = ctypes.POINTER(ctypes.c_int64)


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


EXPORTS = [
    "prism_default_options", "prism_create", "prism_destroy", "prism_last_error", "prism_abi_version",
    "prism_polar_workspace", "prism_polar", "prism_sqrt_workspace", "prism_sqrt_invsqrt",
    "prism_polar_host", "prism_sqrt_invsqrt_host", "prism_sign_workspace", "prism_sign", "prism_sign_host",
    "prism_inv_root_workspace", "prism_inv_root", "prism_inv_root_host",
                     "prism_chebyshev_inverse", "prism_chebyshev_inverse_host", "prism_db_newton",
                     "prism_db_newton_host",
    "prism_chebyshev_inverse_workspace", "prism_chebyshev_inverse", "prism_chebyshev_inverse_host",
    "prism_db_newton_workspace", "prism_db_newton", "prism_db_newton_host",
    "prism_lpt_partition", "prism_polar_flops_per_iter", "prism_sqrt_flops_per_iter",
    "prism_launch_count", "prism_profile_enable", "prism_profile_read",
    "prism_rowblock_workspace", "prism_rowblock_begin", "prism_rowblock_gram", "prism_rowblock_update",
    "prism_rowblock_end",
    "prism_debug_gemm", "prism_debug_sketch", "prism_debug_argmin",
    "prism_debug_trace_gemm", "prism_debug_trace_chain",
]

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
        vp, i32, i64, dbl, u64, sz = (ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double,
                                      ctypes.c_uint64, ctypes.c_size_t)
        L.prism_default_options.argtypes = [ctypes.POINTER(Options)]
        L.prism_default_options.restype = None
        L.prism_create.argtypes = [ctypes.POINTER(vp)]
        L.prism_destroy.argtypes = [vp]
        L.prism_last_error.restype = ctypes.c_char_p
        L.prism_abi_version.restype = i32
        L.prism_polar_workspace.argtypes = [vp, i32, c_i64p, c_i64p, ctypes.POINTER(Options)]
        L.prism_polar_workspace.restype = sz
        L.prism_polar.argtypes = [vp, i32, c_i64p, c_i64p, ctypes.POINTER(vp), c_i64p, ctypes.POINTER(vp), c_i64p,
                                  c_i64p, ctypes.POINTER(Options), ctypes.POINTER(Report), vp, sz, vp]
        L.prism_polar_host.argtypes = [vp, i32, c_i64p, c_i64p, ctypes.POINTER(vp), c_i64p, ctypes.POINTER(vp),
                                       c_i64p, c_i64p, ctypes.POINTER(Options), ctypes.POINTER(Report), vp]
        L.prism_sqrt_invsqrt_host.argtypes = [vp, i32, c_i64p, ctypes.POINTER(vp), c_i64p, ctypes.POINTER(vp),
                                              ctypes.POINTER(vp), c_i64p, c_i64p, ctypes.POINTER(Options),
                                              ctypes.POINTER(Report), vp]
        L.prism_sqrt_workspace.argtypes = [vp, i32, c_i64p, ctypes.POINTER(Options)]
        L.prism_sqrt_workspace.restype = sz
        L.prism_sqrt_invsqrt.argtypes = [vp, i32, c_i64p, ctypes.POINTER(vp), c_i64p, ctypes.POINTER(vp),
                                         ctypes.POINTER(vp), c_i64p, c_i64p, ctypes.POINTER(Options),
                                         ctypes.POINTER(Report), vp, sz, vp]
        L.prism_sign_workspace.argtypes = [vp, i32, c_i64p, ctypes.POINTER(Options)]
        L.prism_sign_workspace.restype = sz
        L.prism_sign.argtypes = [vp, i32, c_i64p, ctypes.POINTER(vp), c_i64p, ctypes.POINTER(vp), c_i64p, c_i64p,
                                 ctypes.POINTER(Options), ctypes.POINTER(Report), vp, sz, vp]
        L.prism_sign_host.argtypes = [vp, i32, c_i64p, ctypes.POINTER(vp), c_i64p, ctypes.POINTER(vp), c_i64p,
                                      c_i64p, ctypes.POINTER(Options), ctypes.POINTER(Report), vp]
        L.prism_inv_root_workspace.argtypes = [vp, i32, c_i64p, i32, ctypes.POINTER(Options)]
        L.prism_inv_root_workspace.restype = sz
        L.prism_inv_root.argtypes = [vp, i32, c_i64p, i32, ctypes.POINTER(vp), c_i64p, ctypes.POINTER(vp), c_i64p,
                                     c_i64p, ctypes.POINTER(Options), ctypes.POINTER(Report), vp, sz, vp]
        L.prism_inv_root_host.argtypes = [vp, i32, c_i64p, i32, ctypes.POINTER(vp), c_i64p, ctypes.POINTER(vp),
                                          c_i64p, c_i64p, ctypes.POINTER(Options), ctypes.POINTER(Report), vp]
        L.prism_chebyshev_inverse_workspace.argtypes = [vp, i32, c_i64p, ctypes.POINTER(Options)]
        L.prism_chebyshev_inverse_workspace.restype = sz
        L.prism_chebyshev_inverse.argtypes = [vp, i32, c_i64p, ctypes.POINTER(vp), c_i64p, ctypes.POINTER(vp), c_i64p,
                                              c_i64p, ctypes.POINTER(Options), ctypes.POINTER(Report), vp, sz, vp]
        L.prism_chebyshev_inverse_host.argtypes = [vp, i32, c_i64p, ctypes.POINTER(vp), c_i64p, ctypes.POINTER(vp),
                                                   c_i64p, c_i64p, ctypes.POINTER(Options), ctypes.POINTER(Report),
                                                   vp]
        L.prism_db_newton_workspace.argtypes = [vp, i32, c_i64p, ctypes.POINTER(Options)]
        L.prism_db_newton_workspace.restype = sz
        L.prism_db_newton.argtypes = [vp, i32, c_i64p, ctypes.POINTER(vp), c_i64p, ctypes.POINTER(vp),
                                      ctypes.POINTER(vp), c_i64p, c_i64p, ctypes.POINTER(Options),
                                      ctypes.POINTER(Report), vp, sz, vp]
        L.prism_db_newton_host.argtypes = [vp, i32, c_i64p, ctypes.POINTER(vp), c_i64p, ctypes.POINTER(vp),
                                           ctypes.POINTER(vp), c_i64p, c_i64p, ctypes.POINTER(Options),
                                           ctypes.POINTER(Report), vp]
        L.prism_lpt_partition.argtypes = [i32, ctypes.POINTER(dbl), i32, ctypes.POINTER(ctypes.c_int32)]
        L.prism_polar_flops_per_iter.argtypes = [i64, i64, i32, i32]
        L.prism_polar_flops_per_iter.restype = dbl
        L.prism_sqrt_flops_per_iter.argtypes = [i64, i32, i32]
        L.prism_sqrt_flops_per_iter.restype = dbl
        L.prism_debug_gemm.argtypes = [vp, i32, i32, i32, i32, i32, i32, i32, vp, vp, i64, vp, vp, i64, vp, vp, i64,
                                       vp, vp, i64, vp, ctypes.c_float, i32, vp, vp, vp, sz, vp]
        L.prism_launch_count.argtypes = [vp]
        L.prism_launch_count.restype = i64
        L.prism_profile_enable.argtypes = [vp, i32]
        L.prism_profile_read.argtypes = [vp, ctypes.POINTER(dbl), ctypes.POINTER(i64), i32]
        L.prism_rowblock_workspace.argtypes = [vp, i64, i64, ctypes.POINTER(Options)]
        L.prism_rowblock_workspace.restype = sz
        L.prism_rowblock_begin.argtypes = [vp, i64, i64, vp, i64, vp, i64, vp, vp, ctypes.POINTER(Options), vp, sz, vp]
        L.prism_rowblock_gram.argtypes = [vp, i32, vp, vp]
        L.prism_rowblock_update.argtypes = [vp, i32, vp, vp, vp]
        L.prism_rowblock_end.argtypes = [vp, ctypes.POINTER(Report), vp]
        L.prism_debug_sketch.argtypes = [u64, i64, i32, i32, i32, vp, vp]
        L.prism_debug_argmin.argtypes = [i32, vp, dbl, dbl, dbl, vp, vp]
        L.prism_debug_trace_gemm.argtypes = [vp, i32]
        L.prism_debug_trace_chain.argtypes = [vp]
        for name in ("prism_create", "prism_destroy", "prism_polar", "prism_sqrt_invsqrt", "prism_lpt_partition",
                     "prism_polar_host", "prism_sqrt_invsqrt_host", "prism_sign", "prism_sign_host", "prism_inv_root", "prism_inv_root_host",
                     "prism_debug_gemm", "prism_debug_sketch", "prism_debug_argmin",
                     "prism_debug_trace_gemm", "prism_debug_trace_chain", "prism_profile_enable", "prism_profile_read", "prism_rowblock_begin",
                     "prism_rowblock_gram", "prism_rowblock_update", "prism_rowblock_end"):
            getattr(L, name).restype = i32
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
    """A prism_handle plus a reusable device workspace (per device)."""

    def __init__(self):
        h = ctypes.c_void_p()
        check(lib().prism_create(ctypes.byref(h)), "prism_create")
        self.h = h
        self._ws = {}

    def __del__(self):
        try:
            if self.h and _lib is not None:
                _lib.prism_destroy(self.h)
        except Exception:
            pass

    KINDS = ("gram", "square", "apply", "sketch_chain", "alpha", "norm_final")

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

    def workspace(self, nbytes: int, device):
        import torch
        key = str(device)
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
    for t in ts:
        if t.dtype != want or t.is_cuda == on_host or t.dim() != 2 or t.stride(1) != 1:
            raise PrismError(f"inputs must be 2-D {where} {want} tensors with unit column stride")


def _report_buffers(batch, max_iters, device):
    import torch
    return {
        "iters": torch.zeros(batch, dtype=torch.int32, device=device),
        "resid": torch.zeros(batch, dtype=torch.float32, device=device),
        "status": torch.full((batch,), -1, dtype=torch.int32, device=device),
        "alphas": torch.full((batch, max_iters), float("nan"), dtype=torch.float64, device=device),
        "resid_hist": torch.full((batch, max_iters + 1), float("nan"), dtype=torch.float32, device=device),
    }


def _report_struct(rb):
    r = Report()
    r.iters = rb["iters"].data_ptr()
    r.resid = rb["resid"].data_ptr()
    r.status = rb["status"].data_ptr()
    r.alphas = rb["alphas"].data_ptr()
    r.resid_hist = rb["resid_hist"].data_ptr()
    return r


def polar(mats, degree=5, max_iters=30, sketch_size=8, tol=1e-6, seed=42, precision=None, fit="sketched",
          warmup_iters=0, alpha_lo=None, alpha_hi=None, out=None, matrix_ids=None, stream=None, handle=None):
    """Polar factors of a batch of CUDA matrices via prism_polar.

    Returns (outputs, report) where report holds device tensors iters, resid,
    status, alphas [batch, max_iters], resid_hist [batch, max_iters+1].
    Asynchronous on `stream` (default: torch's current stream).
    """
    import torch
    mats = list(mats)
    if not mats:
        return [], {}
    precision = _precision_of(mats[0], precision)
    _check_dtype(mats, precision)
    dev = mats[0].device
    h = handle or default_handle()
    o = make_options(degree, max_iters, sketch_size, tol, seed, precision, fit, warmup_iters, alpha_lo, alpha_hi)
    B = len(mats)
    m = _i64([t.shape[0] for t in mats])
    n = _i64([t.shape[1] for t in mats])
    if out is None:
        out = [torch.empty_like(t) for t in mats]
    _check_dtype(out, precision)
    need = lib().prism_polar_workspace(h.h, B, m, n, ctypes.byref(o))
    if need == 0:
        raise PrismError("prism_polar_workspace rejected the arguments: " + lib().prism_last_error().decode())
    ws = h.workspace(need, dev)
    rb = _report_buffers(B, max_iters, dev)
    rep = _report_struct(rb)
    ids = _i64(matrix_ids) if matrix_ids is not None else None
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    check(lib().prism_polar(h.h, B, m, n, _ptrs(mats), _i64([t.stride(0) for t in mats]), _ptrs(out),
                            _i64([t.stride(0) for t in out]), ids, ctypes.byref(o), ctypes.byref(rep),
                            ws.data_ptr(), ws.numel(), ctypes.c_void_p(st.cuda_stream)), "prism_polar")
    return out, rb


def _check_pinned(ts, what):
    for t in ts:
        if t.device.type != "cpu" or not t.is_pinned():
            raise PrismError(f"{what}: host-path tensors must be pinned CPU tensors (tensor.pin_memory())")


def polar_host(mats, degree=5, max_iters=30, sketch_size=8, tol=1e-6, seed=42, precision=None, fit="sketched",
               warmup_iters=0, alpha_lo=None, alpha_hi=None, out=None, matrix_ids=None, stream=None, handle=None,
               device=None):
    """Polar factors of pinned HOST matrices via prism_polar_host (end-to-end path).

    Uploads, solves and downloads on the handle's internal streams; returns
    (outputs, report) immediately — outputs (pinned host tensors) and the device
    report are valid once `stream` (default: the current stream of `device`)
    reaches this call.  Successive calls on one handle overlap copies with solves.
    """
    import torch
    mats = list(mats)
    if not mats:
        return [], {}
    _check_pinned(mats, "polar_host")
    precision = _precision_of(mats[0], precision)
    _check_dtype(mats, precision, on_host=True)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    h = handle or default_handle()
    o = make_options(degree, max_iters, sketch_size, tol, seed, precision, fit, warmup_iters, alpha_lo, alpha_hi)
    B = len(mats)
    if out is None:
        out = [torch.empty_like(t).pin_memory() for t in mats]
    _check_pinned(out, "polar_host")
    _check_dtype(out, precision, on_host=True)
    rb = _report_buffers(B, max_iters, dev)
    rep = _report_struct(rb)
    ids = _i64(matrix_ids) if matrix_ids is not None else None
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    check(lib().prism_polar_host(h.h, B, _i64([t.shape[0] for t in mats]), _i64([t.shape[1] for t in mats]),
                                 _ptrs(mats), _i64([t.stride(0) for t in mats]), _ptrs(out),
                                 _i64([t.stride(0) for t in out]), ids, ctypes.byref(o), ctypes.byref(rep),
                                 ctypes.c_void_p(st.cuda_stream)), "prism_polar_host")
    return out, rb


def sqrt_invsqrt_host(mats, degree=5, max_iters=30, sketch_size=8, tol=1e-6, seed=42, precision=None,
                      fit="sketched", warmup_iters=0, alpha_lo=None, alpha_hi=None, want_sqrt=True,
                      want_invsqrt=True, matrix_ids=None, stream=None, handle=None, device=None):
    """A^{1/2}, A^{-1/2} of pinned HOST SPD matrices via prism_sqrt_invsqrt_host."""
    import torch
    mats = list(mats)
    if not mats:
        return [], [], {}
    _check_pinned(mats, "sqrt_invsqrt_host")
    precision = _precision_of(mats[0], precision)
    _check_dtype(mats, precision, on_host=True)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    h = handle or default_handle()
    o = make_options(degree, max_iters, sketch_size, tol, seed, precision, fit, warmup_iters, alpha_lo, alpha_hi)
    B = len(mats)
    sq = [torch.empty_like(t).pin_memory() for t in mats] if want_sqrt else None
    isq = [torch.empty_like(t).pin_memory() for t in mats] if want_invsqrt else None
    rb = _report_buffers(B, max_iters, dev)
    rep = _report_struct(rb)
    ids = _i64(matrix_ids) if matrix_ids is not None else None
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    check(lib().prism_sqrt_invsqrt_host(h.h, B, _i64([t.shape[0] for t in mats]), _ptrs(mats),
                                        _i64([t.stride(0) for t in mats]), _ptrs(sq) if sq else None,
                                        _ptrs(isq) if isq else None, _i64([t.shape[1] for t in mats]), ids,
                                        ctypes.byref(o), ctypes.byref(rep), ctypes.c_void_p(st.cuda_stream)),
          "prism_sqrt_invsqrt_host")
    return sq, isq, rb


def _outputs(mats, want, given, what):
    """Output matrices: the caller's (same shape / dtype / device as the inputs, unit column
    stride) or fresh ones.  Reusing the same output buffers across calls keeps the handle's
    plan (keyed by every pointer it bakes into its tables) and its CUDA graph warm."""
    import torch
    if not want:
        return None
    if given is None:
        return [torch.empty_like(t) for t in mats]
    given = list(given)
    if len(given) != len(mats):
        raise PrismError(f"{what}: {len(given)} outputs for {len(mats)} matrices")
    for g, t in zip(given, mats):
        if g.shape != t.shape or g.dtype != t.dtype or g.device != t.device or g.stride(1) != 1:
            raise PrismError(f"{what}: each output must match its input's shape, dtype and device, rows contiguous")
    return given


def _ld_out(sq, isq, mats, what):
    a = sq if sq is not None else isq
    if a is None:
        return _i64([t.shape[1] for t in mats])
    if sq is not None and isq is not None and any(x.stride(0) != y.stride(0) for x, y in zip(sq, isq)):
        raise PrismError(f"{what}: the two outputs of a matrix must share one row stride")
    return _i64([t.stride(0) for t in a])


def sqrt_invsqrt(mats, degree=5, max_iters=30, sketch_size=8, tol=1e-6, seed=42, precision=None, fit="sketched",
                 warmup_iters=0, alpha_lo=None, alpha_hi=None, want_sqrt=True, want_invsqrt=True, matrix_ids=None,
                 stream=None, handle=None, out_sqrt=None, out_invsqrt=None):
    """A^{1/2}, A^{-1/2} of a batch of SPD CUDA matrices via prism_sqrt_invsqrt (outputs into
    out_sqrt / out_invsqrt when given)."""
    import torch
    mats = list(mats)
    if not mats:
        return [], [], {}
    precision = _precision_of(mats[0], precision)
    _check_dtype(mats, precision)
    dev = mats[0].device
    h = handle or default_handle()
    o = make_options(degree, max_iters, sketch_size, tol, seed, precision, fit, warmup_iters, alpha_lo, alpha_hi)
    B = len(mats)
    n = _i64([t.shape[0] for t in mats])
    sq = _outputs(mats, want_sqrt, out_sqrt, "sqrt_invsqrt")
    isq = _outputs(mats, want_invsqrt, out_invsqrt, "sqrt_invsqrt")
    ld_out = _ld_out(sq, isq, mats, "sqrt_invsqrt")
    need = lib().prism_sqrt_workspace(h.h, B, n, ctypes.byref(o))
    if need == 0:
        raise PrismError("prism_sqrt_workspace rejected the arguments: " + lib().prism_last_error().decode())
    ws = h.workspace(need, dev)
    rb = _report_buffers(B, max_iters, dev)
    rep = _report_struct(rb)
    ids = _i64(matrix_ids) if matrix_ids is not None else None
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    check(lib().prism_sqrt_invsqrt(h.h, B, n, _ptrs(mats), _i64([t.stride(0) for t in mats]),
                                   _ptrs(sq) if sq else None, _ptrs(isq) if isq else None, ld_out, ids,
                                   ctypes.byref(o), ctypes.byref(rep), ws.data_ptr(), ws.numel(),
                                   ctypes.c_void_p(st.cuda_stream)), "prism_sqrt_invsqrt")
    return sq, isq, rb


def sign(mats, degree=5, max_iters=30, sketch_size=8, tol=1e-6, seed=42, precision=None, fit="sketched",
         warmup_iters=0, alpha_lo=None, alpha_hi=None, out=None, matrix_ids=None, stream=None, handle=None):
    """Matrix signs of a batch of square CUDA matrices via prism_sign."""
    import torch
    mats = list(mats)
    if not mats:
        return [], {}
    precision = _precision_of(mats[0], precision)
    _check_dtype(mats, precision)
    for t in mats:
        if t.shape[0] != t.shape[1]:
            raise PrismError("sign: matrices must be square")
    dev = mats[0].device
    h = handle or default_handle()
    o = make_options(degree, max_iters, sketch_size, tol, seed, precision, fit, warmup_iters, alpha_lo, alpha_hi)
    B = len(mats)
    n = _i64([t.shape[0] for t in mats])
    if out is None:
        out = [torch.empty_like(t) for t in mats]
    _check_dtype(out, precision)
    need = lib().prism_sign_workspace(h.h, B, n, ctypes.byref(o))
    if need == 0:
        raise PrismError("prism_sign_workspace rejected the arguments: " + lib().prism_last_error().decode())
    ws = h.workspace(need, dev)
    rb = _report_buffers(B, max_iters, dev)
    rep = _report_struct(rb)
    ids = _i64(matrix_ids) if matrix_ids is not None else None
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    check(lib().prism_sign(h.h, B, n, _ptrs(mats), _i64([t.stride(0) for t in mats]), _ptrs(out),
                           _i64([t.stride(0) for t in out]), ids, ctypes.byref(o), ctypes.byref(rep),
                           ws.data_ptr(), ws.numel(), ctypes.c_void_p(st.cuda_stream)), "prism_sign")
    return out, rb


def sign_host(mats, degree=5, max_iters=30, sketch_size=8, tol=1e-6, seed=42, precision=None, fit="sketched",
              warmup_iters=0, alpha_lo=None, alpha_hi=None, out=None, matrix_ids=None, stream=None, handle=None,
              device=None):
    """Matrix signs of pinned HOST square matrices via prism_sign_host (as polar_host)."""
    import torch
    mats = list(mats)
    if not mats:
        return [], {}
    _check_pinned(mats, "sign_host")
    precision = _precision_of(mats[0], precision)
    _check_dtype(mats, precision, on_host=True)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    h = handle or default_handle()
    o = make_options(degree, max_iters, sketch_size, tol, seed, precision, fit, warmup_iters, alpha_lo, alpha_hi)
    B = len(mats)
    if out is None:
        out = [torch.empty_like(t).pin_memory() for t in mats]
    _check_pinned(out, "sign_host")
    _check_dtype(out, precision, on_host=True)
    rb = _report_buffers(B, max_iters, dev)
    rep = _report_struct(rb)
    ids = _i64(matrix_ids) if matrix_ids is not None else None
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    check(lib().prism_sign_host(h.h, B, _i64([t.shape[0] for t in mats]), _ptrs(mats),
                                _i64([t.stride(0) for t in mats]), _ptrs(out), _i64([t.stride(0) for t in out]), ids,
                                ctypes.byref(o), ctypes.byref(rep), ctypes.c_void_p(st.cuda_stream)),
          "prism_sign_host")
    return out, rb


def inv_root(mats, q=4, max_iters=30, sketch_size=8, tol=1e-6, seed=42, precision=None, fit="sketched",
             warmup_iters=0, alpha_lo=None, alpha_hi=None, out=None, matrix_ids=None, stream=None, handle=None):
    """A^{-1/q} of a batch of SPD CUDA matrices via prism_inv_root (coupled inverse
    Newton; q in 1..4)."""
    import torch
    mats = list(mats)
    if not mats:
        return [], {}
    precision = _precision_of(mats[0], precision)
    _check_dtype(mats, precision)
    for t in mats:
        if t.shape[0] != t.shape[1]:
            raise PrismError("inv_root: matrices must be square")
    dev = mats[0].device
    h = handle or default_handle()
    o = make_options(5, max_iters, sketch_size, tol, seed, precision, fit, warmup_iters, alpha_lo, alpha_hi)
    B = len(mats)
    n = _i64([t.shape[0] for t in mats])
    if out is None:
        out = [torch.empty_like(t) for t in mats]
    _check_dtype(out, precision)
    need = lib().prism_inv_root_workspace(h.h, B, n, int(q), ctypes.byref(o))
    if need == 0:
        raise PrismError("prism_inv_root_workspace rejected the arguments: " + lib().prism_last_error().decode())
    ws = h.workspace(need, dev)
    rb = _report_buffers(B, max_iters, dev)
    rep = _report_struct(rb)
    ids = _i64(matrix_ids) if matrix_ids is not None else None
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    check(lib().prism_inv_root(h.h, B, n, int(q), _ptrs(mats), _i64([t.stride(0) for t in mats]), _ptrs(out),
                               _i64([t.stride(0) for t in out]), ids, ctypes.byref(o), ctypes.byref(rep),
                               ws.data_ptr(), ws.numel(), ctypes.c_void_p(st.cuda_stream)), "prism_inv_root")
    return out, rb


def inv_root_host(mats, q=4, max_iters=30, sketch_size=8, tol=1e-6, seed=42, precision=None, fit="sketched",
                  warmup_iters=0, alpha_lo=None, alpha_hi=None, out=None, matrix_ids=None, stream=None,
                  handle=None, device=None):
    """A^{-1/q} of pinned HOST SPD matrices via prism_inv_root_host (as polar_host)."""
    import torch
    mats = list(mats)
    if not mats:
        return [], {}
    _check_pinned(mats, "inv_root_host")
    precision = _precision_of(mats[0], precision)
    _check_dtype(mats, precision, on_host=True)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    h = handle or default_handle()
    o = make_options(5, max_iters, sketch_size, tol, seed, precision, fit, warmup_iters, alpha_lo, alpha_hi)
    B = len(mats)
    if out is None:
        out = [torch.empty_like(t).pin_memory() for t in mats]
    _check_pinned(out, "inv_root_host")
    _check_dtype(out, precision, on_host=True)
    rb = _report_buffers(B, max_iters, dev)
    rep = _report_struct(rb)
    ids = _i64(matrix_ids) if matrix_ids is not None else None
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    check(lib().prism_inv_root_host(h.h, B, _i64([t.shape[0] for t in mats]), int(q), _ptrs(mats),
                                    _i64([t.stride(0) for t in mats]), _ptrs(out), _i64([t.stride(0) for t in out]),
                                    ids, ctypes.byref(o), ctypes.byref(rep), ctypes.c_void_p(st.cuda_stream)),
          "prism_inv_root_host")
    return out, rb


def _square_solve(fn_ws, fn, name, mats, q, max_iters, sketch_size, tol, seed, precision, fit, warmup_iters,
                  alpha_lo, alpha_hi, out, matrix_ids, stream, handle):
    import torch
    mats = list(mats)
    if not mats:
        return [], {}
    precision = _precision_of(mats[0], precision)
    _check_dtype(mats, precision)
    for t in mats:
        if t.shape[0] != t.shape[1]:
            raise PrismError(f"{name}: matrices must be square")
    dev = mats[0].device
    h = handle or default_handle()
    o = make_options(5, max_iters, sketch_size, tol, seed, precision, fit, warmup_iters, alpha_lo, alpha_hi)
    B = len(mats)
    n = _i64([t.shape[0] for t in mats])
    if out is None:
        out = [torch.empty_like(t) for t in mats]
    _check_dtype(out, precision)
    need = fn_ws(h.h, B, n, ctypes.byref(o))
    if need == 0:
        raise PrismError(f"{name} workspace query rejected the arguments: " + lib().prism_last_error().decode())
    ws = h.workspace(need, dev)
    rb = _report_buffers(B, max_iters, dev)
    rep = _report_struct(rb)
    ids = _i64(matrix_ids) if matrix_ids is not None else None
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    check(fn(h.h, B, n, _ptrs(mats), _i64([t.stride(0) for t in mats]), _ptrs(out), _i64([t.stride(0) for t in out]),
             ids, ctypes.byref(o), ctypes.byref(rep), ws.data_ptr(), ws.numel(), ctypes.c_void_p(st.cuda_stream)),
          name)
    return out, rb


def chebyshev_inverse(mats, max_iters=40, sketch_size=8, tol=1e-6, seed=42, precision=None, fit="sketched",
                      warmup_iters=0, alpha_lo=None, alpha_hi=None, out=None, matrix_ids=None, stream=None,
                      handle=None):
    """A^{-1} of a batch of square CUDA matrices via prism_chebyshev_inverse."""
    return _square_solve(lib().prism_chebyshev_inverse_workspace, lib().prism_chebyshev_inverse,
                         "prism_chebyshev_inverse", mats, 0, max_iters, sketch_size, tol, seed, precision, fit,
                         warmup_iters, alpha_lo, alpha_hi, out, matrix_ids, stream, handle)


def chebyshev_inverse_host(mats, max_iters=40, sketch_size=8, tol=1e-6, seed=42, precision=None, fit="sketched",
                           warmup_iters=0, alpha_lo=None, alpha_hi=None, out=None, matrix_ids=None, stream=None,
                           handle=None, device=None):
    """A^{-1} of pinned HOST square matrices via prism_chebyshev_inverse_host (as polar_host)."""
    import torch
    mats = list(mats)
    if not mats:
        return [], {}
    _check_pinned(mats, "chebyshev_inverse_host")
    precision = _precision_of(mats[0], precision)
    _check_dtype(mats, precision, on_host=True)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    h = handle or default_handle()
    o = make_options(5, max_iters, sketch_size, tol, seed, precision, fit, warmup_iters, alpha_lo, alpha_hi)
    B = len(mats)
    if out is None:
        out = [torch.empty_like(t).pin_memory() for t in mats]
    _check_pinned(out, "chebyshev_inverse_host")
    _check_dtype(out, precision, on_host=True)
    rb = _report_buffers(B, max_iters, dev)
    rep = _report_struct(rb)
    ids = _i64(matrix_ids) if matrix_ids is not None else None
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    check(lib().prism_chebyshev_inverse_host(h.h, B, _i64([t.shape[0] for t in mats]), _ptrs(mats),
                                             _i64([t.stride(0) for t in mats]), _ptrs(out),
                                             _i64([t.stride(0) for t in out]), ids, ctypes.byref(o),
                                             ctypes.byref(rep), ctypes.c_void_p(st.cuda_stream)),
          "prism_chebyshev_inverse_host")
    return out, rb


def db_newton(mats, max_iters=30, tol=1e-6, precision="fp32", fit="sketched", warmup_iters=0, want_sqrt=True,
              want_invsqrt=True, matrix_ids=None, stream=None, handle=None, out_sqrt=None, out_invsqrt=None):
    """A^{1/2}, A^{-1/2} of a batch of SPD CUDA fp32 matrices via prism_db_newton (PRISM DB
    Newton, product form; the fit is exact and unsketched; outputs into out_sqrt /
    out_invsqrt when given)."""
    import torch
    mats = list(mats)
    if not mats:
        return [], [], {}
    _check_dtype(mats, precision)
    dev = mats[0].device
    h = handle or default_handle()
    o = make_options(5, max_iters, 8, tol, 42, precision, fit, warmup_iters)
    B = len(mats)
    n = _i64([t.shape[0] for t in mats])
    sq = _outputs(mats, want_sqrt, out_sqrt, "db_newton")
    isq = _outputs(mats, want_invsqrt, out_invsqrt, "db_newton")
    ld_out = _ld_out(sq, isq, mats, "db_newton")
    need = lib().prism_db_newton_workspace(h.h, B, n, ctypes.byref(o))
    if need == 0:
        raise PrismError("prism_db_newton_workspace rejected the arguments: " + lib().prism_last_error().decode())
    ws = h.workspace(need, dev)
    rb = _report_buffers(B, max_iters, dev)
    rep = _report_struct(rb)
    ids = _i64(matrix_ids) if matrix_ids is not None else None
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    check(lib().prism_db_newton(h.h, B, n, _ptrs(mats), _i64([t.stride(0) for t in mats]),
                                _ptrs(sq) if sq else None, _ptrs(isq) if isq else None, ld_out, ids,
                                ctypes.byref(o), ctypes.byref(rep), ws.data_ptr(), ws.numel(),
                                ctypes.c_void_p(st.cuda_stream)), "prism_db_newton")
    return sq, isq, rb


def db_newton_host(mats, max_iters=30, tol=1e-6, precision="fp32", fit="sketched", warmup_iters=0, want_sqrt=True,
                   want_invsqrt=True, matrix_ids=None, stream=None, handle=None, device=None):
    """A^{1/2}, A^{-1/2} of pinned HOST SPD fp32 matrices via prism_db_newton_host."""
    import torch
    mats = list(mats)
    if not mats:
        return [], [], {}
    _check_pinned(mats, "db_newton_host")
    _check_dtype(mats, precision, on_host=True)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    h = handle or default_handle()
    o = make_options(5, max_iters, 8, tol, 42, precision, fit, warmup_iters)
    B = len(mats)
    sq = [torch.empty_like(t).pin_memory() for t in mats] if want_sqrt else None
    isq = [torch.empty_like(t).pin_memory() for t in mats] if want_invsqrt else None
    rb = _report_buffers(B, max_iters, dev)
    rep = _report_struct(rb)
    ids = _i64(matrix_ids) if matrix_ids is not None else None
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    check(lib().prism_db_newton_host(h.h, B, _i64([t.shape[0] for t in mats]), _ptrs(mats),
                                     _i64([t.stride(0) for t in mats]), _ptrs(sq) if sq else None,
                                     _ptrs(isq) if isq else None, _i64([t.shape[1] for t in mats]), ids,
                                     ctypes.byref(o), ctypes.byref(rep), ctypes.c_void_p(st.cuda_stream)),
          "prism_db_newton_host")
    return sq, isq, rb


class RowBlockSolver:
    """C-ABI steps of the row-block split (prism_rowblock_*): marshalling only."""

    def __init__(self, A_rows, degree=5, max_iters=30, sketch_size=8, tol=1e-6, seed=42, precision=None,
                 fit="sketched", warmup_iters=0, alpha_lo=None, alpha_hi=None, handle=None, stream=None):
        import torch
        precision = _precision_of(A_rows, precision)
        _check_dtype([A_rows], precision)
        self.A = A_rows
        self.dev = A_rows.device
        self.h = handle or Handle()
        self.o = make_options(degree, max_iters, sketch_size, tol, seed, precision, fit, warmup_iters, alpha_lo,
                              alpha_hi)
        self.max_iters = max_iters
        rows, n = A_rows.shape
        self.Q = torch.empty_like(A_rows)
        self.G = torch.empty(n, n, dtype=torch.float32, device=self.dev)
        self.fro2 = torch.zeros(1, dtype=torch.float64, device=self.dev)
        self.done = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.rb = _report_buffers(1, max_iters, self.dev)
        need = lib().prism_rowblock_workspace(self.h.h, rows, n, ctypes.byref(self.o))
        if need == 0:
            raise PrismError("prism_rowblock_workspace rejected the arguments: " + lib().prism_last_error().decode())
        self.ws = self.h.workspace(need, self.dev)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.dev)
        self._s = ctypes.c_void_p(self.stream.cuda_stream)

    def begin(self):
        rows, n = self.A.shape
        check(lib().prism_rowblock_begin(self.h.h, rows, n, self.A.data_ptr(), self.A.stride(0), self.Q.data_ptr(),
                                         self.Q.stride(0), self.G.data_ptr(), self.fro2.data_ptr(),
                                         ctypes.byref(self.o), self.ws.data_ptr(), self.ws.numel(), self._s),
              "prism_rowblock_begin")

    def gram(self, k):
        check(lib().prism_rowblock_gram(self.h.h, int(k), self.fro2.data_ptr(), self._s), "prism_rowblock_gram")

    def update(self, k):
        check(lib().prism_rowblock_update(self.h.h, int(k), self.G.data_ptr(), self.done.data_ptr(), self._s),
              "prism_rowblock_update")

    def end(self):
        rep = _report_struct(self.rb)
        check(lib().prism_rowblock_end(self.h.h, ctypes.byref(rep), self._s), "prism_rowblock_end")
        return self.Q, self.rb


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
