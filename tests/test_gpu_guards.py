"""Guard-band checks of every device entry point (the pool refuses compute-sanitizer, so
out-of-bounds accesses are caught by construction instead):

* every input is a strided view into a larger buffer whose other elements (row padding,
  rows above and below) hold a NaN canary: a kernel that reads outside the matrix feeds a
  NaN into the iteration, and the result is compared with the fp64 oracle;
* every output is a strided view into a canary-filled buffer: after the solve every element
  outside the view must still hold the canary bit pattern (a stray write anywhere in the
  band fails, including TMA stores and the mirrored blocks of the symmetric epilogues).
"""

import numpy as np
import pytest
import torch

import paper_2601_22137_b200 as P
from oracle import prism
from paper_2601_22137_b200 import workloads as W

pytestmark = pytest.mark.gpu

CANARY = {torch.bfloat16: (0x7FA5, torch.int16), torch.float32: (0x7FC0DEAD, torch.int32)}
PAD_R, PAD_C = 5, 24   # rows above / below and columns of padding around each view (16-B aligned views)


def _banded(m, n, dt, host=False):
    """(base buffer filled with the canary, view of shape m x n with row stride n + 2 PAD_C)."""
    bits, it = CANARY[dt]
    base = torch.empty(m + 2 * PAD_R, n + 2 * PAD_C, dtype=dt, device="cpu" if host else "cuda")
    base.view(it).fill_(bits if bits < 2 ** 31 else bits - 2 ** 32)
    if host:
        base = base.pin_memory()
    return base, base[PAD_R:PAD_R + m, PAD_C:PAD_C + n]


def _input(a, dt, host=False):
    base, view = _banded(a.shape[0], a.shape[1], dt, host)
    view.copy_(torch.tensor(a).to(dt))
    return base, view


def _assert_band_intact(base, view):
    bits, it = CANARY[base.dtype]
    want = bits if bits < 2 ** 31 else bits - 2 ** 32
    raw = base.view(it).cpu()
    mask = torch.ones_like(raw, dtype=torch.bool)
    r0, c0 = PAD_R, PAD_C
    mask[r0:r0 + view.shape[0], c0:c0 + view.shape[1]] = False
    bad = (raw[mask] != want).sum().item()
    assert bad == 0, f"{bad} elements outside the output view were written"


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("prec,shapes,bound", [
    ("bf16", [(300, 200), (200, 520), (768, 768), (130, 66)], 2e-2),
    ("fp32", [(300, 200), (96, 160), (256, 256)], 1e-5),
    ("tf32", [(300, 200), (160, 96)], 5e-3)])
def test_polar_guard_bands(prec, shapes, bound):
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    tol = {"bf16": 3e-2, "fp32": 1e-5, "tf32": 1e-2}[prec]
    ins = [_input(W.gaussian(m, n, seed=90 + i), dt) for i, (m, n) in enumerate(shapes)]
    outs = [_banded(m, n, dt) for (m, n) in shapes]
    Q, rep = P.polar([v for _, v in ins], out=[v for _, v in outs], degree=5, tol=tol, max_iters=30,
                     precision=prec, matrix_ids=list(range(len(shapes))))
    torch.cuda.synchronize()
    for i, ((m, n), (bo, vo), (_, vi)) in enumerate(zip(shapes, outs, ins)):
        _assert_band_intact(bo, vo)
        Qo, _ = prism.polar(vi.double().cpu().numpy(), d=2, p=8, tol=tol, max_iters=30, seed=42, b=i)
        assert _rel(vo.double().cpu().numpy(), Qo) <= bound


def test_sqrt_and_dbnewton_guard_bands():
    n = [200, 96]
    ins = [_input(W.spd_logspaced(k, 1e2, seed=95 + i), torch.float32) for i, k in enumerate(n)]
    for f in (P.sqrt_invsqrt, P.db_newton):
        o1 = [_banded(k, k, torch.float32) for k in n]
        o2 = [_banded(k, k, torch.float32) for k in n]
        X, Y, rep = f([v for _, v in ins], out_sqrt=[v for _, v in o1], out_invsqrt=[v for _, v in o2], tol=1e-5,
                      max_iters=40, matrix_ids=[0, 1])
        torch.cuda.synchronize()
        for (b1, v1), (b2, v2), (_, vi) in zip(o1, o2, ins):
            _assert_band_intact(b1, v1)
            _assert_band_intact(b2, v2)
            A = vi.double().cpu().numpy()
            w, V = np.linalg.eigh(A)
            assert _rel(v1.double().cpu().numpy(), (V * np.sqrt(w)) @ V.T) <= 1e-5
            assert _rel(v2.double().cpu().numpy(), (V / np.sqrt(w)) @ V.T) <= 1e-5


@pytest.mark.parametrize("kind", ["sign", "inv_root", "chebyshev"])
def test_other_kinds_guard_bands(kind):
    n = [192, 72]
    if kind == "sign":
        dt, mats = torch.bfloat16, [W.sym_indefinite(k, 1e-1, seed=97 + i) for i, k in enumerate(n)]
    elif kind == "inv_root":
        dt, mats = torch.float32, [W.spd_logspaced(k, 1e1, seed=97 + i) for i, k in enumerate(n)]
    else:
        dt, mats = torch.bfloat16, [W.logspaced(k, k, 0.3, seed=97 + i) for i, k in enumerate(n)]
    ins = [_input(a, dt) for a in mats]
    outs = [_banded(k, k, dt) for k in n]
    kw = dict(out=[v for _, v in outs], tol=3e-2 if dt == torch.bfloat16 else 1e-5, max_iters=40,
              precision="bf16" if dt == torch.bfloat16 else "fp32", matrix_ids=list(range(len(n))))
    if kind == "sign":
        Y, rep = P.sign([v for _, v in ins], **kw)
    elif kind == "inv_root":
        Y, rep = P.inv_root([v for _, v in ins], q=2, **kw)
    else:
        Y, rep = P.chebyshev_inverse([v for _, v in ins], **kw)
    torch.cuda.synchronize()
    bf = dt == torch.bfloat16
    tol = 3e-2 if bf else 1e-5
    for i, ((bo, vo), (_, vi)) in enumerate(zip(outs, ins)):
        _assert_band_intact(bo, vo)
        A = vi.double().cpu().numpy()
        if kind == "sign":
            ref, _ = prism.sign(A, d=2, p=8, tol=tol, max_iters=40, seed=42, b=i)
        elif kind == "inv_root":
            ref, _ = prism.inv_root(A, q=2, p=8, tol=tol, max_iters=40, seed=42, b=i)
        else:
            ref, _ = prism.chebyshev_inverse(A, p=8, tol=tol, max_iters=40, seed=42, b=i)
        assert _rel(vo.double().cpu().numpy(), ref) <= (2e-2 if bf else 1e-5)


def test_host_path_guard_bands():
    shapes = [(300, 200), (200, 520)]
    ins = [_input(W.gaussian(m, n, seed=99 + i), torch.bfloat16, host=True) for i, (m, n) in enumerate(shapes)]
    outs = [_banded(m, n, torch.bfloat16, host=True) for (m, n) in shapes]
    Q, rep = P.polar_host([v for _, v in ins], out=[v for _, v in outs], degree=5, tol=3e-2, max_iters=30,
                          precision="bf16", matrix_ids=[0, 1])
    torch.cuda.synchronize()
    for i, ((bo, vo), (_, vi)) in enumerate(zip(outs, ins)):
        _assert_band_intact(bo, vo)
        Qo, _ = prism.polar(vi.double().numpy(), d=2, p=8, tol=3e-2, max_iters=30, seed=42, b=i)
        assert _rel(vo.double().numpy(), Qo) <= 2e-2


def test_workspace_guard_bands():
    """Every workspace sub-buffer of every kind is followed by a 256-B band (library switch
    prism_debug_workspace_guards); after a solve no band byte may have changed."""
    import ctypes
    from paper_2601_22137_b200 import binding as B
    from paper_2601_22137_b200 import dist as D
    L = B.lib()
    st = torch.cuda.current_stream()
    g = lambda shp, dt, s: torch.tensor(W.gaussian(*shp, seed=s)).to(dt).cuda()  # noqa: E731
    spd = lambda n, s: torch.tensor(W.spd_logspaced(n, 1e2, seed=s)).float().cuda()  # noqa: E731
    mixed = [g((300, 200), torch.bfloat16, 1), g((200, 520), torch.bfloat16, 2), g((768, 768), torch.bfloat16, 3)]
    cases = {
        "polar bf16 (folded)": lambda h: P.polar(mixed, tol=3e-2, handle=h),
        "polar fp32 d=3": lambda h: P.polar([g((300, 200), torch.float32, 4)], degree=3, tol=1e-5, precision="fp32",
                                            handle=h),
        "polar tf32": lambda h: P.polar([g((160, 96), torch.float32, 5)], tol=1e-2, precision="tf32", handle=h),
        "polar bf16 p=16": lambda h: P.polar([g((512, 384), torch.bfloat16, 6)], tol=3e-2, sketch_size=16, handle=h),
        "sqrt fp32": lambda h: P.sqrt_invsqrt([spd(200, 7), spd(96, 8)], tol=1e-5, handle=h),
        "sign bf16": lambda h: P.sign([torch.tensor(W.sym_indefinite(192, 1e-1, seed=9)).to(torch.bfloat16).cuda()],
                                      tol=3e-2, precision="bf16", handle=h),
        "inv_root q=3": lambda h: P.inv_root([spd(128, 10)], q=3, tol=1e-5, precision="fp32", handle=h),
        "chebyshev bf16": lambda h: P.chebyshev_inverse(
            [torch.tensor(W.logspaced(160, 160, 0.3, seed=11)).to(torch.bfloat16).cuda()], tol=3e-2, precision="bf16",
            handle=h),
        "db_newton": lambda h: P.db_newton([spd(128, 12)], tol=1e-5, handle=h),
    }
    B.check(L.prism_debug_workspace_guards(1), "guards on")
    try:
        for name, run in cases.items():
            h = P.Handle()
            run(h)                      # builds the guarded plan (and its graph)
            torch.cuda.synchronize()
            B.check(L.prism_debug_guards_fill(h.h, ctypes.c_void_p(st.cuda_stream)), "fill")
            run(h)                      # the same plan, bands armed
            bad, n = ctypes.c_int64(-1), ctypes.c_int64(0)
            B.check(L.prism_debug_guards_check(h.h, ctypes.byref(bad), ctypes.byref(n),
                                               ctypes.c_void_p(st.cuda_stream)), "check")
            assert n.value > 0, name
            assert bad.value == 0, f"{name}: {bad.value} guard-band bytes written"
            if name.startswith("polar bf16 (folded)"):   # positive control: the checker sees a poke
                B.check(L.prism_debug_guards_poke(h.h, n.value // 2, ctypes.c_void_p(st.cuda_stream)), "poke")
                B.check(L.prism_debug_guards_check(h.h, ctypes.byref(bad), ctypes.byref(n),
                                                   ctypes.c_void_p(st.cuda_stream)), "check")
                assert bad.value == 1
        # row block over a one-rank NCCL communicator (the library's multi-GPU driver)
        comm = D.Comm()
        try:
            A = g((600, 300), torch.float32, 13)
            h = P.Handle()
            D.polar_rowblock(A, comm, m_global=600, row0=0, tol=1e-5, precision="fp32", handle=h)
            torch.cuda.synchronize()
            B.check(L.prism_debug_guards_fill(h.h, ctypes.c_void_p(st.cuda_stream)), "fill")
            D.polar_rowblock(A, comm, m_global=600, row0=0, tol=1e-5, precision="fp32", handle=h)
            bad, n = ctypes.c_int64(-1), ctypes.c_int64(0)
            B.check(L.prism_debug_guards_check(h.h, ctypes.byref(bad), ctypes.byref(n),
                                               ctypes.c_void_p(st.cuda_stream)), "check")
            assert n.value > 0 and bad.value == 0, ("rowblock", bad.value)
        finally:
            comm.close()
    finally:
        B.check(L.prism_debug_workspace_guards(0), "guards off")
