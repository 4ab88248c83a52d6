"""GPU kernel unit cases shared by tests/test_gpu_kernels.py and scripts/probe_gpu.py.

Each case runs one tcgen05 GEMM through the C-ABI test hook prism_debug_gemm
and compares it with a plain PyTorch fp64 reference of the same op.
"""

import ctypes

import torch

from paper_2601_22137_b200 import binding as B


def tf32_split(x):
    hi = (x.view(torch.int32) & -8192).view(torch.float32)   # clear 13 low mantissa bits
    return hi, x - hi


def padded(t, dev):
    """Copy of t with a leading dimension padded to 64 elements (16-B vector stores)."""
    r, c = t.shape
    ld = (c + 63) // 64 * 64
    buf = torch.zeros(r, ld, dtype=t.dtype, device=dev)
    buf[:, :c] = t.to(dev)
    return buf[:, :c]


def gemm_case(prec, b_mn, mode, sym, M, N, K, seed=0, alpha=0.7, c1=0.5, scale_by_alpha=1):
    """Returns dict of errors for one GEMM problem (prec: 0 bf16, 1 3xTF32, 2 tf32)."""
    dev = "cuda"
    g = torch.Generator(device="cpu").manual_seed(seed)
    dt = torch.bfloat16 if prec == 0 else torch.float32
    A = (torch.randn(M, K, generator=g) / K ** 0.5)
    if sym:
        Bm = A.clone()                      # out = I - A A^T style (K-major B = A)
        N = M
    else:
        Bm = torch.randn(K, N, generator=g) / K ** 0.5 if b_mn else torch.randn(N, K, generator=g) / K ** 0.5
    C = torch.randn(M, N, generator=g)
    if sym and mode == 1:
        C = C + C.T
    A = padded(A.to(dt), dev)
    Bm = padded(Bm.to(dt), dev)
    Cd = padded(C.to(dt), dev)
    lo = {}
    if prec == 1:
        A, lo["A"] = [padded(x, dev) for x in tf32_split(A)]
        Bm, lo["B"] = [padded(x, dev) for x in tf32_split(Bm)]
        Cd, lo["C"] = [padded(x, dev) for x in tf32_split(Cd)]
    ref_A = A.double() + (lo["A"].double() if prec == 1 else 0)
    ref_B = Bm.double() + (lo["B"].double() if prec == 1 else 0)
    ref_C = Cd.double() + (lo["C"].double() if prec == 1 else 0)
    D = ref_A @ (ref_B if b_mn else ref_B.T)
    if mode == 0:
        ref = torch.eye(M, N, dtype=torch.float64, device=dev) - D
    elif mode == 1:
        ref = c1 * ref_C + alpha * D
    elif mode == 2:
        ref = ref_C + (alpha if scale_by_alpha else 1.0) * D
    else:
        ref = D
    out = padded(torch.full((M, N), float("nan"), dtype=dt), dev)
    out_lo = padded(torch.zeros(M, N, dtype=torch.float32), dev) if prec == 1 else None
    alpha_t = torch.tensor([alpha], dtype=torch.float64, device=dev)
    tiles_m = (M + 127) // 128
    BN = 256 if prec == 0 else 128
    tiles_n = (N + BN - 1) // BN
    norm_part = torch.zeros(tiles_m * tiles_n, dtype=torch.float32, device=dev)
    gdiag = torch.zeros(M, dtype=torch.float32, device=dev)
    ws = torch.zeros(1 << 22, dtype=torch.uint8, device=dev)
    h = B.default_handle()
    st = torch.cuda.current_stream()
    p = lambda t: None if t is None else t.data_ptr()  # noqa: E731
    B.check(B.lib().prism_debug_gemm(
        h.h, prec, b_mn, mode, sym, M, N, K, p(A), p(lo.get("A")), A.stride(0), p(Bm), p(lo.get("B")),
        Bm.stride(0), p(Cd), p(lo.get("C")), Cd.stride(0), p(out), p(out_lo), out.stride(0),
        p(alpha_t), ctypes.c_float(c1), scale_by_alpha, p(norm_part), p(gdiag), p(ws), ws.numel(),
        ctypes.c_void_p(st.cuda_stream)), "prism_debug_gemm")
    torch.cuda.synchronize()
    got = out.double() + (out_lo.double() if prec == 1 else 0)
    err = (got - ref).abs()
    res = {
        "nan": int(torch.isnan(got).sum().item()),
        "max_abs": float(err.nan_to_num(1e30).max().item()),
        # relative to the larger of |out| and |A B| (I - D is small when D ~ I)
        "rel_fro": float((err.nan_to_num(1e30).norm() / max(ref.norm(), D.norm())).item()),
        "ref_max": float(ref.abs().max().item()),
    }
    if mode == 0:
        res["norm_rel"] = abs(float(norm_part.double().sum().item()) - float((ref ** 2).sum().item())) / float(
            (ref ** 2).sum().item())
        if sym or M == N:
            res["gdiag_max_abs"] = float((gdiag.double() - torch.diagonal(D)).abs().max().item())
    return res
