"""Warm, event-timed microbenchmark of one tcgen05 GEMM through prism_debug_gemm."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_22137_b200 import binding as B  # noqa: E402


def run(M, N, K, b_mn=0, mode=3, sym=0, prec=0, reps=20):
    dt = torch.bfloat16 if prec == 0 else torch.float32
    A = torch.randn(M, K, device="cuda").to(dt)
    Bm = (torch.randn(K, N, device="cuda") if b_mn else torch.randn(N, K, device="cuda")).to(dt)
    if sym:
        Bm = A
    C = torch.randn(M, N, device="cuda").to(dt)
    out = torch.empty(M, N, device="cuda", dtype=dt)
    lo = lambda t: torch.zeros_like(t) if prec == 1 else None  # noqa: E731
    Al, Bl, Cl, Ol = lo(A), lo(Bm), lo(C), lo(out)
    alpha = torch.tensor([0.5], dtype=torch.float64, device="cuda")
    norm = torch.zeros(4096, device="cuda")
    gd = torch.zeros(M, device="cuda")
    ws = torch.zeros(1 << 24, dtype=torch.uint8, device="cuda")
    h = B.default_handle()
    p = lambda t: None if t is None else t.data_ptr()  # noqa: E731
    st = torch.cuda.current_stream()

    def call():
        B.check(B.lib().prism_debug_gemm(h.h, prec, b_mn, mode, sym, M, N, K, p(A), p(Al), A.stride(0), p(Bm), p(Bl),
                                         Bm.stride(0), p(C), p(Cl), C.stride(0), p(out), p(Ol), out.stride(0),
                                         p(alpha), ctypes.c_float(0.5), 1, p(norm), p(gd), p(ws), ws.numel(),
                                         ctypes.c_void_p(st.cuda_stream)), "gemm")
    for _ in range(3):
        call()
    times = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        call()
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    t = sorted(times)[len(times) // 2]
    flops = 2.0 * M * N * K * (0.5 if sym else 1.0)
    return {"M": M, "N": N, "K": K, "b_mn": b_mn, "sym": sym, "prec": prec, "ms": t, "tflops": flops / t / 1e9}


if __name__ == "__main__":
    res = [run(4096, 4096, 4096), run(4096, 4096, 4096, b_mn=1), run(8192, 8192, 8192), run(4096, 4096, 4096, mode=0, sym=1),
           run(3072, 768, 768), run(4096, 4096, 4096, prec=1)]
    a, b = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16), torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        a @ b
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        a @ b
    e1.record()
    torch.cuda.synchronize()
    res.append({"cublas_8192": 2 * 8192 ** 3 * 10 / e0.elapsed_time(e1) / 1e9})
    for r in res:
        print(json.dumps(r))
