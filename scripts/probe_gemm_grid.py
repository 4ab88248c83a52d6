"""Is the long-K GEMM mainloop bound per SM or chip-wide?  One 8192^3 bf16 GEMM through
prism_debug_gemm with the persistent grid capped at 148 / 112 / 74 / 48 CTAs: the k-block
period of each tile's mainloop (timeline hook) against the grid size (diagnostics)."""
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_22137_b200 import binding as B  # noqa: E402

M = N = K = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
Bm = torch.randn(N, K, device="cuda").to(torch.bfloat16)
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
ws = torch.zeros(1 << 24, dtype=torch.uint8, device="cuda")
h = B.default_handle()
st = torch.cuda.current_stream()
L = B.lib()
W = 376
buf = torch.zeros(148 * W, dtype=torch.int64, device="cuda")


def call():
    B.check(L.prism_debug_gemm(h.h, 0, 0, 3, 0, M, N, K, A.data_ptr(), None, A.stride(0), Bm.data_ptr(), None,
                               Bm.stride(0), None, None, 0, out.data_ptr(), None, out.stride(0), None,
                               ctypes.c_float(1.0), 0, None, None, ws.data_ptr(), ws.numel(),
                               ctypes.c_void_p(st.cuda_stream)), "gemm")


for cap in (148, 112, 74, 48):
    B.check(L.prism_debug_gemm_max_ctas(cap), "cap")
    for _ in range(2):
        call()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        call()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    buf.zero_()
    B.check(L.prism_debug_trace_gemm(ctypes.c_void_p(buf.data_ptr()), 3), "trace")
    call()
    torch.cuda.synchronize()
    B.check(L.prism_debug_trace_gemm(None, -1), "trace off")
    T = buf.view(148, W).cpu().double()
    per = []
    for c in range(148):
        for j in range(8):
            ms, me = float(T[c, 192 + 4 * j]), float(T[c, 192 + 4 * j + 1])
            if ms > 0 and me > ms:
                per.append((me - ms) / (K / 64))
    t = statistics.median(ts)
    print(f"{M}^3 grid cap {cap:3d}: {t:.3f} ms ({2.0 * M * N * K / t / 1e9:.0f} TF/s), k-block period median "
          f"{statistics.median(per):.0f} ns over {len(per)} tiles", flush=True)
B.check(L.prism_debug_gemm_max_ctas(0), "cap")
