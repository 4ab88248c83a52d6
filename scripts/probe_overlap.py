"""Does a concurrent PCIe copy slow the solve?  Solve on the current stream, optionally
with a large D2H and/or H2D copy running on side streams."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_22137_b200 as P  # noqa: E402

name, shapes, mats_np, opts, desc, kind = bench.workload("gpt2", 0)
dev = [torch.tensor(a).to(torch.bfloat16).cuda() for a in mats_np]
h = P.Handle()
n = 512 * 1024 * 1024 // 2
hbuf = torch.empty(n, dtype=torch.bfloat16).pin_memory()
dbuf = torch.empty(n, dtype=torch.bfloat16, device="cuda")
dbuf2 = torch.empty(n, dtype=torch.bfloat16, device="cuda")
hbuf2 = torch.empty(n, dtype=torch.bfloat16).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    P.polar(dev, handle=h, **opts)
torch.cuda.synchronize()
for label, d2h, h2d in [("alone", 0, 0), ("with d2h", 1, 0), ("with h2d", 0, 1), ("with both", 1, 1), ("alone", 0, 0)]:
    ts = []
    for rep in range(3):
        torch.cuda.synchronize()
        if d2h:
            with torch.cuda.stream(s1):
                hbuf.copy_(dbuf, non_blocking=True)
        if h2d:
            with torch.cuda.stream(s2):
                dbuf2.copy_(hbuf2, non_blocking=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        P.polar(dev, handle=h, **opts)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"solve {label}: " + " ".join(f"{t:.2f}" for t in ts) + " ms")

a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
for label, h2d in [("matmul alone", 0), ("matmul with h2d", 1), ("matmul alone", 0)]:
    ts = []
    for rep in range(3):
        torch.cuda.synchronize()
        if h2d:
            with torch.cuda.stream(s2):
                dbuf2.copy_(hbuf2, non_blocking=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            a @ a
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{label}: " + " ".join(f"{t:.2f}" for t in ts) + " ms (10 x 8192^3)")
