"""Per-CTA timeline of the thin chain GEMM passes (prism_debug_trace) for one bench
workload: entry, setup done, first/last TMA issue, MMA k-block arrivals, epilogue."""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_22137_b200 as P  # noqa: E402
from paper_2601_22137_b200 import binding as B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="square4096")
a = ap.parse_args()
name, shapes, mats_np, opts, desc, kind = bench.workload(a.workload, 0)
dt = torch.bfloat16 if opts["precision"] == "bf16" else torch.float32
mats = [torch.tensor(m).to(dt).cuda() for m in mats_np]
h = P.Handle()
run = (lambda: P.polar(mats, handle=h, **opts)) if kind == "polar" else (lambda: P.sqrt_invsqrt(mats, handle=h, **opts))
run()
torch.cuda.synchronize()
buf = torch.zeros(5 * 1024 * 80, dtype=torch.int64, device="cuda")
B.check(B.lib().prism_debug_trace(ctypes.c_void_p(buf.data_ptr())), "trace")
run()
torch.cuda.synchronize()
B.check(B.lib().prism_debug_trace(None), "trace")
T = buf.view(5, 1024, 80).cpu().numpy().astype(np.float64)
for p in range(5):
    blk = T[p]
    used = blk[:, 0] > 0
    if not used.any():
        continue
    b = blk[used]
    t0 = b[:, 0].min()
    rel = lambda c: (b[:, c] - t0) / 1000.0
    print(f"pass {p}: CTAs {used.sum()}  kernel span {(b[:, 5].max() - t0) / 1000:.2f} us")
    for c, nm in [(0, "entry"), (1, "setup"), (2, "tma first"), (3, "tma last"), (6, "mma done"), (4, "epi tfull"), (5, "epi end"), (74, "part sent"), (75, "part recv")]:
        sel = b[:, c] > 0
        if not sel.any():
            continue
        v = (b[sel, c] - t0) / 1000.0
        print(f"   {nm:10s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f}")
    kb = (b[:, 8:72] - t0) / 1000.0
    nkb = int((b[0, 8:72] > 0).sum())
    med = np.median(kb[:, :nkb], axis=0)
    print("   mma full-arrival (median over CTAs) every 4th kb:", " ".join(f"{x:.2f}" for x in med[::4]))
