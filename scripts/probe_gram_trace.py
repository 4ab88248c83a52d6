"""Tile timeline of the Gram launches for a batch of 24 tall 3072x768 bf16 matrices."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2601_22137_b200 as P
from paper_2601_22137_b200 import binding as B
from paper_2601_22137_b200 import workloads as W
shape = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "3072x768").split("x"))
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
mats = [torch.tensor(W.gaussian(*shape, seed=i)).to(torch.bfloat16).cuda() for i in range(24)]
h = P.Handle()
opts = dict(degree=5, max_iters=6, tol=1e-9, precision="bf16")
P.polar(mats, handle=h, **opts); torch.cuda.synchronize()
buf = torch.zeros(148 * 376, dtype=torch.int64, device="cuda")
B.check(B.lib().prism_debug_trace_gemm(ctypes.c_void_p(buf.data_ptr()), mode), "trace")
P.polar(mats, handle=h, **opts); torch.cuda.synchronize()
B.check(B.lib().prism_debug_trace_gemm(None, -1), "trace")
T = buf.view(148, 376).cpu().numpy().astype(np.float64)
tiles = T[:, 192:224].reshape(148, 8, 4)
lead = tiles[:, 0, 0] > 0
tz = tiles[lead]
t0 = tz[:, 0, 0].min()
rel = np.where(tz > 0, (tz - t0) / 1e3, np.nan)
print("per-tile [mma start, mma end, epi start, epi end] us (CTAs 0..3):")
for c in range(4):
    print("  cta", c, "  ".join("[" + ",".join(f"{x:6.2f}" for x in rel[c, j]) + "]" for j in range(8) if not np.isnan(rel[c, j, 0])))
mma = rel[:, :, 1] - rel[:, :, 0]
epi = rel[:, :, 3] - rel[:, :, 2]
print("median tile mma span", np.nanmedian(mma), "epi span", np.nanmedian(epi), "kernel end", np.nanmax(rel[:, :, 3]))
iss, full = T[lead, :64], T[lead, 64:128]
nkb = int((iss[0] > 0).sum())
F = (full[:, :nkb] - full[:, :1]) / 1e3
print("k-blocks traced", nkb, "first-tile full arrival (median) every 8th:", " ".join(f"{x:.2f}" for x in np.median(F, 0)[::8]))
