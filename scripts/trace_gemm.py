"""k-block timeline of the main GEMM launches (prism_debug_trace_gemm): producer issue,
MMA full-barrier arrival and MMA issue per k-block, first tile of every CTA."""
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
for mode, nm in [(0, "gram/resid"), (1, "square/poly"), (2, "apply")]:
    buf = torch.zeros(148 * 376, dtype=torch.int64, device="cuda")
    B.check(B.lib().prism_debug_trace_gemm(ctypes.c_void_p(buf.data_ptr()), mode), "trace")
    run()
    torch.cuda.synchronize()
    B.check(B.lib().prism_debug_trace_gemm(None, -1), "trace")
    T = buf.view(148, 376).cpu().numpy().astype(np.float64)
    iss, full, done = T[:, :64], T[:, 64:128], T[:, 128:192]
    tiles = T[:, 192:224].reshape(148, 8, 4)
    lead = (full[:, 0] > 0)
    nkb = int((iss[0] > 0).sum())
    if not lead.any() or nkb < 4:
        print(nm, "no data")
        continue
    t0 = iss[lead, 0][:, None]
    I = (iss[lead, :nkb] - t0) / 1e3
    F = (full[lead, :nkb] - t0) / 1e3
    D = (done[lead, :nkb] - t0) / 1e3
    print(f"== {nm}: leader CTAs {lead.sum()}, k-blocks traced {nkb}")
    print("   median over CTAs, us since first issue; every 4th k-block")
    print("   issue :", " ".join(f"{x:6.2f}" for x in np.median(I, 0)[::4]))
    print("   full  :", " ".join(f"{x:6.2f}" for x in np.median(F, 0)[::4]))
    print("   mma   :", " ".join(f"{x:6.2f}" for x in np.median(D, 0)[::4]))
    lat = np.median(F - I)
    rate = np.median(np.diff(F, axis=1)[:, 8:])
    print(f"   latency issue->full median {lat:.3f} us; steady full->full {rate * 1e3:.0f} ns per k-block;"
          f" mma issue->done {np.median(D - F) * 1e3:.0f} ns; producer stall (issue gap) {np.median(np.diff(I, axis=1)[:, 8:]) * 1e3:.0f} ns")
    tz = tiles[lead]
    tz0 = tz[:, 0, 0][:, None, None]
    rel = np.where(tz > 0, (tz - tz0) / 1e3, np.nan)
    print("   per-tile [mma start, mma end, epi start, epi end] us, CTAs 0,1,2 (leaders) and median:")
    for c in range(min(3, rel.shape[0])):
        print("     cta", c, "  ".join("[" + ",".join(f"{x:6.2f}" for x in rel[c, j]) + "]" for j in range(8) if not np.isnan(rel[c, j, 0])))
    med = np.nanmedian(rel, 0)
    print("     med  ", "  ".join("[" + ",".join(f"{x:6.2f}" for x in med[j]) + "]" for j in range(8) if not np.isnan(med[j, 0])))
    ends = np.nanmax(rel[:, :, 3], axis=1)
    print(f"   kernel end (last epilogue) median {np.nanmedian(ends):.2f} max {np.nanmax(ends):.2f} us")
    ch = T[lead, 224:232]
    chr_ = np.where(ch > 0, (ch - tz[:, 0, 2][:, None]) / 1e3, np.nan)
    print("   first-tile epilogue chunks, us after epi start [tmem ready, stored] x4 (median):",
          " ".join(f"{x:5.2f}" for x in np.nanmedian(chr_, 0)))
    cf = T[lead, 240:244]
    cfr = np.where(cf > 0, (cf - tz[:, 0, 2][:, None]) / 1e3, np.nan)
    print("   first-tile epilogue chunks, C ready (us after epi start, median):", " ".join(f"{x:5.2f}" for x in np.nanmedian(cfr, 0)))
    W = T[lead, 248:376].reshape(-1, 8, 4, 4)
    base = W[:, :, 0:1, 0:1]
    Wr = np.where(W > 0, W - base, np.nan)
    print("   per-warp chunks (CTA-median) [start, tmem ready, C ready, stored] SM cycles after the warp's first chunk:")
    med = np.nanmedian(Wr, 0)
    for e in range(8):
        print(f"     warp {e}:", "  ".join("[" + ",".join(f"{x:6.0f}" for x in med[e, c]) + "]" for c in range(4)))
