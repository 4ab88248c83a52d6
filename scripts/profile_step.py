"""One PRISM solve of a bench workload, for ncu (no warm-up: ncu serialises and
flushes caches per kernel, so compare kernel SHARES, not absolute times)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_22137_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="gpt2")
ap.add_argument("--solves", type=int, default=1)
ap.add_argument("--direct", action="store_true", help="direct launches (profiling mode) instead of the CUDA graph")
a = ap.parse_args()
name, shapes, mats_np, opts, desc, kind = bench.workload(a.workload, 0)
dt = torch.bfloat16 if opts["precision"] == "bf16" else torch.float32
mats = [torch.tensor(m).to(dt).cuda() for m in mats_np]
h = P.Handle()
if a.direct:
    h.profile(True)
for _ in range(a.solves):
    if kind == "polar":
        Q, rep = P.polar(mats, handle=h, **opts)
    elif kind == "sign":
        Q, rep = P.sign(mats, handle=h, **opts)
    elif kind == "inv_root":
        Q, rep = P.inv_root(mats, handle=h, **opts)
    elif kind == "chebyshev":
        Q, rep = P.chebyshev_inverse(mats, handle=h, **opts)
    elif kind == "db_newton":
        X, Y, rep = P.db_newton(mats, handle=h, **{k: v for k, v in opts.items() if k != "sketch_size"})
    else:
        X, Y, rep = P.sqrt_invsqrt(mats, handle=h, **opts)
torch.cuda.synchronize()
print("iters", rep["iters"].tolist())
