"""Gram/apply time for tall (MN-major operands) vs wide (K-major) batches of equal flops."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2601_22137_b200 as P
from paper_2601_22137_b200 import workloads as W
for label, shape in [("tall 3072x768 (MN-major gram)", (3072, 768)), ("wide 768x3072 (K-major gram)", (768, 3072)),
                     ("square 768x768", (768, 768))]:
    mats = [torch.tensor(W.gaussian(*shape, seed=i)).to(torch.bfloat16).cuda() for i in range(24)]
    h = P.Handle()
    opts = dict(degree=5, max_iters=6, tol=1e-9, precision="bf16")
    P.polar(mats, handle=h, **opts); torch.cuda.synchronize()
    h.profile(True); h.profile_read(reset=True)
    for _ in range(3):
        P.polar(mats, handle=h, **opts)
    torch.cuda.synchronize()
    prof = h.profile_read(reset=True); h.profile(False)
    print(label, {k: round(v["ms"] / 3, 3) for k, v in prof.items() if k in ("gram", "square", "apply", "sketch_chain")})
