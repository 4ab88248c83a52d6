"""Run-to-run and batch-vs-single bit identity of the polar solve (diagnostics): the same
batch twice, each matrix alone twice, and where the first alpha differs.

usage: python scripts/determinism.py [--prec fp32|bf16] [--deg 5]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2601_22137_b200 as P  # noqa: E402
from paper_2601_22137_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--prec", default="fp32")
ap.add_argument("--deg", type=int, default=5)
ap.add_argument("--direct", action="store_true")
a = ap.parse_args()
dt = torch.float32 if a.prec != "bf16" else torch.bfloat16
tol = 1e-5 if a.prec == "fp32" else 3e-2
shapes = [(300, 200), (128, 256), (256, 256), (520, 136)]
mats = [torch.tensor(W.gaussian(m, n, seed=i)).to(dt).cuda() for i, (m, n) in enumerate(shapes)]
h = P.Handle()
h.profile(a.direct)
kw = dict(degree=a.deg, tol=tol, precision=a.prec, handle=h)
Q1, r1 = P.polar(mats, **kw)
Q2, r2 = P.polar(mats, **kw)
torch.cuda.synchronize()
print("batch run-to-run equal:", all(torch.equal(x, y) for x, y in zip(Q1, Q2)),
      torch.equal(torch.nan_to_num(r1["alphas"]), torch.nan_to_num(r2["alphas"])))
for i, t in enumerate(mats):
    Qs, rs = P.polar([t], matrix_ids=[i], **kw)
    Qt, rt = P.polar([t], matrix_ids=[i], **kw)
    torch.cuda.synchronize()
    a_b = r1["alphas"][i].double().cpu()
    a_s = rs["alphas"][0].double().cpu()
    diff = [k for k in range(a_b.numel()) if not (a_b[k] == a_s[k] or (a_b[k] != a_b[k] and a_s[k] != a_s[k]))]
    print(f"matrix {i} {tuple(t.shape)}: single run-to-run {torch.equal(Qs[0], Qt[0])}, batch==single "
          f"{torch.equal(Qs[0], Q1[i])}, iters {int(r1['iters'][i])}/{int(rs['iters'][0])}, first alpha diff "
          f"{diff[:1]} {[(float(a_b[k]), float(a_s[k])) for k in diff[:2]]}")
