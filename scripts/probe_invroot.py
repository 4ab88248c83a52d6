"""Diagnostics: device vs oracle inverse Newton — iterations, residual and alpha histories."""
import numpy as np
import torch

import paper_2601_22137_b200 as P
from oracle import prism
from paper_2601_22137_b200 import workloads as W

for prec, tol, cases in (("fp32", 1e-5, [(1, 64), (2, 64), (4, 200), (3, 517)]), ("bf16", 3e-2, [(2, 1024), (4, 1024)])):
    for q, n in cases:
        A = W.spd_logspaced(n, 1e2, seed=100 * q + n)
        dt = torch.bfloat16 if prec == "bf16" else torch.float32
        At = torch.tensor(A).to(dt).cuda()
        X, rep = P.inv_root([At], q=q, tol=tol, max_iters=40, seed=42, precision=prec)
        torch.cuda.synchronize()
        Xo, ro = prism.inv_root(At.double().cpu().numpy(), q=q, p=8, tol=tol, max_iters=40, seed=42)
        x = X[0].double().cpu().numpy()
        it = int(rep["iters"][0])
        print(prec, "q", q, "n", n, "iters dev", it, "oracle", ro.iters, "status", int(rep["status"][0]),
              "rel", np.linalg.norm(x - Xo) / np.linalg.norm(Xo))
        print("  resid dev", np.array2string(rep["resid_hist"][0, :it + 1].cpu().numpy(), precision=3))
        print("  resid orc", np.array2string(np.array(ro.resid), precision=3))
        print("  alpha dev", np.array2string(rep["alphas"][0, :it].cpu().numpy(), precision=5))
        print("  alpha orc", np.array2string(np.array(ro.alphas), precision=5))
