"""Parity diagnostics (round 2): measured device-vs-oracle errors for the cases the
round-1 verdict asked to tighten.  Prints one JSON line per case.

  * FP32 polar (north_star bar 1e-5)
  * coupled sqrt / inv-sqrt FP32 at kappa <= 1e2 (north_star bar 1e-5 on both outputs)
  * DB Newton A^{-1/2} FP32
  * the exact mixed GPT-2 batch bench.py times (all 48 matrices vs the oracle)
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2601_22137_b200 as P  # noqa: E402
from oracle import prism  # noqa: E402
from paper_2601_22137_b200 import workloads as W  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def exact_sqrt(A):
    w, V = np.linalg.eigh(A)
    return (V * np.sqrt(w)) @ V.T, (V / np.sqrt(w)) @ V.T


def sqrt_cases(which):
    for n, kappa, deg in [(256, 1e2, 5), (200, 1e2, 3), (640, 1e2, 5), (1024, 1e2, 5), (2048, 1e2, 5)]:
        A = W.spd_logspaced(n, kappa, seed=n if n != 1024 else n + 1)
        At = torch.tensor(A).float().cuda()
        Aq = At.double().cpu().numpy()
        tol = 1e-5
        if which == "sqrt":
            X, Y, rep = P.sqrt_invsqrt([At], degree=deg, max_iters=40, tol=tol, seed=42, precision="fp32")
            torch.cuda.synchronize()
            Xo, Yo, ro = prism.sqrt_invsqrt(Aq, d=1 if deg == 3 else 2, p=8, tol=tol, max_iters=40, seed=42)
            oit, ohist = ro.iters, ro.resid
        else:
            X, Y, rep = P.db_newton([At], max_iters=40, tol=tol, precision="fp32")
            torch.cuda.synchronize()
            Xo, Yo, ro = prism.db_newton(Aq, tol=tol, max_iters=40)
            oit, ohist = ro.iters, ro.resid
        Xe, Ye = exact_sqrt(Aq)
        x, y = X[0].double().cpu().numpy(), Y[0].double().cpu().numpy()
        print(json.dumps({"case": which, "n": n, "kappa": kappa, "deg": deg,
                          "iters": int(rep["iters"][0]), "oracle_iters": oit,
                          "rel_X_oracle": rel(x, Xo), "rel_Y_oracle": rel(y, Yo),
                          "rel_X_exact": rel(x, Xe), "rel_Y_exact": rel(y, Ye),
                          "oracle_rel_X_exact": rel(Xo, Xe), "oracle_rel_Y_exact": rel(Yo, Ye),
                          "dev_resid_hist": [float(v) for v in rep["resid_hist"][0].cpu().numpy()[: int(rep["iters"][0]) + 1]],
                          "oracle_resid_hist": [float(v) for v in np.asarray(ohist)[: oit + 1]]}), flush=True)


def polar_fp32():
    for (m, n) in [(300, 200), (200, 520), (256, 256), (640, 384), (1024, 1024)]:
        A = W.gaussian(m, n, seed=m + n)
        At = torch.tensor(A).float().cuda()
        Q, rep = P.polar([At], degree=5, max_iters=40, tol=1e-5, seed=42, precision="fp32")
        torch.cuda.synchronize()
        Qo, ro = prism.polar(At.double().cpu().numpy(), d=2, p=8, tol=1e-5, max_iters=40, seed=42)
        print(json.dumps({"case": "polar_fp32", "shape": [m, n], "iters": int(rep["iters"][0]),
                          "oracle_iters": ro.iters, "rel_oracle": rel(Q[0].double().cpu().numpy(), Qo)}), flush=True)


def gpt2_mixed():
    shapes = W.gpt2_small_shapes()
    mats_np = W.muon_batch(shapes, seed=1, kind="mixed")
    mats = [torch.tensor(a).to(torch.bfloat16).cuda() for a in mats_np]
    Q, rep = P.polar(mats, degree=5, max_iters=20, tol=3e-2, seed=42, precision="bf16", matrix_ids=list(range(48)))
    torch.cuda.synchronize()
    t0 = time.time()
    rows = []
    for i in range(48):
        Qo, ro = prism.polar(mats[i].double().cpu().numpy(), d=2, p=8, tol=3e-2, max_iters=20, seed=42, b=i)
        rows.append({"i": i, "shape": list(shapes[i]), "kind": "mp" if i % 2 == 0 else "htmp",
                     "iters": int(rep["iters"][i]), "oracle_iters": ro.iters,
                     "status": int(rep["status"][i]), "rel": rel(Q[i].double().cpu().numpy(), Qo)})
    print(json.dumps({"case": "gpt2_mixed", "oracle_s": time.time() - t0, "rows": rows}), flush=True)


if __name__ == "__main__":
    what = sys.argv[1:] or ["polar32", "sqrt", "db", "gpt2"]
    if "polar32" in what:
        polar_fp32()
    if "sqrt" in what:
        sqrt_cases("sqrt")
    if "db" in what:
        sqrt_cases("db")
    if "gpt2" in what:
        gpt2_mixed()
