"""Alpha-trajectory audit (diagnostics): for every kind and precision, the device's fitted
alpha per iteration against the fp64 oracle's on the same input (a precision-starved fit —
e.g. a residual ~ I below the compute dtype's resolution — shows up as alphas jumping to the
other end of the interval).  Prints iterations, max |alpha_dev - alpha_oracle| and the output
error.

usage: python scripts/alpha_audit.py [--n 1024]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_22137_b200 as P  # noqa: E402
from oracle import prism  # noqa: E402
from paper_2601_22137_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
a = ap.parse_args()
n = a.n
TOL = {"bf16": 3e-2, "tf32": 1e-2, "fp32": 1e-5}


def rel(x, y):
    return float(np.linalg.norm(x - y) / np.linalg.norm(y))


def report(name, prec, dev_out, rep, orc_out, ro):
    k = min(int(rep["iters"][0]), ro.iters)
    al = rep["alphas"][0, :k].double().cpu().numpy()
    da = float(np.max(np.abs(al - np.array(ro.alphas[:k])))) if k else 0.0
    print(f"{name:10s} {prec:5s} iters {int(rep['iters'][0]):2d}/{ro.iters:2d}  max|da| {da:.2e}  "
          f"rel {rel(dev_out, orc_out):.2e}", flush=True)


for prec in ("bf16", "tf32", "fp32"):
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    tol = TOL[prec]
    for label, A in (("polar-ls", W.logspaced(n, n // 2, 1e-3, seed=1)), ("polar-g", W.gaussian(n, n, seed=2))):
        t = torch.tensor(A).to(dt).cuda()
        Q, rep = P.polar([t], degree=5, tol=tol, max_iters=30, precision=prec, matrix_ids=[0])
        torch.cuda.synchronize()
        Qo, ro = prism.polar(t.double().cpu().numpy(), d=2, p=8, tol=tol, max_iters=30, seed=42, b=0)
        report(label, prec, Q[0].double().cpu().numpy(), rep, Qo, ro)
    t = torch.tensor(W.sym_indefinite(n, 1e-2, seed=3)).to(dt).cuda()
    S, rep = P.sign([t], tol=tol, max_iters=30, precision=prec, matrix_ids=[0])
    torch.cuda.synchronize()
    So, ro = prism.sign(t.double().cpu().numpy(), d=2, p=8, tol=tol, max_iters=30, seed=42, b=0)
    report("sign", prec, S[0].double().cpu().numpy(), rep, So, ro)
    t = torch.tensor(W.spd_logspaced(n, 1e2, seed=4)).to(dt).cuda()
    for q in (2, 4):
        X, rep = P.inv_root([t], q=q, tol=tol, max_iters=30, precision=prec, matrix_ids=[0])
        torch.cuda.synchronize()
        Xo, ro = prism.inv_root(t.double().cpu().numpy(), q=q, p=8, tol=tol, max_iters=30, seed=42, b=0)
        report(f"invroot{q}", prec, X[0].double().cpu().numpy(), rep, Xo, ro)
    if prec != "bf16":
        X, Y, rep = P.sqrt_invsqrt([t], tol=tol, max_iters=30, precision=prec, matrix_ids=[0])
        torch.cuda.synchronize()
        Xo, Yo, ro = prism.sqrt_invsqrt(t.double().cpu().numpy(), d=2, p=8, tol=tol, max_iters=30, seed=42, b=0)
        report("sqrt", prec, Y[0].double().cpu().numpy(), rep, Yo, ro)
