"""The paper's Fig. 1 in B200 device time: PRISM-5 against classical Newton-Schulz
(NS-5 = the same iteration with the Taylor coefficient, fit="taylor") on the same kernels,
4096^2 inputs with log-spaced spectra, sigma_min in {1e-12, 1e-9, 1e-6, 1e-3, 1e-1, 1/2}:

  polar: A = U diag(sigma) V^T, sigma log-spaced in [sigma_min, 1]
  sqrt:  SPD A = Q diag(lambda) Q^T, lambda log-spaced in [sigma_min, 1]

Each (kind, sigma_min, precision, fit) is solved to tolerance (FP32 3xTF32: tol 1e-5, 3e-4
for the sqrt panel below sigma_min = 1e-3 where fp32 cannot reach 1e-5; BF16: tol 3e-2),
timed with CUDA events on the launching stream (1 warm-up, median of 3), and reported with
its iteration count and status.  Next to it: the fp64 oracle's iteration counts at 256^2 on
the same spectra (the SURVEY App.N13 setting), as the paper-side reference for the ratio.

usage: python scripts/fig1.py [--out profiles/r2_fig1.json] [--quick]
"""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SIGMAS = [1e-12, 1e-9, 1e-6, 1e-3, 1e-1, 0.5]


def spd(n, smin, seed):
    from paper_2601_22137_b200 import workloads as W
    lam = np.logspace(0.0, np.log10(smin), n)
    Q = W.haar(n, n, seed)
    A = (Q * lam[None, :]) @ Q.T
    return 0.5 * (A + A.T)


def device_runs(n, quick):
    import torch
    import paper_2601_22137_b200 as P
    from paper_2601_22137_b200 import workloads as W
    h = P.Handle()
    rows = []
    for kind in ("polar", "sqrt"):
        for smin in SIGMAS:
            A = W.logspaced(n, n, smin, seed=11) if kind == "polar" else spd(n, smin, seed=11)
            for prec in ("fp32", "bf16"):
                dt = torch.float32 if prec == "fp32" else torch.bfloat16
                At = torch.tensor(A).to(dt).cuda()
                tol = 3e-2 if prec == "bf16" else (3e-4 if kind == "sqrt" and smin < 1e-3 else 1e-5)
                res = {}
                for fit in ("sketched", "taylor"):
                    kw = dict(degree=5, tol=tol, max_iters=100, precision=prec, fit=fit, handle=h)
                    out = [torch.empty_like(At)]
                    out2 = [torch.empty_like(At)]

                    def run():
                        if kind == "polar":
                            return P.polar([At], out=out, **kw)[1]
                        return P.sqrt_invsqrt([At], out_sqrt=out, out_invsqrt=out2, **kw)[2]
                    run()
                    torch.cuda.synchronize()
                    ts = []
                    for _ in range(1 if quick else 3):
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record()
                        rep = run()
                        e1.record()
                        torch.cuda.synchronize()
                        ts.append(e0.elapsed_time(e1))
                    res[fit] = {"ms": statistics.median(ts), "iters": int(rep["iters"][0]),
                                "status": int(rep["status"][0]), "resid": float(rep["resid"][0])}
                rows.append({"kind": kind, "sigma_min": smin, "precision": prec, "tol": tol, **res,
                             "speedup_time": res["taylor"]["ms"] / res["sketched"]["ms"],
                             "iter_ratio": res["taylor"]["iters"] / max(1, res["sketched"]["iters"])})
                print(json.dumps(rows[-1]), flush=True)
    return rows


def oracle_runs(n=256):
    from oracle import prism
    from paper_2601_22137_b200 import workloads as W
    rows = []
    for kind in ("polar", "sqrt"):
        for smin in SIGMAS:
            A = W.logspaced(n, n, smin, seed=11) if kind == "polar" else spd(n, smin, seed=11)
            it = {}
            for fit in ("sketched", "taylor"):
                f = prism.polar if kind == "polar" else prism.sqrt_invsqrt
                r = f(A, d=2, p=8, tol=1e-6, max_iters=200, seed=42, fit=fit)[-1]
                it[fit] = r.iters
            rows.append({"kind": kind, "sigma_min": smin, "n": n, "tol": 1e-6, "prism5": it["sketched"],
                         "ns5": it["taylor"], "ratio": it["taylor"] / max(1, it["sketched"])})
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "fig1.json"))
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    t0 = time.time()
    dev = device_runs(a.n, a.quick)
    ora = oracle_runs()
    res = {"what": "PRISM-5 vs NS-5 (same kernels, fit=taylor) to tolerance, 1 x B200, device time (CUDA events)",
           "n": a.n, "device": dev, "oracle_fp64_256": ora, "wall_s": time.time() - t0}
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print("wrote", a.out)


if __name__ == "__main__":
    main()
