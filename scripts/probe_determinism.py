"""Repeatability of split-chain solves: same input solved repeatedly / in different batches."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2601_22137_b200 as P  # noqa: E402
from paper_2601_22137_b200 import workloads as W  # noqa: E402

for prec, dt in [("fp32", torch.float32), ("bf16", torch.bfloat16)]:
    A = torch.tensor(W.gaussian(2048, 2048, seed=10)).to(dt).cuda()
    B = torch.tensor(W.gaussian(1536, 1024, seed=11)).to(dt).cuda()
    tol = 1e-5 if prec == "fp32" else 3e-2
    outs = []
    for r in range(3):
        Q, rep = P.polar([A], degree=5, tol=tol, precision=prec, matrix_ids=[0])
        torch.cuda.synchronize()
        outs.append((Q[0].clone(), rep["alphas"][0].clone(), int(rep["iters"][0])))
    Qb, rb = P.polar([A, B], degree=5, tol=tol, precision=prec)
    torch.cuda.synchronize()
    print(prec, "single repeat equal:", all(torch.equal(outs[0][0], o[0]) for o in outs[1:]),
          "alphas equal:", all(torch.equal(outs[0][1], o[1]) for o in outs[1:]), "iters", [o[2] for o in outs])
    print(prec, "batch vs single:", torch.equal(Qb[0], outs[0][0]), "alpha diff",
          float((rb["alphas"][0] - outs[0][1]).abs().max()), "iters", int(rb["iters"][0]))
    print("  alphas single", outs[0][1][:6].tolist())
    print("  alphas batch ", rb["alphas"][0][:6].tolist())
