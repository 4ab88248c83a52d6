"""Small solves of every entry point for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck), s in {64, 128, 256}, direct launches (profiling mode) and the CUDA-graph loop.

usage: compute-sanitizer --tool memcheck python scripts/sanitize_cases.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2601_22137_b200 as P  # noqa: E402
from paper_2601_22137_b200 import dist as D  # noqa: E402
from paper_2601_22137_b200 import workloads as W  # noqa: E402


def main():
    for direct in (True, False):
        h = P.Handle()
        h.profile(direct)
        for s in (64, 128, 256):
            for prec in ("bf16", "fp32"):
                dt = torch.bfloat16 if prec == "bf16" else torch.float32
                tol = 3e-2 if prec == "bf16" else 1e-5
                A = torch.tensor(W.gaussian(s + 40, s, seed=s)).to(dt).cuda()
                B = torch.tensor(W.gaussian(s, s + 72, seed=s + 1)).to(dt).cuda()
                P.polar([A, B], degree=5, tol=tol, max_iters=12, precision=prec, handle=h)
                P.polar([A], degree=3, tol=tol, max_iters=12, precision=prec, handle=h, sketch_size=16)
                S = torch.tensor(W.spd_logspaced(s, 1e2, seed=s)).to(dt).cuda()
                P.sign([torch.tensor(W.sym_indefinite(s, 1e-1, seed=s)).to(dt).cuda()], tol=tol, max_iters=12,
                       precision=prec, handle=h)
                P.chebyshev_inverse([torch.tensor(W.logspaced(s, s, 0.3, seed=s)).to(dt).cuda()], tol=tol,
                                    max_iters=12, precision=prec, handle=h)
                if prec == "fp32":
                    P.sqrt_invsqrt([S], degree=5, tol=tol, max_iters=12, precision=prec, handle=h)
                    P.inv_root([S], q=4, tol=tol, max_iters=12, precision=prec, handle=h)
                    P.db_newton([S], tol=tol, max_iters=12, handle=h)
                torch.cuda.synchronize()
        h.profile(False)
    # multi-GPU entry points through a 1-rank NCCL communicator
    comm = D.Comm()
    mats = [torch.tensor(W.gaussian(m, n, seed=3)).to(torch.bfloat16).cuda() for m, n in ((200, 128), (128, 320))]
    D.polar_sharded(mats, comm, nbuckets=2, tol=3e-2, max_iters=12)
    A = torch.tensor(W.gaussian(300, 256, seed=5)).float().cuda()
    D.polar_rowblock(A, comm, m_global=300, row0=0, tol=1e-5, max_iters=12, precision="fp32")
    torch.cuda.synchronize()
    comm.close()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
