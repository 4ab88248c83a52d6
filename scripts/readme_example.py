"""The README usage example, with a check of its results (runs on a GPU)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2601_22137_b200 as P
G = [torch.randn(768, 3072, device="cuda", dtype=torch.bfloat16) for _ in range(4)]
Q, rep = P.polar(G, degree=5, tol=3e-2, max_iters=20)
A = [torch.eye(1024, device="cuda") * 2]
X, Y, rep2 = P.sqrt_invsqrt(A, tol=1e-5, precision="fp32")
torch.cuda.synchronize()
q = Q[0].float()
print("polar ok", q.shape, float((q @ q.T - torch.eye(768, device="cuda")).norm() / 768 ** 0.5), rep["iters"].tolist())
print("sqrt ok", float((X[0] - 2 ** 0.5 * torch.eye(1024, device="cuda")).abs().max()), rep2["iters"].tolist())
