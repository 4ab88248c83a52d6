import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2601_22137_b200 as P
from oracle import prism
from paper_2601_22137_b200 import workloads as W
A = torch.tensor(W.gaussian(768, 768, seed=31)).to(torch.bfloat16).cuda()
Q, rep = P.polar([A], degree=3, tol=3e-2, max_iters=30, precision="bf16")
torch.cuda.synchronize()
print("single-path d=1 768^2 bf16 iters", int(rep["iters"][0]), rep["resid_hist"][0].cpu().numpy())
Qo, ro = prism.polar(A.double().cpu().numpy(), d=1, p=8, tol=3e-2, max_iters=30, seed=42)
print("oracle", ro.iters, np.array(ro.resid))
