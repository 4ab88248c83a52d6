import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2601_22137_b200 as P
from paper_2601_22137_b200 import workloads as W
shapes = [(2048, 2048), (1536, 1024), (300, 200)]
mats = [torch.tensor(W.gaussian(m, n, seed=10 + i)).float().cuda() for i, (m, n) in enumerate(shapes)]
single = []
for i, t in enumerate(mats):
    Q, r = P.polar([t], degree=5, tol=1e-5, precision="fp32", matrix_ids=[i])
    torch.cuda.synchronize()
    single.append((Q[0].clone(), r["alphas"][0][: int(r["iters"][0])].clone(), int(r["iters"][0])))
for combo in [[0, 1, 2], [0, 2], [1, 2], [0, 1], [2, 0]]:
    Qb, rb = P.polar([mats[i] for i in combo], degree=5, tol=1e-5, precision="fp32", matrix_ids=combo)
    torch.cuda.synchronize()
    res = []
    for j, i in enumerate(combo):
        it = int(rb["iters"][j])
        a = rb["alphas"][j][:it]
        res.append((i, torch.equal(Qb[j], single[i][0]), it == single[i][2],
                    float((a - single[i][1]).abs().max()) if it == single[i][2] else None))
    print(combo, res)
