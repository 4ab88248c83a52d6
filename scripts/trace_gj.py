"""Timeline of the DB Newton pivot inversions (k_gj_pivot, last matrix of the batch):
start, loads done (first pivot broadcast), pivots done, stored — per sweep step
(diagnostics; uses the chain trace buffer's tail)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_22137_b200 as P  # noqa: E402
from paper_2601_22137_b200 import binding as B  # noqa: E402

name, shapes, mats_np, opts, desc, kind = bench.workload("dbnewton", 0)
mats = [torch.tensor(m).float().cuda() for m in mats_np]
h = P.Handle()
o = {k: v for k, v in opts.items() if k != "sketch_size"}
o["max_iters"] = 1
P.db_newton(mats, handle=h, **o)
torch.cuda.synchronize()
buf = torch.zeros(16 * 1024 * 16, dtype=torch.int64, device="cuda")
B.check(B.lib().prism_debug_trace_chain(ctypes.c_void_p(buf.data_ptr())), "trace")
P.db_newton(mats, handle=h, **o)
torch.cuda.synchronize()
B.check(B.lib().prism_debug_trace_chain(None), "trace")
T = buf[-4096:].view(-1, 4)[:32].cpu().numpy().astype(np.float64)
for j, (a, b, c, d) in enumerate(T):
    if a > 0:
        print(f"step {j:2d}: loads {(b - a) / 1e3:7.2f} us  pivots {(c - b) / 1e3:7.2f} us  store {(d - c) / 1e3:6.2f} us")
