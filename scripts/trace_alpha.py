"""Timeline of k_alpha (block 0) per iteration: stop test done, chain sums done, argmin done
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

wl = sys.argv[1] if len(sys.argv) > 1 else "square4096"
name, shapes, mats_np, opts, desc, kind = bench.workload(wl, 0)
mats = [torch.tensor(m).to(torch.bfloat16).cuda() for m in mats_np]
h = P.Handle()
P.polar(mats, handle=h, **opts)
torch.cuda.synchronize()
buf = torch.zeros(16 * 1024 * 16, dtype=torch.int64, device="cuda")
B.check(B.lib().prism_debug_trace_chain(ctypes.c_void_p(buf.data_ptr())), "trace")
P.polar(mats, handle=h, **opts)
torch.cuda.synchronize()
B.check(B.lib().prism_debug_trace_chain(None), "trace")
T = buf[-8192:].view(-1, 4)[:32].cpu().numpy().astype(np.float64)
for k, (a, b, c, d) in enumerate(T):
    if a > 0:
        print(f"iter {k:2d}: stop test {(b - a) / 1e3:6.2f} us  sums {(c - b) / 1e3 if c else float('nan'):6.2f} us"
              f"  argmin {(d - c) / 1e3 if c else float('nan'):6.2f} us  total {(d - a) / 1e3 if d else float('nan'):6.2f} us")
