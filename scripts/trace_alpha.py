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
T = buf[-8192:].view(-1, 8)[:32].cpu().numpy().astype(np.float64)
Cq = buf[-16384:-8192].view(-1, 8)[:32, :5].cpu().view(torch.float64).numpy()
for k in range(3):
    print("quartic", k, repr(list(Cq[k])))
for k, row in enumerate(T):
    a, b, c, d, e, f = row[:6]
    if a > 0 and d > 0:
        print(f"iter {k:2d}: entry->stop test done {(b - a) / 1e3:6.2f}  ->partials loaded {(e - b) / 1e3:6.2f}"
              f"  ->reduced {(f - e) / 1e3:6.2f}  ->coeffs {(c - f) / 1e3:6.2f}  ->argmin {(d - c) / 1e3:6.2f} us")
