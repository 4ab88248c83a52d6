"""Per-CTA timeline of the chain passes (prism_debug_trace_chain) for one bench workload."""
import argparse
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

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="square4096")
ap.add_argument("--max-iters", type=int, default=0, help="cap the solve (all matrices still active in the traced pass)")
a = ap.parse_args()
name, shapes, mats_np, opts, desc, kind = bench.workload(a.workload, 0)
if a.max_iters:
    opts["max_iters"] = a.max_iters
dt = torch.bfloat16 if opts["precision"] == "bf16" else torch.float32
mats = [torch.tensor(m).to(dt).cuda() for m in mats_np]
h = P.Handle()
run = (lambda: P.polar(mats, handle=h, **opts)) if kind == "polar" else (lambda: P.sqrt_invsqrt(mats, handle=h, **opts))
run()
torch.cuda.synchronize()
buf = torch.zeros(16 * 1024 * 16, dtype=torch.int64, device="cuda")
B.check(B.lib().prism_debug_trace_chain(ctypes.c_void_p(buf.data_ptr())), "trace")
run()
torch.cuda.synchronize()
B.check(B.lib().prism_debug_trace_chain(None), "trace")
T = buf.view(16, 1024, 16).cpu().numpy().astype(np.float64)
names = ["entry", "setup", "pred done", "tma first", "mma done", "acc ready", "sent", "received", "epi done", "epi start"]
for p in range(16):
    blk = T[p]
    used = blk[:, 0] > 0
    if not used.any():
        continue
    b = blk[used]
    t0 = b[:, 0].min()
    print(f"pass code {p}: CTAs {used.sum()}  span {(b[:, :10].max() - t0) / 1e3:.2f} us")
    for c, nm in enumerate(names):
        sel = b[:, c] > 0
        if sel.any():
            v = (b[sel, c] - t0) / 1e3
            print(f"   {nm:10s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f}")

# inter-pass timeline in absolute time: last epilogue of pass j -> release of pass j+1
print("absolute (us from pass-0 entry): pass, last entry, release (pred done) median, last epi done")
base = None
for p in range(16):
    blk = T[p]
    used = blk[:, 0] > 0
    if not used.any():
        continue
    b = blk[used]
    if base is None:
        base = b[:, 0].min()
    last_entry = (b[:, 0].max() - base) / 1e3
    rel = (np.median(b[:, 2]) - base) / 1e3
    epi = b[:, 8][b[:, 8] > 0]
    done = (epi.max() - base) / 1e3 if len(epi) else float("nan")
    print(f"   pass {p}: last entry {last_entry:8.2f}  released {rel:8.2f}  done {done:8.2f}")
