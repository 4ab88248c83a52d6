"""Per-iteration cost of a bench workload: time P.polar (CUDA-graph path) with
max_iters = 1 .. N and print the increments (diagnostics, not part of the library)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_22137_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="gpt2")
ap.add_argument("--subset", type=int, default=0, help="first N matrices only")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
name, shapes, mats_np, opts, desc, kind = bench.workload(a.workload, 0)
if a.subset:
    mats_np = mats_np[:a.subset]
dt = torch.bfloat16 if opts["precision"] == "bf16" else torch.float32
mats = [torch.tensor(m).to(dt).cuda() for m in mats_np]
outs = [torch.empty_like(m) for m in mats]
h = P.Handle()
prev = 0.0
full = opts["max_iters"]
for mi in list(range(1, 12)) + [full]:
    o = dict(opts)
    o["max_iters"] = mi
    for _ in range(3):
        P.polar(mats, out=outs, handle=h, **o)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(a.reps):
        _, rep = P.polar(mats, out=outs, handle=h, **o)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / a.reps
    it = rep["iters"].cpu()
    active = int((it >= mi).sum()) if mi != full else 0
    print(f"max_iters {mi:3d}: {ms * 1e3:9.1f} us  (+{(ms - prev) * 1e3:8.1f})  still active after: {active}")
    prev = ms
