"""Per-step device times of a bench workload's solve (CUDA events around each call), to see
run-to-run spread inside a timed region (diagnostics, not part of the library)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_22137_b200 as P  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "dbnewton"
name, shapes, mats_np, opts, desc, kind = bench.workload(wl, 0)
dt = torch.bfloat16 if opts["precision"] == "bf16" else torch.float32
mats = [torch.tensor(m).to(dt).cuda() for m in mats_np]
h = P.Handle()
o = {k: v for k, v in opts.items() if k != "sketch_size"} if kind == "db_newton" else opts
fn = {"db_newton": P.db_newton, "sqrt": P.sqrt_invsqrt, "polar": P.polar}[kind]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for flush_on in (False, True):
    ts = []
    for s in range(15):
        if flush_on:
            flush.add_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(mats, handle=h, **o)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(wl, "flush" if flush_on else "no flush", " ".join(f"{t:.1f}" for t in ts))
