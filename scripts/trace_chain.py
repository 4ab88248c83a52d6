"""Sketch-chain pass timeline of a bench workload (diagnostics, not part of the library):
one CUDA-graph solve with prism_debug_trace_chain on, then per iteration and pass: CTAs,
entry spread, PDL-wait release, accumulator ready, epilogue end (us from the first pass's
first entry of that iteration), and the gap from a pass's last epilogue to the next pass's
first wait release.

usage: python scripts/trace_chain.py --workload gpt2
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_22137_b200 as P  # noqa: E402
from paper_2601_22137_b200 import binding as B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="gpt2")
ap.add_argument("--iters", type=int, default=4)
a = ap.parse_args()
name, shapes, mats_np, opts, desc, kind = bench.workload(a.workload, 0)
dt = torch.bfloat16 if opts["precision"] == "bf16" else torch.float32
mats = [torch.tensor(m).to(dt).cuda() for m in mats_np]
outs = [torch.empty_like(m) for m in mats]
h = P.Handle()
for _ in range(3):
    P.polar(mats, out=outs, handle=h, **opts)
torch.cuda.synchronize()
buf = torch.zeros(16 * 32 * 160 * 32, dtype=torch.int64, device="cuda")
B.check(B.lib().prism_debug_trace_chain(ctypes.c_void_p(buf.data_ptr())), "trace")
P.polar(mats, out=outs, handle=h, **opts)
torch.cuda.synchronize()
B.check(B.lib().prism_debug_trace_chain(None), "trace off")
T = buf.view(16, 32, 160, 32).cpu().double()
for k in range(a.iters):
    rows = []
    for ps in range(32):
        t = T[k, ps]
        live = t[:, 0] > 0
        if not bool(live.any()):
            continue
        rows.append((ps, t[live]))
    if not rows:
        continue
    base = min(float(r[1][:, 0].min()) for r in rows)
    print(f"iteration {k} ({name}): us from the first chain entry")
    prev_end = None
    for ps, t in rows:
        def us(x):
            return (x - base) / 1e3
        acc = t[:, 2][t[:, 2] > 0]
        epi = t[:, 3][t[:, 3] > 0]
        line = (f"  pass {ps}: ctas {t.shape[0]:3d} entry {us(float(t[:, 0].min())):7.2f}..{us(float(t[:, 0].max())):7.2f}"
                f"  wait-out {us(float(t[:, 1].min())):7.2f}..{us(float(t[:, 1].max())):7.2f}")
        if acc.numel():
            line += f"  acc {us(float(acc.median())):7.2f} (max {us(float(acc.max())):7.2f})"
        if epi.numel():
            line += f"  epi-end max {us(float(epi.max())):7.2f}"
        if prev_end is not None:
            line += f"  | gap {us(float(t[:, 1].min())) - prev_end:6.2f}"
        ok = (t[:, 2] > 0) & (t[:, 4] > 0) & (t[:, 5] > 0) & (t[:, 6] > 0) & (t[:, 7] > 0)
        if bool(ok.any()):
            q = t[ok]
            med = lambda a, b: float((q[:, b] - q[:, a]).median()) / 1e3  # noqa: E731
            line += (f"\n           epilogue: staged {med(2, 4):5.2f}  barrier {med(4, 5):5.2f}  reduce {med(5, 6):5.2f}"
                     f"  rows {med(6, 7):5.2f}  end-barrier {med(7, 3):5.2f} us")
        kbt = t[:, 8:24]
        okk = (kbt[:, 0] > 0) & (t[:, 1] > 0)
        if bool(okk.any()):
            q = kbt[okk]
            w = t[okk, 1]
            arr = [float((q[:, k] - w).median()) / 1e3 for k in range(16) if bool((q[:, k] > 0).all())]
            line += "\n           k-block ready after the PDL wait (us): " + " ".join(f"{x:.2f}" for x in arr)
        if epi.numel():
            prev_end = us(float(epi.max()))
        print(line)
