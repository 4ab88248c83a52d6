"""Main-GEMM timeline of one launch (diagnostics, not part of the library): a direct-launch
solve with prism_debug_trace_gemm on for one epilogue mode (0 residual, 1 poly, 2 apply);
the buffer keeps the LAST launch of that mode.  Prints, over the leader CTAs: the first
tile's k-block period at the MMA (full-barrier arrival), the TMA latency (producer issue ->
full arrival), and per tile the mainloop and epilogue spans.

usage: python scripts/trace_gemm.py --workload square4096 --mode 2
"""
import argparse
import ctypes
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_22137_b200 as P  # noqa: E402
from paper_2601_22137_b200 import binding as B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="square4096")
ap.add_argument("--mode", type=int, default=2)
ap.add_argument("--max-iters", type=int, default=0)
a = ap.parse_args()
name, shapes, mats_np, opts, desc, kind = bench.workload(a.workload, 0)
if a.max_iters:
    opts = dict(opts, max_iters=a.max_iters)
dt = torch.bfloat16 if opts["precision"] == "bf16" else torch.float32
mats = [torch.tensor(m).to(dt).cuda() for m in mats_np]
outs = [torch.empty_like(m) for m in mats]
h = P.Handle()
h.profile(True)
for _ in range(2):
    P.polar(mats, out=outs, handle=h, **opts)
torch.cuda.synchronize()
W = 376
buf = torch.zeros(148 * W, dtype=torch.int64, device="cuda")
B.check(B.lib().prism_debug_trace_gemm(ctypes.c_void_p(buf.data_ptr()), a.mode), "trace")
P.polar(mats, out=outs, handle=h, **opts)
torch.cuda.synchronize()
B.check(B.lib().prism_debug_trace_gemm(None, -1), "trace off")
T = buf.view(148, W).cpu().double()
lead = [c for c in range(148) if T[c, 64] > 0]
t0 = min(float(T[c, 64]) for c in lead)
periods, lat, issue = [], [], []
for c in lead:
    f = [float(T[c, 64 + k]) for k in range(64) if T[c, 64 + k] > 0]
    p = [float(T[c, k]) for k in range(64) if T[c, k] > 0]
    d = [float(T[c, 128 + k]) for k in range(64) if T[c, 128 + k] > 0]
    periods += [(f[k + 1] - f[k]) for k in range(4, len(f) - 1)]
    lat += [(f[k] - p[k]) for k in range(min(len(f), len(p)))]
    issue += [(d[k] - f[k]) for k in range(min(len(f), len(d)))]
print(f"{name} mode {a.mode}: {len(lead)} leader CTAs")
if periods:
    print(f"  first-tile k-block period at the MMA (kb >= 4): median {statistics.median(periods):.0f} ns, "
          f"p90 {sorted(periods)[int(0.9 * len(periods))]:.0f} ns")
    print(f"  producer issue -> full arrival: median {statistics.median(lat):.0f} ns, "
          f"p90 {sorted(lat)[int(0.9 * len(lat))]:.0f} ns")
    print(f"  MMA issue (full -> commit issued): median {statistics.median(issue):.0f} ns")
spans = {}
for c in lead:
    for j in range(8):
        ms, me, es, ee = (float(T[c, 192 + 4 * j + x]) for x in range(4))
        if ms > 0:
            spans.setdefault(j, []).append(((ms - t0) / 1e3, (me - ms) / 1e3, (es - t0) / 1e3 if es else 0.0,
                                            (ee - es) / 1e3 if ee and es else 0.0))
for j, v in sorted(spans.items()):
    print(f"  tile #{j}: {len(v):3d} CTAs, MMA start median {statistics.median(x[0] for x in v):7.2f} us, "
          f"mainloop median {statistics.median(x[1] for x in v):6.2f} us, epilogue median "
          f"{statistics.median(x[3] for x in v):6.2f} us (max {max(x[3] for x in v):6.2f})")
end = max(float(T[c, 192 + 4 * j + 3]) for c in lead for j in range(8) if T[c, 192 + 4 * j + 3] > 0)
print(f"  launch span (first MMA -> last epilogue end): {(end - t0) / 1e3:.2f} us")
# per-chunk epilogue marks of the second tile (leader CTAs; warps 4 and 11), with the
# instrumentation patch applied: [0] step start, [1] C ready, [2] output buffer free,
# [3] values, [4] staged, [5] transposed, [6] stores issued, [7] next chunk's TMEM load done
for wi, base in ((4, 224), (11, 288)):
    rows = []
    for c in lead:
        for x in range(8):
            m = [float(T[c, base + 8 * x + k]) for k in range(8)]
            if m[0] > 0:
                rows.append([x] + [(m[k] - m[k - 1]) if m[k] and m[k - 1] else 0.0 for k in range(1, 8)])
    for x in sorted(set(r[0] for r in rows)):
        rr = [r for r in rows if r[0] == x]
        print(f"  warp {wi} chunk {x}: " + " ".join(f"{statistics.median(r[k] for r in rr):5.0f}" for k in range(1, 8)))
