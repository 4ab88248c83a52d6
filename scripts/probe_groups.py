"""Concurrency probe (diagnostics): the GPT-2 batch solved as G sub-batches on G streams
(each its own handle, plan and CUDA graph, so their iteration loops run concurrently and a
group's latency-bound sketch chain can overlap another group's GEMMs), against one call.

usage: python scripts/probe_groups.py [--workload gpt2] [--groups 1 2 3 4]
"""
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
ap.add_argument("--groups", type=int, nargs="+", default=[1, 2, 3, 4])
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--caps", type=int, nargs="+", default=[0], help="GEMM grid caps (prism_debug_gemm_max_ctas)")
a = ap.parse_args()
name, shapes, mats_np, opts, desc, kind = bench.workload(a.workload, 0)
dt = torch.bfloat16 if opts["precision"] == "bf16" else torch.float32
mats = [torch.tensor(m).to(dt).cuda() for m in mats_np]
outs = [torch.empty_like(m) for m in mats]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
main = torch.cuda.current_stream()
from paper_2601_22137_b200 import binding as B  # noqa: E402
ref = None
import itertools  # noqa: E402
for cap, G in itertools.product(a.caps, a.groups):
    B.check(B.lib().prism_debug_gemm_max_ctas(cap), "cap")
    idx = [list(range(g, len(mats), G)) for g in range(G)]   # interleaved: every group the same shape mix
    hs = [P.Handle() for _ in range(G)]
    sts = [torch.cuda.Stream() for _ in range(G)]

    def run():
        ev0 = torch.cuda.Event()
        ev0.record(main)
        evs = []
        for g in range(G):
            sts[g].wait_event(ev0)
            P.polar([mats[i] for i in idx[g]], out=[outs[i] for i in idx[g]], matrix_ids=idx[g], handle=hs[g],
                    stream=sts[g], **opts)
            e = torch.cuda.Event()
            e.record(sts[g])
            evs.append(e)
        for e in evs:
            main.wait_event(e)

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(a.steps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(main)
        run()
        e.record(main)
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    res = [o.clone() for o in outs]
    same = ref is None or all(torch.equal(x, y) for x, y in zip(res, ref))
    ref = ref or res
    print(f"{name}: GEMM cap {cap}: {G} group(s): {tot / a.steps:.3f} ms per step, bits equal to 1 group: {same}", flush=True)
