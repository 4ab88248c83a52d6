"""Tile-order probe (diagnostics): GEMM tiles of a matrix walked in groups of R tile rows,
column by column (prism_debug_raster_rows), against the plain row-major order; per workload
the device time per solve (L2 flushed before each) and bit equality with R = 1.

usage: python scripts/probe_raster.py [--workloads square4096 square8192 gpt2] [--rows 1 4 8]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_22137_b200 as P  # noqa: E402
from paper_2601_22137_b200 import binding as B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workloads", nargs="+", default=["square4096", "square8192", "gpt2"])
ap.add_argument("--rows", type=int, nargs="+", default=[1, 4, 8])
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--rounds", type=int, default=2)
a = ap.parse_args()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for wl in a.workloads:
    name, shapes, mats_np, opts, desc, kind = bench.workload(wl, 0)
    dt = torch.bfloat16 if opts["precision"] == "bf16" else torch.float32
    mats = [torch.tensor(m).to(dt).cuda() for m in mats_np]
    outs = [torch.empty_like(m) for m in mats]
    ref = None
    for rnd in range(a.rounds):
        for R in a.rows:
            B.check(B.lib().prism_debug_raster_rows(R), "raster")
            h = P.Handle()
            for _ in range(3):
                P.polar(mats, out=outs, handle=h, **opts)
            torch.cuda.synchronize()
            tot = 0.0
            for _ in range(a.steps):
                flush.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                P.polar(mats, out=outs, handle=h, **opts)
                e.record()
                torch.cuda.synchronize()
                tot += s.elapsed_time(e)
            res = [o.clone() for o in outs]
            same = ref is None or all(torch.equal(x, y) for x, y in zip(res, ref))
            ref = ref or res
            print(f"{name}: raster rows {R}: {tot / a.steps:.3f} ms per solve, bits equal: {same}", flush=True)
    B.check(B.lib().prism_debug_raster_rows(1), "raster")
