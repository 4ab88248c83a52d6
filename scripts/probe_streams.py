"""Does splitting a batch into G groups solved concurrently on G streams (one handle
each) beat one grouped solve?  (diagnostics, not part of the library)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_22137_b200 as P  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "gpt2"
name, shapes, mats_np, opts, desc, kind = bench.workload(wl, 0)
dt = torch.bfloat16 if opts["precision"] == "bf16" else torch.float32
mats = [torch.tensor(m).to(dt).cuda() for m in mats_np]
outs = [torch.empty_like(m) for m in mats]
B = len(mats)
ids = list(range(B))
main = torch.cuda.current_stream()
for G in (1, 2, 3, 4):
    if B % G:
        continue
    # interleaved groups (each group holds every shape)
    groups = [list(range(g, B, G)) for g in range(G)]
    handles = [P.Handle() for _ in range(G)]
    streams = [torch.cuda.Stream() for _ in range(G)]

    def step():
        ev = torch.cuda.Event()
        ev.record(main)
        done = []
        for g, idx in enumerate(groups):
            s = streams[g]
            s.wait_event(ev)
            P.polar([mats[i] for i in idx], out=[outs[i] for i in idx], matrix_ids=[ids[i] for i in idx],
                    handle=handles[g], stream=s, **opts)
            e = torch.cuda.Event()
            e.record(s)
            done.append(e)
        for e in done:
            main.wait_event(e)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(20):
        step()
    e1.record(main)
    torch.cuda.synchronize()
    print(f"{wl}: {G} group(s) on {G} stream(s): {e0.elapsed_time(e1) / 20 * 1e3:8.1f} us per step")
