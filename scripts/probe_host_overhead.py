"""Host-side cost of one library call vs its device time (diagnostics): the GPT-2 batch
through P.polar, timed on the host (perf_counter, the GPU kept busy) and on the device
(events around each call, and around a burst of calls queued back to back)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_22137_b200 as P  # noqa: E402

name, shapes, mats_np, opts, desc, kind = bench.workload(sys.argv[1] if len(sys.argv) > 1 else "gpt2", 0)
dt = torch.bfloat16 if opts["precision"] == "bf16" else torch.float32
mats = [torch.tensor(m).to(dt).cuda() for m in mats_np]
outs = [torch.empty_like(m) for m in mats]
ids = list(range(len(mats)))
h = P.Handle()
for _ in range(5):
    P.polar(mats, out=outs, handle=h, matrix_ids=ids, **opts)
torch.cuda.synchronize()
# host cost per call with the GPU busy (a long kernel in front keeps it from draining)
hog = torch.empty(1 << 28, device="cuda")
host = []
for _ in range(20):
    hog.mul_(1.0)
    t0 = time.perf_counter()
    P.polar(mats, out=outs, handle=h, matrix_ids=ids, **opts)
    host.append((time.perf_counter() - t0) * 1e6)
torch.cuda.synchronize()
# device time: one call between events vs a burst of 20 queued back to back
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
one = []
for _ in range(10):
    torch.cuda.synchronize()
    e0.record()
    P.polar(mats, out=outs, handle=h, matrix_ids=ids, **opts)
    e1.record()
    torch.cuda.synchronize()
    one.append(e0.elapsed_time(e1) * 1e3)
hog.mul_(1.0)
hog.mul_(1.0)
e0.record()
for _ in range(20):
    P.polar(mats, out=outs, handle=h, matrix_ids=ids, **opts)
e1.record()
torch.cuda.synchronize()
burst = e0.elapsed_time(e1) * 1e3 / 20
host.sort()
one.sort()
print(f"{name}: host per call median {host[len(host) // 2]:.0f} us (min {host[0]:.0f}); device one call "
      f"median {one[len(one) // 2]:.0f} us; device per call in a queued burst {burst:.0f} us")
