"""Host-path e2e probe: host submission time vs completion time for K pipelined calls."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_22137_b200 as P  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "gpt2"
name, shapes, mats_np, opts, desc, kind = bench.workload(w, 0)
dt = torch.bfloat16 if opts["precision"] == "bf16" else torch.float32
host = [torch.tensor(a).to(dt).pin_memory() for a in mats_np]
out = [torch.empty_like(x).pin_memory() for x in host]
h = P.Handle()
dev = [x.cuda() for x in host]
for _ in range(4):   # every staging slot and its plan warmed
    P.polar_host(host, out=out, handle=h, **opts)
    P.polar(dev, handle=h, **opts)
torch.cuda.synchronize()
K = 10
for label, fn in [("device", lambda: P.polar(dev, handle=h, **opts)), ("host", lambda: P.polar_host(host, out=out, handle=h, **opts))]:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(K):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{label}: submit {(t1 - t0) / K * 1e3:.2f} ms/call, complete {(t2 - t0) / K * 1e3:.2f} ms/call")
t0 = time.perf_counter()
for _ in range(K):
    lib = P.lib()
    import ctypes
    o = P.make_options(opts["degree"], opts["max_iters"], opts["sketch_size"], opts["tol"], 42, opts["precision"], "sketched", 0, None, None)
    from paper_2601_22137_b200.binding import _i64
    lib.prism_polar_workspace(h.h, len(host), _i64([x.shape[0] for x in host]), _i64([x.shape[1] for x in host]), ctypes.byref(o))
t1 = time.perf_counter()
print(f"workspace query {(t1 - t0) / K * 1e3:.2f} ms/call")
