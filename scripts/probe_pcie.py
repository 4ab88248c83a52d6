"""PCIe copy bandwidth probe: H2D, D2H alone and concurrently (pinned, 170 MB)."""
import torch

n = 170 * 1024 * 1024 // 2
h_in = torch.empty(n, dtype=torch.bfloat16).pin_memory()
h_out = torch.empty(n, dtype=torch.bfloat16).pin_memory()
d_a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
d_b = torch.empty(n, dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for label, do_in, do_out in [("h2d", 1, 0), ("d2h", 0, 1), ("both", 1, 1)]:
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s1.wait_event(e0)
        s2.wait_event(e0)
        if do_in:
            with torch.cuda.stream(s1):
                d_a.copy_(h_in, non_blocking=True)
        if do_out:
            with torch.cuda.stream(s2):
                h_out.copy_(d_b, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    gb = n * 2 * (do_in + do_out) / 1e9
    print(f"{label}: {ms:.2f} ms, {gb / ms * 1e3:.1f} GB/s total")

# per-copy overhead: 48 copies of ~3.5 MB vs one 170 MB copy (H2D)
chunks = [h_in[i * (n // 48):(i + 1) * (n // 48)] for i in range(48)]
dch = [d_a[i * (n // 48):(i + 1) * (n // 48)] for i in range(48)]
for rep in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for d_, h_ in zip(dch, chunks):
        d_.copy_(h_, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
print(f"48 chunked h2d: {e0.elapsed_time(e1):.2f} ms")
