"""Single-thread latency of the device quartic argmin (prism_debug_argmin, n = 1) for
one-real-root and three-real-root cubics, against a trivial launch (diagnostics)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_22137_b200 import binding as B  # noqa: E402

def t_argmin(c, reps=200):
    cd = torch.tensor([c], dtype=torch.float64, device="cuda")
    ad = torch.empty(1, dtype=torch.float64, device="cuda")
    for _ in range(5):
        B.lib().prism_debug_argmin(1, cd.data_ptr(), 0.375, 1.45, 0.375, ad.data_ptr(), None)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        B.lib().prism_debug_argmin(1, cd.data_ptr(), 0.375, 1.45, 0.375, ad.data_ptr(), None)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3, float(ad.item())

x = torch.zeros(1, device="cuda")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200):
    x.add_(1)
e1.record()
torch.cuda.synchronize()
print(f"trivial launch: {e0.elapsed_time(e1) / 200 * 1e3:.2f} us")
# m(a) = c1 a + c2 a^2 + c3 a^3 + c4 a^4 ; m'(a) = c1 + 2 c2 a + 3 c3 a^2 + 4 c4 a^3
# one real root of m' (monotone-ish): c4 > 0, m' = 4(a - 1)^3 + small
print("1 root :", t_argmin([0.0, -4.0, 12.0 / 2, -12.0 / 3, 4.0 / 4]))
# three real roots of m' at 0.5, 0.9, 1.3: m' = 4 (a-0.5)(a-0.9)(a-1.3)
r = np.poly([0.5, 0.9, 1.3]) * 4    # 4 a^3 + ...
print("3 roots:", t_argmin([0.0, r[3], r[2] / 2, r[1] / 3, r[0] / 4]))
