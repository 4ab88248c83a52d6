"""Device sketch vs oracle bits, device argmin vs oracle argmin."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch, ctypes
from oracle import philox, prism
from paper_2601_22137_b200 import binding as B
out = {}
bad = 0
for (seed, b, k, p, s) in [(0, 0, 0, 8, 512), (42, 3, 7, 8, 768), (2**40 + 5, 17, 2, 5, 1001), (7, 1, 0, 1, 33)]:
    S = torch.empty(p * s, dtype=torch.float32, device="cuda")
    B.check(B.lib().prism_debug_sketch(seed, b, k, p, s, S.data_ptr(), None), "sketch")
    torch.cuda.synchronize()
    ref = philox.gaussian_sketch(seed, b, k, p, s).reshape(-1)
    got = S.cpu().numpy()
    nd = int(np.sum(got.view(np.uint32) != ref.view(np.uint32)))
    bad += nd
    out[f"sketch_{seed}_{b}_{k}_{p}_{s}_mismatch"] = nd
g = np.random.default_rng(0)
cs = g.standard_normal((500, 5)) * 10.0 ** g.uniform(-6, 3, (500, 5))
cd = torch.tensor(cs, dtype=torch.float64, device="cuda").contiguous()
ad = torch.empty(500, dtype=torch.float64, device="cuda")
B.check(B.lib().prism_debug_argmin(500, cd.data_ptr(), 0.375, 1.45, 0.375, ad.data_ptr(), None), "argmin")
torch.cuda.synchronize()
ref = np.array([prism.argmin_quartic(c, 0.375, 1.45, 0.375) for c in cs])
out["argmin_max_abs"] = float(np.max(np.abs(ad.cpu().numpy() - ref)))
print(json.dumps(out))
