"""Write tests/golden/sketch_seed0_b0_k0.txt — calls only oracle/.

The first 256 float32 words (hex bit patterns) of S_0 for seed 0, matrix 0,
p = 8, s = 512 (R8).  The device sketch kernel must reproduce them
bit for bit (tests/test_gpu_kernels.py).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import philox  # noqa: E402

S = philox.gaussian_sketch(0, 0, 0, 8, 512).reshape(-1)[:256].view("uint32")
path = os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "sketch_seed0_b0_k0.txt")
with open(path, "w") as f:
    f.write("# S_0[0:256] (row-major), seed=0 b=0 k=0 p=8 s=512, float32 bit patterns\n")
    f.write("# written by scripts/make_golden.py (oracle/philox.py only)\n")
    for i in range(0, 256, 8):
        f.write(" ".join(f"{int(v):08x}" for v in S[i:i + 8]) + "\n")
