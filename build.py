"""Build libprism.so (all CUDA for sm_100a) in-tree: paper_2601_22137_b200/_lib/libprism.so."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(ROOT, "paper_2601_22137_b200", "csrc")
OUT = os.path.join(ROOT, "paper_2601_22137_b200", "_lib", "libprism.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def build(verbose: bool = False) -> str:
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    srcs = [os.path.join(SRC, "prism.cu")]
    deps = srcs + [os.path.join(SRC, f) for f in os.listdir(SRC)] + [os.path.join(ROOT, "include", "prism.h")]
    if os.path.exists(OUT) and all(os.path.getmtime(OUT) >= os.path.getmtime(d) for d in deps):
        return OUT
    cmd = [NVCC] + FLAGS + ["-I", os.path.join(ROOT, "include"), "-o", OUT] + srcs
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed")
    with open(os.path.join(os.path.dirname(OUT), "ptxas.log"), "w") as f:
        # without the per-function compile times, so the log only changes with the code
        f.write("".join(l for l in r.stderr.splitlines(True) if "Compile time" not in l))
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
