"""Build libprism.so (all CUDA for sm_100a) in-tree: paper_2601_22137_b200/_lib/libprism.so.

Each translation unit of paper_2601_22137_b200/csrc (host side + SIMT kernels in prism.cu,
the tcgen05 GEMM and sketch-chain kernels per precision in gemm_*.cu / chain_*.cu) is
compiled to an object in parallel, then linked into one shared library.
"""
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(ROOT, "paper_2601_22137_b200", "csrc")
LIBDIR = os.path.join(ROOT, "paper_2601_22137_b200", "_lib")
OBJ = os.path.join(LIBDIR, "obj")
OUT = os.path.join(LIBDIR, "libprism.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                "-Xptxas", "-v"]


def _compile(src):
    obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
    cmd = [NVCC] + FLAGS + ["-I", os.path.join(ROOT, "include"), "-c", "-o", obj, src]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return src, obj, r


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(SRC, "*.cu")))
    headers = glob.glob(os.path.join(SRC, "*.cuh")) + glob.glob(os.path.join(SRC, "*.h")) + \
        [os.path.join(ROOT, "include", "prism.h")]
    newest_hdr = max(os.path.getmtime(h) for h in headers)
    stale = []
    for s in srcs:
        obj = os.path.join(OBJ, os.path.basename(s)[:-3] + ".o")
        if not os.path.exists(obj) or os.path.getmtime(obj) < max(newest_hdr, os.path.getmtime(s)):
            stale.append(s)
    objs = [os.path.join(OBJ, os.path.basename(s)[:-3] + ".o") for s in srcs]
    for o in glob.glob(os.path.join(OBJ, "*.o")):   # objects of removed sources
        if o not in objs:
            os.remove(o)
    if not stale and os.path.exists(OUT) and all(os.path.getmtime(OUT) >= os.path.getmtime(o) for o in objs):
        return OUT
    logs = {}
    with cf.ThreadPoolExecutor(max_workers=min(len(stale), os.cpu_count() or 4) or 1) as ex:
        for src, obj, r in ex.map(_compile, stale):
            if verbose or r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed on {os.path.basename(src)}")
            # without the per-function compile times, so the log only changes with the code
            logs[os.path.basename(src)] = "".join(l for l in r.stderr.splitlines(True) if "Compile time" not in l)
    r = subprocess.run([NVCC] + ARCH + ["-shared", "-Xcompiler", "-fPIC", "-o", OUT] + objs + ["-ldl"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    logdir = os.path.join(LIBDIR, "ptxas")
    os.makedirs(logdir, exist_ok=True)
    for name, text in logs.items():
        with open(os.path.join(logdir, name + ".log"), "w") as f:
            f.write(text)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
