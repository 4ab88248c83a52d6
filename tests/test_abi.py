"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every
symbol include/prism.h declares, and validates arguments on the host."""
import ctypes
import os
import re

import pytest

from paper_2601_22137_b200 import binding as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "prism.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(prism_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = B.lib()
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert set(B.EXPORTS) == set(names)


def test_abi_version_and_defaults():
    lib = B.lib()
    assert lib.prism_abi_version() == 1
    o = B.Options()
    lib.prism_default_options(ctypes.byref(o))
    assert (o.degree, o.sketch_size, o.max_iters, o.precision, o.fit) == (5, 8, 30, 0, 0)


def test_workspace_query_and_validation():
    lib = B.lib()
    h = B.Handle()
    m = (ctypes.c_int64 * 2)(768, 3072)
    n = (ctypes.c_int64 * 2)(2304, 768)
    o = B.make_options(precision="bf16")
    ws = lib.prism_polar_workspace(h.h, 2, m, n, ctypes.byref(o))
    assert ws > 2 * 768 * 2304 * 2 * 2
    o_fp32 = B.make_options(precision="fp32")
    assert lib.prism_polar_workspace(h.h, 2, m, n, ctypes.byref(o_fp32)) > ws
    bad = B.make_options(degree=4)
    assert lib.prism_polar_workspace(h.h, 2, m, n, ctypes.byref(bad)) == 0
    bad = B.make_options(sketch_size=65)
    assert lib.prism_polar_workspace(h.h, 2, m, n, ctypes.byref(bad)) == 0
    nn = (ctypes.c_int64 * 1)(1024)
    assert lib.prism_sqrt_workspace(h.h, 1, nn, ctypes.byref(o_fp32)) > 4 * 1024 * 1024 * 4 * 2


def test_host_errors_before_any_launch():
    lib = B.lib()
    h = B.Handle()
    o = B.make_options()
    m = (ctypes.c_int64 * 1)(64)
    n = (ctypes.c_int64 * 1)(32)
    st = lib.prism_polar(h.h, 0, m, n, None, None, None, None, None, ctypes.byref(o), None, None, 0, None)
    assert st == 1 and b"batch" in lib.prism_last_error()
    A = (ctypes.c_void_p * 1)(256)
    ld = (ctypes.c_int64 * 1)(16)      # lda < n
    st = lib.prism_polar(h.h, 1, m, n, A, ld, A, ld, None, ctypes.byref(o), None, ctypes.c_void_p(4096), 1 << 20, None)
    assert st == 1 and b"lda" in lib.prism_last_error()


def test_lpt_partition_deterministic_and_balanced():
    own = B.lpt_partition([5, 4, 3, 3, 2, 1], 2)
    assert own == [0, 1, 1, 0, 1, 0]
    costs = [float(c) for c in range(1, 97)]
    own = B.lpt_partition(costs, 8)
    loads = [sum(c for c, o in zip(costs, own) if o == r) for r in range(8)]
    assert max(loads) - min(loads) <= max(costs) and sorted(set(own)) == list(range(8))


def test_flop_counts():
    # F_min: 4096^2 polar d=2 ~ 277 GFLOP per iteration
    f = B.polar_flops_per_iter(4096, 4096, 5, 8)
    assert abs(f / 1e9 - 277) < 2
    assert B.sqrt_flops_per_iter(1024, 5, 8) == pytest.approx(8 * 1024 ** 3, rel=2e-2)
