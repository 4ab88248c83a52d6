"""The bench's extra workloads at their full size and in bench.py's launch configuration
(the same batch, options and entry point), checked against the fp64 oracle on sampled
matrices: one per distinct block size, the 4096^2 members included.  Slow (the oracle
solves 4096^2 problems in fp64)."""

import numpy as np
import pytest
import torch

import bench
import paper_2601_22137_b200 as P
from oracle import prism

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _batch(name):
    _, shapes, mats_np, opts, _, kind = bench.workload(name, 0)
    dt = torch.bfloat16 if opts["precision"] == "bf16" else torch.float32
    return shapes, [torch.tensor(a).to(dt).cuda() for a in mats_np], opts, kind


def _samples(shapes):
    seen, idx = set(), []
    for i, s in enumerate(shapes):
        if s not in seen and s[0] != 2048:   # 2048 blocks: covered by the smaller parity tests
            seen.add(s)
            idx.append(i)
    return idx


def test_sign4096_bench_workload():
    shapes, mats, opts, _ = _batch("sign4096")
    S, rep = P.sign(mats, matrix_ids=[0], **opts)
    torch.cuda.synchronize()
    So, ro = prism.sign(mats[0].double().cpu().numpy(), d=2, p=8, tol=opts["tol"], max_iters=opts["max_iters"],
                        seed=42, b=0)
    assert int(rep["status"][0]) == prism.CONVERGED
    assert abs(int(rep["iters"][0]) - ro.iters) <= 1
    assert _rel(S[0].double().cpu().numpy(), So) <= 2e-2


def test_cheb4096_bench_workload():
    shapes, mats, opts, _ = _batch("cheb4096")
    X, rep = P.chebyshev_inverse(mats, matrix_ids=[0], **opts)
    torch.cuda.synchronize()
    Xo, ro = prism.chebyshev_inverse(mats[0].double().cpu().numpy(), p=8, tol=opts["tol"],
                                     max_iters=opts["max_iters"], seed=42, b=0)
    assert int(rep["status"][0]) == prism.CONVERGED
    assert abs(int(rep["iters"][0]) - ro.iters) <= 1
    assert _rel(X[0].double().cpu().numpy(), Xo) <= 2e-2


def test_shampoo_sqrt_bench_workload():
    shapes, mats, opts, _ = _batch("shampoo")
    ids = list(range(len(mats)))
    X, Y, rep = P.sqrt_invsqrt(mats, matrix_ids=ids, **opts)
    torch.cuda.synchronize()
    for i in _samples(shapes):
        Xo, Yo, ro = prism.sqrt_invsqrt(mats[i].double().cpu().numpy(), d=2, p=8, tol=opts["tol"],
                                        max_iters=opts["max_iters"], seed=42, b=i)
        assert int(rep["status"][i]) == prism.CONVERGED
        assert abs(int(rep["iters"][i]) - ro.iters) <= 1
        assert _rel(X[i].double().cpu().numpy(), Xo) <= 1e-5
        assert _rel(Y[i].double().cpu().numpy(), Yo) <= 1e-5


def test_invroot4_bench_workload():
    shapes, mats, opts, _ = _batch("invroot")
    q = opts.pop("q")
    ids = list(range(len(mats)))
    X, rep = P.inv_root(mats, q=q, matrix_ids=ids, **opts)
    torch.cuda.synchronize()
    for i in _samples(shapes):
        Xo, ro = prism.inv_root(mats[i].double().cpu().numpy(), q=q, p=8, tol=opts["tol"],
                                max_iters=opts["max_iters"], seed=42, b=i)
        assert int(rep["status"][i]) == prism.CONVERGED
        assert abs(int(rep["iters"][i]) - ro.iters) <= 1
        assert _rel(X[i].double().cpu().numpy(), Xo) <= 1e-5


def test_dbnewton_bench_workload():
    shapes, mats, opts, _ = _batch("dbnewton")
    ids = list(range(len(mats)))
    X, Y, rep = P.db_newton(mats, matrix_ids=ids, **opts)
    torch.cuda.synchronize()
    for i in _samples(shapes):
        Xo, Yo, ro = prism.db_newton(mats[i].double().cpu().numpy(), tol=opts["tol"], max_iters=opts["max_iters"])
        assert int(rep["status"][i]) == prism.CONVERGED
        assert abs(int(rep["iters"][i]) - ro.iters) <= 1
        assert _rel(X[i].double().cpu().numpy(), Xo) <= 1e-5
        assert _rel(Y[i].double().cpu().numpy(), Yo) <= 1e-5
