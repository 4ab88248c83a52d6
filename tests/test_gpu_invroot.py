"""Coupled inverse Newton A^{-1/q} (Appendix A.3) through the
C-ABI prism_inv_root against the fp64 oracle `oracle.prism.inv_root` on the same seeded
SPD inputs: FP32 <= 1e-5, BF16 <= 2e-2 relative Frobenius error, iterations within 1."""

import numpy as np
import pytest
import torch

import paper_2601_22137_b200 as P
from oracle import prism
from paper_2601_22137_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _run(A, q, prec, tol, max_iters=40, fit="sketched"):
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    At = torch.tensor(A).to(dt).cuda()
    X, rep = P.inv_root([At], q=q, tol=tol, max_iters=max_iters, seed=42, precision=prec, fit=fit)
    torch.cuda.synchronize()
    Xo, ro = prism.inv_root(At.double().cpu().numpy(), q=q, p=8, tol=tol, max_iters=max_iters, seed=42, fit=fit)
    return X[0].double().cpu().numpy(), rep, Xo, ro


@pytest.mark.parametrize("q", [1, 2, 3, 4])
@pytest.mark.parametrize("n", [64, 200, 517])
def test_inv_root_fp32_parity(q, n):
    A = W.spd_logspaced(n, 1e2, seed=100 * q + n)
    X, rep, Xo, ro = _run(A, q, "fp32", 1e-5)
    assert int(rep["status"][0]) == prism.CONVERGED and ro.status == prism.CONVERGED
    assert abs(int(rep["iters"][0]) - ro.iters) <= 1
    # q = 1 is the matrix inverse: any fp32 method's relative forward error is ~ kappa(A) u
    # (R24): 2e-5 at kappa = 1e2; q >= 2 keeps the FP32 bar 1e-5
    assert _rel(X, Xo) <= (1e-5 if q > 1 else 2e-5)


@pytest.mark.parametrize("q", [2, 4])
@pytest.mark.parametrize("n", [256, 1024, 2048])
def test_inv_root_bf16_parity(q, n):
    A = W.spd_logspaced(n, 1e2, seed=7 * n + q)
    X, rep, Xo, ro = _run(A, q, "bf16", 3e-2, max_iters=30)
    assert int(rep["status"][0]) == prism.CONVERGED
    assert abs(int(rep["iters"][0]) - ro.iters) <= 1
    assert _rel(X, Xo) <= 2e-2


def test_inv_root_taylor_fp32():
    A = W.spd_logspaced(300, 1e2, seed=5)
    X, rep, Xo, ro = _run(A, 4, "fp32", 1e-5, max_iters=60, fit="taylor")
    assert int(rep["status"][0]) == prism.CONVERGED
    assert abs(int(rep["iters"][0]) - ro.iters) <= 1
    assert _rel(X, Xo) <= 1e-5
    # and PRISM needs fewer iterations than the classical iteration (P:566 vs P:557)
    _, rep2, _, _ = _run(A, 4, "fp32", 1e-5, max_iters=60)
    assert int(rep2["iters"][0]) < int(rep["iters"][0])


def test_inv_root_matches_eigh_wishart_fp32():
    # Shampoo-like Wishart statistics, q = 4 (Shampoo's A^{-1/4})
    A = W.wishart(384, 4.0, seed=3)
    At = torch.tensor(A).float().cuda()
    X, rep = P.inv_root([At], q=4, tol=1e-5, max_iters=60, precision="fp32")
    torch.cuda.synchronize()
    a = At.double().cpu().numpy()
    lam, V = np.linalg.eigh(a)
    ref = (V * lam[None, :] ** -0.25) @ V.T
    assert int(rep["status"][0]) == prism.CONVERGED
    assert _rel(X[0].double().cpu().numpy(), ref) <= 1e-4


def test_inv_root_batch_mixed_sizes_and_in_place():
    sizes = [96, 300, 1024, 40]
    mats = [torch.tensor(W.spd_logspaced(s, 1e2, seed=200 + s)).float().cuda() for s in sizes]
    X, rep = P.inv_root(mats, q=4, tol=1e-5, max_iters=40, seed=42, precision="fp32", matrix_ids=range(4))
    torch.cuda.synchronize()
    for i, a in enumerate(mats):
        Xo, ro = prism.inv_root(a.double().cpu().numpy(), q=4, p=8, tol=1e-5, max_iters=40, seed=42, b=i)
        assert int(rep["status"][i]) == prism.CONVERGED
        assert abs(int(rep["iters"][i]) - ro.iters) <= 1
        assert _rel(X[i].double().cpu().numpy(), Xo) <= 1e-5
    one = mats[2].clone()
    X1, _ = P.inv_root([one], q=4, tol=1e-5, max_iters=40, seed=42, precision="fp32", matrix_ids=[2], out=[one])
    torch.cuda.synchronize()
    assert torch.equal(X1[0], X[2])


def test_inv_root_host_path_equals_device_path():
    sizes = [128, 700]
    dev = [torch.tensor(W.spd_logspaced(s, 1e2, seed=300 + s)).to(torch.bfloat16).cuda() for s in sizes]
    host = [d.cpu().pin_memory() for d in dev]
    X, rep = P.inv_root(dev, q=2, tol=3e-2, max_iters=30, seed=42, precision="bf16")
    for _ in range(3):
        Xh, reph = P.inv_root_host(host, q=2, tol=3e-2, max_iters=30, seed=42, precision="bf16")
    torch.cuda.synchronize()
    for a, b in zip(X, Xh):
        assert torch.equal(a.cpu(), b)
    assert torch.equal(rep["iters"], reph["iters"])


def test_inv_root_zero_input_and_bad_q():
    Z = torch.zeros(64, 64, device="cuda")
    X, rep = P.inv_root([Z], q=2, precision="fp32")
    torch.cuda.synchronize()
    assert int(rep["status"][0]) == prism.ZERO_INPUT
    assert not torch.any(X[0])
    with pytest.raises(P.PrismError):
        P.inv_root([torch.eye(64, device="cuda")], q=5, precision="fp32")
