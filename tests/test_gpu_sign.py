"""Matrix sign (the paper's case study P:145-199) through the C-ABI
prism_sign against the fp64 oracle `oracle.prism.sign` on the same seeded inputs:
FP32 <= 1e-5, BF16 <= 2e-2 relative Frobenius error, iteration counts within 1."""

import numpy as np
import pytest
import torch

import paper_2601_22137_b200 as P
from oracle import prism
from paper_2601_22137_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _run(A, prec, degree=5, tol=1e-5, max_iters=40, **kw):
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    At = torch.tensor(A).to(dt).cuda()
    S, rep = P.sign([At], degree=degree, tol=tol, max_iters=max_iters, seed=42, precision=prec, **kw)
    torch.cuda.synchronize()
    So, ro = prism.sign(At.double().cpu().numpy(), d=(degree - 1) // 2, p=8, tol=tol, max_iters=max_iters,
                        seed=42)
    return S[0].double().cpu().numpy(), rep, So, ro


@pytest.mark.parametrize("n,degree", [(40, 5), (200, 5), (200, 3), (517, 5)])
def test_sign_fp32_parity(n, degree):
    A = W.sym_indefinite(n, 1e-2, seed=n + degree)
    S, rep, So, ro = _run(A, "fp32", degree=degree)
    assert int(rep["status"][0]) == prism.CONVERGED and ro.status == prism.CONVERGED
    assert abs(int(rep["iters"][0]) - ro.iters) <= 1
    assert _rel(S, So) <= 1e-5


@pytest.mark.parametrize("n", [256, 1024, 2048])
def test_sign_bf16_parity(n):
    A = W.sym_indefinite(n, 1e-2, seed=7 * n)
    S, rep, So, ro = _run(A, "bf16", tol=3e-2, max_iters=30)
    assert int(rep["status"][0]) == prism.CONVERGED
    assert abs(int(rep["iters"][0]) - ro.iters) <= 1
    assert _rel(S, So) <= 2e-2


def test_sign_block_matrix_square_roots():
    # sign([[0, A], [I, 0]]) = [[0, A^{1/2}], [A^{-1/2}, 0]] for SPD A
    n = 150
    A = W.spd_logspaced(n, 1e2, seed=11)
    Z = np.zeros((n, n))
    X0 = np.block([[Z, A], [np.eye(n), Z]])
    S, rep, So, ro = _run(X0, "fp32", max_iters=60)
    assert int(rep["status"][0]) == prism.CONVERGED
    assert abs(int(rep["iters"][0]) - ro.iters) <= 1
    assert _rel(S, So) <= 1e-5
    lam, V = np.linalg.eigh(A)
    sq = (V * np.sqrt(lam)[None, :]) @ V.T
    assert _rel(S[:n, n:], sq) <= 1e-4


def test_sign_batch_mixed_sizes_and_in_place():
    sizes = [64, 300, 1024, 33]
    mats = [torch.tensor(W.sym_indefinite(s, 5e-2, seed=100 + s)).float().cuda() for s in sizes]
    S, rep = P.sign(mats, tol=1e-5, max_iters=40, seed=42, precision="fp32", matrix_ids=range(len(sizes)))
    torch.cuda.synchronize()
    for i, a in enumerate(mats):
        So, ro = prism.sign(a.double().cpu().numpy(), d=2, p=8, tol=1e-5, max_iters=40, seed=42, b=i)
        assert int(rep["status"][i]) == prism.CONVERGED
        assert abs(int(rep["iters"][i]) - ro.iters) <= 1
        assert _rel(S[i].double().cpu().numpy(), So) <= 1e-5
    # one matrix alone (same matrix id) gives the same bits; output may alias the input
    one = mats[2].clone()
    S1, _ = P.sign([one], tol=1e-5, max_iters=40, seed=42, precision="fp32", matrix_ids=[2], out=[one])
    torch.cuda.synchronize()
    assert torch.equal(S1[0], S[2])


def test_sign_zero_input():
    Z = torch.zeros(96, 96, device="cuda")
    S, rep = P.sign([Z], precision="fp32")
    torch.cuda.synchronize()
    assert int(rep["status"][0]) == prism.ZERO_INPUT
    assert not torch.any(S[0])


def test_sign_host_path_equals_device_path():
    sizes = [128, 700]
    dev = [torch.tensor(W.sym_indefinite(s, 5e-2, seed=300 + s)).to(torch.bfloat16).cuda() for s in sizes]
    host = [d.cpu().pin_memory() for d in dev]
    S, rep = P.sign(dev, tol=3e-2, max_iters=30, seed=42, precision="bf16")
    for _ in range(3):   # pipelined successive calls over the staging slots
        Sh, reph = P.sign_host(host, tol=3e-2, max_iters=30, seed=42, precision="bf16")
    torch.cuda.synchronize()
    for a, b in zip(S, Sh):
        assert torch.equal(a.cpu(), b)
    assert torch.equal(rep["iters"], reph["iters"])
