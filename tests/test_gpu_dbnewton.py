"""PRISM DB Newton, product form (Appendix A.2), through the
C-ABI prism_db_newton against the fp64 oracle `oracle.prism.db_newton` on the same seeded
SPD inputs (FP32): relative Frobenius error <= 1e-5 (A^{1/2}) and the kappa-scaled bound
for A^{-1/2}, iterations within 1."""

import numpy as np
import pytest
import torch

import paper_2601_22137_b200 as P
from oracle import prism
from paper_2601_22137_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("n", [40, 128, 200, 517])
@pytest.mark.parametrize("fit", ["sketched", "taylor"])
def test_db_newton_fp32_parity(n, fit):
    A = W.spd_logspaced(n, 1e2, seed=n + 3)
    At = torch.tensor(A).float().cuda()
    X, Y, rep = P.db_newton([At], tol=1e-5, max_iters=40, fit=fit)
    torch.cuda.synchronize()
    Xo, Yo, ro = prism.db_newton(At.double().cpu().numpy(), tol=1e-5, max_iters=40,
                                 fit="taylor" if fit == "taylor" else "exact")
    assert int(rep["status"][0]) == prism.CONVERGED and ro.status == prism.CONVERGED
    assert abs(int(rep["iters"][0]) - ro.iters) <= 1
    assert _rel(X[0].double().cpu().numpy(), Xo) <= 1e-5
    assert _rel(Y[0].double().cpu().numpy(), Yo) <= 1e-5


def test_db_newton_alpha_trajectory_matches_oracle():
    A = W.spd_logspaced(300, 1e3, seed=9)
    At = torch.tensor(A).float().cuda()
    X, Y, rep = P.db_newton([At], tol=1e-5, max_iters=40)
    torch.cuda.synchronize()
    _, _, ro = prism.db_newton(At.double().cpu().numpy(), tol=1e-5, max_iters=40)
    it = min(int(rep["iters"][0]), ro.iters)
    al = rep["alphas"][0, :it].cpu().numpy()
    assert np.allclose(al, np.array(ro.alphas[:it]), rtol=1e-3, atol=1e-4)


def test_db_newton_vs_eigh_1024():
    n = 1024
    A = W.spd_logspaced(n, 1e2, seed=4)
    At = torch.tensor(A).float().cuda()
    X, Y, rep = P.db_newton([At], tol=1e-5, max_iters=40)
    torch.cuda.synchronize()
    a = At.double().cpu().numpy()
    lam, V = np.linalg.eigh(a)
    assert int(rep["status"][0]) == prism.CONVERGED
    assert _rel(X[0].double().cpu().numpy(), (V * np.sqrt(lam)) @ V.T) <= 1e-5
    assert _rel(Y[0].double().cpu().numpy(), (V / np.sqrt(lam)) @ V.T) <= 1e-5


def test_db_newton_batch_mixed_sizes_and_bits():
    sizes = [96, 300, 700, 33]
    mats = [torch.tensor(W.spd_logspaced(s, 1e2, seed=600 + s)).float().cuda() for s in sizes]
    X, Y, rep = P.db_newton(mats, tol=1e-5, max_iters=40)
    torch.cuda.synchronize()
    for i, a in enumerate(mats):
        Xo, Yo, ro = prism.db_newton(a.double().cpu().numpy(), tol=1e-5, max_iters=40)
        assert int(rep["status"][i]) == prism.CONVERGED
        assert abs(int(rep["iters"][i]) - ro.iters) <= 1
        assert _rel(X[i].double().cpu().numpy(), Xo) <= 1e-5
    X1, Y1, _ = P.db_newton([mats[2]], tol=1e-5, max_iters=40)
    torch.cuda.synchronize()
    assert torch.equal(X1[0], X[2]) and torch.equal(Y1[0], Y[2])


def test_db_newton_host_path_equals_device_path():
    sizes = [128, 500]
    dev = [torch.tensor(W.spd_logspaced(s, 1e2, seed=700 + s)).float().cuda() for s in sizes]
    host = [d.cpu().pin_memory() for d in dev]
    X, Y, rep = P.db_newton(dev, tol=1e-5, max_iters=40)
    for _ in range(3):
        Xh, Yh, reph = P.db_newton_host(host, tol=1e-5, max_iters=40)
    torch.cuda.synchronize()
    for a, b in zip(X + Y, Xh + Yh):
        assert torch.equal(a.cpu(), b)


def test_db_newton_zero_input_and_precision():
    Z = torch.zeros(64, 64, device="cuda")
    X, Y, rep = P.db_newton([Z])
    torch.cuda.synchronize()
    assert int(rep["status"][0]) == prism.ZERO_INPUT
    with pytest.raises(P.PrismError):
        P.db_newton([torch.eye(64, device="cuda").to(torch.bfloat16)], precision="bf16")


def test_db_newton_caller_outputs_equal_fresh_outputs():
    sizes = [100, 260]
    mats = [torch.tensor(W.spd_logspaced(s, 1e2, seed=800 + s)).float().cuda() for s in sizes]
    X, Y, _ = P.db_newton(mats, tol=1e-5, max_iters=40)
    osq = [torch.full_like(m, float("nan")) for m in mats]
    oisq = [torch.full_like(m, float("nan")) for m in mats]
    for _ in range(2):   # the same buffers twice: the handle's plan is reused
        X2, Y2, _ = P.db_newton(mats, tol=1e-5, max_iters=40, out_sqrt=osq, out_invsqrt=oisq)
    torch.cuda.synchronize()
    assert X2[0] is osq[0] and Y2[1] is oisq[1]
    for a, b in zip(X + Y, X2 + Y2):
        assert torch.equal(a, b)
    with pytest.raises(P.PrismError):
        P.db_newton(mats, out_sqrt=osq[:1])
