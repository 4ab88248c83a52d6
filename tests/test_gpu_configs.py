"""BASELINE.json configs at their full sizes, in the launch configuration bench.py
times (one call per batch), against the fp64 oracle where it finishes in seconds and
otherwise through properties that hold at any size.

  configs[0]  64 x 32, PRISM-5, p = 8, <= 15 iterations            -> oracle parity (FP32)
  configs[2]  Shampoo SPD blocks 1024-4096, kappa up to 1e6, FP32    -> oracle parity / properties
  configs[3]  8192 x 8192 BF16, row-block split                      -> tests/test_gpu_multigpu.py
  configs[4]  1.2B-param GPT Muon batch (96 matrices) BF16           -> sampled oracle + properties
  north star  4096 x 4096 BF16 (bench --workload square4096)         -> full oracle parity
"""

import numpy as np
import pytest
import torch

import paper_2601_22137_b200 as P
from oracle import prism
from paper_2601_22137_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _orth_err(q):
    """||Q^T Q - I||_F / sqrt(s) on the small side (any size, on the device, fp64)."""
    q = q.double()
    G = q.T @ q if q.shape[0] >= q.shape[1] else q @ q.T
    s = G.shape[0]
    return float(torch.linalg.norm(G - torch.eye(s, device=G.device, dtype=G.dtype))) / s ** 0.5


def test_config0_64x32_fp32_parity():
    A = W.gaussian(64, 32, seed=1000)
    At = torch.tensor(A).float().cuda()
    Q, rep = P.polar([At], degree=5, sketch_size=8, max_iters=15, tol=1e-5, seed=42, precision="fp32")
    torch.cuda.synchronize()
    Qo, ro = prism.polar(At.double().cpu().numpy(), d=2, p=8, tol=1e-5, max_iters=15, seed=42)
    assert int(rep["status"][0]) == prism.CONVERGED and ro.status == prism.CONVERGED
    assert abs(int(rep["iters"][0]) - ro.iters) <= 1
    assert _rel(Q[0].double().cpu().numpy(), Qo) <= 1e-5
    # and the fp64 oracle's own limit: the SVD polar factor (tol 1e-10, native fp64)
    Qn, rn = prism.polar(A, d=2, p=8, tol=1e-10, max_iters=15, seed=42)
    U, _, Vt = np.linalg.svd(A, full_matrices=False)
    assert rn.status == prism.CONVERGED and _rel(Qn, U @ Vt) <= 1e-9


@pytest.mark.parametrize("n,kappa", [(1024, 1e2), (2048, 1e4)])
def test_config2_shampoo_sqrt_parity(n, kappa):
    A = W.spd_logspaced(n, kappa, seed=n + 1)
    At = torch.tensor(A).float().cuda()
    tol = 1e-5 if kappa <= 1e2 else 3e-5
    X, Y, rep = P.sqrt_invsqrt([At], degree=5, max_iters=40, tol=tol, seed=42, precision="fp32")
    torch.cuda.synchronize()
    Xo, Yo, ro = prism.sqrt_invsqrt(At.double().cpu().numpy(), d=2, p=8, tol=tol, max_iters=40, seed=42)
    assert int(rep["status"][0]) == prism.CONVERGED
    assert abs(int(rep["iters"][0]) - ro.iters) <= 1
    assert _rel(X[0].double().cpu().numpy(), Xo) <= 1e-5
    assert _rel(Y[0].double().cpu().numpy(), Yo) <= (1e-5 if kappa <= 1e2 else 3e-4)


def test_config2_shampoo_4096_kappa1e6_properties():
    # kappa = 1e6: SURVEY §8(c) "report only" row (cond(A^{-1/2}) ~ 1e3); checked by the
    # defining properties (A^{1/2})^2 = A and A^{1/2} A^{-1/2} = I at full size
    n = 4096
    A = torch.tensor(W.spd_logspaced(n, 1e6, seed=7)).float().cuda()
    X, Y, rep = P.sqrt_invsqrt([A], degree=5, max_iters=40, tol=3e-4, seed=42, precision="fp32")
    torch.cuda.synchronize()
    assert int(rep["status"][0]) in (prism.CONVERGED, prism.MAX_ITERS)
    x, y, a = X[0].double(), Y[0].double(), A.double()
    assert float(torch.linalg.norm(x @ x - a) / torch.linalg.norm(a)) <= 1e-3
    eye = torch.eye(n, device=a.device, dtype=a.dtype)
    assert float(torch.linalg.norm(x @ y - eye)) / n ** 0.5 <= 1e-3


def test_config4_gpt1b_batch_sampled():
    """configs[4] batch (96 matrices, 1.2B parameters) in one BF16 call: every matrix by
    the polar property, one per shape against the oracle."""
    shapes = W.gpt_1b_shapes()
    mats_np = W.muon_batch(shapes, seed=1, kind="gaussian")
    mats = [torch.tensor(a).to(torch.bfloat16).cuda() for a in mats_np]
    Q, rep = P.polar(mats, degree=5, max_iters=20, tol=3e-2, seed=42, precision="bf16")
    torch.cuda.synchronize()
    assert torch.all(rep["status"] == prism.CONVERGED)
    for q in Q:
        assert _orth_err(q) <= 0.06
    for i in (0, 1, 2, 3):
        Qo, ro = prism.polar(mats[i].double().cpu().numpy(), d=2, p=8, tol=3e-2, max_iters=20, seed=42, b=i)
        assert abs(int(rep["iters"][i]) - ro.iters) <= 1
        assert _rel(Q[i].double().cpu().numpy(), Qo) <= 2e-2


def test_north_star_4096_bf16_full_parity():
    A = torch.tensor(W.gaussian(4096, 4096, seed=4096)).to(torch.bfloat16).cuda()
    Q, rep = P.polar([A], degree=5, max_iters=25, tol=3e-2, seed=42, precision="bf16")
    torch.cuda.synchronize()
    Qo, ro = prism.polar(A.double().cpu().numpy(), d=2, p=8, tol=3e-2, max_iters=25, seed=42)
    assert int(rep["status"][0]) == prism.CONVERGED
    assert abs(int(rep["iters"][0]) - ro.iters) <= 1
    assert _rel(Q[0].double().cpu().numpy(), Qo) <= 2e-2


@pytest.mark.slow
def test_polar_4096_fp32_full_parity():
    """The extra block's second workload (the paper's precision): 4096^2 FP32
    (3xTF32, 128-row chain tiles) against the fp64 oracle at tol 1e-5."""
    A = torch.tensor(W.gaussian(4096, 4096, seed=4096)).float().cuda()
    Q, rep = P.polar([A], degree=5, max_iters=25, tol=1e-5, seed=42, precision="fp32")
    torch.cuda.synchronize()
    Qo, ro = prism.polar(A.double().cpu().numpy(), d=2, p=8, tol=1e-5, max_iters=25, seed=42)
    assert int(rep["status"][0]) == prism.CONVERGED
    assert abs(int(rep["iters"][0]) - ro.iters) <= 1
    assert _rel(Q[0].double().cpu().numpy(), Qo) <= 1e-5


@pytest.mark.slow
def test_polar_8192_bf16_single_gpu_parity():
    """configs[3]'s matrix through the single-GPU path (the extra block's third workload)."""
    A = torch.tensor(W.gaussian(8192, 8192, seed=3000)).to(torch.bfloat16).cuda()
    Q, rep = P.polar([A], degree=5, max_iters=25, tol=3e-2, seed=42, precision="bf16")
    torch.cuda.synchronize()
    Qo, ro = prism.polar(A.double().cpu().numpy(), d=2, p=8, tol=3e-2, max_iters=25, seed=42)
    assert int(rep["status"][0]) == prism.CONVERGED
    assert abs(int(rep["iters"][0]) - ro.iters) <= 1
    assert _rel(Q[0].double().cpu().numpy(), Qo) <= 2e-2
