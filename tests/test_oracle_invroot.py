"""Pins of the coupled inverse Newton oracle (oracle.prism.inv_root, Appendix A.3
P:527-594) against what the paper and the mathematics fix:
the paper's printed q = 1, 2 coefficient formulas, the direct loss, the
eigendecomposition A^{-1/q}, the uncoupled inverse Newton recurrence, a dense
grid for the companion-matrix argmin."""

import math

import numpy as np
import pytest

from oracle import prism
from oracle.philox import gaussian_sketch
from paper_2601_22137_b200 import workloads as W


def test_interval_brackets_taylor():
    for q in range(1, 9):
        lo, hi, aT = prism.inv_root_interval(q)
        assert lo < aT < hi and math.isclose(aT, 1.0 / q)


def test_coeffs_match_paper_printed_q1_q2():
    # the paper's printed c_1..c_2q for q = 1 and q = 2
    rng = np.random.default_rng(0)
    for _ in range(20):
        t = rng.standard_normal(7)
        c = prism.inv_root_loss_coeffs(t, 1)
        assert c.size == 3
        assert math.isclose(c[1], 2 * t[3] - 2 * t[2], rel_tol=1e-12, abs_tol=1e-12)
        assert math.isclose(c[2], t[4] - 2 * t[3] + t[2], rel_tol=1e-12, abs_tol=1e-12)
        c = prism.inv_root_loss_coeffs(t, 2)
        assert c.size == 5
        ref = [4 * t[3] - 4 * t[2], 6 * t[4] - 10 * t[3] + 4 * t[2], 4 * t[5] - 8 * t[4] + 4 * t[3],
               t[6] - 2 * t[5] + t[4]]
        for k in range(4):
            assert math.isclose(c[k + 1], ref[k], rel_tol=1e-12, abs_tol=1e-12)


@pytest.mark.parametrize("q", [1, 2, 3, 4, 5])
def test_coeffs_equal_direct_loss(q):
    # m(a) from the coefficients = ||S (I - (I + aR)^q (I - R))||_F^2 evaluated directly
    # (R_{k+1} = I - M_{k+1}), R symmetric
    n, p = 40, 8
    A = W.spd_logspaced(n, 1e3, seed=q)
    cq = 2 * np.linalg.norm(A) / (q + 1)
    R = np.eye(n) - A / cq
    S = gaussian_sketch(7, 0, 0, p, n).astype(np.float64)
    c = prism.inv_root_loss_coeffs(prism.sketched_traces(R, S, 2 * q + 2), q)
    for a in (0.05, 0.2, 0.5, 1.0, 1.7):
        Rn = np.eye(n) - np.linalg.matrix_power(np.eye(n) + a * R, q) @ (np.eye(n) - R)
        direct = float(np.sum((S @ Rn) ** 2))
        poly = float(sum(c[i] * a ** i for i in range(c.size)))
        assert abs(poly - direct) <= 1e-9 * max(1.0, abs(direct))


@pytest.mark.parametrize("q", [1, 2, 3, 4])
@pytest.mark.parametrize("fit", ["sketched", "exact"])
def test_inv_root_vs_eigh(q, fit):
    # A^{-1/q} = V diag(lambda^{-1/q}) V^T for SPD A
    A = W.spd_logspaced(64, 1e4, seed=10 + q)
    lam, V = np.linalg.eigh(A)
    ref = (V * lam[None, :] ** (-1.0 / q)) @ V.T
    X, rep = prism.inv_root(A, q=q, tol=1e-11, max_iters=80, fit=fit)
    assert rep.status == prism.CONVERGED
    assert np.linalg.norm(X - ref) / np.linalg.norm(ref) <= 1e-9


@pytest.mark.parametrize("q", [1, 2, 4])
def test_taylor_mode_is_uncoupled_inverse_newton(q):
    # X_{k+1} = ((q+1) X_k - X_k^{q+1} A) / q, from X_0 = I/c
    n = 24
    A = W.spd_logspaced(n, 1e2, seed=q)
    c = (2 * np.linalg.norm(A) / (q + 1)) ** (1.0 / q)
    X = np.eye(n) / c
    for _ in range(5):
        X = ((q + 1) * X - np.linalg.matrix_power(X, q + 1) @ A) / q
    Xo, rep = prism.inv_root(A, q=q, fit="taylor", max_iters=5, tol=1e-300)
    assert rep.iters == 5
    assert np.abs(Xo - X).max() <= 1e-12 * np.abs(X).max()


def test_argmin_poly_companion_vs_grid():
    rng = np.random.default_rng(5)
    grid = np.linspace(0.1, 0.9, 40001)
    for trial in range(300):
        deg = 2 * int(rng.integers(3, 7))
        c = rng.standard_normal(deg + 1)
        c[-1] = abs(c[-1]) + 0.1
        a = prism.argmin_poly(c, 0.1, 0.9, 0.3)
        mg = np.polyval(c[::-1], grid)
        assert np.polyval(c[::-1], a) <= mg.min() + 1e-9 * max(1.0, abs(mg).max())
        assert 0.1 <= a <= 0.9


def test_exact_fit_step_not_worse_than_taylor():
    # exact fit minimises ||R_{k+1}||_F over [l, u], which contains the Taylor a
    for q in (1, 2, 3, 4):
        n = 48
        A = W.spd_logspaced(n, 1e5, seed=20 + q)
        lo, hi, aT = prism.inv_root_interval(q)
        cq = 2 * np.linalg.norm(A) / (q + 1)
        M = A / cq
        for k in range(6):
            R = np.eye(n) - M
            a = prism.argmin_poly(prism.inv_root_loss_coeffs(prism.exact_traces(R, 2 * q + 2), q), lo, hi, aT)

            def nxt(al):
                return np.linalg.matrix_power(np.eye(n) + al * R, q) @ M
            rf = np.linalg.norm(np.eye(n) - nxt(a))
            for al in (lo, aT, hi, 0.5 * (lo + hi)):
                assert rf <= np.linalg.norm(np.eye(n) - nxt(al)) * (1 + 1e-10)
            M = nxt(a)


def test_sketched_close_to_exact_and_faster_than_taylor():
    # P:225 (p = 8 sketch ~ exact fit); PRISM needs fewer iterations than Taylor
    for q in (2, 4):
        A = W.spd_logspaced(96, 1e6, seed=q)
        _, rs = prism.inv_root(A, q=q, tol=1e-9, max_iters=80, fit="sketched")
        _, re = prism.inv_root(A, q=q, tol=1e-9, max_iters=80, fit="exact")
        _, rt = prism.inv_root(A, q=q, tol=1e-9, max_iters=80, fit="taylor")
        assert abs(rs.iters - re.iters) <= 1
        assert rs.iters < rt.iters


def test_zero_input():
    X, rep = prism.inv_root(np.zeros((8, 8)), q=4)
    assert rep.status == prism.ZERO_INPUT and not X.any()
