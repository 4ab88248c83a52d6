"""Pins of the PRISM Chebyshev inverse oracle (oracle.prism.chebyshev_inverse, Appendix
A.4 P:596-629): the printed trace-form coefficients (symmetric R), the
next-residual identity of the loss, numpy's inverse, the textbook Chebyshev recurrence."""

import math

import numpy as np
import pytest

from oracle import prism
from oracle.philox import gaussian_sketch
from paper_2601_22137_b200 import workloads as W


def test_coeffs_match_printed_trace_form_symmetric():
    # P:622-627 (valid for symmetric R): c1 = -2 t4 + 2 t5, c2 = t4 - 2 t5 + t6
    n, p = 50, 8
    A = W.spd_logspaced(n, 1e2, seed=1)
    R = np.eye(n) - A / np.linalg.norm(A, 2)
    S = gaussian_sketch(3, 0, 0, p, n).astype(np.float64)
    t = prism.sketched_traces(R, S, 6)
    c = prism.chebyshev_loss_coeffs(R, S)
    assert math.isclose(c[1], -2 * t[4] + 2 * t[5], rel_tol=1e-10, abs_tol=1e-12)
    assert math.isclose(c[2], t[4] - 2 * t[5] + t[6], rel_tol=1e-10, abs_tol=1e-12)
    assert math.isclose(c[0], t[4], rel_tol=1e-10)


@pytest.mark.parametrize("sketched", [True, False])
def test_loss_is_next_residual_general_A(sketched):
    # m(a) = ||S R_{k+1}(a)||_F^2 with R_{k+1} = I - A X_k (I + R_k + a R_k^2) computed directly
    n, p = 40, 8
    A = W.gaussian(n, n, seed=2)
    An = A / np.linalg.norm(A)
    X = An.T.copy()
    for _ in range(3):
        X = X @ (2 * np.eye(n) - An @ X)   # move away from X_0 (any X works for the identity)
    R = np.eye(n) - An @ X
    S = gaussian_sketch(5, 1, 2, p, n).astype(np.float64) if sketched else None
    c = prism.chebyshev_loss_coeffs(R, S)
    for a in (0.3, 0.5, 1.0, 1.5, 2.0):
        Rn = np.eye(n) - An @ X @ (np.eye(n) + R + a * R @ R)
        direct = float(np.sum(((S @ Rn) if sketched else Rn) ** 2))
        assert abs(c[0] + c[1] * a + c[2] * a * a - direct) <= 1e-10 * max(1.0, direct)


@pytest.mark.parametrize("kind", ["gaussian", "logspaced", "spd"])
@pytest.mark.parametrize("fit", ["sketched", "exact"])
def test_chebyshev_vs_numpy_inverse(kind, fit):
    n = 64
    A = {"gaussian": W.gaussian(n, n, seed=7), "logspaced": W.logspaced(n, n, 1e-2, seed=8),
         "spd": W.spd_logspaced(n, 1e3, seed=9)}[kind]
    Ainv, rep = prism.chebyshev_inverse(A, tol=1e-12, max_iters=80, fit=fit)
    assert rep.status == prism.CONVERGED
    ref = np.linalg.inv(A)
    assert np.linalg.norm(Ainv - ref) / np.linalg.norm(ref) <= 1e-9


def test_taylor_mode_is_textbook_chebyshev():
    # X_{k+1} = 3X - 3XAX + XAXAX from X_0 = A^T (normalised A)
    n = 24
    A = W.logspaced(n, n, 0.2, seed=3)
    An = A / np.linalg.norm(A)
    X = An.T.copy()
    for _ in range(6):
        XA = X @ An
        X = 3 * X - 3 * XA @ X + XA @ XA @ X
    Xo, rep = prism.chebyshev_inverse(A, fit="taylor", max_iters=6, tol=1e-300)
    assert rep.iters == 6
    assert np.abs(Xo * np.linalg.norm(A) - X).max() <= 1e-12 * np.abs(X).max()


def test_exact_fit_step_minimises_next_residual():
    n = 48
    A = W.logspaced(n, n, 1e-2, seed=4)
    An = A / np.linalg.norm(A)
    X = An.T.copy()
    lo, hi, aT = prism.chebyshev_interval()
    for _ in range(8):
        R = np.eye(n) - An @ X
        a = prism.argmin_quartic(np.concatenate([prism.chebyshev_loss_coeffs(R, None), [0, 0]]), lo, hi, aT)

        def nxt(al):
            return X @ (np.eye(n) + R + al * R @ R)
        best = np.linalg.norm(np.eye(n) - An @ nxt(a))
        for al in np.linspace(lo, hi, 31):
            assert best <= np.linalg.norm(np.eye(n) - An @ nxt(al)) * (1 + 1e-10)
        X = nxt(a)


def test_prism_fewer_iterations_than_taylor_and_sketch_close():
    A = W.logspaced(96, 96, 1e-3, seed=5)
    _, rs = prism.chebyshev_inverse(A, tol=1e-9, max_iters=100, fit="sketched")
    _, re = prism.chebyshev_inverse(A, tol=1e-9, max_iters=100, fit="exact")
    _, rt = prism.chebyshev_inverse(A, tol=1e-9, max_iters=100, fit="taylor")
    assert abs(rs.iters - re.iters) <= 1 and rs.iters < rt.iters


def test_zero_input():
    X, rep = prism.chebyshev_inverse(np.zeros((8, 8)))
    assert rep.status == prism.ZERO_INPUT and not X.any()
