"""Pins of the PRISM DB Newton oracle (oracle.prism.db_newton, product form, Appendix
A.2 P:466-525): the printed trace-form loss against the direct
||I - M_{k+1}(a)||^2, numpy eigh A^{+-1/2}, the classical two-inverse DB iteration."""

import numpy as np
import pytest

from oracle import prism
from paper_2601_22137_b200 import workloads as W


def _spd(n, kappa, seed):
    return W.spd_logspaced(n, kappa, seed=seed)


@pytest.mark.parametrize("kappa", [1e1, 1e3, 1e6])
def test_coeffs_equal_direct_next_residual(kappa):
    # ||I - M_{k+1}(a)||_F^2 with M_{k+1} = 2a(1-a)I + (1-a)^2 M + a^2 M^{-1}
    n = 30
    M = _spd(n, kappa, seed=int(np.log10(kappa)))
    Mi = np.linalg.inv(M)
    c = prism.db_newton_coeffs(M, Mi)
    for a in (-0.5, 0.0, 0.1, 0.5, 0.9, 1.7):
        Mn = 2 * a * (1 - a) * np.eye(n) + (1 - a) ** 2 * M + a * a * Mi
        direct = float(np.sum((np.eye(n) - Mn) ** 2))
        poly = float(sum(c[i] * a ** i for i in range(5)))
        assert abs(poly - direct) <= 1e-9 * max(1.0, direct)


@pytest.mark.parametrize("kappa", [1e2, 1e6])
@pytest.mark.parametrize("fit", ["exact", "taylor"])
def test_db_newton_vs_eigh(kappa, fit):
    A = _spd(64, kappa, seed=3)
    lam, V = np.linalg.eigh(A)
    sq = (V * np.sqrt(lam)[None, :]) @ V.T
    isq = (V / np.sqrt(lam)[None, :]) @ V.T
    X, Y, rep = prism.db_newton(A, tol=1e-12, max_iters=60, fit=fit)
    assert rep.status == prism.CONVERGED
    assert np.linalg.norm(X - sq) / np.linalg.norm(sq) <= 1e-9
    assert np.linalg.norm(Y - isq) / np.linalg.norm(isq) <= 1e-9 * max(1.0, np.sqrt(kappa) / 10)


def test_taylor_mode_is_classical_db_newton():
    # X_{k+1} = (X + Y^{-1})/2, Y_{k+1} = (Y + X^{-1})/2 (two inverses per step)
    n = 20
    A = _spd(n, 1e2, seed=5)
    X, Y = A.copy(), np.eye(n)
    for _ in range(4):
        X, Y = 0.5 * (X + np.linalg.inv(Y)), 0.5 * (Y + np.linalg.inv(X))
    Xo, Yo, rep = prism.db_newton(A, fit="taylor", max_iters=4, tol=1e-300)
    assert rep.iters == 4
    assert np.abs(Xo - X).max() <= 1e-10 * np.abs(X).max()
    assert np.abs(Yo - Y).max() <= 1e-10 * np.abs(Y).max()


def test_argmin_quartic_free_vs_grid():
    rng = np.random.default_rng(9)
    grid = np.linspace(-6, 6, 240001)
    for _ in range(300):
        c = rng.standard_normal(5)
        c[4] = abs(c[4]) + 0.05
        a = prism.argmin_quartic_free(c, 0.5)
        mg = np.polyval(c[::-1], grid)
        if grid[np.argmin(mg)] in (grid[0], grid[-1]):
            continue   # minimiser outside the grid window
        assert np.polyval(c[::-1], a) <= mg.min() + 1e-9 * max(1.0, abs(mg).max())


def test_exact_fit_beats_taylor_step_and_iterations():
    A = _spd(80, 1e5, seed=7)
    M = A.copy()
    for _ in range(4):
        Mi = np.linalg.inv(M)
        a = prism.argmin_quartic_free(prism.db_newton_coeffs(M, Mi), 0.5)

        def nxt(al):
            return 2 * al * (1 - al) * np.eye(80) + (1 - al) ** 2 * M + al * al * Mi
        assert np.linalg.norm(np.eye(80) - nxt(a)) <= np.linalg.norm(np.eye(80) - nxt(0.5)) * (1 + 1e-12)
        M = nxt(a)
    _, _, re = prism.db_newton(A, tol=1e-10, max_iters=60)
    _, _, rt = prism.db_newton(A, tol=1e-10, max_iters=60, fit="taylor")
    assert re.iters < rt.iters


def test_coupling_and_zero_input():
    A = _spd(32, 1e3, seed=8)
    X, Y, rep = prism.db_newton(A, tol=1e-12, max_iters=60)
    assert np.linalg.norm(X @ Y - np.eye(32)) <= 1e-9 and np.linalg.norm(X @ X - A) <= 1e-9 * np.linalg.norm(A)
    X, Y, rep = prism.db_newton(np.zeros((8, 8)))
    assert rep.status == prism.ZERO_INPUT
