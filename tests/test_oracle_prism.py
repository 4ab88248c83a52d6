"""Pins for the fp64 PRISM oracle (oracle/prism.py) against what the paper
and mathematics fix — never against the oracle itself.

Each test names the pin it uses: paper-printed values (tests/golden/
paper_values.txt), closed forms, textbook special cases, library routines
(numpy SVD / eigh), brute force (grid search), and invariants/theorems.
"""

import math

import numpy as np
import pytest

from oracle import prism
from oracle.philox import gaussian_sketch
from paper_2601_22137_b200 import workloads as W


# ---------------------------------------------------------------- Lemma 1 / Fig 2

def test_lemma1_printed_values():
    # P:692, P:737, P:746, P:754 (tests/golden/paper_values.txt)
    assert prism.h_scalar(0.5, 1.0, 1) == -0.125
    assert abs((1 - prism.h_scalar(0.5, 0.5, 1)) - 25 / 32) < 1e-15
    assert abs((1 - prism.h_scalar(1 / 3, 1.0, 1)) - 32 / 27) < 1e-15
    assert abs((1 - prism.h_scalar(-0.2, 1.0, 1)) - 96 / 125) < 1e-15


def test_lemma1_closed_forms_claim1():
    # P:680 h(x,1/2) = 3/4 x^2 + 1/4 x^3 ; P:684 h(x,1) = -x + x^2 + x^3
    x = np.linspace(-1, 1, 101)
    assert np.allclose(prism.h_scalar(x, 0.5, 1), 0.75 * x ** 2 + 0.25 * x ** 3, atol=1e-15)
    assert np.allclose(prism.h_scalar(x, 1.0, 1), -x + x ** 2 + x ** 3, atol=1e-15)


def test_lemma1_items_1_2_grid():
    # h in [-1/5, x^2] on [1/2,1]x[1/2,1]; in [-1/5, 1/4] on [-1/5,1/2]x[1/2,1]
    a = np.linspace(0.5, 1.0, 201)[None, :]
    x1 = np.linspace(0.5, 1.0, 401)[:, None]
    h1 = prism.h_scalar(x1, a, 1)
    assert np.all(h1 >= -0.2 - 1e-15) and np.all(h1 <= x1 ** 2 + 1e-15)
    x2 = np.linspace(-0.2, 0.5, 401)[:, None]
    h2 = prism.h_scalar(x2, a, 1)
    assert np.all(h2 >= -0.2 - 1e-15) and np.all(h2 <= 0.25 + 1e-15)


def test_lemma1_item3_constant():
    # x_i in [-1/4,1/4], a* = argmin_{[1/2,1]} sum h(x_i,a)^2
    # => max|h(x_i,a*)| <= C max x_i^2 with C < 1.71.  a* from the oracle's
    # exact-trace coefficients (R = diag(x)) and quartic argmin.
    g = np.random.default_rng(5)
    for _ in range(300):
        n = int(g.integers(1, 12))
        x = g.uniform(-0.25, 0.25, n)
        c = prism.loss_coeffs(prism.exact_traces(np.diag(x), 6), 1)
        a = prism.argmin_quartic(c, 0.5, 1.0, 0.5)
        assert 0.5 <= a <= 1.0
        assert np.max(np.abs(prism.h_scalar(x, a, 1))) <= 1.71 * np.max(x ** 2) + 1e-15


def test_fig2_one_step_values():
    # 1 - x1^2 = 3/4 xi^2 + 1/4 xi^3 ~ 1 - 9/4 x0^2 ; P:169 (alpha=1) ~ 1 - 4 x0^2
    x0 = 1e-6
    xi = 1 - x0 * x0
    t = prism.h_scalar(xi, 0.5, 1)
    assert abs(t - (0.75 * xi ** 2 + 0.25 * xi ** 3)) < 1e-15
    assert abs((1 - t) / x0 ** 2 - 9 / 4) < 1e-3
    t1 = prism.h_scalar(xi, 1.0, 1)
    assert abs(t1 - (xi ** 2 + xi ** 3 - xi)) < 1e-15
    assert abs((1 - t1) / x0 ** 2 - 4.0) < 1e-3


def test_matrix_iteration_on_diagonal_is_scalar_recurrence():
    # A diagonal: R_k is diagonal and each entry follows x <- x g_d(1 - x^2)
    sig = np.array([1.0, 0.5, 0.1, 0.01, 1e-3])
    A = np.diag(sig)
    for d in (1, 2):
        Q, rep = prism.polar(A, d=d, fit="taylor", tol=1e-13, max_iters=60)
        x = sig / np.linalg.norm(sig)
        aT = prism.interval(d)[2]
        for _ in range(rep.iters):
            x = x * prism.g_scalar(1 - x * x, aT, d)
        assert np.allclose(np.diag(Q), x, atol=1e-14, rtol=0)
        assert np.allclose(Q, np.diag(np.diag(Q)), atol=0)


# ---------------------------------------------------------------- coefficients

def _direct_sketched_loss(R, S, a, d):
    """|| S (I - (I - R) g_d(R;a)^2) ||_F^2 with explicit matrices (eq. (4))."""
    n = R.shape[0]
    I = np.eye(n)
    G = I + a * R if d == 1 else I + 0.5 * R + a * R @ R
    H = I - (I - R) @ G @ G
    return float(np.sum((S.astype(np.float64) @ H) ** 2))


@pytest.mark.parametrize("d", [1, 2])
def test_coefficients_match_direct_loss(d):
    # the polynomial with the paper's c_i equals the directly
    # evaluated sketched loss at 5 alphas, rel <= 1e-9
    g = np.random.default_rng(11 + d)
    for trial in range(5):
        n = 32
        B = g.standard_normal((n, n))
        R = 0.9 * (B + B.T) / np.linalg.norm(B + B.T, 2)
        S = gaussian_sketch(99, trial, 0, 8, n)
        c = prism.loss_coeffs(prism.sketched_traces(R, S, 4 * d + 2), d)
        for a in (0.3, 0.5, 0.75, 1.0, 1.45):
            poly = sum(c[i] * a ** i for i in range(5))
            ref = _direct_sketched_loss(R, S, a, d)
            assert abs(poly - ref) <= 1e-9 * abs(ref)


@pytest.mark.parametrize("d", [1, 2])
def test_exact_coefficients_match_eigenvalue_form(d):
    # eq. (3): m(a) = sum_i (1 - (1 - l_i) g(l_i;a)^2)^2, l_i from numpy eigvalsh
    g = np.random.default_rng(21 + d)
    B = g.standard_normal((24, 24))
    R = (B + B.T) / np.linalg.norm(B + B.T, 2)
    lam = np.linalg.eigvalsh(R)
    c = prism.loss_coeffs(prism.exact_traces(R, 4 * d + 2), d)
    for a in np.linspace(0.2, 1.6, 8):
        poly = sum(c[i] * a ** i for i in range(5))
        ref = float(np.sum(prism.h_scalar(lam, a, d) ** 2))
        assert abs(poly - ref) <= 1e-9 * max(abs(ref), 1e-300)


def test_sketched_traces_identity_and_zero():
    # R = I -> t_i = tr(S S^T); R = 0 -> t_i = 0 for i >= 1 (S: sketched_power_traces)
    S = gaussian_sketch(1, 0, 0, 5, 20).astype(np.float64)
    t = prism.sketched_traces(np.eye(20), S, 6)
    assert np.allclose(t, np.sum(S * S), rtol=1e-14)
    t0 = prism.sketched_traces(np.zeros((20, 20)), S, 6)
    assert np.all(t0[1:] == 0)


def test_sketched_traces_vs_dense_powers():
    g = np.random.default_rng(8)
    B = g.standard_normal((32, 32))
    R = (B + B.T) / 16
    S = gaussian_sketch(5, 0, 0, 8, 32).astype(np.float64)
    t = prism.sketched_traces(R, S, 10)
    P = np.eye(32)
    for i in range(11):
        assert abs(t[i] - np.trace(S @ P @ S.T)) <= 1e-10 * max(1.0, abs(t[i]))
        P = P @ R


# ---------------------------------------------------------------- argmin

def _beta(lam, d):
    # closed form of the perfect fit (1-l) g_d(l;a)^2 = 1 for a single eigenvalue
    if d == 1:
        return (1 / math.sqrt(1 - lam) - 1) / lam              # P:856 beta(M)
    return ((1 - lam) ** -0.5 - 1 - lam / 2) / lam ** 2


@pytest.mark.parametrize("d", [1, 2])
def test_argmin_single_eigenvalue_closed_form(d):
    lo, hi, aT = prism.interval(d)
    for lam in (0.05, 0.2, 0.4, 0.6, 0.8, 0.95, 0.999):
        R = lam * np.eye(6)
        _, c = prism.fit_alpha(R, d, "exact", None, lo, hi, aT)
        a = prism.argmin_quartic(c, lo, hi, aT)
        want = min(max(_beta(lam, d), lo), hi)
        assert abs(a - want) < 1e-7, (lam, a, want)


def test_argmin_simple_quadratics():
    # (a - 0.7)^2 on [0.5, 1] -> 0.7 ; (a - 2)^2 on [0.5, 1] -> 1 (S: minimize_quartic examples)
    assert abs(prism.argmin_quartic([0.49, -1.4, 1.0, 0, 0], 0.5, 1.0, 0.5) - 0.7) < 1e-14
    assert prism.argmin_quartic([4.0, -4.0, 1.0, 0, 0], 0.5, 1.0, 0.5) == 1.0
    # degenerate (constant) loss -> Taylor coefficient
    assert prism.argmin_quartic([3.0, 0, 0, 0, 0], 0.375, 1.45, 0.375) == 0.375


def test_argmin_against_grid():
    g = np.random.default_rng(2)
    lo, hi = 0.375, 1.45
    grid = np.linspace(lo, hi, 4097)
    for _ in range(2000):
        c = g.standard_normal(5) * 10.0 ** g.uniform(-6, 3, 5)
        if g.random() < 0.5:
            c[4] = abs(c[4])
        a = prism.argmin_quartic(c, lo, hi, 0.375)
        assert lo <= a <= hi
        mv = lambda x: c[1] * x + c[2] * x ** 2 + c[3] * x ** 3 + c[4] * x ** 4  # noqa: E731
        gmin = np.min(mv(grid))
        scale = np.max(np.abs(c[1:]))
        assert mv(a) <= gmin + 1e-12 * scale
        assert mv(a) <= mv(lo) + 1e-15 * scale and mv(a) <= mv(hi) + 1e-15 * scale


def test_cubic_roots_known():
    g = np.random.default_rng(4)
    for _ in range(500):
        r = np.sort(g.uniform(-3, 3, 3))
        a3 = g.uniform(0.5, 2) * (1 if g.random() < 0.5 else -1)
        co = a3 * np.poly(r)  # a3 x^3 + a2 x^2 + a1 x + a0
        got = np.sort(prism._real_roots_cubic(*co))
        if np.min(np.diff(r)) > 1e-3:
            assert len(got) == 3
            assert np.allclose(got, r, atol=1e-6)


# ---------------------------------------------------------------- whole iteration

def _equal_sigma_trajectory(s, d, tol):
    """Independent scalar recurrence for A = c Q (all sigma equal): R_k = l_k I,
    l_0 = 1 - 1/s, a_k = clamp(beta_d(l_k)), l_{k+1} = 1 - (1-l)(g_d(l;a))^2."""
    lo, hi, _ = prism.interval(d)
    lam = 1.0 - 1.0 / s
    alphas = []
    while abs(lam) * math.sqrt(s) > tol * math.sqrt(s):
        a = min(max(_beta(lam, d), lo), hi)
        alphas.append(a)
        g = 1 + a * lam if d == 1 else 1 + 0.5 * lam + a * lam * lam
        lam = 1 - (1 - lam) * g * g
        if len(alphas) > 60:
            break
    return alphas


@pytest.mark.parametrize("d,s,m", [(1, 32, 64), (2, 32, 64), (2, 256, 256), (1, 256, 512)])
def test_equal_sigma_closed_form(d, s, m):
    A = W.equal_sigma(m, s, 3.7, seed=1)
    Q, rep = prism.polar(A, d=d, p=8, tol=1e-12, max_iters=40, seed=42)
    want = _equal_sigma_trajectory(s, d, 1e-12)
    assert rep.status == prism.CONVERGED
    assert rep.iters == len(want)
    assert np.allclose(rep.alphas, want, atol=1e-6)
    assert np.linalg.norm(Q - A / 3.7) < 1e-10


def test_equal_sigma_survey_counts():
    # SURVEY App.N10 (scalar recurrence): d=1 s=32 -> 3, d=2 s=32 -> 2, d=2 s=768 -> 4
    assert len(_equal_sigma_trajectory(32, 1, 1e-12)) == 3
    assert len(_equal_sigma_trajectory(32, 2, 1e-12)) == 2
    tr = _equal_sigma_trajectory(768, 2, 1e-12)
    assert len(tr) == 4 and abs(tr[0] - 1.45) < 1e-15 and abs(tr[3] - 0.5229) < 1e-4


@pytest.mark.parametrize("shape", [(40, 24), (24, 40), (30, 30)])
@pytest.mark.parametrize("d", [1, 2])
def test_polar_limit_vs_svd(shape, d):
    A = W.gaussian(*shape, seed=3)
    Q, rep = prism.polar(A, d=d, p=8, tol=1e-13, max_iters=80, seed=1)
    U, _, Vt = np.linalg.svd(A, full_matrices=False)
    assert rep.status == prism.CONVERGED
    assert np.linalg.norm(Q - U @ Vt) < 1e-10
    s = min(shape)
    G = Q.T @ Q if shape[0] >= shape[1] else Q @ Q.T
    assert np.linalg.norm(G - np.eye(s)) < 1e-11


@pytest.mark.parametrize("d", [1, 2])
@pytest.mark.parametrize("kappa", [1e2, 1e4])
def test_sqrt_vs_eigh(d, kappa):
    A = 3.0 * W.spd_logspaced(32, kappa, seed=4)
    X, Y, rep = prism.sqrt_invsqrt(A, d=d, p=8, tol=1e-12, max_iters=80, seed=3)
    lam, V = np.linalg.eigh(A)
    sq = (V * np.sqrt(lam)) @ V.T
    isq = (V / np.sqrt(lam)) @ V.T
    assert rep.status == prism.CONVERGED
    assert np.linalg.norm(X - sq) / np.linalg.norm(sq) < 1e-10
    assert np.linalg.norm(Y - isq) / np.linalg.norm(isq) < 1e-8
    assert np.linalg.norm(X @ Y - np.eye(32)) < 1e-9


def test_taylor_mode_is_classical_newton_schulz():
    # textbook NS (Higham): d=1: 3/2 X - 1/2 X X^T X ; d=2: X(15/8 I - 5/4 G + 3/8 G^2)
    A = W.gaussian(20, 12, seed=9)
    X0 = A / np.linalg.norm(A)
    G = X0.T @ X0
    one = 1.5 * X0 - 0.5 * X0 @ G
    two = X0 @ (15 / 8 * np.eye(12) - 5 / 4 * G + 3 / 8 * G @ G)
    Q1, r1 = prism.polar(A, d=1, fit="taylor", max_iters=1, tol=1e-30)
    Q2, r2 = prism.polar(A, d=2, fit="taylor", max_iters=1, tol=1e-30)
    assert r1.iters == 1 and r2.iters == 1
    assert np.allclose(Q1, one, atol=1e-15) and np.allclose(Q2, two, atol=1e-15)


@pytest.mark.parametrize("d", [1, 2])
def test_exact_fit_residual_non_increasing(d):
    # the minimiser never increases ||R||_F (alpha_T is a feasible candidate
    # at least as good as Taylor, and Taylor contracts on [0,1) spectra)
    A = W.logspaced(48, 32, 1e-4, seed=2)
    _, rep = prism.polar(A, d=d, fit="exact", tol=1e-13, max_iters=60)
    r = np.array(rep.resid)
    assert np.all(np.diff(r) <= 1e-15)


def test_theorem1_bound_d1_exact():
    # P:199 (Theorem 1, via Theorem 4 P:277-279 for polar): ||R_k||_2 <= ||R_0||_2^(2^(k-2))
    for seed in range(5):
        A = W.logspaced(40, 24, 10 ** -(seed + 1), seed=seed)
        X = A / np.linalg.norm(A)
        r0 = np.linalg.norm(np.eye(24) - X.T @ X, 2)
        for k in range(2, 30):
            Q, rep = prism.polar(A, d=1, fit="exact", tol=1e-300, max_iters=k)
            rk = np.linalg.norm(np.eye(24) - Q.T @ Q, 2)
            bound = r0 ** (2.0 ** (k - 2))
            assert rk <= bound + 1e-13
            if rk < 1e-13:
                break


def test_theorem2_bound_d1_sketched():
    # P:229 (Theorem 2, empirical at p = 8): ||R_k||_2 <= ||R_0||_2^(2^(k-3)) w.h.p.
    fails = 0
    for seed in range(20):
        A = W.logspaced(40, 24, 1e-3, seed=100 + seed)
        X = A / np.linalg.norm(A)
        r0 = np.linalg.norm(np.eye(24) - X.T @ X, 2)
        Q, rep = prism.polar(A, d=1, p=8, seed=seed, tol=1e-300, max_iters=12)
        X = A / np.linalg.norm(A)
        ok = True
        for k, a in enumerate(rep.alphas):
            X = X @ (np.eye(24) + a * (np.eye(24) - X.T @ X))
            rk = np.linalg.norm(np.eye(24) - X.T @ X, 2)
            if k + 1 >= 3 and rk > r0 ** (2.0 ** (k + 1 - 3)) + 1e-13:
                ok = False
        fails += not ok
    assert fails <= 1


@pytest.mark.parametrize("d", [1, 2])
def test_sketched_close_to_exact(d):
    # S: |a_sketch - a_exact| <= 0.15 in >= 90% of steps, counts within +-1
    close = total = 0
    for seed in range(6):
        A = W.gaussian(96, 64, seed=seed)
        _, re = prism.polar(A, d=d, fit="exact", tol=1e-8, max_iters=60)
        _, rs = prism.polar(A, d=d, fit="sketched", p=8, seed=seed, tol=1e-8, max_iters=60)
        assert abs(re.iters - rs.iters) <= 1
        # compare alpha on the same residuals: refit exact on the sketched path's R_k
        X = A / np.linalg.norm(A)
        lo, hi, aT = prism.interval(d)
        for k, a in enumerate(rs.alphas):
            R = np.eye(64) - X.T @ X
            ae, _ = prism.fit_alpha(R, d, "exact", None, lo, hi, aT)
            close += abs(ae - a) <= 0.15
            total += 1
            X = X @ prism.g_matrix(R, a, d)
    assert close >= 0.9 * total


def test_warmup_and_status_codes():
    A = W.gaussian(30, 20, seed=1)
    _, rep = prism.polar(A, d=2, warmup=3, tol=1e-10, max_iters=30)
    assert rep.alphas[:3] == [1.45, 1.45, 1.45]
    _, rep = prism.polar(np.zeros((5, 3)))
    assert rep.status == prism.ZERO_INPUT
    v = W.haar(12, 1, seed=3)             # ||v||_F = 1: X_0 = v, R_0 = 0 (R10)
    Q, rep = prism.polar(5.0 * v, tol=1e-12)
    assert rep.iters == 0 and rep.status == prism.CONVERGED and np.allclose(Q, v)
    _, rep = prism.polar(A, d=2, tol=1e-14, max_iters=2)
    assert rep.status == prism.MAX_ITERS and rep.iters == 2 and len(rep.resid) == 3


def test_sqrt_non_spd_diverges_exactly_as_the_scalar_recurrence():
    # A diagonal A keeps every iterate diagonal, so the Taylor-mode coupled iteration is one
    # scalar recurrence per eigenvalue (P:246-250 with g_2(r) = 1 + r/2 + 3/8 r^2):
    # x_0 = lambda / ||A||_F, y_0 = 1, r = 1 - y x, x <- x g(r), y <- g(r) y.  The negative
    # eigenvalue makes ||R_k||_F grow at every step, so the DIVERGED rule (5 consecutive
    # increases) stops it at k = 5, with the residual history of the recurrence.
    lam = [1.0, 0.5, -0.3, 0.2]
    A = np.diag(lam)
    c = math.sqrt(sum(v * v for v in lam))
    x, y = [v / c for v in lam], [1.0] * 4
    hist = []
    for _ in range(6):
        r = [1.0 - yi * xi for xi, yi in zip(x, y)]
        hist.append(math.sqrt(sum(v * v for v in r)) / 2.0)      # ||R||_F / sqrt(s), s = 4
        g = [1.0 + 0.5 * v + 0.375 * v * v for v in r]
        x = [xi * gi for xi, gi in zip(x, g)]
        y = [gi * yi for gi, yi in zip(g, y)]
    assert all(b > a for a, b in zip(hist, hist[1:]))
    for fit in ("taylor", "sketched"):
        _, _, rep = prism.sqrt_invsqrt(A, d=2, tol=1e-10, max_iters=40, fit=fit)
        assert rep.status == prism.DIVERGED and rep.iters == 5, fit
        np.testing.assert_allclose(rep.resid, hist, rtol=1e-12)
    # PRISM-3 (d = 1, g_1(r) = 1 + r/2) on a 64 x 64 diagonal: ||R_k|| first falls, then
    # grows five times in a row from k = 5, staying finite in fp32 (the device test's case)
    lam64 = [1.0, 0.5, -0.03, 0.2] * 16
    c = math.sqrt(sum(v * v for v in lam64))
    x, y = [v / c for v in lam64], [1.0] * 64
    hist = []
    for _ in range(10):
        r = [1.0 - yi * xi for xi, yi in zip(x, y)]
        hist.append(math.sqrt(sum(v * v for v in r)) / 8.0)
        x = [xi * (1.0 + 0.5 * v) for xi, v in zip(x, r)]
        y = [(1.0 + 0.5 * v) * yi for v, yi in zip(r, y)]
    assert hist[5] > hist[4] and all(b > a for a, b in zip(hist[4:], hist[5:]))
    _, _, rep = prism.sqrt_invsqrt(np.diag(lam64), d=1, tol=1e-10, max_iters=40, fit="taylor")
    assert rep.status == prism.DIVERGED and rep.iters == 9
    np.testing.assert_allclose(rep.resid, hist, rtol=1e-12)
    # the counter restarts after a decrease: 4 increases, a drop, 4 increases never diverge
    rep, incr, r_prev = prism.Report(), 0, math.inf
    for k, r in enumerate([1, 2, 3, 4, 5, 0.5, 1, 2, 3, 4]):
        stop, incr = prism._status_update(rep, k, float(r), r_prev, 1, 1e-12, 40, incr)
        r_prev = float(r)
        assert not stop, k
    stop, incr = prism._status_update(rep, 10, 5.0, r_prev, 1, 1e-12, 40, incr)
    assert stop and rep.status == prism.DIVERGED


def test_sqrt_iterates_commute():
    # Theorem 3: X_k, Y_k are polynomials in A, so X_k Y_k = Y_k X_k
    A = W.wishart(24, 2.0, seed=5)
    for iters in (1, 2, 4):
        X, Y, _ = prism.sqrt_invsqrt(A, d=2, tol=1e-300, max_iters=iters)
        assert np.linalg.norm(X @ Y - Y @ X) <= 1e-12 * np.linalg.norm(X) * np.linalg.norm(Y)


# ---------------------------------------------------------------- matrix sign
def _sym_indefinite(n, seed, lo=1e-3):
    """Q diag(lam) Q^T with |lam| log-spaced in [lo, 1] and alternating signs."""
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.logspace(0, np.log10(lo), n) * np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    return (Q * lam[None, :]) @ Q.T


@pytest.mark.parametrize("d", [1, 2])
def test_sign_vs_eigh(d):
    # sign(A) = V sign(Lambda) V^T for symmetric A (definition P:145 with A^2 = A^T A)
    A = _sym_indefinite(40, seed=d)
    lam, V = np.linalg.eigh(A)
    ref = (V * np.sign(lam)[None, :]) @ V.T
    S, rep = prism.sign(A, d=d, p=8, tol=1e-12, max_iters=80)
    assert rep.status == prism.CONVERGED
    assert np.linalg.norm(S - ref) / np.linalg.norm(ref) <= 1e-10


def test_sign_taylor_mode_is_classical_newton_schulz():
    # textbook Newton-Schulz for the sign (Higham 2008, eq. 5.22): X (3I - X^2) / 2
    A = _sym_indefinite(16, seed=3, lo=0.05)
    X = A / np.linalg.norm(A)
    for _ in range(3):
        X = 0.5 * X @ (3 * np.eye(16) - X @ X)
    S, rep = prism.sign(A, d=1, fit="taylor", max_iters=3, tol=1e-300)
    assert rep.iters == 3 and np.allclose(S, X, atol=1e-14)


def test_sign_theorem1_bound_d1_exact():
    # Theorem 1: d = 1, exact fit on [1/2, 1]: ||I - X_k^2||_2 <= ||I - A^2||_2^(2^(k-2))
    for seed in range(4):
        A = _sym_indefinite(30, seed=10 + seed, lo=10.0 ** -(seed + 1))
        X0 = A / np.linalg.norm(A)
        r0 = np.linalg.norm(np.eye(30) - X0 @ X0, 2)
        for k in range(2, 40):
            S, rep = prism.sign(A, d=1, fit="exact", tol=1e-300, max_iters=k)
            rk = np.linalg.norm(np.eye(30) - S @ S, 2)
            assert rk <= r0 ** (2.0 ** (k - 2)) + 1e-13
            if rk < 1e-13:
                break


def test_sign_block_matrix_gives_square_roots():
    # for X_0 = [[0, A], [I, 0]] (A SPD; X_0^2 symmetric),
    # sign(X_0) = [[0, A^{1/2}], [A^{-1/2}, 0]]
    n = 12
    A = W.spd_logspaced(n, 1e2, seed=4)
    Z = np.zeros((n, n))
    X0 = np.block([[Z, A], [np.eye(n), Z]])
    S, rep = prism.sign(X0, d=2, p=8, tol=1e-12, max_iters=80)
    lam, V = np.linalg.eigh(A)
    sq = (V * np.sqrt(lam)[None, :]) @ V.T
    isq = (V / np.sqrt(lam)[None, :]) @ V.T
    assert rep.status == prism.CONVERGED
    assert np.abs(S[:n, :n]).max() < 1e-10 and np.abs(S[n:, n:]).max() < 1e-10
    assert np.linalg.norm(S[:n, n:] - sq) / np.linalg.norm(sq) <= 1e-9
    assert np.linalg.norm(S[n:, :n] - isq) / np.linalg.norm(isq) <= 1e-9


def test_sign_zero_input():
    S, rep = prism.sign(np.zeros((8, 8)))
    assert rep.status == prism.ZERO_INPUT and not S.any()


def test_argmin_badly_scaled_cubic_against_dense_grid():
    """Regression pin (R16): quartics whose c4 is ~1e-10 of c3 — the closed-form Cardano
    roots lost the moderate root and the argmin returned an interval end with a larger
    loss.  The argmin must match a 200001-point brute-force grid."""
    cases = [([19.544087647012184, -44.43517630092626, -114.43158552440468, 132.84099703384126,
               1.5172433851677812e-08], 0.375, 1.45),
             ([19.544087647012184, -44.43517630092626, -114.43158552440468, 132.84099703384126,
               1.5172433851677812e-08], 0.5, 1.0),
             ([3.4403680645019565e-08, 6.009257289921177e-07, -8.716852875631071, 4.452838746516632,
               1.0848522704284619e-08], 0.375, 1.45)]
    for c, lo, hi in cases:
        c = np.array(c)
        m = lambda x: c[1] * x + c[2] * x ** 2 + c[3] * x ** 3 + c[4] * x ** 4  # noqa: E731
        xs = np.linspace(lo, hi, 200001)
        a = prism.argmin_quartic(c, lo, hi, lo)
        assert lo <= a <= hi
        assert m(a) <= m(xs).min() + 1e-12 * np.max(np.abs(c[1:]))
        assert abs(a - xs[np.argmin(m(xs))]) <= 2 * (hi - lo) / 200000


def test_argmin_against_companion_roots():
    """Pin of argmin_quartic (R16) by an independent method: the critical points as
    the eigenvalues of the companion matrix of m'(a) (numpy.roots), the interval ends, and
    the smallest loss among them.  The oracle's argmin splits [lo, hi] at the roots of m''
    and bisects m' (the same design as the device's), so this shares nothing with it; the
    two must reach the same minimal loss (the minimiser itself may differ on flat ties)."""
    g = np.random.default_rng(7)
    for lo, hi in ((0.375, 1.45), (0.5, 1.0)):
        for _ in range(3000):
            c = g.standard_normal(5) * 10.0 ** g.uniform(-8, 3, 5)
            if g.random() < 0.6:
                c[4] = abs(c[4])
            scale = float(np.max(np.abs(c[1:])))
            m = lambda x: c[1] * x + c[2] * x ** 2 + c[3] * x ** 3 + c[4] * x ** 4  # noqa: E731
            cands = [lo, hi]
            for r in np.roots([4.0 * c[4], 3.0 * c[3], 2.0 * c[2], c[1]]):
                if abs(r.imag) <= 1e-7 * (1.0 + abs(r.real)) and lo <= r.real <= hi:
                    cands.append(float(r.real))
            best = min(m(x) for x in cands)
            a = prism.argmin_quartic(c, lo, hi, lo)
            assert lo <= a <= hi
            assert m(a) <= best + 1e-11 * scale, (c.tolist(), lo, hi, a, m(a), best)
