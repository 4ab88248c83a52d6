"""PRISM Newton–Schulz iterations in fp64 — TEST INFRASTRUCTURE ONLY.

Plain transcription of the paper (arXiv 2601.22137, /root/reference/PAPER.md,
``P:<line>``).  Every step below follows the paper's order and notation;
library primitives (numpy matmul) are used as steps, with no blocking, fusion
or reordering.  Where the paper is silent or garbled, the DESIGN.md reading
(R1..R20) named in the comment is used.

Polar (Table 1 rows P:252-254; Appendix A.1):
    X_0 = A/||A||_F (R10)
    R_k = I - X_k^T X_k
    X_{k+1} = X_k g_d(R_k; a_k),  g_1 = I + a R,  g_2 = I + R/2 + a R^2
Coupled square root (Table 1 rows P:246-250, Theorem 3; R11):
    X_0 = A/||A||_F, Y_0 = I, R_k = I - Y_k X_k
    X_{k+1} = X_k g_d(R_k; a_k),  Y_{k+1} = g_d(R_k; a_k) Y_k
    A^{1/2} ~ sqrt(c) X,  A^{-1/2} ~ Y / sqrt(c)
Matrix sign (the paper's case study, eq. 2; A^2 symmetric):
    X_0 = A/||A||_F, R_k = I - X_k^2, X_{k+1} = X_k g_d(R_k; a_k)
Coupled inverse Newton A^{-1/q} (Appendix A.3; q = the paper's p):
    c = (2||A||_F/(q+1))^{1/q}, X_0 = I/c, M_0 = A/c^q, R_k = I - M_k
    X_{k+1} = X_k (I + a_k R_k),  M_{k+1} = (I + a_k R_k)^q M_k
    loss of degree 2q, argmin analytic for q <= 2, companion-matrix
    roots of m' for q >= 3; interval [1/(2q), 2/q] (R22).
Chebyshev inverse A^{-1} (Appendix A.4):
    A' = A/||A||_F, X_0 = A'^T, R_k = I - A' X_k, X_{k+1} = X_k (I + R_k + a_k R_k^2),
    a_k = argmin_{[1/2,2]} ||S_k (R_k^2 - a (R_k^2 - R_k^3))||_F^2 (quadratic; R25, R26).
DB Newton, product form (Appendix A.2), SPD A:
    M_0 = X_0 = A, Y_0 = I, M_{k+1} = 2a(1-a)I + (1-a)^2 M_k + a^2 M_k^{-1},
    X_{k+1} = (1-a)X_k + a X_k M_k^{-1}, Y likewise; a = unconstrained argmin of the
    exact quartic ||I - M_{k+1}||_F^2 (trace form, no sketch; R27, R28).
Coefficient a_k (eq. (4)):
    a_k = argmin_{a in [l,u]} || S_k (I - (I-R_k) g_d(R_k;a)^2) ||_F^2
        = argmin m(a),  m(a) = c0 + c1 a + c2 a^2 + c3 a^3 + c4 a^4
    with c_i linear in t_i = tr(S_k R_k^i S_k^T), the t_i from
    the chain S R(...(R(R S^T))), and the argmin from the real
    roots of the cubic m'(a) = 0.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .philox import gaussian_sketch

# status codes (shared meaning with include/prism.h, defined independently)
CONVERGED, MAX_ITERS, DIVERGED, NONFINITE, ZERO_INPUT = 0, 1, 2, 3, 4

FIT_SKETCHED, FIT_TAYLOR, FIT_EXACT = "sketched", "taylor", "exact"


def interval(d: int) -> tuple[float, float, float]:
    """(l, u, a_Taylor) for degree parameter d.

    d=1: [1/2, 1] (the "[1, 1/2]" of P:454/P:461 is read
    as [1/2, 1], R2); Taylor coefficient 1/2 = binomial coefficient of xi in
    (1-xi)^{-1/2}.  d=2: [3/8, 29/20]; Taylor 3/8 (R3).
    """
    if d == 1:
        return 0.5, 1.0, 0.5
    if d == 2:
        return 0.375, 1.45, 0.375
    raise ValueError("d must be 1 or 2")


# --------------------------------------------------------------------------
# scalar forms
# --------------------------------------------------------------------------

def g_scalar(xi, alpha, d: int):
    """g_d(xi; a) = f_{d-1}(xi) + a xi^d with f_0 = 1, f_1 = 1 + xi/2."""
    if d == 1:
        return 1.0 + alpha * xi
    return 1.0 + 0.5 * xi + alpha * xi * xi


def h_scalar(xi, alpha, d: int):
    """Next residual eigenvalue: 1 - (1 - xi) g_d(xi; a)^2 (eq. (3)).

    For d=1 this is Lemma 1's h(x, a) = 1 - (1-x)(1+a x)^2.
    """
    g = g_scalar(xi, alpha, d)
    return 1.0 - (1.0 - xi) * g * g


# --------------------------------------------------------------------------
# matrix pieces
# --------------------------------------------------------------------------

def g_matrix(R: np.ndarray, alpha: float, d: int) -> np.ndarray:
    """g_d(R; a) as a matrix (Table 1 'Iteration' column)."""
    n = R.shape[0]
    I = np.eye(n)
    if d == 1:
        return I + alpha * R
    return I + 0.5 * R + alpha * (R @ R)


def sketched_traces(R: np.ndarray, S: np.ndarray, imax: int) -> np.ndarray:
    """t_i = tr(S R^i S^T), i = 0..imax, by the chain of P:442-446.

    V_0 = S^T, V_i = R V_{i-1}, t_i = <S^T, V_i>_F: imax products of an
    n x n by an n x p matrix, never an n x n by n x n product.
    """
    St = S.T.astype(np.float64)
    V = St.copy()
    t = np.zeros(imax + 1)
    t[0] = float(np.sum(St * V))
    for i in range(1, imax + 1):
        V = R @ V
        t[i] = float(np.sum(St * V))
    return t


def exact_traces(R: np.ndarray, imax: int) -> np.ndarray:
    """t_i = tr(R^i) (the unsketched eq. (3); S = I)."""
    n = R.shape[0]
    P = np.eye(n)
    t = np.zeros(imax + 1)
    t[0] = float(n)
    for i in range(1, imax + 1):
        P = P @ R
        t[i] = float(np.trace(P))
    return t


def loss_coeffs(t: np.ndarray, d: int) -> np.ndarray:
    """(c0, c1, c2, c3, c4) of m(a) from the trace table t.

    d=1, d=2.  c0 is not printed ("c_5" typo);
    derived as c0 = t2 (d=1) and 9/16 t4 + 3/8 t5 + 1/16 t6 (d=2) (R18).
    """
    if d == 1:
        c0 = t[2]
        c1 = 4 * t[3] - 4 * t[2]
        c2 = 6 * t[4] - 10 * t[3] + 4 * t[2]
        c3 = 4 * t[5] - 8 * t[4] + 4 * t[3]
        c4 = t[6] - 2 * t[5] + t[4]
    else:
        c0 = 9.0 / 16.0 * t[4] + 3.0 / 8.0 * t[5] + 1.0 / 16.0 * t[6]
        c1 = 0.5 * t[7] + 2 * t[6] + 0.5 * t[5] - 3 * t[4]
        c2 = 1.5 * t[8] + 3 * t[7] - 4.5 * t[6] - 4 * t[5] + 4 * t[4]
        c3 = 2 * t[9] - 6 * t[7] + 4 * t[6]
        c4 = t[10] - 2 * t[9] + t[8]
    return np.array([c0, c1, c2, c3, c4], dtype=np.float64)


def _real_roots_cubic(a3: float, a2: float, a1: float, a0: float) -> list[float]:
    """Real roots of a3 x^3 + a2 x^2 + a1 x + a0 (closed form, R16).

    Degrades to the quadratic / linear case when the leading coefficient is
    negligible (|a3| <= 1e-12 max(|a2|,|a1|,|a0|)); quadratic via the stable
    q = -(b + sign(b) sqrt(disc))/2 form; cubic via the depressed form with
    the trigonometric branch for three real roots and Cardano otherwise.
    """
    big = max(abs(a2), abs(a1), abs(a0))
    if abs(a3) <= 1e-12 * big:
        if abs(a2) <= 1e-12 * max(abs(a1), abs(a0)):
            return [-a0 / a1] if a1 != 0.0 else []
        disc = a1 * a1 - 4.0 * a2 * a0
        if disc < 0.0:
            return []
        sq = math.sqrt(disc)
        q = -0.5 * (a1 + (sq if a1 >= 0.0 else -sq))
        roots = [q / a2]
        if q != 0.0:
            roots.append(a0 / q)
        return roots
    b, c, d = a2 / a3, a1 / a3, a0 / a3
    p = c - b * b / 3.0
    q = 2.0 * b * b * b / 27.0 - b * c / 3.0 + d
    shift = -b / 3.0
    disc = (q / 2.0) ** 2 + (p / 3.0) ** 3
    if disc > 0.0:
        sq = math.sqrt(disc)
        A = -math.copysign(1.0, q) * math.pow(abs(q) / 2.0 + sq, 1.0 / 3.0)
        t = A - p / (3.0 * A) if A != 0.0 else 0.0
        return [t + shift]
    if p == 0.0:
        return [shift]
    r = 2.0 * math.sqrt(-p / 3.0)
    arg = (3.0 * q / (2.0 * p)) * math.sqrt(-3.0 / p)
    arg = min(1.0, max(-1.0, arg))
    phi = math.acos(arg) / 3.0
    return [r * math.cos(phi - 2.0 * math.pi * j / 3.0) + shift for j in range(3)]


def argmin_quartic(c: np.ndarray, lo: float, hi: float, alpha_taylor: float) -> float:
    """argmin_{a in [lo, hi]} m(a) from the roots of m'(a) = 0 (R15, R16).

    1. degenerate loss (max|c1..c4| = 0 or <= 1e-14 |c0|) -> Taylor a;
    2. divide c1..c4 by max|c1..c4|;
    3. the real roots of m''(a) = 2c2 + 6c3 a + 12c4 a^2 inside (lo, hi) cut [lo, hi]
       into pieces on which m' is monotone, so a piece holds a root of m' where m has a
       local minimum iff m' < 0 at its left end and m' >= 0 at its right end; that root
       is bisected to the last bit (R16: the closed-form Cardano roots lost the moderate
       roots when |c4| << |c3|, e.g. c4/c3 = 1e-10, and missed the minimum);
    4. candidates {lo, hi} U those roots; return the candidate with the smallest m
       (ties -> smaller a).
    """
    c = np.asarray(c, dtype=np.float64)
    scale = float(np.max(np.abs(c[1:])))
    if not np.isfinite(scale):
        return alpha_taylor
    if scale == 0.0 or scale <= 1e-14 * abs(float(c[0])):
        return alpha_taylor
    d1, d2, d3, d4 = (float(x) / scale for x in c[1:])

    def mprime(a):
        return ((4.0 * d4 * a + 3.0 * d3) * a + 2.0 * d2) * a + d1

    def m(a):  # c0 dropped: argmin-invariant
        return (((d4 * a + d3) * a + d2) * a + d1) * a

    # roots of m''(a) = 12 d4 a^2 + 6 d3 a + 2 d2 (stable quadratic formula)
    A, B, C = 12.0 * d4, 6.0 * d3, 2.0 * d2
    crit = []
    if A != 0.0:
        disc = B * B - 4.0 * A * C
        if disc >= 0.0:
            q = -0.5 * (B + math.copysign(math.sqrt(disc), B))
            crit.append(q / A)
            if q != 0.0:
                crit.append(C / q)
    elif B != 0.0:
        crit.append(-C / B)
    breaks = [lo] + sorted(x for x in crit if lo < x < hi) + [hi]
    cands = [lo, hi]
    for x0, x1 in zip(breaks[:-1], breaks[1:]):
        if not (mprime(x0) < 0.0 <= mprime(x1)):
            continue
        while True:   # bisection keeping m'(x0) < 0 <= m'(x1)
            xm = 0.5 * (x0 + x1)
            if xm <= x0 or xm >= x1:
                break
            if mprime(xm) < 0.0:
                x0 = xm
            else:
                x1 = xm
        cands.append(x1)
    cands.sort()
    best, best_m = cands[0], m(cands[0])
    for a in cands[1:]:
        ma = m(a)
        if ma < best_m:
            best, best_m = a, ma
    return best


def fit_alpha(R: np.ndarray, d: int, fit: str, S: np.ndarray | None,
              lo: float, hi: float, alpha_taylor: float) -> tuple[float, np.ndarray]:
    """Sketched (eq. (4)) or exact (eq. (3)) a_k for residual R; returns (a, c)."""
    imax = 4 * d + 2                      # powers up to 4d+2
    if fit == FIT_EXACT:
        t = exact_traces(R, imax)
    else:
        t = sketched_traces(R, S, imax)
    c = loss_coeffs(t, d)
    return argmin_quartic(c, lo, hi, alpha_taylor), c


@dataclass
class Report:
    iters: int = 0
    status: int = MAX_ITERS
    resid: list = field(default_factory=list)    # ||R_k||_F / sqrt(s), k = 0..iters
    alphas: list = field(default_factory=list)   # a_k, k = 0..iters-1
    coeffs: list = field(default_factory=list)   # (c0..c4) per fitted k


def _choose_alpha(k, R, d, fit, p, seed, b, s, warmup, lo, hi, aT, rep):
    if k < warmup:                        # a = u for the first iterations (R20)
        return hi
    if fit == FIT_TAYLOR:                 # classical Newton-Schulz
        return aT
    S = None
    if fit == FIT_SKETCHED:
        S = gaussian_sketch(seed, b, k, p, s)       # fresh S_k per k (R8)
    a, c = fit_alpha(R, d, fit, S, lo, hi, aT)
    rep.coeffs.append(c)
    return a


def _status_update(rep, k, r, r_prev, s, tol, max_iters, incr):
    """Stop test before the update (R12): returns (stop, incr).

    converged if ||R_k||_F <= tol sqrt(s); non-finite; diverged after 5
    consecutive increases of ||R_k||_F; max_iters when k = max_iters.
    """
    rep.resid.append(r / math.sqrt(s))
    if not math.isfinite(r):
        rep.status = NONFINITE
        return True, incr
    if r <= tol * math.sqrt(s):
        rep.status = CONVERGED
        return True, incr
    incr = incr + 1 if (k >= 1 and r > r_prev) else 0
    if incr >= 5:
        rep.status = DIVERGED
        return True, incr
    if k == max_iters:
        rep.status = MAX_ITERS
        return True, incr
    return False, incr


def polar(A, d: int = 2, p: int = 8, tol: float = 1e-10, max_iters: int = 50,
          seed: int = 0, b: int = 0, warmup: int = 0, fit: str = FIT_SKETCHED,
          alpha_lo: float | None = None, alpha_hi: float | None = None):
    """PRISM Newton–Schulz polar factor U V^T of A (m x n) in fp64.

    Wide inputs are handled as A^T (P:456 assumes m >= n; R14).  Returns
    (Q, Report) with Q of A's shape.
    """
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    wide = m < n
    X = A.T.copy() if wide else A.copy()       # L x s, L >= s
    s = X.shape[1]
    lo, hi, aT = interval(d)
    lo = lo if alpha_lo is None else alpha_lo
    hi = hi if alpha_hi is None else alpha_hi
    rep = Report()
    c = math.sqrt(float(np.sum(X * X)))        # ||A||_F
    if c == 0.0:
        rep.status = ZERO_INPUT
        return np.zeros_like(A), rep
    X = X / c                                  # X_0 = A/||A||_F
    I = np.eye(s)
    incr = 0
    r_prev = math.inf
    k = 0
    while True:
        R = I - X.T @ X                        # R_k = I - X_k^T X_k
        r = float(np.linalg.norm(R, "fro"))
        stop, incr = _status_update(rep, k, r, r_prev, s, tol, max_iters, incr)
        r_prev = r
        if stop:
            break
        a = _choose_alpha(k, R, d, fit, p, seed, b, s, warmup, lo, hi, aT, rep)
        rep.alphas.append(a)
        X = X @ g_matrix(R, a, d)              # X_{k+1} = X_k g_d(R_k; a_k)
        k += 1
    rep.iters = k
    return (X.T.copy() if wide else X), rep


def sqrt_invsqrt(A, d: int = 2, p: int = 8, tol: float = 1e-10, max_iters: int = 50,
                 seed: int = 0, b: int = 0, warmup: int = 0, fit: str = FIT_SKETCHED,
                 alpha_lo: float | None = None, alpha_hi: float | None = None):
    """PRISM coupled Newton–Schulz A^{1/2}, A^{-1/2} of an SPD A in fp64.

    Theorem-3 ordering R_k = I - Y_k X_k (R11).  Returns
    (Asqrt, Ainvsqrt, Report).
    """
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    lo, hi, aT = interval(d)
    lo = lo if alpha_lo is None else alpha_lo
    hi = hi if alpha_hi is None else alpha_hi
    rep = Report()
    c = math.sqrt(float(np.sum(A * A)))
    if c == 0.0:
        rep.status = ZERO_INPUT
        return np.zeros_like(A), np.zeros_like(A), rep
    X = A / c                                  # X_0 = A/||A||_F (R10)
    I = np.eye(n)
    Y = I.copy()                               # Y_0 = I
    incr = 0
    r_prev = math.inf
    k = 0
    while True:
        R = I - Y @ X                          # R_k = I - Y_k X_k (Thm 3, R11)
        r = float(np.linalg.norm(R, "fro"))
        stop, incr = _status_update(rep, k, r, r_prev, n, tol, max_iters, incr)
        r_prev = r
        if stop:
            break
        a = _choose_alpha(k, R, d, fit, p, seed, b, n, warmup, lo, hi, aT, rep)
        rep.alphas.append(a)
        P = g_matrix(R, a, d)
        X = X @ P                              # X_{k+1} = X_k g_d(R_k; a_k)
        Y = P @ Y                              # Y_{k+1} = g_d(R_k; a_k) Y_k
        k += 1
    rep.iters = k
    sc = math.sqrt(c)
    return sc * X, Y / sc, rep


def sign(A, d: int = 2, p: int = 8, tol: float = 1e-10, max_iters: int = 50,
         seed: int = 0, b: int = 0, warmup: int = 0, fit: str = FIT_SKETCHED,
         alpha_lo: float | None = None, alpha_hi: float | None = None):
    """PRISM Newton–Schulz matrix sign sign(A) = A (A^2)^{-1/2} of a square A in fp64.

    The paper's case study (eq. 2): X_0 = A/||A||_F (R10),
    R_k = I - X_k^2, X_{k+1} = X_k g_d(R_k; a_k), with the loss of eq. (4) fitted on
    R_k exactly as for polar / sqrt ("identical formulas; only R differs").  A^2
    symmetric is the paper's standing assumption: then R_k is symmetric for all
    k.  Returns (S, Report).
    """
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    lo, hi, aT = interval(d)
    lo = lo if alpha_lo is None else alpha_lo
    hi = hi if alpha_hi is None else alpha_hi
    rep = Report()
    c = math.sqrt(float(np.sum(A * A)))
    if c == 0.0:
        rep.status = ZERO_INPUT
        return np.zeros_like(A), rep
    X = A / c                                  # X_0 = A/||A||_F
    I = np.eye(n)
    incr = 0
    r_prev = math.inf
    k = 0
    while True:
        R = I - X @ X                          # R_k = I - X_k^2 (eq. 2)
        r = float(np.linalg.norm(R, "fro"))
        stop, incr = _status_update(rep, k, r, r_prev, n, tol, max_iters, incr)
        r_prev = r
        if stop:
            break
        a = _choose_alpha(k, R, d, fit, p, seed, b, n, warmup, lo, hi, aT, rep)
        rep.alphas.append(a)
        X = X @ g_matrix(R, a, d)              # X_{k+1} = X_k g_d(R_k; a_k)
        k += 1
    rep.iters = k
    return X, rep


# --------------------------------------------------------------------------
# Coupled inverse Newton for A^{-1/p} (Appendix A.3)
# --------------------------------------------------------------------------
# The root order is called q here (the paper's p) because p already
# names the sketch size (the paper's m; R6).

def inv_root_interval(q: int) -> tuple[float, float, float]:
    """(l, u, a_Taylor) for the inverse q-th root: [1/(2q), 2/q], Taylor 1/q.

    The paper defines a_k with a constraint a in [l, u] but never states
    the interval (R22).  Taylor: f_1(xi) = 1 + xi/q.  The bracket [a_T/2,
    2 a_T] mirrors d=1's [1/2, 1] around its Taylor 1/2; with M_0's
    spectrum in (0, (q+1)/2] it keeps 1 + a xi > 0.
    """
    if q < 1:
        raise ValueError("q >= 1")
    return 0.5 / q, 2.0 / q, 1.0 / q


def inv_root_loss_coeffs(t: np.ndarray, q: int) -> np.ndarray:
    """c_0..c_{2q} of m(a) = ||S (R + sum_{i=1}^q C(q,i) a^i (R^{i+1} - R^i))||_F^2.

    P:562-566 (loss), expanded for symmetric R: the bracket is
    sum_i a^i B_i with B_0 = R, B_i = C(q,i)(R^{i+1} - R^i) (polynomials in R),
    so m(a) = sum_{i,j} a^{i+j} tr(S B_i B_j S^T) and each product is a
    combination of t_j = tr(S R^j S^T), j = 2..2q+2.  P:570-590 print the
    result for q = 1, 2 (pinned against it in the tests).
    """
    # B_i as coefficient vectors over powers of R (index = power)
    B = []
    b0 = np.zeros(q + 2)
    b0[1] = 1.0
    B.append(b0)
    for i in range(1, q + 1):
        bi = np.zeros(q + 2)
        bi[i + 1] += math.comb(q, i)
        bi[i] -= math.comb(q, i)
        B.append(bi)
    c = np.zeros(2 * q + 1)
    for i in range(q + 1):
        for j in range(q + 1):
            prod = np.convolve(B[i], B[j])          # B_i B_j as powers of R
            c[i + j] += float(np.dot(prod, t[: prod.size]))
    return c


def argmin_poly(c: np.ndarray, lo: float, hi: float, alpha_taylor: float) -> float:
    """argmin_{a in [lo, hi]} of m(a) = sum_i c_i a^i (degree 2q).

    Degree <= 4 (q <= 2, "analytically"): argmin_quartic.  Degree > 4
    (q >= 3): the real roots of m'(a) = 0 as eigenvalues of its companion
    matrix (numpy.roots), then m at {lo, hi} and the roots inside,
    smallest m wins (ties -> smaller a); degenerate loss -> Taylor (R15).
    """
    c = np.asarray(c, dtype=np.float64)
    if c.size <= 5:
        return argmin_quartic(np.concatenate([c, np.zeros(5 - c.size)]), lo, hi, alpha_taylor)
    scale = float(np.max(np.abs(c[1:])))
    if not np.isfinite(scale):
        return alpha_taylor
    if scale == 0.0 or scale <= 1e-14 * abs(float(c[0])):
        return alpha_taylor
    d = c / scale
    deriv = np.array([i * d[i] for i in range(1, d.size)])          # m' coefficients, ascending
    nz = np.nonzero(np.abs(deriv) > 1e-12 * np.max(np.abs(deriv)))[0]
    deriv = deriv[: nz[-1] + 1]
    roots = np.roots(deriv[::-1]) if deriv.size > 1 else np.array([])

    def m(a):  # c0 dropped: argmin-invariant
        return float(np.polyval(d[:0:-1], a) * a)

    cands = [lo, hi]
    for r in roots:
        if abs(r.imag) <= 1e-9 * (1.0 + abs(r.real)) and lo <= r.real <= hi:
            cands.append(float(r.real))
    cands.sort()
    best, best_m = cands[0], m(cands[0])
    for a in cands[1:]:
        ma = m(a)
        if ma < best_m:
            best, best_m = a, ma
    return best


def inv_root(A, q: int = 4, p: int = 8, tol: float = 1e-10, max_iters: int = 50,
             seed: int = 0, b: int = 0, warmup: int = 0, fit: str = FIT_SKETCHED,
             alpha_lo: float | None = None, alpha_hi: float | None = None):
    """PRISM coupled inverse Newton A^{-1/q} of an SPD A in fp64.

        c = (2 ||A||_F / (q+1))^{1/q},  X_0 = I/c,  M_0 = A/c^q
        R_k = I - M_k
        X_{k+1} = X_k (I + a_k R_k),  M_{k+1} = (I + a_k R_k)^q M_k
        a_k = argmin_{[l,u]} ||S_k (R_k + sum_i C(q,i) a^i (R_k^{i+1} - R_k^i))||_F^2

    Stop test, sketch and statuses as polar (R8, R12); Taylor a = 1/q is the
    classical coupled inverse Newton.  Returns (X, Report).
    """
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    lo, hi, aT = inv_root_interval(q)
    lo = lo if alpha_lo is None else alpha_lo
    hi = hi if alpha_hi is None else alpha_hi
    rep = Report()
    nrm = math.sqrt(float(np.sum(A * A)))
    if nrm == 0.0:
        rep.status = ZERO_INPUT
        return np.zeros_like(A), rep
    cq = 2.0 * nrm / (q + 1)                   # c^q
    c = cq ** (1.0 / q)
    I = np.eye(n)
    X = I / c                                  # X_0 = I/c
    M = A / cq                                 # M_0 = A/c^q
    incr = 0
    r_prev = math.inf
    k = 0
    while True:
        R = I - M                              # R_k = I - M_k
        r = float(np.linalg.norm(R, "fro"))
        stop, incr = _status_update(rep, k, r, r_prev, n, tol, max_iters, incr)
        r_prev = r
        if stop:
            break
        if k < warmup:
            a = hi
        elif fit == FIT_TAYLOR:
            a = aT
        else:
            if fit == FIT_EXACT:
                t = exact_traces(R, 2 * q + 2)
            else:
                t = sketched_traces(R, gaussian_sketch(seed, b, k, p, n), 2 * q + 2)
            cf = inv_root_loss_coeffs(t, q)
            rep.coeffs.append(cf)
            a = argmin_poly(cf, lo, hi, aT)
        rep.alphas.append(a)
        G = I + a * R                          # I + a_k R_k
        X = X @ G                              # X_{k+1} = X_k (I + a_k R_k)
        M = np.linalg.matrix_power(G, q) @ M   # M_{k+1} = (I + a_k R_k)^q M_k
        k += 1
    rep.iters = k
    return X, rep


# --------------------------------------------------------------------------
# PRISM Chebyshev iteration for A^{-1} (Appendix A.4)
# --------------------------------------------------------------------------

def chebyshev_interval() -> tuple[float, float, float]:
    """(l, u, a_Taylor) = (1/2, 2, 1): [1/2, 2]; f_2's xi^2 coefficient 1."""
    return 0.5, 2.0, 1.0


def chebyshev_loss_coeffs(R: np.ndarray, S: np.ndarray | None) -> np.ndarray:
    """(c0, c1, c2) of m(a) = ||S (R^2 - a (R^2 - R^3))||_F^2, S = I if None.

    Written from the definition for a general (non-symmetric) R, as the section allows
    (P:598): U = S R^2, V = S (R^2 - R^3) = U - U R, m(a) = ||U - a V||^2.  For symmetric
    R it equals the printed trace form c1 = -2 t4 + 2 t5, c2 = t4 - 2 t5 + t6 (
    pinned in the tests) (R26).
    """
    U = R @ R if S is None else (S.astype(np.float64) @ R) @ R
    V = U - U @ R
    return np.array([float(np.sum(U * U)), -2.0 * float(np.sum(U * V)), float(np.sum(V * V))])


def chebyshev_inverse(A, p: int = 8, tol: float = 1e-10, max_iters: int = 50, seed: int = 0, b: int = 0,
                      warmup: int = 0, fit: str = FIT_SKETCHED, alpha_lo: float | None = None,
                      alpha_hi: float | None = None):
    """PRISM-accelerated Chebyshev iteration for A^{-1} of a square full-rank A in fp64.

        c = ||A||_F, A' = A/c (||A'||_2 <= 1),  X_0 = A'^T           (R25)
        R_k = I - A' X_k,  X_{k+1} = X_k (I + R_k + a_k R_k^2)
        a_k = argmin_{[1/2, 2]} ||S_k (R_k^2 - a (R_k^2 - R_k^3))||_F^2
        A^{-1} = A'^{-1} / c.
    Stop test, sketch and statuses as polar (R8, R12).  Returns (Ainv, Report).
    """
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    lo, hi, aT = chebyshev_interval()
    lo = lo if alpha_lo is None else alpha_lo
    hi = hi if alpha_hi is None else alpha_hi
    rep = Report()
    c = math.sqrt(float(np.sum(A * A)))
    if c == 0.0:
        rep.status = ZERO_INPUT
        return np.zeros_like(A), rep
    An = A / c
    X = An.T.copy()                            # X_0 = A^T (of the normalised A)
    I = np.eye(n)
    incr = 0
    r_prev = math.inf
    k = 0
    while True:
        R = I - An @ X                         # R_k = I - A X_k
        r = float(np.linalg.norm(R, "fro"))
        stop, incr = _status_update(rep, k, r, r_prev, n, tol, max_iters, incr)
        r_prev = r
        if stop:
            break
        if k < warmup:
            a = hi
        elif fit == FIT_TAYLOR:
            a = aT
        else:
            S = None if fit == FIT_EXACT else gaussian_sketch(seed, b, k, p, n)
            cf = chebyshev_loss_coeffs(R, S)
            rep.coeffs.append(cf)
            a = argmin_quartic(np.concatenate([cf, [0.0, 0.0]]), lo, hi, aT)   # closed form
        rep.alphas.append(a)
        X = X @ (I + R + a * (R @ R))          # X_{k+1} = X_k (I + R_k + a_k R_k^2)
        k += 1
    rep.iters = k
    return X / c, rep


# --------------------------------------------------------------------------
# PRISM DB Newton, product form, for A^{1/2}, A^{-1/2} (Appendix A.2; f3)
# --------------------------------------------------------------------------

def db_newton_coeffs(M: np.ndarray, Minv: np.ndarray) -> np.ndarray:
    """(c0..c4) of m(a) = ||I - M_{k+1}(a)||_F^2 for symmetric M.

    c1..c4 are the paper's trace forms; traces of squares are sums of squared entries
    (P:521).  c0 (not printed) = ||I - M||_F^2 (the a = 0 value).
    """
    n = M.shape[0]
    tM, tMi = float(np.trace(M)), float(np.trace(Minv))
    tM2, tMi2 = float(np.sum(M * M)), float(np.sum(Minv * Minv))
    c0 = n - 2 * tM + tM2
    c1 = -4 * n + 8 * tM - 4 * tM2
    c2 = 10 * n - 14 * tM + 6 * tM2 - 2 * tMi
    c3 = -12 * n + 12 * tM - 4 * tM2 + 4 * tMi
    c4 = 6 * n - 4 * tM + tM2 - 4 * tMi + tMi2
    return np.array([c0, c1, c2, c3, c4])


def argmin_quartic_free(c: np.ndarray, alpha_default: float) -> float:
    """Unconstrained argmin over the reals of m(a) = sum c_i a^i (no interval).

    The global minimum of a quartic with c4 > 0 is at a real root of the cubic m'(a) = 0
    (P:213); candidates = those roots (two Newton polishes, as argmin_quartic), smallest
    m wins (ties -> smaller a).  c4 <= 0 or a degenerate loss -> the default (1/2, the
    classical DB Newton step) (R27).
    """
    c = np.asarray(c, dtype=np.float64)
    scale = float(np.max(np.abs(c[1:])))
    if not np.isfinite(scale) or scale == 0.0 or scale <= 1e-14 * abs(float(c[0])) or c[4] <= 0.0:
        return alpha_default
    d1, d2, d3, d4 = (float(x) / scale for x in c[1:])

    def mprime(a):
        return ((4.0 * d4 * a + 3.0 * d3) * a + 2.0 * d2) * a + d1

    def msecond(a):
        return (12.0 * d4 * a + 6.0 * d3) * a + 2.0 * d2

    def m(a):
        return (((d4 * a + d3) * a + d2) * a + d1) * a

    cands = []
    for r in _real_roots_cubic(4.0 * d4, 3.0 * d3, 2.0 * d2, d1):
        for _ in range(2):
            m2 = msecond(r)
            if m2 != 0.0:
                nr = r - mprime(r) / m2
                if math.isfinite(nr):
                    r = nr
        if math.isfinite(r):
            cands.append(r)
    if not cands:
        return alpha_default
    cands.sort()
    best, best_m = cands[0], m(cands[0])
    for a in cands[1:]:
        ma = m(a)
        if ma < best_m:
            best, best_m = a, ma
    return best


def db_newton(A, tol: float = 1e-10, max_iters: int = 50, fit: str = FIT_EXACT):
    """PRISM DB Newton, product form, for an SPD A in fp64.

        M_0 = A, X_0 = A, Y_0 = I
        M_{k+1} = 2a(1-a) I + (1-a)^2 M_k + a^2 M_k^{-1}
        X_{k+1} = (1-a) X_k + a X_k M_k^{-1},  Y_{k+1} = (1-a) Y_k + a Y_k M_k^{-1}
        a_k = argmin_a ||I - M_{k+1}||_F^2 (exact, unsketched, unconstrained)
    fit="taylor" keeps a = 1/2 (Cheng et al.'s product form).  Residual R_k =
    I - M_k; stop test and statuses as polar (R12, R28).  Returns (X ~ A^{1/2},
    Y ~ A^{-1/2}, Report).  No sketch: the coefficients are O(n^2) traces.
    """
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    rep = Report()
    if not np.any(A):
        rep.status = ZERO_INPUT
        return np.zeros_like(A), np.zeros_like(A), rep
    I = np.eye(n)
    M, X, Y = A.copy(), A.copy(), I.copy()
    incr = 0
    r_prev = math.inf
    k = 0
    while True:
        r = float(np.linalg.norm(I - M, "fro"))     # residual I - M_k (M_k = X_k Y_k -> I)
        stop, incr = _status_update(rep, k, r, r_prev, n, tol, max_iters, incr)
        r_prev = r
        if stop:
            break
        Minv = np.linalg.inv(M)
        if fit == FIT_TAYLOR:
            a = 0.5
        else:
            cf = db_newton_coeffs(M, Minv)
            rep.coeffs.append(cf)
            a = argmin_quartic_free(cf, 0.5)
        rep.alphas.append(a)
        X = (1 - a) * X + a * (X @ Minv)
        Y = (1 - a) * Y + a * (Y @ Minv)
        M = 2 * a * (1 - a) * I + (1 - a) ** 2 * M + a * a * Minv
        k += 1
    rep.iters = k
    return X, Y, rep
