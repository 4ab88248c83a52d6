"""Gaussian sketch generator for the oracle — TEST INFRASTRUCTURE ONLY.

The paper draws a fresh i.i.d. Gaussian sketch S_k in R^{p x n} at every
iteration (eq. (4) "S_k", "simple random Gaussian matrices
appear to be sufficient", P:1170 union bound over k).  It does not say which
random generator.  DESIGN.md reading R8 fixes one so that the oracle and the
device draw the *same* S_k, each with its own implementation:

* Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as
  1, 2, 3"), pinned by its published known-answer vectors
  (tests/test_oracle_philox.py).
* element (i, j) of S_k for matrix b: q = i*s + j, pair e = q >> 1,
  counter = (e, k, b, 0x534B4348 "SKCH"), key = (seed_lo, seed_hi).
* u1 = (K1 + 1) 2^-53 in (0, 1], u2 = K2 2^-53 in [0, 1) with
  K1 = (o0>>5) 2^26 + (o1>>6), K2 = (o2>>5) 2^26 + (o3>>6).
* z = sqrt(-2 ln u1) * (cos 2pi u2 if q even else sin 2pi u2), with ln, sin,
  cos evaluated by the fixed, IEEE-exact-operation routines below (no fused
  multiply-add, fixed evaluation order) so both sides produce the same bits;
  S[i, j] = float32(z) (round to nearest even).

The scale of S does not change the argmin of eq. (4), so N(0, 1) is used
instead of the printed N(1, 1/p) (reading R7).
"""

from __future__ import annotations

import math

import numpy as np

MASK32 = np.uint64(0xFFFFFFFF)
PHILOX_M0 = np.uint64(0xD2511F53)
PHILOX_M1 = np.uint64(0xCD9E8D57)
PHILOX_W0 = np.uint64(0x9E3779B9)
PHILOX_W1 = np.uint64(0xBB67AE85)

TAG_SKETCH = 0x534B4348  # "SKCH"


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32 with 10 rounds on arrays of 32-bit words (held in uint64).

    Round: (hi0, lo0) = M0*c0, (hi1, lo1) = M1*c2,
    c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0); the key is bumped by the
    Weyl constants (W0, W1) before every round after the first.
    """
    c0 = np.asarray(c0, dtype=np.uint64) & MASK32
    c1 = np.asarray(c1, dtype=np.uint64) & MASK32
    c2 = np.asarray(c2, dtype=np.uint64) & MASK32
    c3 = np.asarray(c3, dtype=np.uint64) & MASK32
    k0 = np.asarray(k0, dtype=np.uint64) & MASK32
    k1 = np.asarray(k1, dtype=np.uint64) & MASK32
    for r in range(10):
        if r > 0:
            k0 = (k0 + PHILOX_W0) & MASK32
            k1 = (k1 + PHILOX_W1) & MASK32
        p0 = PHILOX_M0 * c0  # < 2^64, exact in uint64
        p1 = PHILOX_M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0), lo1, (hi0 ^ c3 ^ k1), lo0
    return c0, c1, c2, c3


# --- portable fp64 elementary functions (IEEE +,-,*,/,sqrt only) ----------

LN2_HI = 6.93147180369123816490e-01  # 0x3FE62E42FEE00000 (trailing zeros: e*LN2_HI exact)
LN2_LO = 1.90821492927058770002e-10  # 0x3DEA39EF35793C76
SQRT_HALF = 0.70710678118654752440
PIO2 = 1.5707963267948966  # fp64(pi/2)

# Horner coefficients, each the correctly rounded fp64 of the exact rational
_LN_C = [1.0 / (2 * j + 1) for j in range(11)]                      # 1/(2j+1)
_SIN_C = [(-1.0) ** j / math.factorial(2 * j + 1) for j in range(11)]  # x^(2j+1)/(2j+1)!
_COS_C = [(-1.0) ** j / math.factorial(2 * j) for j in range(12)]      # x^(2j)/(2j)!


def portable_log(u):
    """ln u for u in (0, 1] (arrays), fixed operation order.

    u = m 2^e with m in [sqrt(1/2), sqrt(2)); f = m - 1, t = f/(2+f);
    ln m = 2t * sum_{j=0..10} t^(2j)/(2j+1) (atanh series, |t| <= 0.1716,
    truncation < 1e-18); ln u = e*LN2_HI + (e*LN2_LO + ln m).
    """
    u = np.asarray(u, dtype=np.float64)
    m, e = np.frexp(u)                       # u = m * 2^e, m in [0.5, 1)
    small = m < SQRT_HALF
    m = np.where(small, m * 2.0, m)          # exact
    e = np.where(small, e - 1, e).astype(np.float64)
    f = m - 1.0                              # exact (Sterbenz)
    t = f / (2.0 + f)
    t2 = t * t
    acc = np.full_like(t, _LN_C[10])
    for j in range(9, -1, -1):
        acc = acc * t2
        acc = acc + _LN_C[j]
    lnm = (2.0 * t) * acc
    return e * LN2_HI + (e * LN2_LO + lnm)


def portable_sincos_2pi(K2):
    """(sin, cos) of 2*pi*u2 with u2 = K2 * 2^-53, K2 an integer in [0, 2^53).

    q = round(4 u2) computed on the integer, d = 4u2 - q exactly,
    x = d * fp64(pi/2) in [-pi/4, pi/4]; Taylor polynomials to x^21 (sin) and
    x^22 (cos) by Horner in x^2; then the exact quadrant map.
    """
    K2 = np.asarray(K2, dtype=np.uint64)
    q = (K2 + np.uint64(1 << 50)) >> np.uint64(51)                  # 0..4
    d_int = K2.astype(np.int64) - (q.astype(np.int64) << np.int64(51))  # |.| <= 2^50
    d = d_int.astype(np.float64) * (2.0 ** -51)                     # exact
    x = d * PIO2
    x2 = x * x
    s = np.full_like(x, _SIN_C[10])
    for j in range(9, -1, -1):
        s = s * x2
        s = s + _SIN_C[j]
    s = x * s
    c = np.full_like(x, _COS_C[11])
    for j in range(10, -1, -1):
        c = c * x2
        c = c + _COS_C[j]
    qq = (q & np.uint64(3)).astype(np.int64)
    sin_out = np.select([qq == 0, qq == 1, qq == 2, qq == 3], [s, c, -s, -c])
    cos_out = np.select([qq == 0, qq == 1, qq == 2, qq == 3], [c, -s, -c, s])
    return sin_out, cos_out


def _gauss_from_counter(q, k, b, seed, tag):
    """Gaussian value for flat element index q (array) of draw (k, b)."""
    q = np.asarray(q, dtype=np.uint64)
    e = q >> np.uint64(1)
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    k0, k1 = seed & 0xFFFFFFFF, seed >> 32
    o0, o1, o2, o3 = philox4x32_10(e, np.uint64(k), np.uint64(b), np.uint64(tag), k0, k1)
    K1 = ((o0 >> np.uint64(5)) << np.uint64(26)) + (o1 >> np.uint64(6))
    K2 = ((o2 >> np.uint64(5)) << np.uint64(26)) + (o3 >> np.uint64(6))
    u1 = (K1 + np.uint64(1)).astype(np.float64) * (2.0 ** -53)   # (0, 1], exact
    rad = np.sqrt(-2.0 * portable_log(u1))
    sn, cs = portable_sincos_2pi(K2)
    even = (q & np.uint64(1)) == 0
    return rad * np.where(even, cs, sn)


def gaussian_sketch(seed: int, b: int, k: int, p: int, s: int) -> np.ndarray:
    """S_k for matrix b of a batch: p x s float32 (RNE of the fp64 draw).

    Depends only on (seed, b, k, p, s) (R8), so a batch split
    across GPUs draws the same sketches as one GPU.
    """
    q = np.arange(p * s, dtype=np.uint64)
    z = _gauss_from_counter(q, k, b, seed, TAG_SKETCH)
    return z.astype(np.float32).reshape(p, s)
