"""Seeded synthetic inputs shaped like the paper's workloads.

This module holds none of the method's arithmetic: it only draws input
matrices.  It serves both the CUDA path (tests, bench) and the oracle
(tests), which is the one piece the two sides may share.

Recipes (DESIGN.md §"Input recipe"):
* ``gaussian``      i.i.d. N(0,1) entries — the paper's Gaussian/MP polar
                    inputs with aspect ratio gamma.
* ``spectrum``      U diag(sigma) V^T with Haar U, V — prescribed spectra,
                    e.g. log-spaced sigma in [sigma_min, 1] (Fig. 1).
* ``htmp``          heavy-tailed stand-in for the HTMP ensemble (P:295,
                    P:1274): sigma_i^2 = lambda_i w_i, lambda_i from the
                    Marchenko–Pastur law of the aspect ratio, w_i inverse-gamma
                    (shape kappa+1, scale kappa); smaller kappa = heavier tail.
* ``equal_sigma``   c * Q with orthonormal Q: all singular values equal.
* ``spd_logspaced`` Q diag(lambda) Q^T, lambda_i = kappa^{-i/(n-1)} (Shampoo
                    blocks with condition number kappa; P:1298 analogue).
* ``wishart``       G^T G / rows, G Gaussian rows x n.
* ``sym_indefinite`` Q diag(lambda) Q^T, |lambda_i| log-spaced in [lo, 1] with
                    alternating signs: symmetric indefinite inputs of the
                    matrix-sign case study (A^2 symmetric).
* GPT-2 small / 1B-model Muon batches (BASELINE.json configs[1], [4]).
"""

from __future__ import annotations

import numpy as np


def rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(int(seed))


def gaussian(m: int, n: int, seed: int) -> np.ndarray:
    return rng(seed).standard_normal((m, n))


def haar(n: int, k: int, seed: int) -> np.ndarray:
    """n x k matrix with orthonormal columns (QR of a Gaussian, sign-fixed)."""
    g = rng(seed).standard_normal((n, k))
    q, r = np.linalg.qr(g)
    return q * np.sign(np.diag(r))[None, :]


def spectrum(m: int, n: int, sigma: np.ndarray, seed: int) -> np.ndarray:
    k = min(m, n)
    sigma = np.asarray(sigma, dtype=np.float64)
    assert sigma.shape == (k,)
    U = haar(m, k, seed)
    V = haar(n, k, seed + 7919)
    return (U * sigma[None, :]) @ V.T


def logspaced(m: int, n: int, sigma_min: float, seed: int) -> np.ndarray:
    k = min(m, n)
    sigma = np.logspace(0.0, np.log10(sigma_min), k)
    return spectrum(m, n, sigma, seed)


def _mp_quantiles(k: int, ratio: float) -> np.ndarray:
    """k quantiles of the Marchenko–Pastur law (variance 1, aspect ratio <= 1)."""
    lam_m, lam_p = (1 - np.sqrt(ratio)) ** 2, (1 + np.sqrt(ratio)) ** 2
    x = np.linspace(lam_m, lam_p, 20001)
    dens = np.sqrt(np.maximum((lam_p - x) * (x - lam_m), 0.0)) / (2 * np.pi * ratio * np.maximum(x, 1e-300))
    cdf = np.concatenate([[0.0], np.cumsum(0.5 * (dens[1:] + dens[:-1]) * np.diff(x))])
    cdf /= cdf[-1]
    u = (np.arange(k) + 0.5) / k
    return np.interp(u, cdf, x)


def htmp(m: int, n: int, kappa: float, seed: int) -> np.ndarray:
    """Heavy-tailed (HTMP-like) matrix, sigma_max normalised to 1."""
    g = rng(seed + 104729)
    k = min(m, n)
    ratio = k / max(m, n)
    lam = _mp_quantiles(k, ratio)
    lam = g.permutation(lam)
    # inverse-gamma(shape kappa+1, scale kappa): mean 1
    w = kappa / g.gamma(kappa + 1.0, 1.0, size=k)
    sig = np.sort(np.sqrt(lam * w))[::-1]
    sig = sig / sig[0]
    return spectrum(m, n, sig, seed)


def equal_sigma(m: int, n: int, c: float, seed: int) -> np.ndarray:
    k = min(m, n)
    U = haar(m, k, seed)
    V = haar(n, k, seed + 7919)
    return c * (U @ V.T)


def spd_logspaced(n: int, kappa: float, seed: int) -> np.ndarray:
    lam = kappa ** (-np.arange(n) / max(n - 1, 1))
    Q = haar(n, n, seed)
    A = (Q * lam[None, :]) @ Q.T
    return 0.5 * (A + A.T)


def sym_indefinite(n: int, lo: float, seed: int) -> np.ndarray:
    lam = np.logspace(0.0, np.log10(lo), n) * np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    Q = haar(n, n, seed)
    A = (Q * lam[None, :]) @ Q.T
    return 0.5 * (A + A.T)


def wishart(n: int, gamma: float, seed: int) -> np.ndarray:
    rows = int(round(gamma * n))
    G = rng(seed).standard_normal((rows, n))
    A = G.T @ G / rows
    return 0.5 * (A + A.T)


# ---- optimizer-step batches (BASELINE.json configs) ------------------------

def gpt2_small_shapes() -> list[tuple[int, int]]:
    """48 GPT-2 small layer matrices: 12 x {c_attn 768x2304, attn proj 768x768,
    mlp fc 768x3072, mlp proj 3072x768} (configs[1])."""
    shapes = []
    for _ in range(12):
        shapes += [(768, 2304), (768, 768), (768, 3072), (3072, 768)]
    return shapes


def gpt_1b_shapes() -> list[tuple[int, int]]:
    """96 matrices of a 1.2B-parameter GPT-style model (d_model 2048, 24
    layers; configs[4])."""
    shapes = []
    for _ in range(24):
        shapes += [(2048, 6144), (2048, 2048), (2048, 8192), (8192, 2048)]
    return shapes


def muon_batch(shapes, seed: int, kind: str = "mixed") -> list[np.ndarray]:
    """Gradient-like matrices: even index Gaussian (MP), odd index HTMP
    kappa=0.5 when kind == 'mixed'."""
    out = []
    for i, (m, n) in enumerate(shapes):
        s = 1000 * seed + i
        if kind == "gaussian" or (kind == "mixed" and i % 2 == 0):
            out.append(gaussian(m, n, s))
        else:
            out.append(htmp(m, n, 0.5, s))
    return out
