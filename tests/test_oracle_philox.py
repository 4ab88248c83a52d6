"""Pins for the oracle's sketch generator (R8).

Philox4x32-10 is pinned by the published known-answer vectors; the portable
ln / sin / cos are pinned against libm; the Box–Muller output against the
moments of N(0,1) and the Johnson–Lindenstrauss identity E||Sx||^2 = p||x||^2.
"""

import math
import os

import numpy as np
import pytest

from oracle import philox

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _kats():
    rows = []
    with open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            rows.append([int(x, 16) for x in line.split()])
    return rows


@pytest.mark.parametrize("row", _kats())
def test_philox_known_answers(row):
    c0, c1, c2, c3, k0, k1 = row[:6]
    out = philox.philox4x32_10(c0, c1, c2, c3, k0, k1)
    assert [int(x) for x in out] == row[6:]


def test_philox_vectorised_matches_scalar():
    e = np.arange(17, dtype=np.uint64)
    vec = philox.philox4x32_10(e, 3, 5, philox.TAG_SKETCH, 11, 13)
    for i in range(17):
        sc = philox.philox4x32_10(i, 3, 5, philox.TAG_SKETCH, 11, 13)
        assert [int(v[i]) for v in vec] == [int(x) for x in sc]


def test_portable_log_against_libm():
    g = np.random.default_rng(0)
    u = np.concatenate([g.random(100000) * (1 - 1e-15) + 1e-15,
                        [1.0, 0.5, 2.0 ** -53, 0.75, 1 - 2.0 ** -53]])
    got = philox.portable_log(u)
    ref = np.array([math.log(x) for x in u])
    # <= 2 ulp of |ln u| away from the correctly rounded value
    assert np.all(np.abs(got - ref) <= 4.5e-16 * np.maximum(np.abs(ref), 1e-300) + 1e-300)
    assert got[-5] == 0.0                      # ln 1 = 0 exactly
    assert abs(got[-4] + math.log(2)) < 2e-16


def test_portable_sincos_against_libm():
    g = np.random.default_rng(1)
    K = g.integers(0, 2 ** 53, 100000, dtype=np.uint64)
    K = np.concatenate([K, np.array([0, 2 ** 51, 2 ** 52, 3 * 2 ** 51, 2 ** 53 - 1], dtype=np.uint64)])
    s, c = philox.portable_sincos_2pi(K)
    a = [2 * math.pi * (int(k) * 2.0 ** -53) for k in K]
    assert np.max(np.abs(s - np.array([math.sin(x) for x in a]))) < 1e-15
    assert np.max(np.abs(c - np.array([math.cos(x) for x in a]))) < 1e-15
    assert s[-5] == 0.0 and c[-5] == 1.0       # u2 = 0
    assert c[-4] == 0.0 or abs(c[-4]) < 1e-300  # u2 = 1/4: cos(pi/2) = 0 exactly by the quadrant map
    assert s[-4] == 1.0


def test_sketch_moments_and_jl():
    S = philox.gaussian_sketch(seed=7, b=0, k=0, p=64, s=4096)
    assert S.dtype == np.float32 and S.shape == (64, 4096)
    n = S.size
    assert abs(float(S.mean())) < 4.0 / math.sqrt(n)
    assert abs(float(S.var()) - 1.0) < 0.02
    # JL identity: E ||S x||^2 = p ||x||^2 for fixed unit x, averaged over draws
    x = np.random.default_rng(3).standard_normal(512)
    x /= np.linalg.norm(x)
    vals = [float(np.sum((philox.gaussian_sketch(42, 0, k, 8, 512).astype(np.float64) @ x) ** 2))
            for k in range(300)]
    assert abs(np.mean(vals) / 8.0 - 1.0) < 0.1


def test_sketch_depends_only_on_seed_b_k():
    a = philox.gaussian_sketch(42, 3, 5, 8, 100)
    assert np.array_equal(a, philox.gaussian_sketch(42, 3, 5, 8, 100))
    assert not np.array_equal(a, philox.gaussian_sketch(42, 3, 6, 8, 100))
    assert not np.array_equal(a, philox.gaussian_sketch(42, 4, 5, 8, 100))
    assert not np.array_equal(a, philox.gaussian_sketch(43, 3, 5, 8, 100))
    # element (i, j) is a function of q = i*s + j: a p=2 draw is the prefix of p=4
    b4 = philox.gaussian_sketch(42, 3, 5, 4, 100)
    assert np.array_equal(b4[:2], philox.gaussian_sketch(42, 3, 5, 2, 100))


def test_sketch_golden_prefix():
    """Regression pin for the device: first values of seed 0 (written by
    scripts/make_golden.py, which calls only oracle/)."""
    path = os.path.join(GOLDEN, "sketch_seed0_b0_k0.txt")
    words = [w for line in open(path) if not line.startswith("#") for w in line.split()]
    want = np.array([int(w, 16) for w in words], dtype=np.uint32)
    S = philox.gaussian_sketch(0, 0, 0, 8, 512)
    assert np.array_equal(S.reshape(-1)[: want.size].view(np.uint32), want)
