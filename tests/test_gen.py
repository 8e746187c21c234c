"""CPU tests of the seeded input generators (gen/).  These pin the
generators to published known answers and to the distributions they claim."""
import math
import os

import numpy as np
import pytest

from gen import configs as G
from gen import ct, rng

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_philox_known_answers():
    for line in open(os.path.join(GOLD, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(t, 16) for t in line.split()]
        out = rng.philox4x32_10(*v[:6])
        assert [int(o) for o in out] == v[6:], line


def test_log_exp_accuracy():
    x = np.concatenate([np.logspace(-300, 300, 2001), np.linspace(0.01, 10, 1001)])
    assert np.max(np.abs(rng.log64(x) - np.log(x)) / np.maximum(1.0, np.abs(np.log(x)))) < 4e-16
    y = np.linspace(-700, 700, 20001)
    assert np.max(np.abs(rng.exp64(y) / np.exp(y) - 1.0)) < 4e-16
    from scipy.special import gammaln
    k = np.arange(0, 100000, dtype=float)
    assert np.max(np.abs(rng.logfact64(k) - gammaln(k + 1)) / np.maximum(1, gammaln(k + 1))) < 1e-12


def test_uniform_open_interval():
    w = np.array([0, 0xFFFFFFFF], dtype=np.uint64)
    u = rng.u01(w, w)
    assert u[0] > 0.0 and u[1] < 1.0


def test_normal_moments_and_determinism():
    z = rng.gaussian_rows(5, rng.STREAM_TEST, np.arange(400), 500)
    assert abs(z.mean()) < 0.01 and abs(z.var() - 1.0) < 0.01
    assert abs(np.mean(z ** 4) - 3.0) < 0.05
    # tail frequency P(|Z|>2) = 0.0455
    assert abs(np.mean(np.abs(z) > 2.0) - 0.0455) < 0.003
    z2 = rng.gaussian_rows(5, rng.STREAM_TEST, np.array([7, 399, 3]), 500)
    assert np.array_equal(z2, z[[7, 399, 3]])  # keyed by global row, order-free
    z3 = rng.gaussian_rows(6, rng.STREAM_TEST, np.array([7]), 500)
    assert not np.array_equal(z3[0], z[7])


def test_poisson_moments():
    for lam in (0.0, 0.7, 3.5, 9.99, 10.0, 25.0, 1e4, 1e6):
        L = np.full(100_000, lam)
        k = rng.poisson(11, rng.STREAM_TEST, L, np.arange(L.size))
        if lam == 0.0:
            assert np.all(k == 0)
            continue
        se = math.sqrt(lam / L.size)
        assert abs(k.mean() - lam) < 5 * se, lam
        assert abs(k.var() / lam - 1.0) < 0.03, lam
    # SPEC.md:74-76 example: mean 1e6, 1e4 draws -> within 4 sqrt(1e6/1e4)
    k = rng.poisson(12, rng.STREAM_TEST, np.full(10_000, 1e6), np.arange(10_000))
    assert abs(k.mean() - 1e6) < 4 * math.sqrt(1e6 / 1e4)


def test_poisson_pmf_small_lambda():
    lam = 2.5
    k = rng.poisson(13, rng.STREAM_TEST, np.full(200_000, lam), np.arange(200_000))
    freq = np.bincount(k, minlength=12)[:8] / k.size
    pmf = np.array([math.exp(-lam) * lam ** j / math.factorial(j) for j in range(8)])
    assert np.max(np.abs(freq - pmf)) < 0.004


def test_spectrum_recipe():
    # Σ_j s_j μ_j values derived in SURVEY.md §8(c) reading #9
    for W, v in ((10, 1.185578), (16, 1.211326), (20, 1.219464), (32, 1.231282)):
        s, mu = G.spectrum(W)
        assert abs(s.sum() - 1.0) < 1e-15
        assert np.all(s > 0) and np.all(s <= 1)
        assert abs(float(np.dot(s, mu)) - v) < 5e-7, W
        assert mu[0] == 2.0 and mu[-1] == 0.5


def test_unit_sphere():
    x = rng.unit_sphere(1, rng.STREAM_XSTAR, 1024, 1.0)
    assert abs(np.linalg.norm(x) - 1.0) < 1e-14


@pytest.fixture(scope="module")
def radon():
    return ct.parallel_beam_csr(256, 360, 367)


def test_radon_structure(radon):
    row_ptr, col, val = radon
    n = 360 * 367
    assert row_ptr.shape == (n + 1,)
    assert np.all(val > 0)
    assert np.all((col >= 0) & (col < 256 * 256))
    lens = np.diff(row_ptr)
    # SURVEY.md §8(c) reading #12: 14,781 empty rows, nnz ≈ 30.2M
    assert int((lens == 0).sum()) == 14781
    assert 29.5e6 < row_ptr[-1] < 30.5e6
    # row weight sums <= diagonal of the unit field of view
    sums = np.add.reduceat(val, row_ptr[:-1][lens > 0])
    assert sums.max() <= math.sqrt(2.0) + 1e-12
    # no pixel appears twice in a row
    for i in np.random.default_rng(0).integers(0, n, 200):
        c = col[row_ptr[i]:row_ptr[i + 1]]
        assert np.unique(c).size == c.size


def test_radon_chord_lengths(radon):
    """A · 1 = in-grid chord length of each ray (geometric identity)."""
    row_ptr, col, val = radon
    lens = np.diff(row_ptr)
    sums = np.zeros(lens.size)
    sums[lens > 0] = np.add.reduceat(val, row_ptr[:-1][lens > 0])
    half = 0.5  # the grid is the square [-128.5/256, 127.5/256]^2
    lo, hi = -128.5 / 256, 127.5 / 256
    for k in (0, 1, 45, 90, 179, 180, 271, 359):
        th = k * math.pi / 360
        for b in (0, 50, 183, 300, 366):
            t = (b - 183) / 256
            px, py = t * math.cos(th), t * math.sin(th)
            ux, uy = -math.sin(th), math.cos(th)
            s0, s1 = -10.0, 10.0
            for p, u in ((px, ux), (py, uy)):
                if abs(u) < 1e-15:
                    if not (lo < p < hi):
                        s0, s1 = 1.0, 0.0
                    continue
                a, c = (lo - p) / u, (hi - p) / u
                s0, s1 = max(s0, min(a, c)), min(s1, max(a, c))
            chord = max(0.0, s1 - s0)
            assert abs(sums[k * 367 + b] - chord) < 1e-12, (k, b)
    assert half > 0


def test_radon_line_integral(radon):
    """Random rays vs a fine midpoint-rule line integral of a smooth image
    sampled piecewise-constant."""
    row_ptr, col, val = radon
    img = ct.ellipse_phantom(3)
    r = np.random.default_rng(1)
    for i in r.integers(0, 360 * 367, 30):
        k, b = divmod(int(i), 367)
        th = k * math.pi / 360
        t = (b - 183) / 256
        s = np.linspace(-1, 1, 400_001)
        sm = 0.5 * (s[1:] + s[:-1])
        x = t * math.cos(th) - sm * math.sin(th)
        y = t * math.sin(th) + sm * math.cos(th)
        c = np.floor(x * 256 + 128.5).astype(np.int64)
        rr = np.floor(y * 256 + 128.5).astype(np.int64)
        ok = (c >= 0) & (c < 256) & (rr >= 0) & (rr < 256)
        ref = np.sum(img[(rr * 256 + c)[ok]]) * (s[1] - s[0])
        got = float(np.dot(val[row_ptr[i]:row_ptr[i + 1]], img[col[row_ptr[i]:row_ptr[i + 1]]]))
        assert abs(got - ref) <= 1e-4 * max(1.0, abs(ref)) + 2e-5, (k, b, got, ref)


def test_phantom():
    x = ct.ellipse_phantom(3)
    assert x.shape == (65536,)
    assert x.min() >= 0.0 and x.max() <= 1.0
    assert 0.05 < np.mean(x > 0) < 0.95
    assert np.array_equal(x, ct.ellipse_phantom(3))
