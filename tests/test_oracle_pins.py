"""Pins of the fp64 oracle to things other than itself:
worked values, closed forms, the finite-difference identity ∇ℓ = F,
monotonicity and Lipschitz bounds, a Monte-Carlo variance identity, the
Appendix A.1 reparameterisation identity, projection properties and the E6
closed loop.  A plausible mistake in the oracle (dropped term, wrong sign or
index, missing ReLU, wrong 1/n) fails at least one of these."""
import math
import os

import numpy as np
import pytest
from scipy.special import erfcx

import oracle
from gen import configs as G
from gen import rng
from oracle import workloads as Wk

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _small(n=300, d=12, W=5, I_bar=50.0, seed=3, relu=1, y_kind="poisson", xs_norm=0.8,
           nonneg=False):
    s, mu = G.spectrum(W)
    A = rng.gaussian_rows(seed, rng.STREAM_TEST, np.arange(n), d)
    if nonneg:
        A = np.abs(A)
    xs = rng.unit_sphere(seed, rng.STREAM_XSTAR, d, xs_norm)
    p0 = oracle.Problem(A=A, y=np.zeros(n), s=s, mu=mu, I_bar=I_bar, d=d, relu=relu)
    lam = p0.mean(xs)
    if y_kind == "poisson":
        y = rng.poisson(seed, rng.STREAM_Y, lam, np.arange(n)).astype(float)
    else:
        y = lam.copy()
    return dict(A=A, s=s, mu=mu, xs=xs, y=y, lam=lam, I_bar=I_bar,
                p=oracle.Problem(A=A, y=y, s=s, mu=mu, I_bar=I_bar, d=d, relu=relu))


# ---------------------------------------------------------------- P1 / P2
def test_P1_P2_link_worked_values():
    for line in open(os.path.join(GOLD, "link_values.txt")):
        if line.startswith("#") or not line.strip():
            continue
        kind, W, s, mu, t, exp, tol = line.split()[:7]
        s = np.array([float(v) for v in s.split(",")])
        mu = np.array([float(v) for v in mu.split(",")])
        assert s.shape[0] == int(W)
        got = oracle.h(s, mu, float(t)) if kind == "h" else oracle.hprime_abs(s, mu, float(t))
        assert abs(got - float(exp)) <= float(tol), line


def test_P1_link_shape():
    s, mu = G.spectrum(20)
    ts = np.linspace(-3, 8, 221)
    hv = np.array([oracle.h(s, mu, t) for t in ts])
    assert np.all(np.diff(hv) <= 0)                      # nonincreasing
    assert np.all(hv > 0) and np.all(hv <= 1 + 1e-15)
    assert np.all(hv[ts <= 0] == hv[0])                   # ReLU: flat on t <= 0
    # without ReLU h(-1) = Σ s_j e^{μ_j} > 1 (Eq. eq:model-orig)
    assert oracle.h(s, mu, -1.0, relu=0) == pytest.approx(float(np.dot(s, np.exp(mu))), rel=1e-14)


def test_P2_hprime_is_derivative():
    s, mu = G.spectrum(7)
    for t in (0.05, 0.5, 1.0, 3.0):
        e = 1e-6
        fd = (oracle.h(s, mu, t + e) - oracle.h(s, mu, t - e)) / (2 * e)
        assert oracle.hprime_abs(s, mu, t) == pytest.approx(-fd, rel=1e-8)
    assert math.isnan(oracle.hprime_abs(s, mu, 0.0))      # SPEC.md:53 rejects t <= 0


def test_H_is_primitive_of_h():
    s, mu = G.spectrum(9)
    for relu in (1, 0):
        for t in (-2.0, -0.3, 0.0, 0.4, 2.5):
            e = 1e-6
            fd = (oracle.H(s, mu, t + e, relu) - oracle.H(s, mu, t - e, relu)) / (2 * e)
            # h has a kink at 0 under the ReLU: central FD error O(e) there
            tol = 1e-6 if (relu and t == 0.0) else 1e-8
            assert fd == pytest.approx(oracle.h(s, mu, t, relu), rel=tol)
        assert oracle.H(s, mu, 0.0, relu) == 0.0


# ---------------------------------------------------------------- P3
def test_P3_noiseless_zero_and_fixed_point():
    w = _small(n=400, d=10, y_kind="noiseless")
    g, _ = w["p"].F(w["xs"])
    g0, _ = w["p"].F(np.zeros(10))
    assert np.linalg.norm(g) <= 1e-12 * np.linalg.norm(g0)   # F̄(x⋆)=0, ζ=0
    p = oracle.Problem(A=w["A"], y=w["y"], s=w["s"], mu=w["mu"], I_bar=w["I_bar"], d=10,
                       set=oracle.SET_BALL, R=4.0, center=w["xs"])
    x, _, bad = p.solve(20, 0.01, x1=w["xs"])
    assert bad == 0 and np.linalg.norm(x - w["xs"]) <= 1e-12


# ---------------------------------------------------------------- P4
def test_P4_monochromatic_single_row_closed_form():
    # W=1: h(t) = e^{-μ t+}, H(t) = (1 - e^{-μ t})/μ for t >= 0, t for t < 0
    mu, I_bar, y = 1.5, 10.0, 5.0
    for a, x in ((2.0, 0.3), (2.0, -0.4), (-1.5, 0.25)):
        p = oracle.Problem(A=np.array([[a]]), y=[y], s=[1.0], mu=[mu], I_bar=I_bar, d=1)
        g, l = p.F([x])
        z = a * x
        hz = math.exp(-mu * z) if z > 0 else 1.0
        Hz = (1 - math.exp(-mu * z)) / mu if z >= 0 else z
        assert g[0] == pytest.approx((y - I_bar * hz) * a, rel=1e-15)
        assert l == pytest.approx(y * z - I_bar * Hz, rel=1e-14)


def test_P4_two_rows_normalisation():
    # two rows, d=2: F = (1/2)[r_1 a_1 + r_2 a_2], written out by hand
    A = np.array([[1.0, 2.0], [0.5, -1.0]])
    x = np.array([0.2, 0.1])
    y = np.array([3.0, 7.0])
    p = oracle.Problem(A=A, y=y, s=[1.0], mu=[1.0], I_bar=4.0, d=2)
    g, _ = p.F(x)
    r1 = 3.0 - 4.0 * math.exp(-0.4)      # z_1 = 0.2 + 0.2 = 0.4
    r2 = 7.0 - 4.0 * 1.0                 # z_2 = 0.1 - 0.1 = 0.0 -> h = 1
    assert g == pytest.approx([(r1 * 1.0 + r2 * 0.5) / 2, (r1 * 2.0 + r2 * -1.0) / 2], rel=1e-15)


# ---------------------------------------------------------------- P4b
def _pop_c(s, mu, sigma):
    # c(σ) = Σ_j s_j μ_j e^{μ_j²σ²/2} Φ(-μ_j σ) = Σ_j s_j μ_j ½ erfcx(μ_j σ/√2)
    return float(np.sum(s * mu * 0.5 * erfcx(mu * sigma / math.sqrt(2.0))))


def test_P4b_population_closed_form_gaussian():
    """Stein's lemma with a ~ N(0, I) (Assumption 3):
    E F(x) = Ī (c(||x||) x - c(||x⋆||) x⋆).  Band 3 × 1.1 sqrt(d/n)."""
    n, d, W, I_bar = 60000, 40, 8, 100.0
    s, mu = G.spectrum(W)
    A = rng.gaussian_rows(21, rng.STREAM_TEST, np.arange(n), d)
    xs = rng.unit_sphere(21, rng.STREAM_XSTAR, d, 0.9)
    p0 = oracle.Problem(A=A, y=np.zeros(n), s=s, mu=mu, I_bar=I_bar, d=d)
    y = rng.poisson(21, rng.STREAM_Y, p0.mean(xs), np.arange(n)).astype(float)
    p = oracle.Problem(A=A, y=y, s=s, mu=mu, I_bar=I_bar, d=d)
    band = 3 * 1.1 * math.sqrt(d / n)
    r = np.random.default_rng(4)
    for trial in range(4):
        x = r.standard_normal(d)
        x *= (0.3 + 0.5 * trial) / np.linalg.norm(x)
        g, _ = p.F(x)
        fbar = I_bar * (_pop_c(s, mu, np.linalg.norm(x)) * x - _pop_c(s, mu, np.linalg.norm(xs)) * xs)
        assert np.linalg.norm(g - fbar) <= band * np.linalg.norm(fbar), trial
        # a flipped sign or dropped ReLU would be far outside the band
        assert np.linalg.norm(-g - fbar) > 5 * band * np.linalg.norm(fbar)


# ---------------------------------------------------------------- P5
@pytest.mark.parametrize("relu", [1, 0])
def test_P5_finite_difference_gradient(relu):
    w = _small(n=60, d=6, relu=relu)
    p = w["p"]
    r = np.random.default_rng(7)
    for _ in range(3):
        x = 0.5 * r.standard_normal(6)
        g, _ = p.F(x)
        fd = np.zeros(6)
        for k in range(6):
            e = np.zeros(6)
            e[k] = 1e-5
            fd[k] = (p.F(x + e)[1] - p.F(x - e)[1]) / 2e-5
        assert np.linalg.norm(fd - g) <= 1e-6 * np.linalg.norm(g)


# ---------------------------------------------------------------- P6 / P7
def test_P6_P7_monotone_and_lipschitz():
    w = _small(n=200, d=10, I_bar=30.0)
    p = w["p"]
    lam, _ = p.lambda_max(tol=1e-12)
    L = w["I_bar"] * lam * float(np.dot(w["s"], w["mu"]))
    r = np.random.default_rng(8)
    worst_ratio = 0.0
    for _ in range(1000):
        x, x2 = r.standard_normal(10), r.standard_normal(10)
        g, _ = p.F(x)
        g2, _ = p.F(x2)
        dx = x - x2
        assert np.dot(g - g2, dx) >= -1e-10 * np.dot(dx, dx)       # Eq.(monotone)
        worst_ratio = max(worst_ratio, np.linalg.norm(g - g2) / np.linalg.norm(dx))
    assert worst_ratio <= L * (1 + 1e-12)


def test_lambda_max_matches_eigvalsh():
    w = _small(n=300, d=15)
    lam, it = w["p"].lambda_max(tol=1e-13, max_it=5000)
    ev = np.linalg.eigvalsh(w["A"].T @ w["A"] / 300)[-1]
    assert lam == pytest.approx(ev, rel=1e-9)


# ---------------------------------------------------------------- P8
@pytest.mark.parametrize("sigma", [0.0, 3.0])
def test_P8_monte_carlo_variance_identity(sigma):
    """E[R^T A A^T R] = Σ_i ||a_i||² E[R_i²] with E[R_i²] = Ī h(<a_i,x⋆>) (+σ²)
    (Appendix A.2; electronic noise PAPER.md:26-41)."""
    n, d, I_bar, K = 1500, 30, 40.0, 150
    s, mu = G.spectrum(6)
    A = rng.gaussian_rows(31, rng.STREAM_TEST, np.arange(n), d)
    xs = rng.unit_sphere(31, rng.STREAM_XSTAR, d, 1.0)
    lam = oracle.Problem(A=A, y=np.zeros(n), s=s, mu=mu, I_bar=I_bar, d=d).mean(xs)
    acc = 0.0
    for k in range(K):
        y = rng.poisson(1000 + k, rng.STREAM_Y, lam, np.arange(n)).astype(float)
        if sigma:
            y = y + sigma * rng.normal(1000 + k, rng.STREAM_NOISE, np.arange(n), 0)
        g, _ = oracle.Problem(A=A, y=y, s=s, mu=mu, I_bar=I_bar, d=d).F(xs)
        acc += np.sum((n * g) ** 2)
    rows2 = np.sum(A * A, axis=1)
    expect = float(np.sum(rows2 * (lam + sigma ** 2)))
    assert acc / K == pytest.approx(expect, rel=0.10)


# ---------------------------------------------------------------- P9
def test_P9_reparameterisation():
    s, mu = np.array([0.5, 0.5]), np.array([0.02, 1.0])
    s0, I0 = oracle.reparam(s, mu, 100.0, np.array([0.0]))
    assert np.allclose(s0[0], s) and I0[0] == pytest.approx(100.0)   # e = 0 → unchanged
    s1, I1 = oracle.reparam(s, mu, 100.0, np.array([50.0]))           # exponents [1, 50]
    assert s1[0, 0] == pytest.approx(1.0, abs=1e-20) and s1[0, 1] < 1e-20
    assert I1[0] == pytest.approx(100.0 * 0.5 * (math.exp(-1) + math.exp(-50)), rel=1e-14)
    # identity: reduced model mean == direct three-material mean
    s, mu = G.spectrum(16)
    r = np.random.default_rng(9)
    b = r.standard_normal(500) * 1.5
    z = r.standard_normal(500)
    sr, Ir = oracle.reparam(s, mu, 5e4, b, clamp=1)
    assert np.allclose(sr.sum(axis=1), 1.0, rtol=0, atol=1e-15)
    for i in range(500):
        red = Ir[i] * oracle.h(sr[i], mu, z[i])
        direct = 5e4 * float(np.sum(s * np.exp(-mu * (max(b[i], 0.0) + max(z[i], 0.0)))))
        assert red == pytest.approx(direct, rel=1e-13)


def test_P9_reduced_F_equals_direct():
    """F of the reduced single-material model == F written directly from the
    three-material means (y - Ī Σ_j s_j e^{-μ_j (b+ + z+)}) a_i."""
    n, d = 400, 8
    s, mu = G.spectrum(5)
    r = np.random.default_rng(10)
    A = r.standard_normal((n, d))
    b = r.standard_normal(n)
    y = r.poisson(300, n).astype(float)
    x = 0.3 * r.standard_normal(d)
    sr, Ir = oracle.reparam(s, mu, 500.0, b)
    g, _ = oracle.Problem(A=A, y=y, s=s, mu=mu, I_bar=500.0, d=d, s_row=sr, I_row=Ir).F(x)
    z = A @ x
    lam = 500.0 * np.exp(-np.outer(np.maximum(b, 0) + np.maximum(z, 0), mu)) @ s
    gd = A.T @ (y - lam) / n
    assert np.linalg.norm(g - gd) <= 1e-12 * np.linalg.norm(gd)


# ---------------------------------------------------------------- P10
def test_P10_permutation_and_shards():
    w = _small(n=9000, d=7)      # > 2 oracle chunks
    x = 0.2 * np.ones(7)
    g, l = w["p"].F(x)
    perm = np.random.default_rng(11).permutation(9000)
    gp, lp = oracle.Problem(A=w["A"][perm], y=w["y"][perm], s=w["s"], mu=w["mu"],
                            I_bar=w["I_bar"], d=7).F(x)
    assert np.allclose(gp, g, rtol=1e-13, atol=1e-13 * np.abs(g).max()) and lp == pytest.approx(l)
    acc, lacc = np.zeros(7), 0.0
    for lo, hi in ((0, 1000), (1000, 4097), (4097, 9000)):
        gs, ls = oracle.Problem(A=w["A"][lo:hi], y=w["y"][lo:hi], s=w["s"], mu=w["mu"],
                                I_bar=w["I_bar"], d=7, n_norm=9000).F(x)
        acc += gs
        lacc += ls
    assert np.allclose(acc, g, rtol=1e-13, atol=1e-13 * np.abs(g).max())
    assert lacc == pytest.approx(l, rel=1e-13)


# ---------------------------------------------------------------- P11
def test_P11_projections():
    r = np.random.default_rng(12)
    c = r.standard_normal(20)
    v = c + 0.1 * r.standard_normal(20)
    assert np.array_equal(oracle.project(oracle.SET_BALL, 5.0, c, v), v)   # inside
    u = r.standard_normal(20)
    u /= np.linalg.norm(u)
    out = oracle.project(oracle.SET_BALL, 2.0, c, c + 4.0 * u)              # at 2R
    assert np.linalg.norm(out - c) == pytest.approx(2.0, rel=1e-15)
    assert np.allclose(out, c + 2.0 * u, rtol=0, atol=1e-15)
    assert np.array_equal(oracle.project(oracle.SET_NONNEG, 0, None, np.array([-1.0, 2.0, -3.0])),
                          [0.0, 2.0, 0.0])
    for st in (oracle.SET_BALL, oracle.SET_NONNEG, oracle.SET_NONNEG_BALL):
        cc = c if st == oracle.SET_BALL else None
        for _ in range(50):
            a, b = 3 * r.standard_normal(20), 3 * r.standard_normal(20)
            pa, pb = oracle.project(st, 2.0, cc, a), oracle.project(st, 2.0, cc, b)
            assert np.allclose(oracle.project(st, 2.0, cc, pa), pa, rtol=0, atol=1e-14)
            assert np.linalg.norm(pa - pb) <= np.linalg.norm(a - b) + 1e-14
            if st == oracle.SET_NONNEG_BALL:
                assert pa.min() >= 0 and np.linalg.norm(pa) <= 2.0 + 1e-14
                # optimality: <a - P a, x - P a> <= 0 for x in the set
                xx = np.abs(r.standard_normal(20))
                xx *= min(1.0, 2.0 / np.linalg.norm(xx))
                assert np.dot(a - pa, xx - pa) <= 1e-12


# ---------------------------------------------------------------- P12
def _iters_to(p, xs, tol, gamma, cap):
    x = np.zeros(xs.shape[0])
    done = 0
    while done < cap:
        x, _, bad = p.solve(50, gamma, x1=x)
        done += 50
        assert bad == 0
        if np.linalg.norm(x - xs) <= tol:
            # refine within the last block
            x2 = x
            return done
    return None


@pytest.mark.slow
def test_P12_E6_closed_loop_iterations_decrease_with_n():
    """E6: W=1, Ī=1, μ=1, d=100, ||x⋆||=3, γ=0.25,
    noiseless, X = B(12; x⋆); iterations to reach 1e-6 are
    nonincreasing in n ("improves up to a threshold")."""
    d = 100
    xs = rng.unit_sphere(0, rng.STREAM_XSTAR, d, 3.0)
    counts = []
    for n in (10 * d, 20 * d, 40 * d):
        A = rng.gaussian_rows(0, rng.STREAM_TEST, np.arange(n), d)
        p0 = oracle.Problem(A=A, y=np.zeros(n), s=[1.0], mu=[1.0], I_bar=1.0, d=d)
        y = p0.mean(xs)
        p = oracle.Problem(A=A, y=y, s=[1.0], mu=[1.0], I_bar=1.0, d=d, set=oracle.SET_BALL,
                           R=12.0, center=xs)
        counts.append(_iters_to(p, xs, 1e-6, 0.25, 20000))
    assert all(c is not None for c in counts), counts
    assert counts[0] >= counts[1] >= counts[2], counts


# ---------------------------------------------------------------- P13
def test_P13_population_trajectory():
    """Large-n EXACT from x_1 = 0 with X = B(R) stays on span{x⋆}, following
    the scalar recursion driven by the Stein closed form (P4b)."""
    n, d, W, I_bar, T = 120_000, 30, 10, 1e4, 40
    s, mu = G.spectrum(W)
    A = rng.gaussian_rows(41, rng.STREAM_TEST, np.arange(n), d)
    xs = rng.unit_sphere(41, rng.STREAM_XSTAR, d, 1.0)
    p0 = oracle.Problem(A=A, y=np.zeros(n), s=s, mu=mu, I_bar=I_bar, d=d)
    y = rng.poisson(41, rng.STREAM_Y, p0.mean(xs), np.arange(n)).astype(float)
    R = 1.0
    p = oracle.Problem(A=A, y=y, s=s, mu=mu, I_bar=I_bar, d=d, set=oracle.SET_BALL, R=R)
    gamma = 1.0 / (4.0 * I_bar * float(np.dot(s, mu)) * 1.05)
    x, _, _ = p.solve(T, gamma)
    rho = np.linalg.norm(xs)
    u = xs / rho

    def Fbar(a):
        return I_bar * (_pop_c(s, mu, abs(a)) * a - _pop_c(s, mu, rho) * rho)

    a = 0.0
    for _ in range(T):
        ah = float(np.clip(a - gamma * Fbar(a), -R, R))
        a = float(np.clip(a - gamma * Fbar(ah), -R, R))
    band = 3 * 1.1 * math.sqrt(d / n)
    assert abs(np.dot(x, u) - a) <= band
    assert np.linalg.norm(x - np.dot(x, u) * u) <= band


# ---------------------------------------------------------------- workloads
def test_workload_c1_counts_and_step():
    w = Wk.build(G.C1)
    assert w["A"].dtype == np.float64 and w["A"].shape == (2000, 100)
    assert np.all(w["counts"] >= 0)
    assert abs(np.linalg.norm(w["x_star"]) - 1.0) < 1e-14
    # counts mean matches the Poisson means (E[y] = Ī h, Eq. model)
    assert abs(np.mean(w["counts"] - w["lam"])) < 4 * math.sqrt(np.mean(w["lam"]) / 2000)
    gam, lam = Wk.step_size(w["problem"], w["s"], w["mu"], G.C1.I_bar)
    # Marchenko–Pastur edge (1 + sqrt(d/n))² for N(0,1) rows
    assert lam == pytest.approx((1 + math.sqrt(100 / 2000)) ** 2, rel=0.1)
    w32 = Wk.build(G.C1F)
    assert np.array_equal(w32["A"], w["A"].astype(np.float32))


def test_workload_rows_subset_consistent():
    full = Wk.build(G.scaled(G.C2, 64))
    sub = Wk.build(G.scaled(G.C2, 64), rows=np.array([5, 17, 63]))
    assert np.array_equal(sub["A"], full["A"][[5, 17, 63]])
    assert np.array_equal(sub["counts"], full["counts"][[5, 17, 63]])


def test_workload_c3_reparam_rows():
    cfg = G.scaled(G.C3, 3000)
    w = Wk.build(cfg)
    assert np.all(w["I_row"] > 0) and np.all(w["I_row"] <= cfg.I_bar * (1 + 1e-6))
    assert np.allclose(w["s_row"].sum(axis=1), 1.0, atol=1e-6)
    # rows with b <= 0 keep the original spectrum (clamp, reading R7)
    neg = w["b"] <= 0
    assert np.allclose(w["I_row"][neg], cfg.I_bar, rtol=1e-7)
