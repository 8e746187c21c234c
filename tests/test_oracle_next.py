"""Pins of the oracle's NEXT-row functions — CPU only.

NEXT-1: stacked multi-window operator (footnote PAPER.md:842)
and the averaged-iterate stopping rule (reading R15).
NEXT-3: the §3.1 comparison objectives L2, L1 and the Poisson NLL
 and their (sub)gradients.

Each function is pinned against something other than itself: the SPEC worked
examples (closed forms), special cases that reduce to the already-pinned
oracle_F, finite differences, the Gaussian population closed form, a
single-row hand evaluation, and the W = 1 identity ∇NLL = μ F.
"""
import math

import numpy as np
import pytest
from scipy.special import erfcx

import oracle
from gen import configs as G
from gen import rng


def _A(n, d, seed=5):
    return rng.gaussian_rows(seed, rng.STREAM_TEST, np.arange(n), d)


def _windows(Om, W, seed=0):
    r = np.random.default_rng(seed)
    s = r.uniform(0.2, 1.0, (Om, W))
    s /= s.sum(axis=1, keepdims=True)
    I = r.uniform(20.0, 80.0, Om)
    return s, I


def _win_problem(n=400, d=10, Om=3, W=6, seed=5, noiseless=False, relu=1, xs_norm=0.8):
    A = _A(n, d, seed)
    _, mu = G.spectrum(W)
    s_win, I_win = _windows(Om, W, seed)
    xs = rng.unit_sphere(seed, rng.STREAM_XSTAR, d, xs_norm)
    ys = []
    for w in range(Om):
        pw = oracle.Problem(A=A, y=np.zeros(n), s=s_win[w], mu=mu, I_bar=I_win[w], d=d, relu=relu)
        lam = pw.mean(xs)
        ys.append(lam if noiseless else
                  rng.poisson(seed + w, rng.STREAM_Y, lam, np.arange(n)).astype(float))
    y_win = np.array(ys)
    p = oracle.Problem(A=A, y=np.zeros(n), s=s_win[0], mu=mu, I_bar=1.0, d=d, relu=relu)
    return dict(A=A, mu=mu, s_win=s_win, I_win=I_win, y_win=y_win, xs=xs, p=p, n=n, d=d)


# ------------------------------------------------------------- averaging
def test_average_spec_worked_examples():
    """constant history -> the constant; t=2 -> mean{x1,x2};
    t=4 -> mean{x2,x3,x4}; plus t=1 and t=5 (window ⌈t/2⌉..t)."""
    r = np.random.default_rng(0)
    H = r.standard_normal((6, 4))
    c = np.tile(r.standard_normal(4), (6, 1))
    assert np.allclose(oracle.average(c, 6), c[0], rtol=0, atol=1e-15)
    assert np.array_equal(oracle.average(H, 1), H[0])
    assert np.allclose(oracle.average(H, 2), (H[0] + H[1]) / 2, rtol=0, atol=1e-15)
    assert np.allclose(oracle.average(H, 4), (H[1] + H[2] + H[3]) / 3, rtol=0, atol=1e-15)
    assert np.allclose(oracle.average(H, 5), (H[2] + H[3] + H[4]) / 3, rtol=0, atol=1e-15)


def _plain_iterates(p, T, gam):
    xs = [p.project(np.zeros(p.d))]
    for _ in range(T):
        x, _, _ = p.solve(1, gam, x1=xs[-1])
        xs.append(x)
    return np.array(xs)


def test_solve_avg_window_and_stop_rule():
    w = _win_problem()
    A, mu = w["A"], w["mu"]
    s, _ = G.spectrum(6)
    y = rng.poisson(3, rng.STREAM_Y, oracle.Problem(A=A, y=np.zeros(400), s=s, mu=mu,
                                                    I_bar=40.0, d=10).mean(w["xs"]),
                    np.arange(400)).astype(float)
    p = oracle.Problem(A=A, y=y, s=s, mu=mu, I_bar=40.0, d=10, set=oracle.SET_BALL, R=1.0)
    gam = 0.01
    T = 40
    H = _plain_iterates(p, T, gam)
    # tol = 0: never stops; returns x̄_{T+1} and x_{T+1}
    xb, xl, it, mv, bad = p.solve_avg(T, gam, tol=0.0)
    assert bad == 0 and it == T
    assert np.allclose(xl, H[T], rtol=0, atol=1e-13)
    lo = (T + 2) // 2                      # ⌈(T+1)/2⌉, 1-based
    assert np.allclose(xb, H[lo - 1:].mean(axis=0), rtol=0, atol=1e-13)
    # movement sequence from the plain iterates; the stop is the first k >= 2
    # with ||x̄_k - x̄_{k-1}|| <= tol
    bars = [H[(k + 1) // 2 - 1:k].mean(axis=0) for k in range(1, T + 2)]
    moves = np.array([np.linalg.norm(bars[k] - bars[k - 1]) for k in range(1, T + 1)])
    tol = float(np.sort(moves)[len(moves) // 2])
    k_stop = int(np.argmax(moves <= tol)) + 2          # iterate index at the stop
    xb2, _, it2, mv2, _ = p.solve_avg(T, gam, tol=tol * (1 + 1e-9))
    assert it2 == k_stop - 1
    assert np.allclose(xb2, bars[k_stop - 1], rtol=0, atol=1e-13)
    assert abs(mv2 - moves[k_stop - 2]) <= 1e-12


def test_solve_avg_noiseless_converges_to_truth():
    """Noiseless, x⋆ interior to X: F(x⋆) = 0 and the
    averaged iterate converges to x⋆."""
    w = _win_problem(n=600, d=8, noiseless=True)
    s, _ = G.spectrum(6)
    p0 = oracle.Problem(A=w["A"], y=np.zeros(600), s=s, mu=w["mu"], I_bar=1.0, d=8)
    y = p0.mean(w["xs"])
    p = oracle.Problem(A=w["A"], y=y, s=s, mu=w["mu"], I_bar=1.0, d=8, set=oracle.SET_BALL,
                       R=4.0)
    xb, xl, it, mv, bad = p.solve_avg(20000, 0.2, tol=1e-9)
    assert bad == 0 and it < 20000 and mv <= 1e-9
    assert np.linalg.norm(xb - w["xs"]) <= 1e-6
    assert np.linalg.norm(xl - w["xs"]) <= 1e-7


# ------------------------------------------------------------- windows
def test_windows_single_window_is_F():
    w = _win_problem(Om=1)
    p1 = oracle.Problem(A=w["A"], y=w["y_win"][0], s=w["s_win"][0], mu=w["mu"],
                        I_bar=w["I_win"][0], d=w["d"])
    for x in (np.zeros(w["d"]), w["xs"], -0.5 * w["xs"]):
        g1, l1 = p1.F(x)
        g, l = w["p"].F_windows(x, w["s_win"], w["I_win"], w["y_win"])
        assert np.allclose(g, g1, rtol=1e-13, atol=1e-14) and math.isclose(l, l1, rel_tol=1e-13)


def test_windows_mean_of_window_operators():
    """Stacking Ω windows of n rays: n_tot = Ω n, so F is the mean of the
    per-window operators (each the pinned single-window oracle_F)."""
    w = _win_problem(Om=3)
    x = 0.4 * w["xs"] + 0.1
    gs, ls = [], []
    for k in range(3):
        pk = oracle.Problem(A=w["A"], y=w["y_win"][k], s=w["s_win"][k], mu=w["mu"],
                            I_bar=w["I_win"][k], d=w["d"])
        g, l = pk.F(x)
        gs.append(g)
        ls.append(l)
    g, l = w["p"].F_windows(x, w["s_win"], w["I_win"], w["y_win"])
    assert np.allclose(g, np.mean(gs, axis=0), rtol=1e-12, atol=1e-14)
    assert math.isclose(l, np.mean(ls), rel_tol=1e-12)
    # a window-index mix-up (y of window 0 with spectrum of window 1) is caught
    g_bad, _ = w["p"].F_windows(x, w["s_win"][[1, 0, 2]], w["I_win"], w["y_win"])
    assert np.linalg.norm(g_bad - g) > 1e-3 * np.linalg.norm(g)


def test_windows_noiseless_zero_fd_and_monotone():
    w = _win_problem(n=120, d=5, Om=3, noiseless=True)
    g, _ = w["p"].F_windows(w["xs"], w["s_win"], w["I_win"], w["y_win"])
    assert np.linalg.norm(g) <= 1e-12 * np.max(w["I_win"])
    wn = _win_problem(n=80, d=5, Om=2)
    r = np.random.default_rng(3)
    for _ in range(3):
        x = 0.5 * r.standard_normal(5)
        g, _ = wn["p"].F_windows(x, wn["s_win"], wn["I_win"], wn["y_win"])
        fd = np.zeros(5)
        for k in range(5):
            e = np.zeros(5)
            e[k] = 1e-5
            fd[k] = (wn["p"].F_windows(x + e, wn["s_win"], wn["I_win"], wn["y_win"])[1] -
                     wn["p"].F_windows(x - e, wn["s_win"], wn["I_win"], wn["y_win"])[1]) / 2e-5
        assert np.linalg.norm(fd - g) <= 1e-6 * np.linalg.norm(g)
    for _ in range(200):
        x, xp = r.standard_normal(5), r.standard_normal(5)
        gx, _ = wn["p"].F_windows(x, wn["s_win"], wn["I_win"], wn["y_win"])
        gp, _ = wn["p"].F_windows(xp, wn["s_win"], wn["I_win"], wn["y_win"])
        assert np.dot(gx - gp, x - xp) >= -1e-10 * np.dot(x - xp, x - xp)


def _pop_c(s, mu, sigma):
    return float(np.sum(s * mu * 0.5 * erfcx(mu * sigma / math.sqrt(2.0))))


def test_windows_population_closed_form():
    """Stein's lemma per window (a ~ N(0, I)):
    E F(x) = (1/Ω) Σ_ω Ī_ω (c_ω(||x||) x - c_ω(||x⋆||) x⋆)."""
    w = _win_problem(n=40000, d=30, Om=3, W=8, seed=11)
    band = 3 * 1.1 * math.sqrt(30 / 40000)
    r = np.random.default_rng(2)
    for t in range(3):
        x = r.standard_normal(30)
        x *= (0.3 + 0.4 * t) / np.linalg.norm(x)
        g, _ = w["p"].F_windows(x, w["s_win"], w["I_win"], w["y_win"])
        fbar = np.mean([w["I_win"][k] * (_pop_c(w["s_win"][k], w["mu"], np.linalg.norm(x)) * x -
                                         _pop_c(w["s_win"][k], w["mu"], np.linalg.norm(w["xs"])) *
                                         w["xs"]) for k in range(3)], axis=0)
        assert np.linalg.norm(g - fbar) <= band * np.linalg.norm(fbar), t


# ------------------------------------------------------------- objectives
def _obj_problem(n=150, d=6, W=4, relu=1, noiseless=False, seed=9, I_bar=60.0):
    A = _A(n, d, seed)
    s, mu = G.spectrum(W)
    xs = rng.unit_sphere(seed, rng.STREAM_XSTAR, d, 0.7)
    lam = oracle.Problem(A=A, y=np.zeros(n), s=s, mu=mu, I_bar=I_bar, d=d, relu=relu).mean(xs)
    y = lam if noiseless else rng.poisson(seed, rng.STREAM_Y, lam, np.arange(n)).astype(float)
    return oracle.Problem(A=A, y=y, s=s, mu=mu, I_bar=I_bar, d=d, relu=relu), xs, A, y, s, mu


@pytest.mark.parametrize("mode", [1, 3])
@pytest.mark.parametrize("relu", [0, 1])
def test_objective_finite_differences(mode, relu):
    p, xs, A, y, s, mu = _obj_problem(relu=relu)
    r = np.random.default_rng(mode + 10 * relu)
    done = 0
    while done < 3:
        x = 0.6 * r.standard_normal(6)
        if relu and np.min(np.abs(A @ x)) < 1e-3:   # stay away from the kink of t_+
            continue
        g, _ = p.objective(x, mode)
        fd = np.zeros(6)
        for k in range(6):
            e = np.zeros(6)
            e[k] = 1e-6
            fd[k] = (p.objective(x + e, mode)[1] - p.objective(x - e, mode)[1]) / 2e-6
        assert np.linalg.norm(fd - g) <= 1e-5 * np.linalg.norm(g), (mode, relu)
        done += 1


def test_objective_l1_subgradient_smooth_points():
    p, xs, A, y, s, mu = _obj_problem(relu=0)
    r = np.random.default_rng(1)
    for _ in range(3):
        x = 0.6 * r.standard_normal(6)
        m = np.array([oracle.h(s, mu, z, relu=0) for z in A @ x]) * 60.0
        assert np.min(np.abs(m - y)) > 1e-3           # no residual at a kink
        g, _ = p.objective(x, 2)
        fd = np.zeros(6)
        for k in range(6):
            e = np.zeros(6)
            e[k] = 1e-8
            fd[k] = (p.objective(x + e, 2)[1] - p.objective(x - e, 2)[1]) / 2e-8
        assert np.linalg.norm(fd - g) <= 1e-5 * np.linalg.norm(g)


def test_objectives_noiseless_truth_is_stationary():
    p, xs, *_ = _obj_problem(noiseless=True)
    for mode in (1, 2, 3):
        g, l = p.objective(xs, mode)
        assert np.linalg.norm(g) <= 1e-12 * 60.0, mode
        if mode in (1, 2):
            assert abs(l) <= 1e-12 * 60.0


def test_objectives_single_row_closed_form():
    """W = 1, d = 1, one row a = 2, relu = 1: h = e^{-μ z+}, h' = -μ e^{-μ z}
    (z > 0).  At x = 0.3 (z = 0.6), Ī = 5, μ = 1.5, y = 3."""
    p = oracle.Problem(A=np.array([[2.0]]), y=np.array([3.0]), s=[1.0], mu=[1.5], I_bar=5.0,
                       d=1)
    z = 0.6
    h = math.exp(-1.5 * z)
    hp = -1.5 * h
    m = 5.0 * h
    g1, l1 = p.objective(np.array([0.3]), 1)
    assert math.isclose(l1, (m - 3.0) ** 2, rel_tol=1e-14)
    assert math.isclose(g1[0], 2.0 * (m - 3.0) * 5.0 * hp * 2.0, rel_tol=1e-14)
    g2, l2 = p.objective(np.array([0.3]), 2)
    assert math.isclose(l2, abs(m - 3.0), rel_tol=1e-14)
    assert math.isclose(g2[0], math.copysign(1.0, m - 3.0) * 5.0 * hp * 2.0, rel_tol=1e-14)
    g3, l3 = p.objective(np.array([0.3]), 3)
    assert math.isclose(l3, m - 3.0 * math.log(m), rel_tol=1e-14)
    assert math.isclose(g3[0], (5.0 - 3.0 / h) * hp * 2.0, rel_tol=1e-14)
    # negative z under relu: h' = 0, so every gradient vanishes
    for mode in (1, 2, 3):
        assert p.objective(np.array([-0.3]), mode)[0][0] == 0.0


def test_objective_W1_nll_gradient_is_mu_F():
    """W = 1, relu = 0: h' = -μ h, so ∇NLL = (Ī - y/h)(-μ h) a = μ (y - Ī h) a,
    i.e. ∇NLL(x) = μ F(x) with F the (pinned) EXACT operator."""
    A = _A(200, 7)
    xs = rng.unit_sphere(2, rng.STREAM_XSTAR, 7, 0.6)
    p0 = oracle.Problem(A=A, y=np.zeros(200), s=[1.0], mu=[1.3], I_bar=40.0, d=7, relu=0)
    y = rng.poisson(2, rng.STREAM_Y, p0.mean(xs), np.arange(200)).astype(float)
    p = oracle.Problem(A=A, y=y, s=[1.0], mu=[1.3], I_bar=40.0, d=7, relu=0)
    x = 0.3 * xs + 0.05
    g, _ = p.objective(x, 3)
    F, _ = p.F(x)
    assert np.allclose(g, 1.3 * F, rtol=1e-12, atol=1e-14)


def test_gd_baseline_descends_and_fixes_truth():
    p, xs, *_ = _obj_problem()
    x0 = np.full(6, 0.05)        # at x = 0 every z_i = 0 and h'(0) = 0 under relu
    l0 = p.objective(x0, 1)[1]
    x1, bad = p.solve_gd(1, 50, 1e-5, x1=x0)
    assert bad == 0 and p.objective(x1, 1)[1] < l0
    pn, xsn, *_ = _obj_problem(noiseless=True)
    for mode in (1, 3):
        x, bad = pn.solve_gd(mode, 10, 1e-4, x1=xsn)
        assert np.linalg.norm(x - xsn) <= 1e-12
