"""Pins of the oracle's TV machinery (NEXT-2) — CPU only.

X = X1 ∩ X2 with X1 = {||x||_TV <= τ}, X2 = R_+^d.  The oracle follows the
paper's recipe: P_X1 approximated by the TV prox of Eq.(TV-regularization)
with λ binary-searched to | ||x̄||_TV - τ | <= tol, and Dykstra's algorithm
Eq.(projection-intersection) for the intersection.  Pinned against: the SPEC
worked examples of tv_norm, the prox's duality gap (a certificate of
optimality independent of the algorithm), closed-form limits (λ = 0, λ -> ∞,
τ = 0), monotonicity of ||prox(z, λ)||_TV in λ, and scipy's SLSQP solution
of the same projections written as smooth QPs (a library routine).
"""
import math

import numpy as np
import pytest
from scipy.optimize import minimize

import oracle


def D_matrix(side):
    """The forward-difference operator, built independently of the oracle."""
    rows = []
    for r in range(side):
        for c in range(side - 1):
            v = np.zeros(side * side)
            v[r * side + c + 1], v[r * side + c] = 1.0, -1.0
            rows.append(v)
    for r in range(side - 1):
        for c in range(side):
            v = np.zeros(side * side)
            v[(r + 1) * side + c], v[r * side + c] = 1.0, -1.0
            rows.append(v)
    return np.array(rows)


def test_tv_norm_worked_examples():
    """constant -> 0; [[0,1],[0,1]] -> 2; |c|-homogeneous."""
    assert oracle.tv_norm(np.full(9, 3.7)) == 0.0
    assert oracle.tv_norm(np.array([[0.0, 1.0], [0.0, 1.0]])) == 2.0
    r = np.random.default_rng(0)
    x = r.standard_normal(25)
    assert np.isclose(oracle.tv_norm(-2.5 * x), 2.5 * oracle.tv_norm(x), rtol=1e-14)
    # 3x3 hand count: rows [0,2,2],[1,1,0],[0,0,0]: horizontal 2+0+0+1+0+0 = 3,
    # vertical |1-0|+|1-2|+|0-2| + |0-1|+|0-1|+|0-0| = 1+1+2+1+1+0 = 6
    assert oracle.tv_norm(np.array([0, 2, 2, 1, 1, 0, 0, 0, 0.0])) == 9.0
    assert np.isclose(oracle.tv_norm(x), np.abs(D_matrix(5) @ x).sum(), rtol=1e-14)


@pytest.mark.parametrize("side,lam", [(2, 0.3), (5, 0.5), (8, 2.0), (16, 0.7)])
def test_prox_duality_gap(side, lam):
    """x = z - D^T u with |u| <= λ/2 and a vanishing gap between the primal
    ||x - z||^2 + λ||Dx||_1 and the dual 2<D^T u, z> - ||D^T u||^2."""
    z = np.random.default_rng(side).standard_normal(side * side)
    x, u, it = oracle.prox_tv(z, lam, rtol=1e-12, max_it=200000)
    D = D_matrix(side)
    assert np.max(np.abs(u)) <= lam / 2 * (1 + 1e-12)
    assert np.allclose(x, z - D.T @ u, atol=1e-12)
    P = np.sum((x - z) ** 2) + lam * np.abs(D @ x).sum()
    Dual = 2 * np.dot(D.T @ u, z) - np.sum((D.T @ u) ** 2)
    assert P - Dual >= -1e-12 and P - Dual <= 1e-7 * P, (P, Dual)


def test_prox_limits_and_monotone_tv():
    z = np.random.default_rng(3).standard_normal(36)
    x0, _, _ = oracle.prox_tv(z, 0.0)
    assert np.array_equal(x0, z)
    xb, _, _ = oracle.prox_tv(z, 1e4, rtol=1e-10, max_it=100000)
    assert np.allclose(xb, z.mean(), atol=1e-4)
    tvs = [oracle.tv_norm(oracle.prox_tv(z, lam, rtol=1e-10, max_it=100000)[0])
           for lam in (0.05, 0.1, 0.3, 0.6, 1.2, 3.0)]
    assert all(a >= b - 1e-7 for a, b in zip(tvs, tvs[1:]))


def _slsqp(z, tau, nonneg):
    """min ||x - z||^2 s.t. ||Dx||_1 <= τ (and x >= 0) as a smooth QP in (x, t),
    -t <= Dx <= t, Σ t <= τ, solved by scipy SLSQP."""
    d = z.shape[0]
    side = int(np.sqrt(d))
    D = D_matrix(side)
    m = D.shape[0]
    f = lambda v: np.sum((v[:d] - z) ** 2)  # noqa: E731
    jac = lambda v: np.concatenate([2 * (v[:d] - z), np.zeros(m)])  # noqa: E731
    cons = [{"type": "ineq", "fun": lambda v: v[d:] - D @ v[:d],
             "jac": lambda v: np.hstack([-D, np.eye(m)])},
            {"type": "ineq", "fun": lambda v: v[d:] + D @ v[:d],
             "jac": lambda v: np.hstack([D, np.eye(m)])},
            {"type": "ineq", "fun": lambda v: np.array([tau - v[d:].sum()]),
             "jac": lambda v: np.concatenate([np.zeros(d), -np.ones(m)])[None, :]}]
    bounds = [(0, None) if nonneg else (None, None)] * d + [(0, None)] * m
    v0 = np.concatenate([np.full(d, max(z.mean(), 0.0)), np.zeros(m)])
    res = minimize(f, v0, jac=jac, constraints=cons, bounds=bounds, method="SLSQP",
                   options={"ftol": 1e-14, "maxiter": 2000})
    assert res.success, res.message
    return res.x[:d]


def test_project_tv_matches_qp_and_limits():
    r = np.random.default_rng(5)
    z = r.standard_normal(9)
    tau = 0.4 * oracle.tv_norm(z)
    x, steps = oracle.project_tv(z, tau, tv_tol=1e-9, rtol=1e-13, max_it=200000)
    assert steps >= 1 and abs(oracle.tv_norm(x) - tau) <= 1e-8
    assert np.allclose(x, _slsqp(z, tau, nonneg=False), atol=1e-5)
    # inside the ball: unchanged; τ = 0: the constant image at mean(z)
    x_in, st = oracle.project_tv(z, 2 * oracle.tv_norm(z))
    assert st == 0 and np.array_equal(x_in, z)
    x0, _ = oracle.project_tv(z, 0.0, tv_tol=1e-6, rtol=1e-12, max_it=400000)
    assert np.allclose(x0, z.mean(), atol=1e-5)
    # the paper's tolerance on a larger image
    z8 = r.standard_normal(64)
    x8, _ = oracle.project_tv(z8, 0.5 * oracle.tv_norm(z8))
    assert abs(oracle.tv_norm(x8) - 0.5 * oracle.tv_norm(z8)) <= 0.01


def test_dykstra_tv_nonneg_matches_qp():
    r = np.random.default_rng(6)
    z = r.standard_normal(9) + 0.3
    tau = 0.5 * oracle.tv_norm(z)
    x, it = oracle.project_tv_nonneg(z, tau, tv_tol=1e-10, rtol=1e-13, max_it=200000,
                                     tol=1e-11, max_outer=100000)
    assert it >= 2
    assert x.min() >= 0.0 and oracle.tv_norm(x) <= tau + 1e-6
    assert np.allclose(x, _slsqp(z, tau, nonneg=True), atol=1e-4)
    # already in X1 ∩ X2: returned after one sweep
    zi = np.abs(z)
    xi, it = oracle.project_tv_nonneg(zi, oracle.tv_norm(zi) + 1.0)
    assert it == 1 and np.array_equal(xi, zi)


def test_solve_with_tv_set_reduces_to_orthant_for_large_tau():
    """With τ above any reachable TV, X1 ∩ X2 = X2 and the Dykstra projection
    returns max(z, 0) exactly, so EXACT with the TV set equals EXACT with the
    orthant, iterate for iterate."""
    r = np.random.default_rng(2)
    n, d = 300, 36
    A = np.abs(r.standard_normal((n, d))) / 6
    s, mu = np.array([0.3, 0.7]), np.array([1.5, 0.8])
    xs = np.abs(r.standard_normal(d)) * 0.4
    y = oracle.Problem(A=A, y=np.zeros(n), s=s, mu=mu, I_bar=200.0, d=d).mean(xs)
    p_tv = oracle.Problem(A=A, y=y, s=s, mu=mu, I_bar=200.0, d=d, set=oracle.SET_TV_NONNEG,
                          tv={"tau": 1e9})
    p_nn = oracle.Problem(A=A, y=y, s=s, mu=mu, I_bar=200.0, d=d, set=oracle.SET_NONNEG)
    x1b, _, _ = p_tv.solve(15, 1e-3, x1=np.linspace(-1, 1, d))
    x2b, _, _ = p_nn.solve(15, 1e-3, x1=np.linspace(-1, 1, d))
    assert np.array_equal(x1b, x2b)
    # a binding τ keeps every iterate in X (nonnegative, TV within the tolerance)
    tau = 0.5 * oracle.tv_norm(xs)
    p_b = oracle.Problem(A=A, y=y, s=s, mu=mu, I_bar=200.0, d=d, set=oracle.SET_TV_NONNEG,
                         tv={"tau": tau, "tol": 1e-6, "rtol": 1e-10, "max_it": 100000,
                             "dykstra_tol": 1e-9})
    xb, _, _ = p_b.solve(5, 1e-3, x1=np.linspace(-1, 1, d))
    assert xb.min() >= 0.0 and oracle.tv_norm(xb) <= tau + 1e-5


@pytest.mark.parametrize("k", [2, 3, 8])
def test_kary_search_matches_qp_and_binary(k):
    """Reading R22: k λ values per search round.  The result is still a TV
    prox of z whose TV is within tv_tol of τ, so at tight tolerances it is the
    projection (SLSQP QP) like the binary search's; rounds shrink roughly by
    log2(k + 1); k = 1 is exactly the binary search."""
    r = np.random.default_rng(11)
    z = r.standard_normal(16)
    tau = 0.35 * oracle.tv_norm(z)
    x1, st1 = oracle.project_tv(z, tau, tv_tol=1e-9, rtol=1e-13, max_it=200000, k=1)
    xk, stk = oracle.project_tv(z, tau, tv_tol=1e-9, rtol=1e-13, max_it=200000, k=k)
    assert abs(oracle.tv_norm(xk) - tau) <= 1e-8
    assert np.allclose(xk, _slsqp(z, tau, nonneg=False), atol=1e-5)
    assert np.allclose(xk, x1, atol=1e-6)
    assert stk <= st1 and stk <= math.ceil(st1 / math.log2(k + 1)) + 2
    xb, _ = oracle.project_tv(z, tau, tv_tol=1e-9, rtol=1e-13, max_it=200000)
    assert np.array_equal(xb, x1)          # default k = 1: the binary search itself
    # orthant ∩ TV ball by Dykstra with the k-ary inner search
    zn = z + 0.3
    taun = 0.5 * oracle.tv_norm(np.maximum(zn, 0))
    xn, it = oracle.project_tv_nonneg(zn, taun, tv_tol=1e-10, rtol=1e-13, max_it=200000,
                                      tol=1e-11, max_outer=100000, k=k)
    assert xn.min() >= 0.0 and oracle.tv_norm(xn) <= taun + 1e-6
    assert np.allclose(xn, _slsqp(zn, taun, nonneg=True), atol=1e-4)


def test_kary_bracket_large_lambda():
    """τ far below TV(z): the bracket doubles λ past 2^k; the k-ary bracket
    (2^(gk + j)) lands on the same power-of-two bracket as the doubling loop."""
    r = np.random.default_rng(12)
    z = 40.0 * r.standard_normal(25)
    tau = 1e-3 * oracle.tv_norm(z)
    for k in (1, 3, 5):
        x, st = oracle.project_tv(z, tau, tv_tol=1e-6, rtol=1e-12, max_it=400000, k=k)
        assert abs(oracle.tv_norm(x) - tau) <= 1e-6, (k, oracle.tv_norm(x), tau)


@pytest.mark.parametrize("k", [1, 3])
def test_warm_started_proxes_match_qp(k):
    """Reading R23: each prox of a projection starts FISTA from the previous
    prox's dual solution (clipped to the new box).  The prox itself is the
    same minimiser, so at tight tolerances the projection is unchanged (QP
    certificate); at the paper's tolerances the TV bound still holds and the
    proxes need fewer FISTA iterations than cold starts."""
    r = np.random.default_rng(11)
    z = r.standard_normal(16)
    tau = 0.35 * oracle.tv_norm(z)
    xw, _ = oracle.project_tv(z, tau, tv_tol=1e-9, rtol=1e-13, max_it=200000, k=k, warm=True)
    assert abs(oracle.tv_norm(xw) - tau) <= 1e-8
    assert np.allclose(xw, _slsqp(z, tau, nonneg=False), atol=1e-5)
    zn = z + 0.3
    taun = 0.5 * oracle.tv_norm(np.maximum(zn, 0))
    xn, _ = oracle.project_tv_nonneg(zn, taun, tv_tol=1e-10, rtol=1e-13, max_it=200000, tol=1e-11,
                                     max_outer=100000, k=k, warm=True)
    assert xn.min() >= 0.0 and np.allclose(xn, _slsqp(zn, taun, nonneg=True), atol=1e-4)
    # paper tolerances on a 48 x 48 phantom: fewer FISTA iterations, same guarantees
    from gen import ct
    img = ct.ellipse_phantom(5, 48, 6) + 0.2 * r.standard_normal(48 * 48)
    t = oracle.tv_norm(ct.ellipse_phantom(5, 48, 6))
    oracle.fista_iterations(True)
    xc, _ = oracle.project_tv_nonneg(img, t, k=k)
    n_cold = oracle.fista_iterations(True)
    xh, _ = oracle.project_tv_nonneg(img, t, k=k, warm=True)
    n_warm = oracle.fista_iterations(True)
    assert n_warm < (0.8 if k == 1 else 1.0) * n_cold, (n_warm, n_cold)
    for x in (xc, xh):
        assert x.min() >= 0.0 and oracle.tv_norm(x) <= t + 0.05
    assert np.linalg.norm(xh - xc) <= 1e-3 * np.linalg.norm(xc)
