"""GPU parity at the sizes and kernel instantiations the benchmarks run.

Eq.(operator) per call and Eq.(extragrad-method)
 trajectories, the CUDA path through the C ABI against the
fp64 oracle (BASELINE.json north_star: per call ≤ 1e-4 relative ℓ2, final
iterate ≤ 1e-3, counts bit-exact).

Input sharing: the Gaussian rows of A are the output of the
seeded generator; at these sizes the oracle takes the bytes drawn by the
generator's CUDA twin (libpolysynth) after `oracle.workloads._shared_rows`
has redrawn sampled rows with gen/rng and found them bit-identical.
Everything the method computes from A — the means λ, the Poisson counts, the
A.1 spectra, γ, F and the iterates — the oracle computes itself; its counts
are then compared with the device's bit for bit.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from gen import configs as G  # noqa: E402
from gen import rng  # noqa: E402
from oracle import workloads as OW  # noqa: E402

TOL32 = 1e-4
TOL_ITER = 1e-3


def _W():
    from paper_2503_19925_b200 import workloads as PW
    return PW


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def gpu_F(p, x):
    g, loss = p.loss_grad(torch.tensor(np.asarray(x, dtype=np.float64), device="cuda"))
    return g.cpu().numpy(), loss


def host_rows(t, d):
    return t[:, :d].cpu().numpy()


def eval_pts(wo, prob, cfg, gamma=None, k_iter=0):
    """x = 0, x⋆, P_X(x⋆ + 0.3 u) for 3 unit u, first iterates."""
    xs = wo["x_star"]
    pts = [np.zeros(cfg.d), xs.copy()]
    r = np.random.default_rng(cfg.seed + 100)
    for _ in range(3):
        u = r.standard_normal(cfg.d)
        pts.append(prob.project(xs + 0.3 * u / np.linalg.norm(u)))
    x = np.zeros(cfg.d)
    for _ in range(k_iter):
        x, _, _ = prob.solve(1, gamma, x1=x)
        pts.append(x.copy())
    return pts


def gamma_of(prob, wo, cfg, max_it, tol=1e-8):
    """Reading R5: γ = 1/(4 Ī λ̂max Σ s_j μ_j) (max_i Ī'_i Σ_j s'_ij μ_j with
    per-row spectra), λ̂max by the ORACLE's power iteration; the same double
    is handed to both sides."""
    lam, _ = prob.lambda_max(max_it=max_it, tol=tol)
    if wo.get("I_row") is not None:
        c = float(np.max(wo["I_row"] * (wo["s_row"] @ wo["mu"])))
    else:
        c = cfg.I_bar * float(np.dot(wo["s"], wo["mu"]))
    return 1.0 / (4.0 * lam * c)


# ------------------------------------------------------------------ C2, full size
@pytest.fixture(scope="module")
def c2_both():
    cfg = G.C2
    wg = _W().build(cfg)
    wo = OW.build(cfg, A=host_rows(wg["A"], cfg.d))
    return cfg, wg, wo


def test_c2_full_counts_bit_exact(c2_both):
    cfg, wg, wo = c2_both
    assert np.array_equal(wg["counts"].cpu().numpy(), wo["counts"])


def test_c2_full_per_call_parity(c2_both):
    """All 200,000 rows in the bench's launch configuration (148 CTAs, ~1351
    rows per CTA accumulated in fp32 registers): ≤ 1e-4 at the §8(d) points."""
    cfg, wg, wo = c2_both
    p = _W().make_poly(wg)
    d = p.describe()
    assert (d["grid"], d["V"], d["WPR"], d["full"]) == (148, 8, 1, 1), d
    prob = wo["problem"]
    gam = gamma_of(prob, wo, cfg, max_it=30)
    for x in eval_pts(wo, prob, cfg, gamma=gam, k_iter=3):
        g_ref, l_ref = prob.F(x)
        g, l = gpu_F(p, x)
        assert rel(g, g_ref) <= TOL32, rel(g, g_ref)
        assert abs(l - l_ref) <= TOL32 * abs(l_ref)
    p.close()


def test_c2_full_solve_T200(c2_both):
    """C2 at n = 200,000 and T = 200 (BASELINE configs[1]): final iterate
    x_{T+1} within 1e-3 of the oracle's."""
    cfg, wg, wo = c2_both
    prob = wo["problem"]
    gam = gamma_of(prob, wo, cfg, max_it=30)
    x_ref, _, bad = prob.solve(cfg.T, gam)
    assert bad == 0
    x = torch.zeros(cfg.d, dtype=torch.float64, device="cuda")
    _W().make_poly(wg).solve(x, cfg.T, gam)
    assert rel(x.cpu().numpy(), x_ref) <= TOL_ITER, rel(x.cpu().numpy(), x_ref)


# ------------------------------------------------------------------ C3 block solve
def test_c3_block_solve_T100():
    """C3's recipe on its first 65,536 rows as a problem of its own (rows
    are keyed by global index, so these are C3's rows), T = 100, per-row
    spectra formed by each side's own A.1 reparameterisation."""
    from paper_2503_19925_b200 import synth
    cfg = G.scaled(G.C3, 65_536)
    W = _W()
    wg = W.build(cfg)
    K = torch.empty((cfg.n, 2 * cfg.d), dtype=torch.float32, device="cuda")
    synth.gaussian_matrix(K, 2 * cfg.d, 0, cfg.seed, rng.STREAM_A_KNOWN)
    wo = OW.build(cfg, A=host_rows(wg["A"], cfg.d), A_known=K.cpu().numpy())
    del K
    assert np.array_equal(wg["counts"].cpu().numpy(), wo["counts"])
    p = W.make_poly(wg)
    assert p.describe()["V"] == 4
    prob = wo["problem"]
    gam = gamma_of(prob, wo, cfg, max_it=100)
    for x in eval_pts(wo, prob, cfg)[:3]:
        g_ref, _ = prob.F(x)
        g, _ = gpu_F(p, x)
        assert rel(g, g_ref) <= TOL32, rel(g, g_ref)
    x_ref, _, bad = prob.solve(cfg.T, gam)
    assert bad == 0
    x = torch.zeros(cfg.d, dtype=torch.float64, device="cuda")
    p.solve(x, cfg.T, gam)
    assert rel(x.cpu().numpy(), x_ref) <= TOL_ITER, rel(x.cpu().numpy(), x_ref)
    assert np.linalg.norm(x.cpu().numpy()) <= cfg.radius * (1 + 1e-12)
    p.close()


# ------------------------------------------------------------------ C5 instantiation
C5_BLOCK = 65_536


def test_c5_block_kernel_instantiation_parity():
    """A 65,536-row block of C5 (n_global = 8e6, d = 4096) runs the bench's
    K1 instantiation k_dense_loss_grad<float, 8, 4, 12, 6, *, FULL=1> on 148
    CTAs; per call ≤ 1e-4 at the §8(d) points, counts bit-exact."""
    cfg = G.C5
    r0 = 1_234_567
    W = _W()
    wg = W.build(cfg, row0=r0, n_local=C5_BLOCK)
    p = W.make_poly(wg)
    d = p.describe()
    assert (d["V"], d["WPR"], d["NW"], d["rows_per_stage"], d["full"], d["grid"]) == \
        (8, 4, 12, 6, 1, 148), d
    wo = OW.build(cfg, rows=np.arange(r0, r0 + C5_BLOCK), A=host_rows(wg["A"], cfg.d))
    assert np.array_equal(wg["counts"].cpu().numpy(), wo["counts"])
    prob = wo["problem"]
    assert prob.n_norm == cfg.n
    for x in eval_pts(wo, prob, cfg):
        g_ref, l_ref = prob.F(x)
        g, l = gpu_F(p, x)
        assert rel(g, g_ref) <= TOL32, rel(g, g_ref)
        assert abs(l - l_ref) <= TOL32 * abs(l_ref)
    p.close()


def test_c5_block_solve_T20():
    """C5's recipe on its first 65,536 rows as a problem of its own, in the
    same K1 instantiation, T = 20 (reading R14): final iterate ≤ 1e-3."""
    cfg = G.scaled(G.C5, C5_BLOCK)
    W = _W()
    wg = W.build(cfg)
    p = W.make_poly(wg)
    assert p.describe()["full"] == 1 and p.describe()["WPR"] == 4
    wo = OW.build(cfg, A=host_rows(wg["A"], cfg.d))
    assert np.array_equal(wg["counts"].cpu().numpy(), wo["counts"])
    prob = wo["problem"]
    gam = gamma_of(prob, wo, cfg, max_it=40)
    x_ref, _, bad = prob.solve(cfg.T, gam)
    assert bad == 0
    x = torch.zeros(cfg.d, dtype=torch.float64, device="cuda")
    p.solve(x, cfg.T, gam)
    assert rel(x.cpu().numpy(), x_ref) <= TOL_ITER, rel(x.cpu().numpy(), x_ref)
    p.close()
