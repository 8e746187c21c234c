"""GPU parity of the NEXT rows against the fp64 oracle.

NEXT-1: stacked detector windows (POLY problem.windows, folded into one
spectrum on the device — the oracle evaluates the unfolded double sum) and
the averaged-iterate stopping rule (poly_solve_ex).
NEXT-3: the baseline objectives L2 / L1 / Poisson NLL as modes of the same
fused passes and the projected-GD method.

Tolerances as in test_gpu_parity: fp32 path 1e-4 per call / 1e-3 final
iterate, fp64 path 1e-12 / 1e-10.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from gen import configs as G  # noqa: E402
from gen import rng  # noqa: E402
from oracle import workloads as OW  # noqa: E402


def _P():
    import paper_2503_19925_b200 as P
    return P


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _dense(n, d, seed, dtype):
    per = 4 if dtype == np.float32 else 2
    lda = (d + per - 1) // per * per
    A = np.zeros((n, lda), dtype=dtype)
    A[:, :d] = rng.gaussian_rows(seed, rng.STREAM_TEST, np.arange(n), d).astype(dtype) / np.sqrt(d)
    return A


def _problem(n=3000, d=200, W=8, seed=1, dtype=np.float32, relu=1, I_bar=300.0, noiseless=False):
    A = _dense(n, d, seed, dtype)
    s, mu = G.spectrum(W)
    xs = rng.unit_sphere(seed, rng.STREAM_XSTAR, d, 0.9)
    p0 = oracle.Problem(A=A[:, :d].astype(np.float64), y=np.zeros(n), s=s, mu=mu, I_bar=I_bar,
                        d=d, relu=relu)
    lam = p0.mean(xs)
    y = lam if noiseless else rng.poisson(seed, rng.STREAM_Y, lam, np.arange(n)).astype(np.int32)
    return dict(A=A, d=d, n=n, s=s, mu=mu, xs=xs, y=y, I_bar=I_bar, relu=relu)


def _gpu(pb, **kw):
    P = _P()
    y = torch.tensor(pb["y"], device="cuda")
    return P.Poly(A=torch.tensor(pb["A"], device="cuda"), d=pb["d"], y=y, s=pb["s"], mu=pb["mu"],
                  I_bar=pb["I_bar"], relu=pb["relu"], **kw)


def _orc(pb, **kw):
    return oracle.Problem(A=pb["A"][:, :pb["d"]].astype(np.float64), y=np.asarray(pb["y"], float),
                          s=pb["s"], mu=pb["mu"], I_bar=pb["I_bar"], d=pb["d"], relu=pb["relu"],
                          **kw)


# ------------------------------------------------------------- NEXT-3 modes
@pytest.mark.parametrize("dtype,tol", [(np.float32, 1e-4), (np.float64, 1e-12)])
@pytest.mark.parametrize("mode", [1, 2, 3])
@pytest.mark.parametrize("relu", [0, 1])
def test_modes_dense_parity(dtype, tol, mode, relu):
    pb = _problem(dtype=dtype, relu=relu, seed=mode + 3 * relu)
    p = _gpu(pb, mode=mode, set=G.SET_NONE)
    o = _orc(pb)
    r = np.random.default_rng(mode)
    for x in (np.zeros(pb["d"]), pb["xs"], 0.5 * pb["xs"] + 0.3 * r.standard_normal(pb["d"]) /
              np.sqrt(pb["d"])):
        g_ref, l_ref = o.objective(x, mode)
        g, l = p.loss_grad(torch.tensor(x, device="cuda"))
        if np.linalg.norm(g_ref) == 0.0:
            assert torch.count_nonzero(g).item() == 0
        elif mode == 2:
            # L1: sign(Ī h - y) is decided from z and h, whose summation order
            # differs from the oracle's (fp32 dot: ~1e-6 relative; at x = 0 with
            # relu = 0, Ī h = Ī Σ s_j ties with y = Ī up to rounding); rows with
            # |Ī h - y| inside that band may flip, each moving g by at most
            # 2 Ī |h'| ||a_i|| / n <= 2 Ī Σ s_j μ_j ||a_i|| / n.
            m = o.mean(x)
            A64 = pb["A"][:, :pb["d"]].astype(np.float64)
            tie = np.abs(m - pb["y"]) <= 1e-5 * np.maximum(1.0, m)
            slack = 2 * pb["I_bar"] * float(np.dot(pb["s"], pb["mu"])) * \
                np.linalg.norm(A64[tie], axis=1).sum() / pb["n"]
            err = np.linalg.norm(g.cpu().numpy() - g_ref)
            assert err <= tol * np.linalg.norm(g_ref) + slack, (err, slack, int(tie.sum()))
        else:
            assert rel(g.cpu().numpy(), g_ref) <= tol, (mode, relu, rel(g.cpu().numpy(), g_ref))
        assert abs(l - l_ref) <= tol * max(1.0, abs(l_ref))
    p.close()


@pytest.mark.parametrize("mode", [1, 3])
def test_modes_csr_parity(mode):
    from paper_2503_19925_b200 import workloads as PW
    cfg = G.C4
    wg = PW.build(cfg)
    wo = OW.build(cfg)
    p = PW.make_poly(wg, mode=mode)
    prob = wo["problem"]
    for x in (0.5 * wo["x_star"], wo["x_star"] + 0.01):
        g_ref, l_ref = prob.objective(x, mode)
        g, l = p.loss_grad(torch.tensor(x, device="cuda"))
        assert rel(g.cpu().numpy(), g_ref) <= 1e-4
        assert abs(l - l_ref) <= 1e-4 * abs(l_ref)
    p.close()


def test_gd_method_parity():
    P = _P()
    for dtype, tol in ((np.float64, 1e-10), (np.float32, 1e-3)):
        pb = _problem(dtype=dtype, seed=7)
        p = _gpu(pb, mode=P.POLY_MODE_L2, set=G.SET_BALL, R=1.0)
        o = _orc(pb, set=G.SET_BALL, R=1.0)
        x1 = np.full(pb["d"], 0.02)
        x_ref, bad = o.solve_gd(1, 60, 2e-6, x1=x1)
        x = torch.tensor(x1, device="cuda")
        info = p.solve_ex(x, 60, 2e-6, method=P.POLY_METHOD_GD)
        assert bad == 0 and info.iters == 60 and not info.stopped
        assert rel(x.cpu().numpy(), x_ref) <= tol, (dtype, rel(x.cpu().numpy(), x_ref))
        p.close()


# ------------------------------------------------------------- NEXT-1 windows
def _win(pb, Om=3, seed=0):
    r = np.random.default_rng(seed)
    s = r.uniform(0.2, 1.0, (Om, len(pb["mu"])))
    s /= s.sum(axis=1, keepdims=True)
    I = r.uniform(100.0, 600.0, Om)
    A64 = pb["A"][:, :pb["d"]].astype(np.float64)
    ys = []
    for w in range(Om):
        lam = oracle.Problem(A=A64, y=np.zeros(pb["n"]), s=s[w], mu=pb["mu"], I_bar=I[w],
                             d=pb["d"], relu=pb["relu"]).mean(pb["xs"])
        ys.append(rng.poisson(seed + w, rng.STREAM_Y, lam, np.arange(pb["n"])).astype(np.int32))
    return s, I, np.array(ys)


@pytest.mark.parametrize("dtype,tol", [(np.float32, 1e-4), (np.float64, 1e-12)])
@pytest.mark.parametrize("ykind", ["i32", "f32"])
def test_windows_dense_parity(dtype, tol, ykind):
    P = _P()
    pb = _problem(dtype=dtype, seed=11)
    s, I, Y = _win(pb)
    if ykind == "f32":
        Y = (Y - 3.5).astype(np.float32)       # electronic-noise-like, may be negative
    p = P.Poly(A=torch.tensor(pb["A"], device="cuda"), d=pb["d"], y=torch.tensor(Y, device="cuda"),
               s=s, mu=pb["mu"], I_bar=1.0, I_win=I, set=G.SET_NONE)
    o = _orc(pb)
    for x in (np.zeros(pb["d"]), pb["xs"], -0.4 * pb["xs"]):
        g_ref, l_ref = o.F_windows(x, s, I, Y.astype(np.float64))
        g, l = p.loss_grad(torch.tensor(x, device="cuda"))
        assert rel(g.cpu().numpy(), g_ref) <= tol, rel(g.cpu().numpy(), g_ref)
        assert abs(l - l_ref) <= tol * max(1.0, abs(l_ref))
    p.close()


def test_windows_csr_parity_and_solve():
    P = _P()
    from gen import ct
    side, views, bins = 64, 60, 93
    rp, col, val = ct.parallel_beam_csr(side, views, bins)
    val = val.astype(np.float32)
    n, d = rp.shape[0] - 1, side * side
    _, mu = G.spectrum(8)
    xs = ct.ellipse_phantom(5, side, 6)
    r = np.random.default_rng(1)
    s = r.uniform(0.2, 1.0, (3, 8))
    s /= s.sum(axis=1, keepdims=True)
    I = np.array([2e3, 5e3, 1e3])
    ys = []
    for w in range(3):
        lam = oracle.Problem(row_ptr=rp, col=col, val=val, y=np.zeros(n), s=s[w], mu=mu,
                             I_bar=I[w], d=d).mean(xs)
        ys.append(rng.poisson(20 + w, rng.STREAM_Y, lam, np.arange(n)).astype(np.int32))
    Y = np.array(ys)
    R = float(np.linalg.norm(xs))
    p = P.Poly(row_ptr=torch.tensor(rp, device="cuda"), col=torch.tensor(col, device="cuda"),
               val=torch.tensor(val, device="cuda"), d=d, y=torch.tensor(Y, device="cuda"), s=s,
               mu=mu, I_bar=1.0, I_win=I, set=G.SET_NONNEG_BALL, R=R)
    o = oracle.Problem(row_ptr=rp, col=col, val=val, y=np.zeros(n), s=s[0], mu=mu, I_bar=1.0, d=d,
                       set=G.SET_NONNEG_BALL, R=R)
    g_ref, l_ref = o.F_windows(0.5 * xs, s, I, Y.astype(np.float64))
    g, l = p.loss_grad(torch.tensor(0.5 * xs, device="cuda"))
    assert rel(g.cpu().numpy(), g_ref) <= 1e-4 and abs(l - l_ref) <= 1e-4 * abs(l_ref)
    p.close()


# ------------------------------------------------------------- NEXT-1 averaging
def test_solve_ex_average_fp64_matches_oracle_exactly():
    P = _P()
    pb = _problem(n=2000, d=100, dtype=np.float64, seed=21)
    p = _gpu(pb, set=G.SET_BALL, R=1.0)
    o = _orc(pb, set=G.SET_BALL, R=1.0)
    gam, _ = OW.step_size(o, pb["s"], pb["mu"], pb["I_bar"])
    # tol = 0: runs T_max iterations; x̄ over ⌈k/2⌉..k
    xb_ref, xl_ref, it_ref, mv_ref, _ = o.solve_avg(37, gam, tol=0.0)
    x = torch.zeros(pb["d"], dtype=torch.float64, device="cuda")
    xl = torch.zeros_like(x)
    info = p.solve_ex(x, 37, gam, average=True, tol=0.0, x_last=xl)
    assert info.iters == 37 and not info.stopped
    assert rel(x.cpu().numpy(), xb_ref) <= 1e-10 and rel(xl.cpu().numpy(), xl_ref) <= 1e-10
    assert abs(info.move - mv_ref) <= 1e-8 * max(mv_ref, 1e-300)
    # a tolerance the run crosses: same stopping iteration, same x̄ and x_k
    tol = 1e-4
    xb_ref, xl_ref, it_ref, mv_ref, _ = o.solve_avg(3000, gam, tol=tol)
    assert it_ref < 3000
    x.zero_()
    info = p.solve_ex(x, 3000, gam, average=True, tol=tol, x_last=xl)
    assert info.stopped and info.iters == it_ref, (info.iters, it_ref)
    assert rel(x.cpu().numpy(), xb_ref) <= 1e-10 and rel(xl.cpu().numpy(), xl_ref) <= 1e-10
    assert abs(info.move - mv_ref) <= 1e-6 * mv_ref and info.move <= tol
    p.close()


def test_solve_ex_average_fp32_and_plain_consistency():
    P = _P()
    pb = _problem(n=4000, d=256, dtype=np.float32, seed=22)
    p = _gpu(pb, set=G.SET_BALL, R=1.0)
    o = _orc(pb, set=G.SET_BALL, R=1.0)
    gam, _ = OW.step_size(o, pb["s"], pb["mu"], pb["I_bar"])
    xb_ref, xl_ref, it_ref, mv_ref, _ = o.solve_avg(2000, gam, tol=3e-5)
    x = torch.zeros(pb["d"], dtype=torch.float64, device="cuda")
    info = p.solve_ex(x, 2000, gam, average=True, tol=3e-5)
    assert info.stopped
    assert abs(info.iters - it_ref) <= max(2, 0.02 * it_ref), (info.iters, it_ref)
    assert rel(x.cpu().numpy(), xb_ref) <= 1e-3
    # average off: the last iterate equals poly_solve's, bit for bit
    xa = torch.zeros_like(x)
    xc = torch.zeros_like(x)
    p.solve_ex(xa, 50, gam)
    p.solve(xc, 50, gam)
    assert torch.equal(xa, xc)
    # profile (no graph) path gives the same bits as the graph path
    xd = torch.zeros_like(x)
    p.solve_ex(xd, 50, gam, profile=True)
    assert torch.equal(xa, xd)
    p.close()


def test_solve_ex_average_csr_large_d():
    """d = 65536 exercises the split step tail and a 256-block averaging pass."""
    from paper_2503_19925_b200 import workloads as PW
    cfg = G.C4
    wg = PW.build(cfg)
    wo = OW.build(cfg)
    prob = wo["problem"]
    gam = 1.0 / (4.0 * cfg.I_bar * 4e-5 * float(np.dot(wo["s"], wo["mu"])))
    xb_ref, xl_ref, it_ref, mv_ref, _ = prob.solve_avg(12, gam, tol=0.0)
    p = PW.make_poly(wg)
    x = torch.zeros(cfg.d, dtype=torch.float64, device="cuda")
    xl = torch.zeros_like(x)
    info = p.solve_ex(x, 12, gam, average=True, tol=0.0, x_last=xl)
    assert info.iters == 12
    assert rel(x.cpu().numpy(), xb_ref) <= 1e-3 and rel(xl.cpu().numpy(), xl_ref) <= 1e-3
    p.close()
