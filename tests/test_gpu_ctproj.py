"""GPU parity of the matrix-free parallel-beam projector (SURVEY.md §8(f)
NEXT-4; csrc/ctproj.cuh) against the fp64 oracle on the CSR that gen/ct.py
builds for the same geometry (Siddon lengths, reading R12): the kernels
evaluate the chord length of each ray in each pixel in closed form instead of
streaming A, so F, ℓ and the EXACT iterates must match the CSR problem."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from gen import configs as G  # noqa: E402
from gen import ct, rng  # noqa: E402
from oracle import workloads as OW  # noqa: E402


def _P():
    import paper_2503_19925_b200 as P
    return P


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _pb_poly(w, cfg, **kw):
    P = _P()
    e = cfg.extra
    return P.Poly(pb=dict(side=e["side"], views=e["views"], bins=e["bins"]), y=w["y"], s=w["s"],
                  mu=w["mu"], I_bar=cfg.I_bar, set=cfg.set, R=w["R"], n_global=cfg.n, **kw)


@pytest.fixture(scope="module")
def c4():
    from paper_2503_19925_b200 import workloads as PW
    return PW.build(G.C4), OW.build(G.C4)


def test_pb_matches_csr_and_oracle_c4(c4):
    from paper_2503_19925_b200 import workloads as PW
    wg, wo = c4
    cfg = G.C4
    p_mf = _pb_poly(wg, cfg)
    p_csr = PW.make_poly(wg)
    prob = wo["problem"]
    r = np.random.default_rng(3)
    for x in (0.5 * wo["x_star"], wo["x_star"], np.abs(wo["x_star"] + 0.05 * r.standard_normal(cfg.d))):
        xt = torch.tensor(x, device="cuda")
        g_mf, l_mf = p_mf.loss_grad(xt)
        g_cs, l_cs = p_csr.loss_grad(xt)
        g_ref, l_ref = prob.F(x)
        assert rel(g_mf.cpu().numpy(), g_ref) <= 1e-4, rel(g_mf.cpu().numpy(), g_ref)
        assert abs(l_mf - l_ref) <= 1e-4 * abs(l_ref)
        assert rel(g_mf.cpu().numpy(), g_cs.cpu().numpy()) <= 1e-4
    p_mf.close()
    p_csr.close()


def test_pb_solve_parity_c4(c4):
    wg, wo = c4
    cfg = G.C4
    prob = wo["problem"]
    gam = 1.0 / (4.0 * cfg.I_bar * 4e-5 * float(np.dot(wo["s"], wo["mu"])))
    x_ref, _, _ = prob.solve(10, gam)
    p = _pb_poly(wg, cfg)
    x = torch.zeros(cfg.d, dtype=torch.float64, device="cuda")
    p.solve(x, 10, gam)
    assert rel(x.cpu().numpy(), x_ref) <= 1e-3
    assert x.min().item() >= 0.0
    p.close()


@pytest.mark.parametrize("side,views,bins", [(24, 30, 37), (33, 17, 51), (64, 90, 93)])
def test_pb_small_geometries_and_view_shards(side, views, bins):
    """Odd sides, views that are not a multiple of 4, more bins than needed
    (B odd: rays at whole-pixel offsets, never on a pixel edge, reading R12);
    two handles holding the first and the last views (row_offset) sum to the
    full operator."""
    P = _P()
    rp, col, val = ct.parallel_beam_csr(side, views, bins)
    val = val.astype(np.float32)
    n, d = rp.shape[0] - 1, side * side
    s, mu = G.spectrum(6)
    xs = ct.ellipse_phantom(side, side, 5)
    lam = oracle.Problem(row_ptr=rp, col=col, val=val, y=np.zeros(n), s=s, mu=mu, I_bar=3e3,
                         d=d).mean(xs)
    y = rng.poisson(side, rng.STREAM_Y, lam, np.arange(n)).astype(np.int32)
    o = oracle.Problem(row_ptr=rp, col=col, val=val, y=y.astype(float), s=s, mu=mu, I_bar=3e3,
                       d=d, set=G.SET_NONE)
    geo = dict(side=side, views=views, bins=bins)
    yt = torch.tensor(y, device="cuda")
    p = P.Poly(pb=geo, y=yt, s=s, mu=mu, I_bar=3e3, set=G.SET_NONE)
    x = 0.7 * xs + 0.02
    g, l = p.loss_grad(torch.tensor(x, device="cuda"))
    g_ref, l_ref = o.F(x)
    assert rel(g.cpu().numpy(), g_ref) <= 1e-4 and abs(l - l_ref) <= 1e-4 * abs(l_ref)
    k = views // 3
    parts = [P.Poly(pb=geo, y=yt[:k * bins], s=s, mu=mu, I_bar=3e3, set=G.SET_NONE, n_global=n),
             P.Poly(pb=geo, y=yt[k * bins:], s=s, mu=mu, I_bar=3e3, set=G.SET_NONE, n_global=n,
                    row_offset=k * bins)]
    acc = sum(q.loss_grad(torch.tensor(x, device="cuda"))[0].cpu().numpy() for q in parts)
    assert rel(acc, g.cpu().numpy()) <= 1e-6
    with pytest.raises(P.PolyError):
        P.Poly(pb=geo, y=yt[:bins + 1], s=s, mu=mu, I_bar=3e3)   # not whole views


def test_pb_adjoint_with_rays_on_pixel_edges():
    """B even puts the axis-aligned views' rays on pixel edges (gen/ct.py then
    assigns each to a pixel by the rounding of its own arithmetic); the
    projector assigns them to the pixel on the positive side in both passes,
    so its forward and backward stay exact adjoints.  With Ī -> 0 one
    evaluation gives ℓ = (1/n) <y, A x> (forward pass) and g = (1/n) A^T y
    (backward pass): <x, g> must equal ℓ."""
    P = _P()
    r = np.random.default_rng(0)
    for side, views, bins in ((20, 12, 40), (32, 8, 46), (25, 36, 37)):
        geo = dict(side=side, views=views, bins=bins)
        n, d = views * bins, side * side
        y = torch.tensor(r.standard_normal(n), device="cuda")
        p = P.Poly(pb=geo, y=y, s=[1.0], mu=[1.0], I_bar=1e-300, relu=0, set=G.SET_NONE)
        x = r.random(d)
        g, l = p.loss_grad(torch.tensor(x, device="cuda"))
        assert abs(np.dot(x, g.cpu().numpy()) - l) <= 1e-6 * max(abs(l), 1e-12), (side, views, bins)
        p.close()
