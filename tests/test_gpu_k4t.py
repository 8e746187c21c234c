"""K4t — the tiled CSR layout (csrc/tiled.cuh): which matrices take it, and
oracle parity on each of its branches.

Eq.(operator): F(x) = (1/n) Σ_i [y_i − Ī h(⟨a_i,x⟩)] a_i with
h(t) = Σ_j s_j e^{−μ_j t₊} (Eq. function-h-plus).  K4t computes
the same sums as the SELL paths in a different order: every ⟨a_i, x⟩ as
per-strip partials added in strip order, four products summed in fp32 before
the fp64 accumulator (POLY_TILE_CHAIN), and — when μ is an arithmetic
progression — the W exponentials of a row as one exponential times powers of
a ratio (exact algebra).  All branches are compared with the fp64 oracle at
the north-star per-call tolerance 1e-4 (TOL32 in test_gpu_parity.py)."""
from __future__ import annotations

import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from gen import configs as G  # noqa: E402
from gen import rng  # noqa: E402
from oracle import workloads as OW  # noqa: E402

pytestmark = pytest.mark.gpu

TOL32 = 1e-4


def _P():
    import paper_2503_19925_b200 as P
    return P


def _W():
    from paper_2503_19925_b200 import workloads as PW
    return PW


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def c4():
    return _W().build(G.C4), OW.build(G.C4)


def _grad(p, x):
    g, l = p.loss_grad(torch.tensor(x, device="cuda"))
    return g.cpu().numpy(), float(l)


def test_c4_takes_k4t(c4):
    """The C4 system matrix (fp32, 256 x 256 image, Siddon rows) is re-blocked
    into 3 column strips (89 KB of iterate each) and 32 x TH pixel tiles, TH
    chosen so that two backward CTAs per SM cover the image evenly (148 SMs:
    TH = 7, 37 x 8 = 296 tiles)."""
    wg, _ = c4
    d = _W().make_poly(wg).describe()
    assert d["csr_layout"] == 3
    assert d["rows_per_stage"] == 3
    th = next(t for t in range(8, 3, -1) if -(-256 // t) * 8 == d["stages"])
    assert -(-d["stages"] // (2 * d["sms"])) * th <= 16
    assert d["grid"] % 3 == 0 and d["grid"] <= d["sms"]


def test_c4_k4t_deterministic_and_geometric_bins(c4, monkeypatch):
    """Repeated calls give the same bits (fixed summation orders, no atomics
    in the sums); the geometric bin walk (μ = linspace, checked at poly_init)
    and the per-bin exponentials (POLY_NO_GEO_MU=1) agree to rounding: φ_i
    differs in its last fp64 bits, which can move the fp32 residual r_i the
    backward gathers by one fp32 ulp (6e-8 relative) on a few rows — hence
    1e-8 on g; the objective (1/n) Σ_i [y_i z_i − Ī H(z_i)] sums terms of
    size Ī·H ~ 1e5 that cancel to ~4e3 per row, so its last-bit differences
    show at 1e-11 relative — 1e-10 on ℓ."""
    wg, wo = c4
    W = _W()
    x = 0.7 * wo["x_star"]
    p = W.make_poly(wg)
    g1, l1 = _grad(p, x)
    g2, l2 = _grad(p, x)
    assert np.array_equal(g1, g2) and l1 == l2
    monkeypatch.setenv("POLY_NO_GEO_MU", "1")
    g3, l3 = _grad(W.make_poly(wg), x)
    assert rel(g1, g3) <= 1e-8
    assert abs(l1 - l3) <= 1e-10 * abs(l3)


def test_c4_k4t_non_arithmetic_spectrum(c4):
    """μ not an arithmetic progression (every bin's exponential evaluated) and
    a per-bin spectrum that is not the Gaussian recipe: oracle parity."""
    wg, wo = c4
    P, W = _P(), _W()
    Wb = 16
    mu = np.sort(np.random.default_rng(5).uniform(0.4, 2.2, Wb))[::-1].copy()
    s = np.random.default_rng(6).uniform(0.2, 1.0, Wb)
    s /= s.sum()
    y = wo["y"]
    p = P.Poly(row_ptr=wg["row_ptr"], col=wg["col"], val=wg["val"], d=G.C4.d, y=wg["y"], s=s, mu=mu,
               I_bar=G.C4.I_bar, set=G.SET_NONNEG_BALL, R=wo["R"])
    assert p.describe()["csr_layout"] == 3
    o = oracle.Problem(row_ptr=wo["row_ptr"], col=wo["col"], val=wo["val"], y=y, s=s, mu=mu, I_bar=G.C4.I_bar,
                       d=G.C4.d, set=G.SET_NONNEG_BALL, R=wo["R"])
    for x in (np.zeros(G.C4.d), 0.5 * wo["x_star"], wo["x_star"]):
        g, l = _grad(p, x)
        g_ref, l_ref = o.F(x)
        assert rel(g, g_ref) <= TOL32
        assert abs(l - l_ref) <= TOL32 * abs(l_ref)


def _banded(n, d, seed, width, empty_rows=()):
    """A banded sparse matrix: row i holds up to `width` columns near i·d/n
    (ascending, gaps < 256), so every strip-local and list delta fits 8 bits."""
    r = np.random.default_rng(seed)
    rows, cols = [], []
    for i in range(n):
        if i in empty_rows:
            continue
        c0 = int(i * (d - width) / max(1, n - 1))
        k = int(r.integers(1, width))
        cc = np.sort(r.choice(width, size=k, replace=False)) + c0
        rows += [i] * k
        cols += cc.tolist()
    rows, cols = np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int32)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    return np.cumsum(row_ptr), cols, r.uniform(0.0, 0.05, cols.shape[0]).astype(np.float32)


def _parity(row_ptr, col, val, d, seed, expect_layout=None, W=8):
    P = _P()
    n = row_ptr.shape[0] - 1
    r = np.random.default_rng(seed)
    s = np.linspace(1.0, 2.0, W)
    s /= s.sum()
    mu = np.linspace(2.0, 0.5, W)
    xs = r.uniform(0, 1, d)
    z = np.array([float(val[row_ptr[i]:row_ptr[i + 1]] @ xs[col[row_ptr[i]:row_ptr[i + 1]]]) for i in range(n)])
    lam = 200.0 * np.array([np.dot(s, np.exp(-mu * max(0.0, zi))) for zi in z])
    y = rng.poisson(11, rng.STREAM_TEST, lam, np.arange(n)).astype(np.int32)
    o = oracle.Problem(row_ptr=row_ptr, col=col, val=val, y=y.astype(np.float64), s=s, mu=mu, I_bar=200.0, d=d,
                       set=G.SET_NONE)
    p = P.Poly(row_ptr=torch.tensor(row_ptr, device="cuda"), col=torch.tensor(col, device="cuda"),
               val=torch.tensor(val, device="cuda"), d=d, y=torch.tensor(y, device="cuda"), s=s, mu=mu,
               I_bar=200.0, set=G.SET_NONE)
    if expect_layout is not None:
        assert p.describe()["csr_layout"] == expect_layout
    for x in (np.zeros(d), 0.6 * xs, xs):
        g, l = _grad(p, x)
        g_ref, l_ref = o.F(x)
        assert rel(g, g_ref) <= TOL32
        assert abs(l - l_ref) <= TOL32 * max(1.0, abs(l_ref))
    p.close()


@pytest.mark.parametrize("n,d,width", [(3000, 5000, 60), (777, 70000, 200), (64, 300, 40), (2, 300, 40), (3, 257, 50)])
def test_k4t_generic_banded(n, d, width):
    """A non-square d (one image row of d pixels: strips and tiles of
    consecutive columns), ragged rows, empty rows, ragged last tile, d larger
    than one strip (70000 columns: several strips), two or three rows (the
    sort key's row field narrower than the r-chunk shift): K4t, oracle parity."""
    rp, col, val = _banded(n, d, n + d, width, empty_rows=(3, n // 2))
    _parity(rp, col, val, d, n, expect_layout=3)


def test_k4t_square_image_small():
    """A square d that is not a multiple of the 32 x 8 tile (s = 50): edge tiles
    with empty slots; Siddon rows of a 50 x 50 parallel-beam geometry."""
    from gen import ct
    rp, col, val = ct.parallel_beam_csr(50, 30, 73)
    _parity(rp, col, val.astype(np.float32), 2500, 7, expect_layout=3)


def test_k4t_falls_back_on_wide_gaps():
    """Random columns (strip-local gaps > 255): poly_init keeps the SELL pair."""
    r = np.random.default_rng(3)
    n, d = 500, 20000
    rows, cols = [], []
    for i in range(n):
        k = int(r.integers(1, 30))
        rows += [i] * k
        cols += sorted(r.choice(d, size=k, replace=False).tolist())
    rows, cols = np.array(rows), np.array(cols, dtype=np.int32)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, rows + 1, 1)
    rp = np.cumsum(rp)
    val = r.uniform(0.0, 0.05, cols.shape[0]).astype(np.float32)
    _parity(rp, cols, val, d, 11, expect_layout=1)


def test_c4_solve_bits_repeat(c4):
    """Determinism of the graph-replayed solve (fixed summation order in every
    kernel of Eq. extragrad-method): 300 repetitions of the
    same 25-iteration C4 solve on one handle give identical bits.  (With part of
    the backward's records read evict-last, 1-2 % of such runs differed — that
    option is off.)"""
    wg, _ = c4
    p = _W().make_poly(wg)
    assert p.describe()["csr_layout"] == 3 and p.describe()["l2_keep_bytes"] == 0
    cfg = G.C4
    gam = 1.0 / (4.0 * cfg.I_bar * 4e-5 * float(np.dot(*cfg.spectrum)))
    ref = None
    for _ in range(300):
        x = torch.zeros(cfg.d, dtype=torch.float64, device="cuda")
        p.solve(x, 25, gam)
        if ref is None:
            ref = x.clone()
        else:
            assert torch.equal(ref, x)
    p.close()
