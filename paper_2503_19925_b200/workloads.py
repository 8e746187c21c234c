"""Build a BASELINE.json workload in HBM (product side).

Random draws come from libpolysynth.so (bit-identical twin of gen/rng.py);
the Poisson means λ_i = Ī_i h_i(<a_i, x⋆>) come from the product's own
poly_expected_counts, and the C3 per-row spectra from poly_reparameterize
(Appendix A.1).  Nothing here imports the oracle; tests rebuild sampled rows
on the CPU with gen/ + oracle/ and compare bit for bit.
"""
from __future__ import annotations

import numpy as np
import torch

from gen import configs as G
from gen import ct, rng

from . import poly_reparameterize, synth
from .api import Poly


def padded_lda(d: int, elsize: int) -> int:
    per = 16 // elsize
    return (d + per - 1) // per * per


def x_star(cfg: G.Config) -> np.ndarray:
    if cfg.kind == "csr":
        return ct.ellipse_phantom(cfg.seed, cfg.extra["side"], cfg.extra["ellipses"])
    return rng.unit_sphere(cfg.seed, rng.STREAM_XSTAR, cfg.d, cfg.x_star_radius)


def known_images(cfg: G.Config) -> np.ndarray:
    return np.concatenate([rng.unit_sphere(cfg.seed, rng.STREAM_X1, cfg.d, 1.0),
                           rng.unit_sphere(cfg.seed, rng.STREAM_X2, cfg.d, 1.0)])


def build(cfg: G.Config, row0: int = 0, n_local: int | None = None, device="cuda"):
    """Rows [row0, row0 + n_local) of workload `cfg` on `device`."""
    n_local = cfg.n - row0 if n_local is None else int(n_local)
    s, mu = cfg.spectrum
    xs = x_star(cfg)
    xs_t = torch.tensor(xs, dtype=torch.float64, device=device)
    out = dict(cfg=cfg, s=s, mu=mu, x_star=xs_t, row0=row0, n_local=n_local, n_global=cfg.n,
               s_row=None, I_row=None)
    zeros_y = torch.zeros(max(n_local, 1), dtype=torch.int32, device=device)[:n_local]
    if cfg.kind == "csr":
        e = cfg.extra
        rp, col, val = ct.parallel_beam_csr(e["side"], e["views"], e["bins"])
        lo, hi = row0, row0 + n_local
        rp_l = rp[lo:hi + 1] - rp[lo]
        out["row_ptr"] = torch.tensor(rp_l, dtype=torch.int64, device=device)
        out["col"] = torch.tensor(col[rp[lo]:rp[hi]], dtype=torch.int32, device=device)
        out["val"] = torch.tensor(val[rp[lo]:rp[hi]].astype(np.float32), device=device)
        mat = dict(row_ptr=out["row_ptr"], col=out["col"], val=out["val"], d=cfg.d)
    else:
        dt = torch.float32 if cfg.dtype == "f32" else torch.float64
        lda = padded_lda(cfg.d, 4 if cfg.dtype == "f32" else 8)
        A = torch.empty((n_local, lda), dtype=dt, device=device)
        synth.gaussian_matrix(A, cfg.d, row0, cfg.seed, rng.STREAM_A)
        out["A"] = A
        mat = dict(A=A, d=cfg.d)
    if cfg.kind == "reparam":
        d2 = 2 * cfg.d
        K = torch.empty((n_local, padded_lda(d2, 4)), dtype=torch.float32, device=device)
        synth.gaussian_matrix(K, d2, row0, cfg.seed, rng.STREAM_A_KNOWN)
        xk = torch.tensor(known_images(cfg), dtype=torch.float64, device=device)
        pk = Poly(A=K, d=d2, y=zeros_y, s=s, mu=mu, I_bar=1.0)
        b = pk.forward(xk)
        pk.close()
        del K
        s_row = torch.empty((n_local, cfg.W), dtype=torch.float32, device=device)
        I_row = torch.empty(n_local, dtype=torch.float32, device=device)
        poly_reparameterize(cfg.W, s, mu, cfg.I_bar, n_local, b.data_ptr(), 1, s_row.data_ptr(),
                            I_row.data_ptr(), torch.cuda.current_stream().cuda_stream)
        out.update(s_row=s_row, I_row=I_row, b=b)
    p0 = Poly(y=zeros_y, s=s, mu=mu, I_bar=cfg.I_bar, s_row=out["s_row"], I_row=out["I_row"],
              n_global=cfg.n, **mat)
    lam = p0.expected_counts(xs_t)
    p0.close()
    k = torch.empty(n_local, dtype=torch.int32, device=device)
    synth.poisson(lam, k, row0, cfg.seed, rng.STREAM_Y)
    if cfg.sigma > 0:
        y = torch.empty(n_local, dtype=torch.float32, device=device)
        synth.add_noise(k, y, row0, cfg.sigma, cfg.seed, rng.STREAM_NOISE)
    else:
        y = k
    out["counts"] = k
    out["y"] = y
    out["lam"] = lam
    out["R"] = float(np.sqrt(np.sum(xs * xs))) if cfg.set == G.SET_NONNEG_BALL else cfg.radius
    out["mat"] = mat
    torch.cuda.synchronize()
    return out


def make_poly(w, **kw) -> Poly:
    cfg = w["cfg"]
    args = dict(y=w["y"], s=w["s"], mu=w["mu"], I_bar=cfg.I_bar, s_row=w["s_row"],
                I_row=w["I_row"], set=cfg.set, R=w["R"], n_global=w["n_global"],
                row_offset=w["row0"])
    args.update(w["mat"])
    args.update(kw)
    return Poly(**args)

