"""ORACLE side workload assembly — test infrastructure only.

Builds the oracle's copy of a BASELINE.json workload (or of a subset of its
rows) from the seeded generators in gen/ plus the oracle's own arithmetic for
the expected counts (Eq. model).  It never reads anything
the CUDA path computes; tests compare the two sides' independently built
inputs bit for bit (counts, indices) instead.  The one thing it may take from
the device is the output of the shared seeded generator (the Gaussian rows of
A drawn by its CUDA twin), verified against gen/rng on sampled rows — see
`build(A=...)`.
"""
from __future__ import annotations

import numpy as np

from gen import configs as G
from gen import ct, rng

from . import Problem, SET_NONNEG_BALL


def x_star(cfg: G.Config) -> np.ndarray:
    """x⋆ uniform on the sphere of radius cfg.x_star_radius (BASELINE.json)."""
    if cfg.kind == "csr":
        return ct.ellipse_phantom(cfg.seed, cfg.extra["side"], cfg.extra["ellipses"])
    return rng.unit_sphere(cfg.seed, rng.STREAM_XSTAR, cfg.d, cfg.x_star_radius)


def known_images(cfg: G.Config) -> np.ndarray:
    """C3: [x⋆^1; x⋆^2] (both uniform on the unit sphere, BASELINE.json configs[2])."""
    x1 = rng.unit_sphere(cfg.seed, rng.STREAM_X1, cfg.d, 1.0)
    x2 = rng.unit_sphere(cfg.seed, rng.STREAM_X2, cfg.d, 1.0)
    return np.concatenate([x1, x2])


def dense_rows(cfg: G.Config, rows) -> np.ndarray:
    """Rows of A: iid N(0,1) (reading R10), fp64 draw rounded to cfg.dtype."""
    a = rng.gaussian_rows(cfg.seed, rng.STREAM_A, rows, cfg.d)
    return a.astype(np.float32) if cfg.dtype == "f32" else a


def known_rows(cfg: G.Config, rows) -> np.ndarray:
    """C3: rows of [A^1 | A^2] (n x 2d), stored fp32 on both sides."""
    return rng.gaussian_rows(cfg.seed, rng.STREAM_A_KNOWN, rows, 2 * cfg.d).astype(np.float32)


def csr_matrix(cfg: G.Config):
    e = cfg.extra
    row_ptr, col, val = ct.parallel_beam_csr(e["side"], e["views"], e["bins"])
    return row_ptr, col, val.astype(np.float32)


def _shared_rows(cfg: G.Config, rows, M, d, stream):
    """Accept rows of a generated matrix produced by the generators' CUDA twin
    (libpolysynth, the seeded input generator shared by both sides — it holds
    none of the method's arithmetic) instead of redrawing them
    here with numpy (≈2M draws/s: 4 minutes for full C2).  Sampled rows are
    redrawn from gen/rng and must match bit for bit before the bytes are used."""
    M = np.ascontiguousarray(M[:, :d])
    if M.shape[0] != rows.shape[0]:
        raise ValueError("shared matrix has the wrong number of rows")
    m = rows.shape[0]
    pick = sorted({0, m // 3, m // 2, (2 * m) // 3, m - 1}) if m else []
    ref = rng.gaussian_rows(cfg.seed, stream, rows[pick], d)
    ref = ref.astype(np.float32) if (cfg.dtype == "f32" or stream == rng.STREAM_A_KNOWN) else ref
    if not np.array_equal(M[pick], ref.astype(M.dtype)):
        raise ValueError("shared generator bytes differ from gen/rng on sampled rows")
    return M


def build(cfg: G.Config, rows=None, with_counts=True, A=None, A_known=None):
    """Oracle-side inputs for `cfg` restricted to global row indices `rows`
    (default: all).  Returns a dict of numpy arrays + an oracle Problem with
    n_norm = cfg.n (the full problem's n, reading R4).

    A / A_known (optional, host arrays [len(rows), >= d]): the generated rows
    of A (and, for C3, of [A^1 | A^2]) as drawn by the generators' CUDA twin;
    checked against gen/rng on sampled rows (`_shared_rows`).  Everything the
    method computes from them — λ, counts, s', Ī', F — is the oracle's own."""
    s, mu = cfg.spectrum
    xs = x_star(cfg)
    out = {"s": s, "mu": mu, "x_star": xs}
    if cfg.kind == "csr":
        row_ptr, col, val = csr_matrix(cfg)
        if rows is not None:
            rows = np.asarray(rows, dtype=np.int64)
            lens = row_ptr[rows + 1] - row_ptr[rows]
            rp = np.zeros(rows.shape[0] + 1, dtype=np.int64)
            np.cumsum(lens, out=rp[1:])
            idx = np.concatenate([np.arange(row_ptr[r], row_ptr[r + 1]) for r in rows]) \
                if rows.size else np.zeros(0, dtype=np.int64)
            row_ptr, col, val = rp, col[idx], val[idx]
        else:
            rows = np.arange(cfg.n, dtype=np.int64)
        out.update(row_ptr=row_ptr, col=col, val=val)
        mat = dict(row_ptr=row_ptr, col=col, val=val)
    else:
        rows = np.arange(cfg.n, dtype=np.int64) if rows is None else np.asarray(rows, dtype=np.int64)
        A = dense_rows(cfg, rows) if A is None else _shared_rows(cfg, rows, A, cfg.d, rng.STREAM_A)
        out["A"] = A
        mat = dict(A=A)
    out["rows"] = rows
    s_row = I_row = None
    if cfg.kind == "reparam":
        xk = known_images(cfg)
        Ak = known_rows(cfg, rows) if A_known is None else \
            _shared_rows(cfg, rows, A_known, 2 * cfg.d, rng.STREAM_A_KNOWN)
        pk = Problem(A=Ak, y=np.zeros(rows.shape[0]), s=s, mu=mu, I_bar=1.0, d=2 * cfg.d)
        b = pk.forward(xk)
        from . import reparam
        s64, I64 = reparam(s, mu, cfg.I_bar, b, clamp=1)
        # the problem the solver sees is defined by the stored fp32 values
        s_row = s64.astype(np.float32).astype(np.float64)
        I_row = I64.astype(np.float32).astype(np.float64)
        out.update(b=b, s_row=s_row, I_row=I_row, x_known=xk)
    y = np.zeros(rows.shape[0])
    if with_counts:
        p0 = Problem(y=y, s=s, mu=mu, I_bar=cfg.I_bar, d=cfg.d, s_row=s_row, I_row=I_row,
                     **mat)
        lam = p0.mean(xs)
        k = rng.poisson(cfg.seed, rng.STREAM_Y, lam, rows)
        out["lam"] = lam
        out["counts"] = k
        if cfg.sigma > 0:
            e = rng.normal(cfg.seed, rng.STREAM_NOISE, rows, 0)
            y = (k.astype(np.float64) + cfg.sigma * e).astype(np.float32).astype(np.float64)
        else:
            y = k.astype(np.float64)
    out["y"] = y
    if cfg.set == SET_NONNEG_BALL:
        R = float(np.sqrt(np.sum(xs * xs)))   # oracle radius ||x⋆|| (reading R14)
    else:
        R = cfg.radius
    out["R"] = R
    out["problem"] = Problem(y=y, s=s, mu=mu, I_bar=cfg.I_bar, d=cfg.d, s_row=s_row,
                             I_row=I_row, set=cfg.set, R=R, n_norm=cfg.n, **mat)
    return out


def step_size(problem: Problem, s, mu, I_bar, I_row=None, s_row=None, max_it=2000, tol=1e-10):
    """Default γ = 1 / (4 Ī λmax(Σ) Σ_j s_j μ_j) — Theorem 2's step
    (PAPER.md:1068), reading R5; with per-row spectra max_i Ī'_i Σ_j s'_ij μ_j."""
    lam, _ = problem.lambda_max(max_it=max_it, tol=tol)
    if I_row is not None:
        c = float(np.max(I_row * (s_row @ mu)))
    else:
        c = I_bar * float(np.dot(s, mu))
    return 1.0 / (4.0 * lam * c), lam
