"""CT-like sparse system matrix and phantom for config C4 (BASELINE.json
configs[3]).  Input generation only: geometry and a seeded random-ellipse
phantom.  Readings R12/R13 of DESIGN.md fix what the paper leaves open.

Geometry (parallel beam, reading R12):
  * image side N (256), pixel pitch delta = 1/N (unit field of view);
  * rotation centre = centre of 0-based pixel (N/2, N/2); pixel (r, c) covers
    x in [(c - N/2 - 1/2) delta, (c - N/2 + 1/2) delta], y likewise with r;
  * views theta_k = k pi / V, k = 0..V-1 (V = 360 over 180 degrees);
  * detector bins t_b = (b - (B-1)/2) delta, b = 0..B-1 (B = 367);
  * ray (k, b) = { t_b (cos th, sin th) + s (-sin th, cos th) }, row index
    i = k * B + b; A[i, r*N + c] = length of the ray inside pixel (r, c)
    (Siddon traversal; "fractional contribution of pixel k to
    the line integral").  Zero-length corner crossings dropped;
    entries of a row are stored in traversal order.
"""
from __future__ import annotations

import numpy as np

from . import rng


def parallel_beam_csr(side=256, views=360, bins=367):
    N = side
    delta = 1.0 / N
    c0 = N // 2
    # grid line coordinates (x for columns, y for rows)
    lines = (np.arange(N + 1, dtype=np.float64) - c0 - 0.5) * delta
    lo, hi = lines[0], lines[-1]
    t = (np.arange(bins, dtype=np.float64) - (bins - 1) / 2.0) * delta
    row_len = np.zeros(views * bins, dtype=np.int64)
    cols_all, vals_all = [], []
    for k in range(views):
        th = k * np.pi / views
        ct, st = np.cos(th), np.sin(th)
        ux, uy = -st, ct                      # unit direction
        px, py = t * ct, t * st               # foot points, shape [B]
        params = []
        # slab entry/exit per axis (parametric interval where inside the box)
        smin = np.full(bins, -np.inf)
        smax = np.full(bins, np.inf)
        if abs(ux) > 1e-15:
            a1 = (lo - px) / ux
            a2 = (hi - px) / ux
            smin = np.maximum(smin, np.minimum(a1, a2))
            smax = np.minimum(smax, np.maximum(a1, a2))
            params.append((lines[None, :] - px[:, None]) / ux)
        else:
            inside = (px > lo) & (px < hi)
            smin = np.where(inside, smin, np.inf)
        if abs(uy) > 1e-15:
            b1 = (lo - py) / uy
            b2 = (hi - py) / uy
            smin = np.maximum(smin, np.minimum(b1, b2))
            smax = np.minimum(smax, np.maximum(b1, b2))
            params.append((lines[None, :] - py[:, None]) / uy)
        else:
            inside = (py > lo) & (py < hi)
            smin = np.where(inside, smin, np.inf)
        S = np.concatenate(params, axis=1)
        hit = smax > smin
        S = np.where((S > smin[:, None]) & (S < smax[:, None]), S, np.nan)
        S = np.concatenate([np.where(hit, smin, np.nan)[:, None], S,
                            np.where(hit, smax, np.nan)[:, None]], axis=1)
        S = np.sort(S, axis=1)                # NaNs sort last
        seg = S[:, 1:] - S[:, :-1]
        mid = 0.5 * (S[:, 1:] + S[:, :-1])
        ok = np.isfinite(seg) & (seg > 1e-12 * delta)
        mid = np.where(ok, mid, 0.0)
        mx = px[:, None] + mid * ux
        my = py[:, None] + mid * uy
        cc = np.floor((mx - lo) / delta).astype(np.int64)
        rr = np.floor((my - lo) / delta).astype(np.int64)
        ok &= (cc >= 0) & (cc < N) & (rr >= 0) & (rr < N)
        cnt = ok.sum(axis=1)
        row_len[k * bins:(k + 1) * bins] = cnt
        cols_all.append((rr * N + cc)[ok])
        vals_all.append(seg[ok])
    row_ptr = np.zeros(views * bins + 1, dtype=np.int64)
    np.cumsum(row_len, out=row_ptr[1:])
    col = np.concatenate(cols_all).astype(np.int32)
    val = np.concatenate(vals_all)
    return row_ptr, col, val


def ellipse_phantom(seed, side=256, K=10):
    """Reading R13: K ellipses, centres uniform in the inscribed disc, semi-axes
    U[0.05, 0.35] of the FOV, angle U[0, pi), value U[0, 1], painted in order
    with overwrite, pixel-centre inclusion.  Returns fp64 [side*side], values
    in [0, 1], row-major (r * side + c)."""
    N = side
    c0 = N // 2
    coords = (np.arange(N, dtype=np.float64) - c0) / N
    X, Y = np.meshgrid(coords, coords)       # X varies along columns
    img = np.zeros((N, N))
    e = np.arange(K)
    U = [rng.uniform(seed, rng.STREAM_PHANTOM, e, p) for p in range(6)]
    rad = 0.5 * np.sqrt(U[0])
    phi = 2.0 * np.pi * U[1]
    cx, cy = rad * np.cos(phi), rad * np.sin(phi)
    ax = 0.05 + 0.30 * U[2]
    ay = 0.05 + 0.30 * U[3]
    ang = np.pi * U[4]
    val = U[5]
    for q in range(K):
        ca, sa = np.cos(ang[q]), np.sin(ang[q])
        dx, dy = X - cx[q], Y - cy[q]
        u = (dx * ca + dy * sa) / ax[q]
        v = (-dx * sa + dy * ca) / ay[q]
        img[u * u + v * v <= 1.0] = val[q]
    return img.ravel()
