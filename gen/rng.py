"""Counter-based seeded input generators (numpy side).

This module is the ONLY code shared by the oracle side and the CUDA side, and
it holds none of the method's arithmetic (no h, no F, no projection): it draws
random numbers.  The CUDA side (``paper_2503_19925_b200/csrc/synth.cu``)
implements the *same* generator instruction for instruction, so every draw is
a pure function of (seed, stream, counter) and both sides produce identical
bits without exchanging data.

Bit-exactness rules followed here and in synth.cu:
  * Philox4x32-10 (Salmon et al., SC'11) on 32-bit words;
  * uniforms are built from integer bits, exactly: U = (2*m + 1) * 2^-53 with
    m a 52-bit integer, so U is in (0, 1) and never 0, 1/2 or 1;
  * every floating-point step is a single IEEE-754 fp64 +, -, *, /, sqrt,
    floor, frexp or ldexp (each correctly rounded, hence identical on numpy and
    CUDA compiled with -fmad=false); log/exp are our own polynomial routines
    (``log64``/``exp64``) evaluated in a fixed operation order — never libm.

Distributions:
  * standard normal: Marsaglia's polar method, one variate per counter,
    rejected pairs retried with attempt+1;
  * Poisson(lam): inversion for lam < 10, Hormann's PTRS transformed rejection
    for lam >= 10 (SPEC.md:105 asks for an exact sampler of this kind).
"""
from __future__ import annotations

import math

import numpy as np

MASK32 = np.uint64(0xFFFFFFFF)
_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = 0x9E3779B9
_W1 = 0xBB67AE85

# fp64 constants, written with enough digits to round to the same double on
# every compiler (synth.cu spells the identical literals).
LN2 = 0.6931471805599453
LN2_HI = 6.93147180369123816490e-01
LN2_LO = 1.90821492927058770002e-10
INV_LN2 = 1.4426950408889634
SQRT_HALF = 0.7071067811865476
HALF_LOG_2PI = 0.9189385332046728
TWO_POW_M53 = 1.0 / 9007199254740992.0  # 2^-53, exact

LOG_TERMS = 12  # atanh series terms: |f| <= 0.1716 -> f^26/27 < 1e-21
EXP_TERMS = 13  # Taylor terms for exp(r), |r| <= ln2/2 -> r^14/14! < 1e-20
_LOG_C = [1.0 / float(2 * k + 1) for k in range(LOG_TERMS + 1)]
_EXP_C = [1.0 / float(math.factorial(k)) for k in range(EXP_TERMS + 1)]

POISSON_PTRS_MIN = 10.0
POISSON_INV_MAX_K = 1000

# stream ids (Philox key word 1).  Survey §8(d): A 0, x* 1, y 2, noise 3,
# phantom 4, known-material matrix 5; 7/8 known-material images.
STREAM_A, STREAM_XSTAR, STREAM_Y, STREAM_NOISE, STREAM_PHANTOM = 0, 1, 2, 3, 4
STREAM_A_KNOWN, STREAM_X1, STREAM_X2 = 5, 7, 8
STREAM_TEST = 9


def _u32(a):
    return np.asarray(a, dtype=np.uint64) & MASK32


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32 with 10 rounds.  Arguments are uint32-valued arrays/ints;
    returns four uint64 arrays holding 32-bit words."""
    c0, c1, c2, c3 = _u32(c0), _u32(c1), _u32(c2), _u32(c3)
    k0 = int(k0) & 0xFFFFFFFF
    k1 = int(k1) & 0xFFFFFFFF
    for _ in range(10):
        p0 = _M0 * c0
        p1 = _M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0), lo1,
                          hi0 ^ c3 ^ np.uint64(k1), lo0)
        k0 = (k0 + _W0) & 0xFFFFFFFF
        k1 = (k1 + _W1) & 0xFFFFFFFF
    return c0, c1, c2, c3


def u01(w_hi, w_lo):
    """Two 32-bit words -> uniform in (0,1): (2*m + 1) * 2^-53, m 52-bit."""
    m = ((w_hi >> np.uint64(6)) << np.uint64(26)) | (w_lo >> np.uint64(6))
    return (m.astype(np.float64) * 2.0 + 1.0) * TWO_POW_M53


def log64(x):
    """Natural log for finite x > 0 using only IEEE-exact operations."""
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)
    small = m < SQRT_HALF
    m = np.where(small, m * 2.0, m)
    e = np.where(small, e - 1, e).astype(np.float64)
    f = (m - 1.0) / (m + 1.0)
    f2 = f * f
    p = np.full_like(f, _LOG_C[LOG_TERMS])
    for k in range(LOG_TERMS - 1, -1, -1):
        p = p * f2 + _LOG_C[k]
    return e * LN2 + (2.0 * f) * p


def exp64(x):
    """exp(x) for moderate |x| (< 700) using only IEEE-exact operations."""
    x = np.asarray(x, dtype=np.float64)
    k = np.floor(x * INV_LN2 + 0.5)
    r = (x - k * LN2_HI) - k * LN2_LO
    p = np.full_like(r, _EXP_C[EXP_TERMS])
    for j in range(EXP_TERMS - 1, -1, -1):
        p = p * r + _EXP_C[j]
    return np.ldexp(p, k.astype(np.int64))


def _logfact_table():
    t = np.zeros(16)
    for i in range(2, 16):
        t[i] = t[i - 1] + float(log64(np.float64(i)))
    return t


_LOGFACT_SMALL = _logfact_table()


def logfact64(k):
    """log(k!) for integer-valued k >= 0: table below 16, Stirling above."""
    k = np.asarray(k, dtype=np.float64)
    out = np.empty_like(k)
    small = k < 16.0
    out[small] = _LOGFACT_SMALL[k[small].astype(np.int64)]
    kb = k[~small]
    if kb.size:
        lk = log64(kb)
        r = 1.0 / kb
        r2 = r * r
        t = (kb + 0.5) * lk - kb + HALF_LOG_2PI
        series = r * ((1.0 / 12.0) - r2 * ((1.0 / 360.0) - r2 * (1.0 / 1260.0)))
        out[~small] = t + series
    return out


def _split64(a):
    a = np.asarray(a, dtype=np.int64).astype(np.uint64)
    return a & MASK32, a >> np.uint64(32)


def normal(seed, stream, idx_a, idx_b=0):
    """One N(0,1) variate per (idx_a, idx_b) pair (broadcast), polar method.

    Counter = (idx_b, lo32(idx_a), hi32(idx_a), attempt); key = (seed, stream).
    For a matrix entry A[i, k]: idx_a = global row i, idx_b = column k.
    """
    ia, ib = np.broadcast_arrays(np.asarray(idx_a, dtype=np.int64),
                                 np.asarray(idx_b, dtype=np.int64))
    shape = ia.shape
    a_lo, a_hi = _split64(ia.ravel())
    b = ib.ravel().astype(np.uint64)
    out = np.empty(a_lo.shape[0], dtype=np.float64)
    pending = np.arange(a_lo.shape[0])
    attempt = 0
    while pending.size:
        w0, w1, w2, w3 = philox4x32_10(b[pending], a_lo[pending], a_hi[pending],
                                       attempt, seed, stream)
        u = 2.0 * u01(w0, w1) - 1.0
        v = 2.0 * u01(w2, w3) - 1.0
        s = u * u + v * v
        ok = s < 1.0
        so, uo = s[ok], u[ok]
        out[pending[ok]] = uo * np.sqrt((-2.0 * log64(so)) / so)
        pending = pending[~ok]
        attempt += 1
        if attempt > 64:
            raise RuntimeError("polar method failed to accept in 64 attempts")
    return out.reshape(shape)


def gaussian_rows(seed, stream, rows, d, col0=0):
    """Rows `rows` (global indices) of an iid N(0,1) matrix, fp64 [len, d]."""
    rows = np.asarray(rows, dtype=np.int64)
    return normal(seed, stream, rows[:, None], np.arange(col0, col0 + d)[None, :])


def poisson(seed, stream, lam, idx):
    """Poisson(lam[i]) draw for row index idx[i]; returns int64 array."""
    lam = np.asarray(lam, dtype=np.float64).ravel()
    idx = np.asarray(idx, dtype=np.int64).ravel()
    if lam.shape != idx.shape:
        raise ValueError("lam and idx must have the same shape")
    if np.any(~np.isfinite(lam)) or np.any(lam < 0):
        raise ValueError("Poisson means must be finite and >= 0")
    out = np.zeros(lam.shape[0], dtype=np.int64)
    lo, hi = _split64(idx)

    # --- inversion, lam < 10 -------------------------------------------
    sel = np.nonzero(lam < POISSON_PTRS_MIN)[0]
    if sel.size:
        w0, w1, _, _ = philox4x32_10(0, lo[sel], hi[sel], 0x50000001, seed, stream)
        U = u01(w0, w1)
        L = lam[sel]
        p = exp64(-L)
        F = p.copy()
        k = np.zeros(sel.size)
        act = U > F
        while np.any(act):
            k = np.where(act, k + 1.0, k)
            pn = (p * L) / np.where(act, k, 1.0)
            p = np.where(act, pn, p)
            F = np.where(act, F + p, F)
            act = act & (U > F) & (k < POISSON_INV_MAX_K)
        out[sel] = k.astype(np.int64)

    # --- PTRS, lam >= 10 --------------------------------------------------
    sel = np.nonzero(lam >= POISSON_PTRS_MIN)[0]
    if sel.size:
        L = lam[sel]
        slam = np.sqrt(L)
        loglam = log64(L)
        b = 0.931 + 2.53 * slam
        a = -0.059 + 0.02483 * b
        invalpha = 1.1239 + 1.1328 / (b - 3.4)
        vr = 0.9277 - 3.6224 / (b - 2.0)
        log_invalpha = log64(invalpha)
        pending = np.arange(sel.size)
        attempt = 0
        while pending.size:
            w0, w1, w2, w3 = philox4x32_10(attempt, lo[sel[pending]], hi[sel[pending]],
                                           0x50000000, seed, stream)
            U = u01(w0, w1) - 0.5
            V = u01(w2, w3)
            us = 0.5 - np.abs(U)
            ap, bp, Lp = a[pending], b[pending], L[pending]
            k = np.floor(((2.0 * ap) / us + bp) * U + Lp + 0.43)
            acc = (us >= 0.07) & (V <= vr[pending])
            rej = (k < 0.0) | ((us < 0.013) & (V > us))
            test = ~acc & ~rej
            if np.any(test):
                ti = np.nonzero(test)[0]
                lhs = (log64(V[ti]) + log_invalpha[pending[ti]]) - \
                    log64(ap[ti] / (us[ti] * us[ti]) + bp[ti])
                rhs = (-Lp[ti] + k[ti] * loglam[pending[ti]]) - logfact64(k[ti])
                acc[ti] = lhs <= rhs
            out[sel[pending[acc]]] = k[acc].astype(np.int64)
            pending = pending[~acc]
            attempt += 1
            if attempt > 256:
                raise RuntimeError("PTRS failed to accept in 256 attempts")
    return out


def unit_sphere(seed, stream, d, radius=1.0):
    """x = radius * g / ||g||, g ~ N(0, I_d) from `normal` (host-only data)."""
    g = normal(seed, stream, np.arange(d), 0)
    return radius * g / math.sqrt(float(np.sum(g * g)))


def uniform(seed, stream, idx_a, idx_b=0):
    """Uniform (0,1) per (idx_a, idx_b): counter (idx_b, lo, hi, 0x55000000)."""
    ia, ib = np.broadcast_arrays(np.asarray(idx_a, dtype=np.int64),
                                 np.asarray(idx_b, dtype=np.int64))
    lo, hi = _split64(ia.ravel())
    w0, w1, _, _ = philox4x32_10(ib.ravel().astype(np.uint64), lo, hi,
                                 0x55000000, seed, stream)
    return u01(w0, w1).reshape(ia.shape)
