"""ORACLE — test infrastructure only (see oracle/oracle.c header).

ctypes wrapper over liboracle.so, the plain fp64 C implementation of the
EXACT hot path.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this package.  Nothing here
imports or links the CUDA path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

SET_NONE, SET_BALL, SET_NONNEG, SET_NONNEG_BALL, SET_TV_NONNEG, SET_TV = 0, 1, 2, 3, 4, 5


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (fp64, no contraction, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
               "-shared", "-fPIC", _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class _Problem(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("d", C.c_int64), ("n_norm", C.c_int64),
        ("csr", C.c_int), ("A", C.c_void_p), ("a_f32", C.c_int), ("lda", C.c_int64),
        ("row_ptr", C.c_void_p), ("col", C.c_void_p), ("val", C.c_void_p),
        ("y", C.c_void_p), ("W", C.c_int), ("s", C.c_void_p), ("mu", C.c_void_p),
        ("I_bar", C.c_double), ("s_row", C.c_void_p), ("I_row", C.c_void_p),
        ("relu", C.c_int), ("set", C.c_int), ("R", C.c_double), ("center", C.c_void_p),
        ("tv_side", C.c_int), ("tv_tau", C.c_double), ("tv_tol", C.c_double),
        ("tv_rtol", C.c_double), ("tv_dtol", C.c_double), ("tv_max_it", C.c_int),
        ("tv_max_outer", C.c_int), ("tv_k", C.c_int), ("tv_warm", C.c_int),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.POINTER(_Problem)
        dp = C.POINTER(C.c_double)
        _lib.oracle_h.restype = C.c_double
        _lib.oracle_h.argtypes = [C.c_int, dp, dp, C.c_double, C.c_int]
        _lib.oracle_H.restype = C.c_double
        _lib.oracle_H.argtypes = [C.c_int, dp, dp, C.c_double, C.c_int]
        _lib.oracle_hprime_abs.restype = C.c_double
        _lib.oracle_hprime_abs.argtypes = [C.c_int, dp, dp, C.c_double]
        _lib.oracle_F.argtypes = [P, dp, dp, dp]
        _lib.oracle_forward.argtypes = [P, dp, dp]
        _lib.oracle_mean.argtypes = [P, dp, dp]
        _lib.oracle_project.argtypes = [C.c_int, C.c_int64, C.c_double, dp, dp, dp]
        _lib.oracle_solve.restype = C.c_int
        _lib.oracle_solve.argtypes = [P, C.c_int, C.c_double, dp, dp]
        _lib.oracle_lambda_max.restype = C.c_double
        _lib.oracle_lambda_max.argtypes = [P, C.c_int, C.c_double, C.POINTER(C.c_int)]
        _lib.oracle_reparam.argtypes = [C.c_int, dp, dp, C.c_double, C.c_int64, dp, C.c_int,
                                        dp, dp]
        _lib.oracle_F_windows.argtypes = [P, C.c_int, dp, dp, dp, dp, dp, dp]
        _lib.oracle_average.argtypes = [dp, C.c_int, C.c_int64, dp]
        _lib.oracle_solve_avg.restype = C.c_int
        _lib.oracle_solve_avg.argtypes = [P, C.c_int, C.c_double, C.c_double, dp, dp,
                                          C.POINTER(C.c_int), dp]
        _lib.oracle_objective.argtypes = [P, C.c_int, dp, dp, dp]
        _lib.oracle_solve_gd.restype = C.c_int
        _lib.oracle_solve_gd.argtypes = [P, C.c_int, C.c_int, C.c_double, dp]
        _lib.oracle_tv_norm.restype = C.c_double
        _lib.oracle_tv_norm.argtypes = [C.c_int, dp]
        _lib.oracle_prox_tv.restype = C.c_int
        _lib.oracle_prox_tv.argtypes = [C.c_int, dp, C.c_double, C.c_double, C.c_int, dp, dp]
        _lib.oracle_project_tv.restype = C.c_int
        _lib.oracle_project_tv.argtypes = [C.c_int, dp, C.c_double, C.c_double, C.c_double,
                                           C.c_int, dp]
        _lib.oracle_project_tv_nonneg.restype = C.c_int
        _lib.oracle_project_tv_nonneg.argtypes = [C.c_int, dp, C.c_double, C.c_double, C.c_double,
                                                  C.c_int, C.c_double, C.c_int, dp]
        _lib.oracle_project_tv_k.restype = C.c_int
        _lib.oracle_project_tv_k.argtypes = [C.c_int, dp, C.c_double, C.c_double, C.c_double,
                                             C.c_int, C.c_int, dp]
        _lib.oracle_project_tv_nonneg_kw.restype = C.c_int
        _lib.oracle_project_tv_nonneg_kw.argtypes = [C.c_int, dp, C.c_double, C.c_double, C.c_double,
                                                     C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, dp]
        _lib.oracle_project_tv_k_warm.restype = C.c_int
        _lib.oracle_project_tv_k_warm.argtypes = [C.c_int, dp, C.c_double, C.c_double, C.c_double,
                                                  C.c_int, C.c_int, dp, dp]
        _lib.oracle_fista_iterations.restype = C.c_longlong
        _lib.oracle_fista_iterations.argtypes = [C.c_int]
        _lib.oracle_project_tv_nonneg_k.restype = C.c_int
        _lib.oracle_project_tv_nonneg_k.argtypes = [C.c_int, dp, C.c_double, C.c_double, C.c_double,
                                                    C.c_int, C.c_double, C.c_int, C.c_int, dp]
        _lib.oracle_set_threads.argtypes = [C.c_int]
        _lib.oracle_max_threads.restype = C.c_int
    return _lib


def _dp(a):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def set_threads(t: int) -> None:
    lib().oracle_set_threads(int(t))


def max_threads() -> int:
    return int(lib().oracle_max_threads())


class Problem:
    """Holds the arrays (keeps them alive) and the C struct view of them."""

    def __init__(self, *, y, s, mu, I_bar, d, A=None, row_ptr=None, col=None, val=None,
                 s_row=None, I_row=None, relu=1, set=SET_BALL, R=1.0, center=None,
                 n_norm=None, tv=None):
        self.csr = A is None
        if self.csr:
            self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
            self.col = np.ascontiguousarray(col, dtype=np.int32)
            v = np.asarray(val)
            self.val = np.ascontiguousarray(v, dtype=np.float32 if v.dtype == np.float32 else np.float64)
            self.a_f32 = int(self.val.dtype == np.float32)
            self.n = self.row_ptr.shape[0] - 1
            self.A = None
            self.lda = 0
        else:
            a = np.asarray(A)
            if a.dtype not in (np.float32, np.float64):
                a = a.astype(np.float64)
            self.A = np.ascontiguousarray(a)
            self.a_f32 = int(self.A.dtype == np.float32)
            self.n = self.A.shape[0]
            self.lda = self.A.shape[1]
        self.d = int(d)
        self.y = _f64(y)
        self.s, self.mu = _f64(s), _f64(mu)
        self.W = self.s.shape[0]
        self.I_bar = float(I_bar)
        self.s_row, self.I_row = _f64(s_row), _f64(I_row)
        self.relu, self.set, self.R = int(relu), int(set), float(R)
        self.center = _f64(center)
        self.n_norm = int(self.n if n_norm is None else n_norm)
        assert self.y.shape[0] == self.n
        st = _Problem()
        st.n, st.d, st.n_norm = self.n, self.d, self.n_norm
        st.csr = int(self.csr)
        st.A = None if self.A is None else self.A.ctypes.data
        st.a_f32, st.lda = self.a_f32, self.lda
        if self.csr:
            st.row_ptr, st.col, st.val = (self.row_ptr.ctypes.data, self.col.ctypes.data,
                                          self.val.ctypes.data)
        st.y = self.y.ctypes.data
        st.W = self.W
        st.s, st.mu = self.s.ctypes.data, self.mu.ctypes.data
        st.I_bar = self.I_bar
        st.s_row = None if self.s_row is None else self.s_row.ctypes.data
        st.I_row = None if self.I_row is None else self.I_row.ctypes.data
        st.relu, st.set, st.R = self.relu, self.set, self.R
        st.center = None if self.center is None else self.center.ctypes.data
        if set in (SET_TV_NONNEG, SET_TV):
            tv = dict(tv or {})
            st.tv_side = int(round(np.sqrt(self.d)))
            assert st.tv_side ** 2 == self.d
            st.tv_tau = float(tv["tau"])
            st.tv_tol = float(tv.get("tol", 0.01))
            st.tv_rtol = float(tv.get("rtol", 1e-6))
            st.tv_dtol = float(tv.get("dykstra_tol", 1e-4))
            st.tv_max_it = int(tv.get("max_it", 5000))
            st.tv_max_outer = int(tv.get("max_outer", 1000))
            st.tv_k = int(tv.get("k", 1))
            st.tv_warm = int(tv.get("warm", 0))
        self._st = st

    @property
    def ptr(self):
        return C.byref(self._st)

    def F(self, x):
        x = _f64(x)
        g = np.zeros(self.d)
        loss = C.c_double()
        lib().oracle_F(self.ptr, _dp(x), _dp(g), C.byref(loss))
        return g, loss.value

    def forward(self, x):
        x = _f64(x)
        z = np.zeros(self.n)
        lib().oracle_forward(self.ptr, _dp(x), _dp(z))
        return z

    def mean(self, x):
        x = _f64(x)
        lam = np.zeros(self.n)
        lib().oracle_mean(self.ptr, _dp(x), _dp(lam))
        return lam

    def project(self, v):
        if self.set in (SET_TV_NONNEG, SET_TV):
            t = self._st
            if self.set == SET_TV:
                return project_tv(v, t.tv_tau, t.tv_tol, t.tv_rtol, t.tv_max_it)[0]
            return project_tv_nonneg(v, t.tv_tau, t.tv_tol, t.tv_rtol, t.tv_max_it, t.tv_dtol,
                                     t.tv_max_outer)[0]
        return project(self.set, self.R, self.center, v)

    def solve(self, T, gamma, x1=None, trace=False):
        x = np.zeros(self.d) if x1 is None else np.array(x1, dtype=np.float64)
        tr = np.zeros(2 * T) if trace else None
        bad = lib().oracle_solve(self.ptr, int(T), float(gamma), _dp(x), _dp(tr))
        return x, tr, int(bad)

    def F_windows(self, x, s_win, I_win, y_win):
        """Stacked multi-window operator (oracle_F_windows): s_win [Ω, W],
        I_win [Ω], y_win [Ω, n]."""
        x = _f64(x)
        s_win, I_win, y_win = _f64(s_win), _f64(I_win), _f64(y_win)
        Om = I_win.shape[0]
        assert s_win.shape == (Om, self.W) and y_win.shape == (Om, self.n)
        g = np.zeros(self.d)
        loss = C.c_double()
        lib().oracle_F_windows(self.ptr, Om, _dp(s_win), _dp(I_win), _dp(y_win), _dp(x), _dp(g),
                               C.byref(loss))
        return g, loss.value

    def solve_avg(self, T_max, gamma, tol=1e-5, x1=None):
        """EXACT with the averaged-iterate stop: (x̄, x_last, iters, move, bad)."""
        x = np.zeros(self.d) if x1 is None else np.array(x1, dtype=np.float64)
        xb = np.zeros(self.d)
        it = C.c_int()
        mv = C.c_double()
        bad = lib().oracle_solve_avg(self.ptr, int(T_max), float(gamma), float(tol), _dp(x),
                                     _dp(xb), C.byref(it), C.byref(mv))
        return xb, x, it.value, mv.value, int(bad)

    def objective(self, x, mode):
        """Baseline objective `mode` (1 L2, 2 L1, 3 NLL) and its (sub)gradient."""
        x = _f64(x)
        g = np.zeros(self.d)
        loss = C.c_double()
        lib().oracle_objective(self.ptr, int(mode), _dp(x), _dp(g), C.byref(loss))
        return g, loss.value

    def solve_gd(self, mode, T, gamma, x1=None):
        x = np.zeros(self.d) if x1 is None else np.array(x1, dtype=np.float64)
        bad = lib().oracle_solve_gd(self.ptr, int(mode), int(T), float(gamma), _dp(x))
        return x, int(bad)

    def lambda_max(self, max_it=1000, tol=1e-8):
        it = C.c_int()
        lam = lib().oracle_lambda_max(self.ptr, int(max_it), float(tol), C.byref(it))
        return lam, it.value


def h(s, mu, t, relu=1):
    s, mu = _f64(s), _f64(mu)
    return lib().oracle_h(s.shape[0], _dp(s), _dp(mu), float(t), int(relu))


def H(s, mu, t, relu=1):
    s, mu = _f64(s), _f64(mu)
    return lib().oracle_H(s.shape[0], _dp(s), _dp(mu), float(t), int(relu))


def hprime_abs(s, mu, t):
    s, mu = _f64(s), _f64(mu)
    return lib().oracle_hprime_abs(s.shape[0], _dp(s), _dp(mu), float(t))


def project(set, R, center, v):
    v = _f64(v)
    out = np.empty_like(v)
    lib().oracle_project(int(set), v.shape[0], float(R), _dp(_f64(center)), _dp(v), _dp(out))
    return out


def average(hist, k):
    """Mean of iterates ⌈k/2⌉..k (1-based) of hist [>=k, d]."""
    hist = _f64(hist)
    out = np.zeros(hist.shape[1])
    lib().oracle_average(_dp(hist), int(k), hist.shape[1], _dp(out))
    return out


def _side(z):
    z = _f64(z)
    side = int(round(np.sqrt(z.shape[0])))
    assert side * side == z.shape[0], "TV needs a square image"
    return z, side


def tv_norm(x):
    """Anisotropic TV of a square image (row-major)."""
    x, side = _side(np.ravel(x))
    return float(lib().oracle_tv_norm(side, _dp(x)))


def prox_tv(z, lam, rtol=1e-6, max_it=5000):
    """argmin ||x - z||^2 + lam ||x||_TV: (x, u, iterations)."""
    z, side = _side(np.ravel(z))
    x = np.zeros_like(z)
    u = np.zeros(max(1, 2 * side * (side - 1)))
    it = lib().oracle_prox_tv(side, _dp(z), float(lam), float(rtol), int(max_it), _dp(x), _dp(u))
    return x, u[:2 * side * (side - 1)], int(it)


def fista_iterations(reset=True) -> int:
    """FISTA iterations run by the TV proxes since the last reset."""
    return int(lib().oracle_fista_iterations(1 if reset else 0))


def project_tv(z, tau, tv_tol=0.01, rtol=1e-6, max_it=5000, k=1, warm=False):
    """P onto {||x||_TV <= tau} as the paper computes it; k λ values per search
    round (reading R22; k = 1: the binary search), proxes warm-started from the
    previous prox of the same λ slot (reading R23) if warm.  (x, rounds)."""
    z, side = _side(np.ravel(z))
    x = np.zeros_like(z)
    if warm:
        ust = np.zeros(max(1, int(k)) * 2 * side * (side - 1) + 1)
        steps = lib().oracle_project_tv_k_warm(side, _dp(z), float(tau), float(tv_tol), float(rtol),
                                               int(max_it), int(k), _dp(ust), _dp(x))
    else:
        steps = lib().oracle_project_tv_k(side, _dp(z), float(tau), float(tv_tol), float(rtol),
                                          int(max_it), int(k), _dp(x))
    return x, int(steps)


def project_tv_nonneg(z, tau, tv_tol=0.01, rtol=1e-6, max_it=5000, tol=1e-4, max_outer=100000, k=1,
                      warm=False):
    z, side = _side(np.ravel(z))
    x = np.zeros_like(z)
    it = lib().oracle_project_tv_nonneg_kw(side, _dp(z), float(tau), float(tv_tol), float(rtol),
                                           int(max_it), float(tol), int(max_outer), int(k), int(bool(warm)),
                                           _dp(x))
    return x, int(it)


def reparam(s, mu, I_bar, b, clamp=1):
    s, mu, b = _f64(s), _f64(mu), _f64(b)
    n, W = b.shape[0], s.shape[0]
    s_row = np.zeros((n, W))
    I_row = np.zeros(n)
    lib().oracle_reparam(W, _dp(s), _dp(mu), float(I_bar), n, _dp(b), int(clamp),
                         _dp(s_row), _dp(I_row))
    return s_row, I_row
