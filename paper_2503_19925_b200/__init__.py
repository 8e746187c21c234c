"""B200-native (sm_100a) hot path of EXACT (arXiv 2503.19925).

Thin ctypes binding over libpoly.so (include/poly.h).  The functions below
carry the C names and only marshal arguments; every step of the path runs in
the library's CUDA kernels.  There is no CPU fallback: importing this package
without the built library raises ImportError.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("POLY_LIB_PATH") or os.path.join(_HERE, "libpoly.so")

POLY_OK, POLY_EINVAL, POLY_ECUDA, POLY_ENCCL, POLY_ENONFINITE, POLY_ENOMEM, POLY_EUNSUPPORTED = range(7)
POLY_DENSE, POLY_CSR, POLY_PARALLEL_BEAM = 0, 1, 2
POLY_F32, POLY_F64 = 0, 1
POLY_Y_I32, POLY_Y_F32, POLY_Y_F64 = 0, 1, 2
POLY_SET_NONE, POLY_SET_BALL, POLY_SET_NONNEG, POLY_SET_NONNEG_BALL = 0, 1, 2, 3
POLY_SET_TV_NONNEG, POLY_SET_TV = 4, 5
POLY_FLAG_HOST_INPUTS, POLY_FLAG_NO_GRAPH, POLY_FLAG_NO_PDL, POLY_FLAG_COMM, POLY_FLAG_NO_SMALL = 1, 2, 4, 8, 16
POLY_FLAG_P2P = 32
POLY_FLAG_NVLS = 64
POLY_SOLVE_PROFILE = 1
POLY_MODE_EXACT, POLY_MODE_L2, POLY_MODE_L1, POLY_MODE_NLL = 0, 1, 2, 3
POLY_METHOD_EXTRAGRADIENT, POLY_METHOD_GD = 0, 1

EXPORTED = ["poly_init", "poly_loss_grad", "poly_solve", "poly_forward", "poly_expected_counts",
            "poly_reparameterize", "poly_kernel_times", "poly_describe", "poly_nccl_unique_id",
            "poly_free", "poly_last_error", "poly_abi_version", "poly_solve_ex", "poly_project",
            "poly_stream_probe", "poly_p2p_handle", "poly_p2p_open", "poly_nvls_handle",
            "poly_nvls_open", "poly_share_fd"]


class PolyProblem(C.Structure):
    """Mirror of `poly_problem` (include/poly.h); field order is the ABI."""
    _fields_ = [
        ("n_local", C.c_int64), ("n_global", C.c_int64), ("row_offset", C.c_int64),
        ("d", C.c_int64), ("layout", C.c_int32), ("dtype", C.c_int32),
        ("A", C.c_void_p), ("lda", C.c_int64),
        ("row_ptr", C.c_void_p), ("col", C.c_void_p), ("val", C.c_void_p), ("nnz", C.c_int64),
        ("ytype", C.c_int32), ("W", C.c_int32), ("y", C.c_void_p),
        ("s", C.c_void_p), ("mu", C.c_void_p), ("I_bar", C.c_double),
        ("s_row", C.c_void_p), ("I_row", C.c_void_p),
        ("relu", C.c_int32), ("set", C.c_int32), ("R", C.c_double), ("center", C.c_void_p),
        ("rank", C.c_int32), ("world", C.c_int32), ("nccl_id", C.c_void_p),
        ("stream", C.c_void_p), ("flags", C.c_uint32), ("mode", C.c_int32),
        ("windows", C.c_int32), ("I_win", C.c_void_p),
        ("tv_tau", C.c_double), ("tv_tol", C.c_double), ("tv_rtol", C.c_double),
        ("tv_dykstra_tol", C.c_double), ("tv_max_it", C.c_int32), ("tv_max_outer", C.c_int32),
        ("pb_side", C.c_int32), ("pb_views", C.c_int32), ("pb_bins", C.c_int32),
        ("pb_reserved", C.c_int32), ("tv_k", C.c_int32), ("tv_cold", C.c_int32),
    ]


class PolySolveOpts(C.Structure):
    """Mirror of `poly_solve_opts`."""
    _fields_ = [("T_max", C.c_int32), ("method", C.c_int32), ("gamma", C.c_double),
                ("tol", C.c_double), ("average", C.c_int32), ("flags", C.c_uint32)]


class PolySolveInfo(C.Structure):
    """Mirror of `poly_solve_info`."""
    _fields_ = [("iters", C.c_int32), ("stopped", C.c_int32), ("bad_iter", C.c_int32),
                ("reserved", C.c_int32), ("move", C.c_double)]


class PolyError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"poly error {code}: {msg}")
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with "
                          "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    dp = C.POINTER(C.c_double)
    lib.poly_init.argtypes = [C.POINTER(PolyProblem), C.POINTER(vp)]
    lib.poly_loss_grad.argtypes = [vp, vp, vp, dp]
    lib.poly_solve.argtypes = [vp, vp, C.c_int, dbl, C.c_uint32, dp, C.POINTER(C.c_int)]
    lib.poly_solve_ex.argtypes = [vp, C.POINTER(PolySolveOpts), vp, vp, C.POINTER(PolySolveInfo)]
    lib.poly_forward.argtypes = [vp, vp, vp]
    lib.poly_project.argtypes = [vp, vp, vp, C.POINTER(C.c_int64)]
    lib.poly_stream_probe.argtypes = [vp, i32, dp]
    lib.poly_expected_counts.argtypes = [vp, vp, vp]
    lib.poly_reparameterize.argtypes = [i32, dp, dp, dbl, i64, vp, i32, vp, vp, vp]
    lib.poly_kernel_times.argtypes = [vp, dp, i32]
    lib.poly_describe.argtypes = [vp, C.POINTER(C.c_int64), i32]
    lib.poly_nccl_unique_id.argtypes = [vp]
    lib.poly_p2p_handle.argtypes = [vp, vp]
    lib.poly_p2p_open.argtypes = [vp, vp]
    lib.poly_nvls_handle.argtypes = [vp, vp]
    lib.poly_nvls_open.argtypes = [vp, vp]
    lib.poly_share_fd.argtypes = [i32, i32, C.c_char_p, C.c_int, C.POINTER(C.c_int), dbl]
    lib.poly_free.argtypes = [vp]
    lib.poly_free.restype = None
    lib.poly_last_error.restype = C.c_char_p
    for name in EXPORTED:
        if name not in ("poly_free", "poly_last_error"):
            getattr(lib, name).restype = C.c_int
    return lib


_lib = _load()


def lib():
    return _lib


def _check(rc):
    if rc != POLY_OK:
        raise PolyError(rc, _lib.poly_last_error().decode(errors="replace"))
    return rc


# ----------------------------------------------------------------- C names
def poly_abi_version() -> int:
    return _lib.poly_abi_version()


def poly_last_error() -> str:
    return _lib.poly_last_error().decode(errors="replace")


def poly_init(problem: PolyProblem) -> int:
    h = C.c_void_p()
    _check(_lib.poly_init(C.byref(problem), C.byref(h)))
    return h.value


def poly_loss_grad(h: int, x_ptr: int, g_ptr: int | None, want_loss: bool):
    loss = C.c_double()
    _check(_lib.poly_loss_grad(h, x_ptr, g_ptr, C.byref(loss) if want_loss else None))
    return loss.value if want_loss else None


def poly_solve(h: int, x_ptr: int, T: int, gamma: float, flags: int = 0, trace=None):
    """trace: None or a ctypes double array of length 2T."""
    bad = C.c_int(0)
    rc = _lib.poly_solve(h, x_ptr, int(T), float(gamma), int(flags), trace, C.byref(bad))
    if rc == POLY_ENONFINITE:
        raise PolyError(rc, f"{poly_last_error()} (bad_iter={bad.value})")
    _check(rc)


def poly_solve_ex(h: int, x_ptr: int, opts: PolySolveOpts, x_last_ptr=None) -> PolySolveInfo:
    info = PolySolveInfo()
    rc = _lib.poly_solve_ex(h, C.byref(opts), x_ptr, x_last_ptr, C.byref(info))
    if rc == POLY_ENONFINITE:
        raise PolyError(rc, f"{poly_last_error()} (bad_iter={info.bad_iter})")
    _check(rc)
    return info


def poly_project(h: int, v_ptr: int, x_ptr: int):
    """x = P_X(v); returns the TV statistics (Dykstra sweeps, bisection steps,
    FISTA iterations) — zeros for the other sets."""
    st = (C.c_int64 * 3)()
    _check(_lib.poly_project(h, v_ptr, x_ptr, st))
    return list(st)


def poly_stream_probe(h: int, reps: int = 20) -> float:
    """K8: ms per read-only pass over the handle's A."""
    ms = C.c_double()
    _check(_lib.poly_stream_probe(h, int(reps), C.byref(ms)))
    return ms.value


def poly_forward(h: int, x_ptr: int, z_ptr: int):
    _check(_lib.poly_forward(h, x_ptr, z_ptr))


def poly_expected_counts(h: int, x_ptr: int, lam_ptr: int):
    _check(_lib.poly_expected_counts(h, x_ptr, lam_ptr))


def poly_reparameterize(W, s, mu, I_bar, n, b_ptr, clamp, s_row_ptr, I_row_ptr, stream=None):
    sa = (C.c_double * W)(*s)
    ma = (C.c_double * W)(*mu)
    _check(_lib.poly_reparameterize(W, sa, ma, float(I_bar), int(n), b_ptr, int(clamp),
                                    s_row_ptr, I_row_ptr, stream))


def poly_kernel_times(h: int):
    out = (C.c_double * 5)()
    _check(_lib.poly_kernel_times(h, out, 5))
    return list(out)


def poly_describe(h: int):
    out = (C.c_int64 * 14)()
    _check(_lib.poly_describe(h, out, 14))
    return dict(zip(["grid", "threads", "rows_per_stage", "stages", "smem", "sms", "V", "WPR", "NW",
                     "full", "comm_ranks", "k9", "csr_layout", "l2_keep_bytes"], list(out)))


def poly_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.poly_nccl_unique_id(buf))
    return buf.raw


def poly_p2p_handle(h: int) -> bytes:
    """This rank's 64-byte peer-reduce window handle (POLY_FLAG_P2P)."""
    buf = C.create_string_buffer(64)
    _check(_lib.poly_p2p_handle(h, buf))
    return buf.raw


def poly_p2p_open(h: int, handles: bytes):
    """Map every rank's window (world * 64 bytes in rank order): K9 replaces
    ncclAllReduce for this handle from the next evaluation on."""
    buf = C.create_string_buffer(bytes(handles), len(handles))
    _check(_lib.poly_p2p_open(h, buf))


def poly_nvls_handle(h: int) -> bytes:
    """Rank 0: create the NVLink multicast object; its 64-byte descriptor
    (POLY_FLAG_NVLS).  Other ranks get bytes they pass on unused."""
    buf = C.create_string_buffer(64)
    _check(_lib.poly_nvls_handle(h, buf))
    return buf.raw


def poly_nvls_open(h: int, desc: bytes):
    """Join rank 0's multicast object (desc = rank 0's descriptor, on every
    rank): K9-NVLS replaces ncclAllReduce for this handle."""
    buf = C.create_string_buffer(bytes(desc), 64)
    _check(_lib.poly_nvls_open(h, buf))


def poly_share_fd(rank: int, world: int, name: str, fd_in: int, timeout_s: float = 30.0) -> int:
    """Same-node fd hand-off of poly_nvls_open (rank 0 -> the others)."""
    out = C.c_int(-1)
    _check(_lib.poly_share_fd(int(rank), int(world), name.encode(), int(fd_in), C.byref(out),
                              float(timeout_s)))
    return out.value


def poly_free(h: int):
    _lib.poly_free(h)


from .api import Poly  # noqa: E402,F401
