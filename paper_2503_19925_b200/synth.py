"""ctypes binding of libpolysynth.so (include/polysynth.h): the CUDA twin of
the seeded generators in gen/rng.py.  Input generation only."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpolysynth.so")
EXPORTED = ["polysynth_gaussian_matrix", "polysynth_poisson", "polysynth_add_noise",
            "polysynth_last_error"]

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, u32 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32
        L.polysynth_gaussian_matrix.argtypes = [vp, i32, i64, i64, i64, i64, i64, u32, u32, vp]
        L.polysynth_poisson.argtypes = [vp, vp, i64, i64, u32, u32, vp]
        L.polysynth_add_noise.argtypes = [vp, vp, i64, i64, C.c_double, u32, u32, vp]
        L.polysynth_last_error.restype = C.c_char_p
        for n in EXPORTED[:-1]:
            getattr(L, n).restype = C.c_int
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise RuntimeError("polysynth: " + lib().polysynth_last_error().decode())


def _stream():
    import torch
    return torch.cuda.current_stream().cuda_stream


def gaussian_matrix(A, d, row0, seed, stream_id, col0=0):
    """Fill torch tensor A [n, lda] (float32/float64, cuda) with N(0,1) draws."""
    import torch
    dt = 0 if A.dtype == torch.float32 else 1
    _check(lib().polysynth_gaussian_matrix(A.data_ptr(), dt, A.shape[0], int(d), A.stride(0),
                                           int(row0), int(col0), int(seed), int(stream_id),
                                           _stream()))


def poisson(lam, y, row0, seed, stream_id):
    _check(lib().polysynth_poisson(lam.data_ptr(), y.data_ptr(), lam.numel(), int(row0),
                                   int(seed), int(stream_id), _stream()))


def add_noise(k, y, row0, sigma, seed, stream_id):
    _check(lib().polysynth_add_noise(k.data_ptr(), y.data_ptr(), k.numel(), int(row0),
                                     float(sigma), int(seed), int(stream_id), _stream()))
