"""Torch-tensor convenience wrapper over the C ABI (marshalling only).

torch provides device memory and the current stream; the computation is the
library's.  Tensors handed to `Poly` are borrowed by the handle (kept alive
by this object) exactly as poly.h describes.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import (POLY_CSR, POLY_DENSE, POLY_F32, POLY_F64, POLY_FLAG_HOST_INPUTS, POLY_PARALLEL_BEAM,
               POLY_METHOD_EXTRAGRADIENT, POLY_SET_BALL, POLY_SOLVE_PROFILE, POLY_Y_F32, POLY_Y_F64,
               POLY_Y_I32, PolyProblem, PolySolveOpts, poly_describe, poly_expected_counts,
               poly_forward, poly_free, poly_init, poly_kernel_times, poly_loss_grad, poly_project,
               poly_solve, poly_solve_ex, poly_stream_probe)

_DT = {torch.float32: POLY_F32, torch.float64: POLY_F64}
_YT = {torch.int32: POLY_Y_I32, torch.float32: POLY_Y_F32, torch.float64: POLY_Y_F64}


def _ptr(t):
    return None if t is None else t.data_ptr()


class Poly:
    """One problem instance: A (dense [n, lda] or CSR), y, spectrum, X.

    Dense A must be row-major with a row pitch (stride(0)) whose byte size is
    a multiple of 16; pass `d` when the rows are padded.
    """

    def __init__(self, *, y, s, mu, I_bar, d=None, A=None, row_ptr=None, col=None, val=None,
                 s_row=None, I_row=None, relu=1, set=POLY_SET_BALL, R=1.0, center=None,
                 n_global=None, row_offset=0, rank=0, world=1, nccl_id=None, stream=None,
                 flags=0, mode=0, I_win=None, tv=None, pb=None):
        p = PolyProblem()
        host = bool(flags & POLY_FLAG_HOST_INPUTS)
        self._keep = [y, A, row_ptr, col, val, s_row, I_row]
        if pb is not None:   # matrix-free parallel beam: pb = dict(side=, views=, bins=)
            p.layout, p.dtype = POLY_PARALLEL_BEAM, POLY_F32
            p.pb_side, p.pb_views, p.pb_bins = int(pb["side"]), int(pb["views"]), int(pb["bins"])
            p.n_local = y.numel() if I_win is None else y.numel() // len(I_win)
            p.d = p.pb_side ** 2
        elif A is not None:
            assert A.dim() == 2 and A.stride(1) == 1, "A must be row-major"
            p.layout, p.dtype = POLY_DENSE, _DT[A.dtype]
            p.n_local = A.shape[0]
            p.d = A.shape[1] if d is None else int(d)
            p.A, p.lda = _ptr(A), A.stride(0)
        else:
            p.layout, p.dtype = POLY_CSR, _DT[val.dtype]
            p.n_local = row_ptr.shape[0] - 1
            p.d = int(d)
            p.row_ptr, p.col, p.val = _ptr(row_ptr), _ptr(col), _ptr(val)
            p.nnz = val.shape[0]
            assert row_ptr.dtype == torch.int64 and col.dtype == torch.int32
        p.n_global = p.n_local if n_global is None else int(n_global)
        p.row_offset = int(row_offset)
        p.ytype, p.y = _YT[y.dtype], _ptr(y)
        if I_win is not None:   # Ω windows: s [Ω, W], y [Ω, n_local] (window-major)
            iw = [float(v) for v in I_win]
            self._iw = (C.c_double * len(iw))(*iw)
            p.windows, p.I_win = len(iw), C.addressof(self._iw)
            assert y.is_contiguous() and y.numel() == len(iw) * p.n_local
            s = [float(v) for row in s for v in row]
        else:
            s = [float(v) for v in s]
        mu = [float(v) for v in mu]
        self._s = (C.c_double * len(s))(*s)
        self._mu = (C.c_double * len(mu))(*mu)
        p.W, p.s, p.mu = len(mu), C.addressof(self._s), C.addressof(self._mu)
        p.mode = int(mode)
        for k, v in (tv or {}).items():   # tv_tau, tv_tol, tv_rtol, tv_dykstra_tol, tv_max_it, ...
            setattr(p, k if k.startswith("tv_") else "tv_" + k, v)
        p.I_bar = float(I_bar)
        if s_row is not None:
            assert s_row.dtype == torch.float32 and I_row.dtype == torch.float32
        p.s_row, p.I_row = _ptr(s_row), _ptr(I_row)
        p.relu, p.set, p.R = int(relu), int(set), float(R)
        if center is not None:
            c = [float(v) for v in (center.tolist() if hasattr(center, "tolist") else center)]
            self._c = (C.c_double * len(c))(*c)
            p.center = C.addressof(self._c)
        p.rank, p.world = int(rank), int(world)
        if nccl_id is not None:
            self._id = C.create_string_buffer(bytes(nccl_id), 128)
            p.nccl_id = C.addressof(self._id)
        if stream is None and not host and torch.cuda.is_available():
            stream = torch.cuda.current_stream().cuda_stream
        p.stream = stream
        p.flags = int(flags)
        self.d = int(p.d)
        self.n_local = int(p.n_local)
        self.problem = p
        self.h = poly_init(p)

    def p2p_setup(self):
        """K9: exchange the peer-reduce window handles (all ranks, collective
        over the default torch.distributed group) and switch this handle's
        cross-rank sum from ncclAllReduce to the NVLink peer-reduce kernel.
        Needs flags with POLY_FLAG_P2P."""
        from . import dist as D
        from . import poly_p2p_handle, poly_p2p_open
        hs = D.gather_handles(poly_p2p_handle(self.h), int(self.problem.rank), int(self.problem.world))
        poly_p2p_open(self.h, hs)

    def nvls_setup(self):
        """K9-NVLS: rank 0 creates the NVLink multicast object, its descriptor
        is broadcast over the default torch.distributed group (world > 1),
        and every rank joins; the cross-rank sum then runs in the switch.
        Needs flags with POLY_FLAG_NVLS."""
        from . import poly_nvls_handle, poly_nvls_open
        desc = poly_nvls_handle(self.h)
        if int(self.problem.world) > 1:
            import torch.distributed as dist
            box = [desc if int(self.problem.rank) == 0 else None]
            dist.broadcast_object_list(box, src=0)
            desc = box[0]
        poly_nvls_open(self.h, desc)

    def close(self):
        if getattr(self, "h", None):
            # K9 / K9-NVLS: a peer may still read this rank's window until it
            # finished its last evaluation, so the ranks meet before freeing
            from . import POLY_FLAG_NVLS, POLY_FLAG_P2P
            if int(self.problem.world) > 1 and int(self.problem.flags) & (POLY_FLAG_P2P | POLY_FLAG_NVLS):
                import torch.distributed as dist
                if dist.is_available() and dist.is_initialized():
                    dist.barrier()
            poly_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- calls
    def loss_grad(self, x, want_loss=True, g=None):
        """F(x) (Eq. operator) and ℓ(x).  x: fp64 tensor (device or host)."""
        assert x.dtype == torch.float64 and x.is_contiguous() and x.numel() == self.d
        if g is None:
            g = torch.empty(self.d, dtype=torch.float64, device=x.device)
        loss = poly_loss_grad(self.h, x.data_ptr(), g.data_ptr(), want_loss)
        return g, loss

    def solve(self, x, T, gamma, trace=False, profile=False):
        """EXACT (Eq. extragrad-method): x is updated in place to x_{T+1}."""
        assert x.dtype == torch.float64 and x.is_contiguous() and x.numel() == self.d
        tr = (C.c_double * (2 * T))() if trace else None
        poly_solve(self.h, x.data_ptr(), T, gamma, POLY_SOLVE_PROFILE if profile else 0, tr)
        return list(tr) if trace else None

    def solve_ex(self, x, T_max, gamma, *, method=POLY_METHOD_EXTRAGRADIENT, average=False,
                 tol=0.0, profile=False, x_last=None):
        """poly_solve_ex: x is overwritten with x̄_k (average) or the last
        iterate; returns the PolySolveInfo (iters, stopped, move, bad_iter)."""
        assert x.dtype == torch.float64 and x.is_contiguous() and x.numel() == self.d
        o = PolySolveOpts()
        o.T_max, o.method, o.gamma, o.tol = int(T_max), int(method), float(gamma), float(tol)
        o.average, o.flags = int(bool(average)), POLY_SOLVE_PROFILE if profile else 0
        return poly_solve_ex(self.h, x.data_ptr(), o, None if x_last is None else x_last.data_ptr())

    def project(self, v, out=None):
        """P_X(v) for the handle's set; returns (x, TV statistics)."""
        assert v.dtype == torch.float64 and v.is_contiguous() and v.numel() == self.d
        out = torch.empty_like(v) if out is None else out
        st = poly_project(self.h, v.data_ptr(), out.data_ptr())
        return out, st

    def forward(self, x):
        z = torch.empty(self.n_local, dtype=torch.float64, device=x.device)
        poly_forward(self.h, x.data_ptr(), z.data_ptr())
        return z

    def expected_counts(self, x):
        lam = torch.empty(self.n_local, dtype=torch.float64, device=x.device)
        poly_expected_counts(self.h, x.data_ptr(), lam.data_ptr())
        return lam

    def stream_probe(self, reps=20):
        """K8 read-only streaming ceiling over this handle's A (ms per pass)."""
        return poly_stream_probe(self.h, reps)

    def kernel_times(self):
        return poly_kernel_times(self.h)

    def describe(self):
        return poly_describe(self.h)
