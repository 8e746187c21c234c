// K4 — CSR loss+gradient for the CT-like sparse system matrix
// (BASELINE.json configs[3]; A nonnegative), two passes:
//
//   K4f k_csr_forward   one warp per row (grid-stride): z_i = Σ_e val_e x[col_e]
//                       (fp64), the W-bin link and residual exactly as K1
//                       (row_residual), r_i stored as fp32, ℓ per block.
//   K4b k_csc_backward  g_k = Σ_{i in column k} val_ik r_i  (Aᵀ r)
//                       from a SELL-32 copy of Aᵀ built once at poly_init: a
//                       slice holds 32 consecutive columns, step s of lane t is
//                       the s-th entry (ascending row) of column 32·slice + t,
//                       so each warp-step is one coalesced 256-byte load and
//                       every lane owns its column's sum in registers — no
//                       atomics, fixed summation order (deterministic).
//
// Why two passes: a one-pass fused kernel must scatter g[col] += r val for
// every nonzero (red.global at ~1 lane/1.3 cycles per SM, B300_MICROARCH.md
// "Atomics"), which caps the scatter near 140 µs for C4's 30M nonzeros; the
// gather formulation reads the values twice (≈ 2x the algorithmic bytes) but
// streams at HBM rate.
#pragma once

#include "dense.cuh"

namespace poly {

template <typename T>
struct CscEnt {
  int32_t row;
  T val;
};

struct CsrFwdArgs {
  const int64_t *row_ptr;
  const int32_t *col;
  const void *val;
  int64_t n;
  int32_t W;
  const void *y;
  int32_t ytype;
  int32_t relu;
  const float *s_row;
  const float *I_row;
  double I_bar;
  const double *x;
  const double *spec;
  float *r;               // [n] residuals r_i (output)
  double *loss_partials;  // [gridDim.x]
};

template <typename T, bool LOSS>
__global__ void __launch_bounds__(256) k_csr_forward(const CsrFwdArgs a) {
  __shared__ double sp[3 * kMaxW];
  __shared__ double wl[8];
  for (int i = threadIdx.x; i < 3 * kMaxW; i += blockDim.x) sp[i] = a.spec[i];
  __syncthreads();
  pdl_wait();  // x is written by the previous kernel; r is read by the previous backward
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const T *val = (const T *)a.val;
  double lacc = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; row < a.n; row += nwarps) {
    const int64_t e0 = a.row_ptr[row], e1 = a.row_ptr[row + 1];
    double p0 = 0.0, p1 = 0.0;
    int64_t e = e0 + lane;
    for (; e + 32 < e1; e += 64) {
      const int32_t c0 = __ldcs(a.col + e), c1 = __ldcs(a.col + e + 32);
      const T v0 = __ldcs(val + e), v1 = __ldcs(val + e + 32);
      p0 = fma((double)v0, a.x[c0], p0);
      p1 = fma((double)v1, a.x[c1], p1);
    }
    if (e < e1) p0 = fma((double)__ldcs(val + e), a.x[__ldcs(a.col + e)], p0);
    const double z = warp_sum(p0 + p1);
    double yv;
    if (a.ytype == 0) yv = (double)((const int32_t *)a.y)[row];
    else if (a.ytype == 1) yv = (double)((const float *)a.y)[row];
    else yv = ((const double *)a.y)[row];
    const double Ii = a.I_row ? (double)a.I_row[row] : a.I_bar;
    const float *srow = a.I_row ? a.s_row + row * a.W : nullptr;
    const double r = row_residual<LOSS>(sp, a.W, a.relu, z, yv, Ii, srow, true, &lacc);
    if (lane == 0) a.r[row] = (float)r;
  }
  // per-block loss partial, warps combined in order (deterministic)
  if (lane == 0) wl[warp] = lacc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double l = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) l += wl[w];
    a.loss_partials[blockIdx.x] = l;
  }
  pdl_trigger();
}

// 4 warps per 32-column slice; warp w takes steps w, w+4, w+8, ...; the four
// warps' sums are combined in warp order.
template <typename T>
__global__ void __launch_bounds__(128) k_csc_backward(const CscEnt<T> *__restrict__ ent,
                                                      const int64_t *__restrict__ slice_off,
                                                      int32_t d, const float *__restrict__ r,
                                                      double *__restrict__ g) {
  __shared__ double part[4][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t s0 = slice_off[blockIdx.x], s1 = slice_off[blockIdx.x + 1];
  const CscEnt<T> *p = ent + s0 * 32 + lane;
  const int64_t len = s1 - s0;
  pdl_wait();  // r is written by the forward pass
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int64_t k = warp;
  for (; k + 12 < len; k += 16) {
    const CscEnt<T> q0 = p[(k) * 32], q1 = p[(k + 4) * 32], q2 = p[(k + 8) * 32],
                    q3 = p[(k + 12) * 32];
    a0 = fma((double)q0.val, (double)__ldg(r + q0.row), a0);
    a1 = fma((double)q1.val, (double)__ldg(r + q1.row), a1);
    a2 = fma((double)q2.val, (double)__ldg(r + q2.row), a2);
    a3 = fma((double)q3.val, (double)__ldg(r + q3.row), a3);
  }
  for (; k < len; k += 4) {
    const CscEnt<T> q = p[k * 32];
    a0 = fma((double)q.val, (double)__ldg(r + q.row), a0);
  }
  part[warp][lane] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  if (warp == 0) {
    const int c = blockIdx.x * 32 + lane;
    const double v = (part[0][lane] + part[1][lane]) + (part[2][lane] + part[3][lane]);
    if (c < d) g[c] = v;
  }
  pdl_trigger();
}

// ---------------------------------------------------------------- SELL build
// (poly_init only) row index of every stored entry
__global__ void k_entry_rows(const int64_t *row_ptr, int64_t n, int32_t *rows) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nw)
    for (int64_t e = row_ptr[i] + lane; e < row_ptr[i + 1]; e += 32) rows[e] = (int32_t)i;
}

__global__ void k_col_count(const int32_t *col, int64_t nnz, int32_t *cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + col[e], 1);
}

// slice length (steps) = longest column of the slice
__global__ void k_slice_len(const int32_t *cnt, int32_t d, int32_t nslices, int64_t *len) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nslices) return;
  int32_t m = 0;
  for (int c = 32 * s; c < min(d, 32 * s + 32); ++c) m = max(m, cnt[c]);
  len[s] = m;
}

// entry k of the column-sorted order (stable: ascending row within a column)
template <typename T>
__global__ void k_sell_fill(const int32_t *sorted_col, const int32_t *perm, const int32_t *rows,
                            const T *val, const int64_t *colptr, const int64_t *slice_off,
                            int64_t nnz, CscEnt<T> *ent) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = sorted_col[k];
    const int32_t e = perm[k];
    const int64_t j = k - colptr[c];
    CscEnt<T> q;
    q.row = rows[e];
    q.val = val[e];
    ent[(slice_off[c >> 5] + j) * 32 + (c & 31)] = q;
  }
}

}  // namespace poly
