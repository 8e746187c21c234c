// K4 — fused CSR loss+gradient kernel for the CT-like sparse system matrix
// (BASELINE.json configs[3]; A nonnegative).
//
// One warp per row (grid-stride): gather z_i = Σ_e val_e x[col_e] (fp64),
// the W-bin link and residual exactly as K1 (row_residual), then scatter
// g[col_e] += r_i val_e with fp64 `red.global.add` into an L2-resident
// accumulator (d = 65536 doubles = 512 KB).  The row's (col, val) pairs stay
// in registers between the gather and the scatter (up to 32*KREG entries;
// longer rows re-read the tail).  The finalize kernel reads the accumulator
// as a single partial row and zeroes it for the next call.
#pragma once

#include "dense.cuh"

namespace poly {

struct CsrArgs {
  const int64_t *row_ptr;
  const int32_t *col;
  const void *val;
  int64_t n;
  int32_t d;
  int32_t W;
  const void *y;
  int32_t ytype;
  int32_t relu;
  const float *s_row;
  const float *I_row;
  double I_bar;
  const double *x;
  const double *spec;
  double *gacc;      // [d], zero on entry
  double *lacc;      // [1], zero on entry
};

template <typename T, int KREG, bool LOSS>
__global__ void __launch_bounds__(256) k_csr_loss_grad(const CsrArgs a) {
  __shared__ double sp[3 * kMaxW];
  for (int i = threadIdx.x; i < 3 * kMaxW; i += blockDim.x) sp[i] = a.spec[i];
  __syncthreads();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const T *val = (const T *)a.val;
  double lacc = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < a.n;
       row += nwarps) {
    const int64_t e0 = a.row_ptr[row], e1 = a.row_ptr[row + 1];
    int32_t cr[KREG];
    T vr[KREG];
    double p = 0.0;
#pragma unroll
    for (int k = 0; k < KREG; ++k) {
      const int64_t e = e0 + lane + 32 * k;
      if (e < e1) {
        cr[k] = __ldg(a.col + e);
        vr[k] = __ldg(val + e);
        p += (double)vr[k] * a.x[cr[k]];
      } else {
        cr[k] = -1;
        vr[k] = (T)0;
      }
    }
    for (int64_t e = e0 + lane + 32 * KREG; e < e1; e += 32) p += (double)__ldg(val + e) * a.x[__ldg(a.col + e)];
    const double z = warp_sum(p);
    double yv;
    if (a.ytype == 0) yv = (double)((const int32_t *)a.y)[row];
    else if (a.ytype == 1) yv = (double)((const float *)a.y)[row];
    else yv = ((const double *)a.y)[row];
    const double Ii = a.I_row ? (double)a.I_row[row] : a.I_bar;
    const float *srow = a.I_row ? a.s_row + row * a.W : nullptr;
    const double r = row_residual<LOSS>(sp, a.W, a.relu, z, yv, Ii, srow, true, &lacc);
#pragma unroll
    for (int k = 0; k < KREG; ++k)
      if (cr[k] >= 0) atomicAdd(a.gacc + cr[k], r * (double)vr[k]);
    for (int64_t e = e0 + lane + 32 * KREG; e < e1; e += 32)
      atomicAdd(a.gacc + __ldg(a.col + e), r * (double)__ldg(val + e));
  }
  if (LOSS && lane == 0 && lacc != 0.0) atomicAdd(a.lacc, lacc);
  pdl_trigger();
}

}  // namespace poly
