// Auxiliary product kernels (not on the timed path): fp64-accurate forward
// projection z = A x, expected counts λ_i = Ī_i h_i(z_i) (Eq. model,
// PAPER.md:867-869), and the Appendix A.1 reparameterisation.
#pragma once

#include "dense.cuh"

namespace poly {

struct AuxArgs {
  int32_t layout;  // 0 dense, 1 csr
  int32_t dtype;   // 0 f32, 1 f64
  const void *A;
  int64_t lda;
  const int64_t *row_ptr;
  const int32_t *col;
  const void *val;
  int64_t n;
  int32_t d;
  int32_t W;
  int32_t relu;
  const float *s_row;
  const float *I_row;
  double I_bar;
  const double *x;
  const double *spec;
  double *out;
  int32_t want_counts;  // 0: z, 1: λ
};

template <typename T>
__device__ __forceinline__ double row_dot_f64(const AuxArgs &a, int64_t row, int lane) {
  double p = 0.0;
  if (a.layout == 0) {
    const T *r = (const T *)a.A + row * a.lda;
    for (int k = lane; k < a.d; k += 32) p += (double)r[k] * a.x[k];
  } else {
    const T *v = (const T *)a.val;
    for (int64_t e = a.row_ptr[row] + lane; e < a.row_ptr[row + 1]; e += 32)
      p += (double)v[e] * a.x[a.col[e]];
  }
  return warp_sum(p);
}

template <typename T>
__global__ void __launch_bounds__(256) k_aux_rows(const AuxArgs a) {
  __shared__ double sp[3 * kMaxW];
  for (int i = threadIdx.x; i < 3 * kMaxW; i += blockDim.x) sp[i] = a.spec[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < a.n;
       row += nwarps) {
    const double z = row_dot_f64<T>(a, row, lane);
    double o = z;
    if (a.want_counts) {
      const double Ii = a.I_row ? (double)a.I_row[row] : a.I_bar;
      const float *srow = a.I_row ? a.s_row + row * a.W : nullptr;
      o = -row_residual<false>(sp, a.W, a.relu, z, 0.0, Ii, srow, false, nullptr);
    }
    if (lane == 0) a.out[row] = o;
  }
}

struct ReparamArgs {
  int32_t W;
  int32_t clamp;
  int64_t n;
  double I_bar;
  double s[kMaxW];
  double mu[kMaxW];
  const double *b;
  float *s_row;
  float *I_row;
};

__global__ void __launch_bounds__(256) k_reparam(const ReparamArgs a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double bi = (a.clamp && a.b[i] < 0.0) ? 0.0 : a.b[i];
    double tot = 0.0;
    for (int j = 0; j < a.W; ++j) tot += a.s[j] * exp(-a.mu[j] * bi);
    for (int j = 0; j < a.W; ++j) a.s_row[i * a.W + j] = (float)(a.s[j] * exp(-a.mu[j] * bi) / tot);
    a.I_row[i] = (float)(a.I_bar * tot);
  }
}

}  // namespace poly
