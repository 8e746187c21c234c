// CUDA twin of gen/rng.py (seeded input generators).  Compiled with
// -fmad=false so every fp64 operation is the single IEEE-rounded operation
// the numpy side performs; the operation order below mirrors gen/rng.py line
// for line.  Not part of the method (see include/polysynth.h).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/polysynth.h"

namespace {

thread_local char g_err[512] = "";

void set_err(const char *what, cudaError_t e) {
  snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
}

constexpr double LN2 = 0.6931471805599453;
constexpr double LN2_HI = 6.93147180369123816490e-01;
constexpr double LN2_LO = 1.90821492927058770002e-10;
constexpr double INV_LN2 = 1.4426950408889634;
constexpr double SQRT_HALF = 0.7071067811865476;
constexpr double HALF_LOG_2PI = 0.9189385332046728;
constexpr double TWO_POW_M53 = 1.0 / 9007199254740992.0;
constexpr int LOG_TERMS = 12;
constexpr int EXP_TERMS = 13;

struct u4 { uint32_t x, y, z, w; };

__device__ __forceinline__ u4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                     uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return {c0, c1, c2, c3};
}

__device__ __forceinline__ double u01(uint32_t hi, uint32_t lo) {
  const uint64_t m = ((uint64_t)(hi >> 6) << 26) | (uint64_t)(lo >> 6);
  return __dmul_rn(__dadd_rn(__dmul_rn((double)m, 2.0), 1.0), TWO_POW_M53);
}

__device__ double log64(double x) {
  int e;
  double m = frexp(x, &e);
  if (m < SQRT_HALF) {
    m = __dmul_rn(m, 2.0);
    e -= 1;
  }
  const double f = __ddiv_rn(__dsub_rn(m, 1.0), __dadd_rn(m, 1.0));
  const double f2 = __dmul_rn(f, f);
  double p = __ddiv_rn(1.0, (double)(2 * LOG_TERMS + 1));
  for (int k = LOG_TERMS - 1; k >= 0; --k)
    p = __dadd_rn(__dmul_rn(p, f2), __ddiv_rn(1.0, (double)(2 * k + 1)));
  return __dadd_rn(__dmul_rn((double)e, LN2), __dmul_rn(__dmul_rn(2.0, f), p));
}

__device__ double exp64(double x) {
  const double k = floor(__dadd_rn(__dmul_rn(x, INV_LN2), 0.5));
  const double r = __dsub_rn(__dsub_rn(x, __dmul_rn(k, LN2_HI)), __dmul_rn(k, LN2_LO));
  double fact[EXP_TERMS + 1];
  fact[0] = 1.0;
  for (int j = 1; j <= EXP_TERMS; ++j) fact[j] = __dmul_rn(fact[j - 1], (double)j);  // exact
  double p = __ddiv_rn(1.0, fact[EXP_TERMS]);
  for (int j = EXP_TERMS - 1; j >= 0; --j) p = __dadd_rn(__dmul_rn(p, r), __ddiv_rn(1.0, fact[j]));
  return ldexp(p, (int)k);
}

__device__ double logfact64(double k) {
  if (k < 16.0) {
    double t = 0.0;
    const int kk = (int)k;
    for (int i = 2; i <= kk; ++i) t = __dadd_rn(t, log64((double)i));
    return t;
  }
  const double lk = log64(k);
  const double r = __ddiv_rn(1.0, k);
  const double r2 = __dmul_rn(r, r);
  const double t = __dadd_rn(__dsub_rn(__dmul_rn(__dadd_rn(k, 0.5), lk), k), HALF_LOG_2PI);
  const double c12 = __ddiv_rn(1.0, 12.0), c360 = __ddiv_rn(1.0, 360.0),
               c1260 = __ddiv_rn(1.0, 1260.0);
  const double series = __dmul_rn(r, __dsub_rn(c12, __dmul_rn(r2, __dsub_rn(c360, __dmul_rn(r2, c1260)))));
  return __dadd_rn(t, series);
}

// polar method, counter (b, lo(a), hi(a), attempt), key (seed, stream)
__device__ double normal_at(uint64_t a, uint32_t b, uint32_t seed, uint32_t sid) {
  for (uint32_t attempt = 0; attempt <= 64; ++attempt) {
    const u4 w = philox(b, (uint32_t)a, (uint32_t)(a >> 32), attempt, seed, sid);
    const double u = __dsub_rn(__dmul_rn(2.0, u01(w.x, w.y)), 1.0);
    const double v = __dsub_rn(__dmul_rn(2.0, u01(w.z, w.w)), 1.0);
    const double s = __dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v));
    if (s < 1.0) return __dmul_rn(u, __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, log64(s)), s)));
  }
  return __longlong_as_double(0x7ff8000000000000ULL);  // unreachable in practice
}

__global__ void k_gaussian_f32(float *A, int64_t n, int64_t d, int64_t lda, int64_t row0,
                               int64_t col0, uint32_t seed, uint32_t sid) {
  const int64_t total = n * lda;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / lda, c = e - r * lda;
    A[e] = c < d ? __double2float_rn(normal_at((uint64_t)(row0 + r), (uint32_t)(col0 + c), seed, sid))
                 : 0.0f;
  }
}

__global__ void k_gaussian_f64(double *A, int64_t n, int64_t d, int64_t lda, int64_t row0,
                               int64_t col0, uint32_t seed, uint32_t sid) {
  const int64_t total = n * lda;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / lda, c = e - r * lda;
    A[e] = c < d ? normal_at((uint64_t)(row0 + r), (uint32_t)(col0 + c), seed, sid) : 0.0;
  }
}

__device__ int64_t poisson_at(double lam, uint64_t idx, uint32_t seed, uint32_t sid) {
  const uint32_t lo = (uint32_t)idx, hi = (uint32_t)(idx >> 32);
  if (lam < 10.0) {
    const u4 w = philox(0u, lo, hi, 0x50000001u, seed, sid);
    const double U = u01(w.x, w.y);
    double p = exp64(-lam);
    double F = p;
    double k = 0.0;
    while (U > F && k < 1000.0) {
      k = __dadd_rn(k, 1.0);
      p = __ddiv_rn(__dmul_rn(p, lam), k);
      F = __dadd_rn(F, p);
    }
    return (int64_t)k;
  }
  const double slam = __dsqrt_rn(lam);
  const double loglam = log64(lam);
  const double b = __dadd_rn(0.931, __dmul_rn(2.53, slam));
  const double a = __dadd_rn(-0.059, __dmul_rn(0.02483, b));
  const double invalpha = __dadd_rn(1.1239, __ddiv_rn(1.1328, __dsub_rn(b, 3.4)));
  const double vr = __dsub_rn(0.9277, __ddiv_rn(3.6224, __dsub_rn(b, 2.0)));
  const double log_invalpha = log64(invalpha);
  for (uint32_t attempt = 0; attempt <= 256; ++attempt) {
    const u4 w = philox(attempt, lo, hi, 0x50000000u, seed, sid);
    const double U = __dsub_rn(u01(w.x, w.y), 0.5);
    const double V = u01(w.z, w.w);
    const double us = __dsub_rn(0.5, fabs(U));
    const double k = floor(__dadd_rn(__dadd_rn(__dmul_rn(__dadd_rn(__ddiv_rn(__dmul_rn(2.0, a), us), b), U),
                                                lam), 0.43));
    if (us >= 0.07 && V <= vr) return (int64_t)k;
    if (k < 0.0 || (us < 0.013 && V > us)) continue;
    const double lhs = __dsub_rn(__dadd_rn(log64(V), log_invalpha),
                                 log64(__dadd_rn(__ddiv_rn(a, __dmul_rn(us, us)), b)));
    const double rhs = __dsub_rn(__dadd_rn(-lam, __dmul_rn(k, loglam)), logfact64(k));
    if (lhs <= rhs) return (int64_t)k;
  }
  return -1;
}

__global__ void k_poisson(const double *lam, int32_t *y, int64_t n, int64_t row0, uint32_t seed,
                          uint32_t sid) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (int32_t)poisson_at(lam[i], (uint64_t)(row0 + i), seed, sid);
}

__global__ void k_noise(const int32_t *k, float *y, int64_t n, int64_t row0, double sigma,
                        uint32_t seed, uint32_t sid) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double e = normal_at((uint64_t)(row0 + i), 0u, seed, sid);
    y[i] = __double2float_rn(__dadd_rn((double)k[i], __dmul_rn(sigma, e)));
  }
}

int grid_for(int64_t work) {
  int64_t g = (work + 255) / 256;
  if (g > 148 * 64) g = 148 * 64;
  if (g < 1) g = 1;
  return (int)g;
}

int finish(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_err(what, e);
    return 1;
  }
  g_err[0] = 0;
  return 0;
}

}  // namespace

extern "C" int polysynth_gaussian_matrix(void *A, int32_t dtype, int64_t n, int64_t d,
                                         int64_t lda, int64_t row0, int64_t col0, uint32_t seed,
                                         uint32_t stream_id, void *stream) {
  if (n < 0 || d < 1 || lda < d || !A) {
    snprintf(g_err, sizeof(g_err), "polysynth_gaussian_matrix: bad arguments");
    return 1;
  }
  if (n == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == 0)
    k_gaussian_f32<<<grid_for(n * lda), 256, 0, st>>>((float *)A, n, d, lda, row0, col0, seed,
                                                      stream_id);
  else
    k_gaussian_f64<<<grid_for(n * lda), 256, 0, st>>>((double *)A, n, d, lda, row0, col0, seed,
                                                       stream_id);
  return finish("polysynth_gaussian_matrix");
}

extern "C" int polysynth_poisson(const double *lam, int32_t *y, int64_t n, int64_t row0,
                                 uint32_t seed, uint32_t stream_id, void *stream) {
  if (n < 0 || (n > 0 && (!lam || !y))) {
    snprintf(g_err, sizeof(g_err), "polysynth_poisson: bad arguments");
    return 1;
  }
  if (n == 0) return 0;
  k_poisson<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(lam, y, n, row0, seed, stream_id);
  return finish("polysynth_poisson");
}

extern "C" int polysynth_add_noise(const int32_t *k, float *y, int64_t n, int64_t row0,
                                   double sigma, uint32_t seed, uint32_t stream_id, void *stream) {
  if (n < 0 || sigma < 0 || (n > 0 && (!k || !y))) {
    snprintf(g_err, sizeof(g_err), "polysynth_add_noise: bad arguments");
    return 1;
  }
  if (n == 0) return 0;
  k_noise<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(k, y, n, row0, sigma, seed, stream_id);
  return finish("polysynth_add_noise");
}

extern "C" const char *polysynth_last_error(void) { return g_err; }
