// K1 — fused dense row-tile loss+gradient kernel (sm_100a).
//
// One pass over A computes, for the rows a CTA owns (PAPER.md:893-896,
// Eq. operator; ℓ per DESIGN.md reading R2):
//   a1  z_i = <a_i, x>                  (fp32 FMA on 4-element chunks, fp64 sum)
//   a2  h(z_i) = Σ_j s_j e^{-μ_j z_i+}   (lanes over bins j, fp64 exp)
//   a3  r_i = y_i - Ī_i h(z_i)           (fp64), ℓ_i = y_i z_i - Ī_i H(z_i)
//   a4  g += r_i a_i                      (the a_i values still in registers)
// and writes one fp64 partial vector per CTA (a5 is the finalize kernel).
//
// Data movement: a persistent grid (one CTA per SM) streams a contiguous row
// range through an S-stage shared-memory ring.  Warp 0 is the producer: lane 0
// issues one 1D bulk copy (TMA engine, L2 evict-first) per stage — a stage is
// RPS consecutive rows, contiguous in HBM because A is row-major — and all 32
// lanes fetch the stage's y / Ī'_i / s'_i· with cp.async, whose completion
// arrives on the same mbarrier.  Consumer warps own a column slab of x and g
// in registers; WPR warps cooperate on one row when d exceeds one slab
// (partial dots exchanged through shared memory, one named barrier per stage).
#pragma once

#include <type_traits>

#include "common.cuh"

namespace poly {

#ifndef POLY_EXP_DEG32
#define POLY_EXP_DEG32 9  // exp polynomial degree of the link for fp32 A (common.cuh exp_nonpos; 0: SFU)
#endif
#ifndef POLY_K1_LINK_SPLIT
#define POLY_K1_LINK_SPLIT 1  // WPR > 1: the row group's warps split the link's bins
#endif

#ifndef POLY_K1_FFMA2
#define POLY_K1_FFMA2 1   // fp32 dot/axpy as packed fma.rn.f32x2 (sm_100): half the FMA issue slots
#endif

// g[0..3] += r * c[0..3] as two packed FMAs (each lane of f32x2 is an IEEE fma: same bits as four scalar FMAs)
__device__ __forceinline__ void axpy4_f32x2(float (&g)[4], float r, const float (&c)[4]) {
  const float2 rr = make_float2(r, r);
  const float2 g0 = __ffma2_rn(rr, make_float2(c[0], c[1]), make_float2(g[0], g[1]));
  const float2 g1 = __ffma2_rn(rr, make_float2(c[2], c[3]), make_float2(g[2], g[3]));
  g[0] = g0.x, g[1] = g0.y, g[2] = g1.x, g[3] = g1.y;
}

constexpr double kK1KeepMB = 64.0;  // MB of A read with L2 evict-last (POLY_K1_KEEP_MB overrides)

struct DenseArgs {
  const void *A;
  int64_t lda;           // row pitch, elements
  int64_t n;             // local rows
  int32_t d;
  int32_t W;
  const void *y;
  int32_t ytype;         // 0 i32, 1 f32, 2 f64
  int32_t relu;
  const float *s_row;    // optional [n*W]
  const float *I_row;    // optional [n]
  double I_bar;
  const double *x;       // fp64 [d]
  const double *spec;    // [3*kMaxW]: s, mu, 1/mu
  double *partials;      // [gridDim.x * d]
  double *loss_partials; // [gridDim.x]
  int32_t stages;
  int32_t side_stride;   // bytes of side data per stage
  int32_t mode;          // POLY_MODE_*
  int32_t keep_stages;   // each CTA's first stages read with L2 evict-last (kept across passes), the rest evict-first
};

// Link + per-row scalar for one row (warp-uniform z).  Lanes take bins
// j = lane, lane+32, ...; fp64 warp sums give h, H (and h' for the baseline
// modes).  Returns φ_i (mode EXACT: r_i = y_i - Ī_i h(z_i)); accumulates the
// row's objective term into *lacc on lane 0 when `count_loss`.
//   mode 0 EXACT  φ = y - Ī h,            ℓ_i = y z - Ī H(z)        (Eq. operator; R2)
//   mode 1 L2     φ = 2 (Ī h - y) Ī h',   (Ī h - y)^2
//   mode 2 L1     φ = sign(Ī h - y) Ī h', |Ī h - y|
//   mode 3 NLL    φ = (Ī - y / h) h',     Ī h - y log(Ī h)
// h'(z) = -Σ_j s_j μ_j e^{-μ_j z}, and 0 for z <= 0 under relu.
template <bool LOSS>
__device__ __forceinline__ double row_residual(const double *sp, int W, int relu, double z,
                                               double yv, double Ii, const float *srow,
                                               bool count_loss, double *lacc, int mode = 0) {
  const int lane = threadIdx.x & 31;
  const bool neg = relu && z < 0.0;
  const double zc = neg ? 0.0 : z;
  double hs = 0.0, Hs = 0.0;
  if (mode == 0) {
    for (int j = lane; j < W; j += 32) {
      const double sj = srow ? (double)srow[j] : sp[j];
      const double e = exp_nonpos(-sp[kMaxW + j] * zc);
      hs += sj * e;
      if (LOSS) Hs += neg ? sj * z : sj * sp[2 * kMaxW + j] * (1.0 - e);
    }
    hs = warp_sum(hs);
    if (LOSS) {
      Hs = warp_sum(Hs);
      if (count_loss && lane == 0) *lacc += yv * z - Ii * Hs;
    }
    return yv - Ii * hs;
  }
  double hp = 0.0;  // Σ s_j μ_j e_j
  for (int j = lane; j < W; j += 32) {
    const double sj = srow ? (double)srow[j] : sp[j];
    const double e = relu ? exp_nonpos(-sp[kMaxW + j] * zc) : exp(-sp[kMaxW + j] * z);
    hs += sj * e;
    hp += sj * sp[kMaxW + j] * e;
  }
  hs = warp_sum(hs);
  hp = -warp_sum(hp);
  if (relu && !(z > 0.0)) hp = 0.0;
  const double m = Ii * hs;
  double phi, l;
  if (mode == 1) {
    phi = 2.0 * (m - yv) * Ii * hp;
    l = (m - yv) * (m - yv);
  } else if (mode == 2) {
    const double r = m - yv;
    phi = (r > 0.0 ? 1.0 : (r < 0.0 ? -1.0 : 0.0)) * Ii * hp;
    l = fabs(r);
  } else {
    phi = (Ii - yv / hs) * hp;
    l = m - yv * log(m);
  }
  if (LOSS && count_loss && lane == 0) *lacc += l;
  return phi;
}

// Mode-0 (EXACT) link for K1, branch-free in the bins: lane j (and j + 32
// when W > 32) evaluates bin j; bins >= W carry s_j = 0 (the spectrum table
// is zero-padded to kMaxW, per-row spectra are masked).  DEG: exp polynomial
// degree (13 for fp64 A, 9 for fp32 A; see exp_nonpos).
template <bool LOSS, int DEG>
__device__ __forceinline__ double link_exact(const double *sp, int W, int relu, double z,
                                             double yv, double Ii, const float *srow,
                                             bool count_loss, double *lacc) {
  const int lane = threadIdx.x & 31;
  const bool neg = relu && z < 0.0;
  const double zc = neg ? 0.0 : z;
  double hs = 0.0, Hs = 0.0;
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    if (b == 1 && W <= 32) break;  // warp-uniform
    const int j = lane + 32 * b;
    const double sj = srow ? (j < W ? (double)srow[j] : 0.0) : sp[j];
    const double e = exp_nonpos<DEG>(-sp[kMaxW + j] * zc);
    hs = fma(sj, e, hs);
    if (LOSS) Hs += neg ? sj * z : sj * sp[2 * kMaxW + j] * (1.0 - e);
  }
  hs = warp_sum(hs);
  if (LOSS) {
    Hs = warp_sum(Hs);
    if (count_loss && lane == 0) *lacc += yv * z - Ii * Hs;
  }
  return yv - Ii * hs;
}

// Two rows' fp64 partial sums reduced in one butterfly (transpose trick):
// returns Σ_lanes p0 in lanes 0-15 and Σ_lanes p1 in lanes 16-31.
__device__ __forceinline__ double pair_sum(double p0, double p1) {
  const bool hi = (threadIdx.x & 16) != 0;
  double v = (hi ? p1 : p0) + __shfl_xor_sync(0xffffffffu, hi ? p0 : p1, 16);
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Mode-0 link of two rows at once (W <= 32): lanes 0-15 take row A's bins
// (j and j + 16), lanes 16-31 row B's, each half reduced on its own.  z, yv, Ii, srow are
// those of the lane's half; returns that half's residual.
template <bool LOSS, int DEG>
__device__ __forceinline__ double link_exact_pair(const double *sp, int W, int relu, double z,
                                                  double yv, double Ii, const float *srow,
                                                  bool count_loss, double *lacc) {
  const bool neg = relu && z < 0.0;
  const double zc = neg ? 0.0 : z;
  double hs = 0.0, Hs = 0.0;
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    if (b == 1 && W <= 16) break;  // warp-uniform
    const int j = (threadIdx.x & 15) + 16 * b;
    const double sj = srow ? (j < W ? (double)srow[j] : 0.0) : sp[j];
    const double e = exp_nonpos<DEG>(-sp[kMaxW + j] * zc);
    hs = fma(sj, e, hs);
    if (LOSS) Hs += neg ? sj * z : sj * sp[2 * kMaxW + j] * (1.0 - e);
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
    hs += __shfl_xor_sync(0xffffffffu, hs, o);
    if (LOSS) Hs += __shfl_xor_sync(0xffffffffu, Hs, o);
  }
  if (LOSS) {  // both halves' terms land on lane 0 (the lane whose lacc is kept)
    const double lt = count_loss ? yv * z - Ii * Hs : 0.0;
    const double lo = __shfl_sync(0xffffffffu, lt, 16);
    if ((threadIdx.x & 31) == 0) *lacc += lt + lo;
  }
  return yv - Ii * hs;
}

// The mode-0 link of two rows split over the WPR warps of a row group (W <=
// 32): warp w evaluates bins j = w + WPR l (l = lane & 15) of row q (lanes
// 0-15) and row q+1 (lanes 16-31), so each exp is computed once per row
// instead of once per warp; returns this half's partial sums Σ s_j e_j and
// Σ (s_j/μ_j)(1 - e_j) (or s_j z under the ReLU) in *hs, *Hs.
template <bool LOSS, int DEG, int WPR>
__device__ __forceinline__ void link_partial_pair(const double *sp, int W, int relu, double z,
                                                  const float *srow, int w, double *hs_out,
                                                  double *Hs_out) {
  const bool neg = relu && z < 0.0;
  const double zc = neg ? 0.0 : z;
  const int j = w + WPR * (threadIdx.x & 15);
  double hs = 0.0, Hs = 0.0;
  if (j < W) {
    const double sj = srow ? (double)srow[j] : sp[j];
    const double e = exp_nonpos<DEG>(-sp[kMaxW + j] * zc);
    hs = sj * e;
    if (LOSS) Hs = neg ? sj * z : sj * sp[2 * kMaxW + j] * (1.0 - e);
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
    hs += __shfl_xor_sync(0xffffffffu, hs, o);
    if (LOSS) Hs += __shfl_xor_sync(0xffffffffu, Hs, o);
  }
  *hs_out = hs;
  *Hs_out = Hs;
}

__device__ __forceinline__ double load_y(const unsigned char *yb, int ytype, int r) {
  if (ytype == 0) return (double)((const int32_t *)yb)[2 * r];
  if (ytype == 1) return (double)((const float *)yb)[2 * r];
  return ((const double *)yb)[r];
}

__device__ __forceinline__ double load_y_global(const void *y, int ytype, int64_t i) {
  if (ytype == 0) return (double)((const int32_t *)y)[i];
  if (ytype == 1) return (double)((const float *)y)[i];
  return ((const double *)y)[i];
}

template <typename T>
struct Vec16;
template <>
struct Vec16<float> {
  using type = float4;
  static constexpr int N = 4;
};
template <>
struct Vec16<double> {
  using type = double2;
  static constexpr int N = 2;
};

template <typename T>
__device__ __forceinline__ void unpack(const typename Vec16<T>::type &v, T *o);
template <>
__device__ __forceinline__ void unpack<float>(const float4 &v, float *o) {
  o[0] = v.x, o[1] = v.y, o[2] = v.z, o[3] = v.w;
}
template <>
__device__ __forceinline__ void unpack<double>(const double2 &v, double *o) {
  o[0] = v.x, o[1] = v.y;
}

// 16-byte chunk of a row at column c0 (smem), zeroing columns >= d.
template <typename T>
__device__ __forceinline__ void load_chunk(const T *rowp, int c0, int d, T *ch) {
  constexpr int VEC = Vec16<T>::N;
  if (c0 < d) {
    const typename Vec16<T>::type t = *reinterpret_cast<const typename Vec16<T>::type *>(rowp + c0);
    unpack<T>(t, ch);
#pragma unroll
    for (int e = 0; e < VEC; ++e)
      if (c0 + e >= d) ch[e] = (T)0;
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e) ch[e] = (T)0;
  }
}

// T: element type of A (float/double); V: 16-byte chunks per lane per slab;
// WPR: warps per row; NW: consumer warps; RPS: rows per stage.
// FULL: d == 32*VEC*V*WPR exactly, so no column masking is needed.
template <typename T, int V, int WPR, int NW, int RPS, bool LOSS, bool FULL>
__global__ void __launch_bounds__(32 * (NW + 1), 1) k_dense_loss_grad(const DenseArgs a) {
  constexpr int VEC = Vec16<T>::N;
  constexpr int SLAB = 32 * VEC * V;  // columns per warp slab
  constexpr int G = NW / WPR;         // row groups
  constexpr int RG = RPS / G;         // rows per group per stage
  static_assert(NW % WPR == 0 && RPS % G == 0, "bad tile");
  // rows handled in pairs (one butterfly for two dots, one link pass for two
  // rows when W <= 32)
  constexpr bool PAIR = (RG % 2 == 0);
  constexpr bool kF2 = POLY_K1_FFMA2 && std::is_same<T, float>::value && VEC == 4;
  using VT = typename Vec16<T>::type;

  extern __shared__ __align__(128) unsigned char smem[];
  const int S = a.stages;
  const int64_t lda = a.lda;
  const size_t stage_elems = (size_t)RPS * (size_t)lda;
  T *ring = reinterpret_cast<T *>(smem);
  unsigned char *side = smem + (size_t)S * stage_elems * sizeof(T);
  double *red = reinterpret_cast<double *>(side + (size_t)S * a.side_stride);  // [2][G][RG][WPR]
  double *hred = red + 2 * G * RG * WPR;                                       // [2][G][RG][WPR][2]
  double *sp = hred + 4 * G * RG * WPR;                                        // [3*kMaxW]
  uint64_t *full = reinterpret_cast<uint64_t *>(sp + 3 * kMaxW);
  uint64_t *empty = full + S;
  double *lsum = reinterpret_cast<double *>(empty + S);  // [NW]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t rb = a.n * (int64_t)blockIdx.x / gridDim.x;
  const int64_t re = a.n * (int64_t)(blockIdx.x + 1) / gridDim.x;
  const int nstage = (int)((re - rb + RPS - 1) / RPS);
  const int yoff = 0, ioff = RPS * 8, soff = RPS * 12;  // side layout: y[8B], I'[4B], s'[4B*W]

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1 + 32);
      mbar_init(&empty[s], NW);
    }
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 3 * kMaxW; i += blockDim.x) sp[i] = a.spec[i];
  __syncthreads();

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // A is immutable, so streaming may start before the previous kernel
    // (programmatic dependent launch) has finished.
    const uint64_t pol_first = l2_evict_first_policy(), pol_last = l2_evict_last_policy();
    const int ysz = a.ytype == 2 ? 8 : 4;
    int slot = 0;
    uint32_t eph = 1;  // toggled to 0 when the ring first wraps: wait for phase 0
    for (int st = 0; st < nstage; ++st) {
      if (st >= S) mbar_wait(&empty[slot], eph);
      const int64_t r0 = rb + (int64_t)st * RPS;
      const int rows = (int)min((int64_t)RPS, re - r0);
      if (lane == 0) {
        const uint32_t bytes = (uint32_t)((size_t)rows * lda * sizeof(T));
        mbar_arrive_expect_tx(&full[slot], bytes);
        bulk_g2s(ring + (size_t)slot * stage_elems, (const T *)a.A + r0 * lda, bytes, &full[slot],
                 st < a.keep_stages ? pol_last : pol_first);
      }
      unsigned char *sd = side + (size_t)slot * a.side_stride;
      const unsigned char *yg = (const unsigned char *)a.y + r0 * ysz;
      for (int r = lane; r < rows; r += 32) {
        if (ysz == 8)
          cp_async8(sd + yoff + 8 * r, yg + 8 * r);
        else
          cp_async4(sd + yoff + 8 * r, yg + 4 * r);
      }
      if (a.I_row) {
        for (int r = lane; r < rows; r += 32) cp_async4(sd + ioff + 4 * r, a.I_row + r0 + r);
        const float *sg = a.s_row + r0 * a.W;
        for (int e = lane; e < rows * a.W; e += 32) cp_async4(sd + soff + 4 * e, sg + e);
      }
      cp_async_mbar_arrive(&full[slot]);
      if (++slot == S) {
        slot = 0;
        eph ^= 1u;
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }

  // ------------------------------------------------------------ consumers
  const int cw = warp - 1;
  const int grp = cw / WPR, w = cw % WPR;
  pdl_wait();  // x is written by the previous kernel

  T xr[V][VEC], gacc[V][VEC];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int c0 = w * SLAB + v * 32 * VEC + lane * VEC;
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      xr[v][e] = (c0 + e < a.d) ? (T)a.x[c0 + e] : (T)0;
      gacc[v][e] = (T)0;
    }
  }
  double lacc = 0.0;
  const bool has_rowspec = a.I_row != nullptr;
  int buf = 0;

  const int lane_off = w * SLAB + lane * VEC;  // + v * 32 * VEC
  int slot = 0;
  uint32_t fph = 0;
  for (int st = 0; st < nstage; ++st) {
    mbar_wait(&full[slot], fph);
    const int64_t r0 = rb + (int64_t)st * RPS;
    const int rows = (int)min((int64_t)RPS, re - r0);
    const T *tile = ring + (size_t)slot * stage_elems;
    const unsigned char *sd = side + (size_t)slot * a.side_stride;

    // Row chunks stay in registers between the dot and the axpy when they are
    // few; otherwise they are re-read from the (still resident) smem tile.
    constexpr bool KEEP = V * VEC * RG <= 16;
    T av[KEEP ? RG : 1][V][VEC];
    double zp[RG];
    double pv[PAIR ? RG : 1], zh[PAIR ? RG / 2 : 1];
    (void)av;
    (void)pv;
    (void)zh;
    // a1: partial dot of this warp's slab for each of its rows: fp32 FMA over
    // pairs of 16-byte chunks, fp64 tree over the pairs, fp64 warp sum.
#pragma unroll
    for (int q = 0; q < RG; ++q) {
      const int lr = grp + G * q;
      double p = 0.0;
      if (lr < rows) {
        const T *rowp = tile + (size_t)lr * lda + lane_off;
        T pp[(V + 1) / 2];
        float2 pp2 = make_float2(0.0f, 0.0f);
        (void)pp2;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          T ch[VEC];
          if (FULL)
            unpack<T>(*reinterpret_cast<const VT *>(rowp + v * 32 * VEC), ch);
          else
            load_chunk<T>(rowp - lane_off, lane_off + v * 32 * VEC, a.d, ch);
          if constexpr (kF2) {
            // even and odd elements in the two lanes of a packed FMA chain; the lanes are added after
            // the pair of chunks
            float2 p2 = (v & 1) ? pp2 : make_float2(0.0f, 0.0f);
            p2 = __ffma2_rn(make_float2(ch[0], ch[1]), make_float2(xr[v][0], xr[v][1]), p2);
            p2 = __ffma2_rn(make_float2(ch[2], ch[3]), make_float2(xr[v][2], xr[v][3]), p2);
            pp2 = p2;
            if ((v & 1) || v == V - 1) pp[v >> 1] = p2.x + p2.y;
          } else {
            T pv = (v & 1) ? pp[v >> 1] : (T)0;
#pragma unroll
            for (int e = 0; e < VEC; ++e) pv = fma(ch[e], xr[v][e], pv);
            pp[v >> 1] = pv;
          }
          if (KEEP) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) av[KEEP ? q : 0][v][e] = ch[e];
          }
        }
        double t[(V + 1) / 2];
#pragma unroll
        for (int k = 0; k < (V + 1) / 2; ++k) t[k] = (double)pp[k];
#pragma unroll
        for (int w2 = 1; w2 < (V + 1) / 2; w2 <<= 1)
#pragma unroll
          for (int k = 0; k + w2 < (V + 1) / 2; k += 2 * w2) t[k] += t[k + w2];
        p = t[0];
      }
      if (PAIR)
        pv[q] = p;
      else
        zp[q] = warp_sum(p);
    }
    if (PAIR) {
#pragma unroll
      for (int q = 0; q < RG; q += 2) {
        const double v2 = pair_sum(pv[q], pv[q + 1]);
        zh[q >> 1] = v2;  // this lane's half: row q (lanes 0-15) or q+1 (16-31)
        if (WPR == 1) {
          zp[q] = __shfl_sync(0xffffffffu, v2, 0);
          zp[q + 1] = __shfl_sync(0xffffffffu, v2, 16);
        }
      }
    }
    if (WPR > 1) {
      double *rb2 = red + (size_t)buf * G * RG * WPR + (size_t)grp * RG * WPR;
      if (PAIR) {
        // lanes 0 and 16 hold this warp's partials of rows q and q+1
        if ((lane & 15) == 0) {
#pragma unroll
          for (int q = 0; q < RG; q += 2) rb2[(q + (lane >> 4)) * WPR + w] = zh[q >> 1];
        }
      } else if (lane == 0) {
#pragma unroll
        for (int q = 0; q < RG; ++q) rb2[q * WPR + w] = zp[q];
      }
      named_bar_sync(1 + grp, 32 * WPR);
      if (PAIR && a.mode == 0 && a.W <= 32) {  // the pair link: each half-warp needs only its row's z
#pragma unroll
        for (int q = 0; q < RG; q += 2) {
          const int qq = q + (lane >> 4);
          double z = 0.0;
#pragma unroll
          for (int k = 0; k < WPR; ++k) z += rb2[qq * WPR + k];
          zh[q >> 1] = z;
        }
      } else {
#pragma unroll
        for (int q = 0; q < RG; ++q) {
          double z = 0.0;
#pragma unroll
          for (int k = 0; k < WPR; ++k) z += rb2[q * WPR + k];
          zp[q] = z;
        }
      }
      buf ^= 1;
    }
    // a2-a4
    if (PAIR && a.mode == 0 && a.W <= 32) {
      // two rows per link: lanes 0-15 row q, lanes 16-31 row q+1; with WPR > 1
      // the group's warps split the bins (link_partial_pair) and exchange the
      // partial sums through shared memory (a second named barrier)
      constexpr int DEG = std::is_same<T, double>::value ? 13 : POLY_EXP_DEG32;
      double *hb = hred + ((size_t)(buf ^ 1) * G + grp) * RG * WPR * 2;  // (buf flipped after the z exchange)
      constexpr bool SPLIT = WPR > 1 && POLY_K1_LINK_SPLIT;
      if (SPLIT) {
#pragma unroll
        for (int q = 0; q < RG; q += 2) {
          const int h = lane >> 4;
          const int lr = grp + G * (q + h);
          const bool valid = lr < rows;
          const float *srow = (valid && has_rowspec) ? (const float *)(sd + soff) + lr * a.W : nullptr;
          double hs, Hs;
          link_partial_pair<LOSS, DEG, WPR>(sp, a.W, a.relu, valid ? zh[q >> 1] : 0.0, srow, w, &hs, &Hs);
          if ((lane & 15) == 0) {
            hb[((q + h) * WPR + w) * 2] = hs;
            if (LOSS) hb[((q + h) * WPR + w) * 2 + 1] = Hs;
          }
        }
        named_bar_sync(1 + grp, 32 * WPR);
      }
#pragma unroll
      for (int q = 0; q < RG; q += 2) {
        const int h = lane >> 4;
        const int lr = grp + G * (q + h);
        const bool valid = lr < rows;
        const double yv = valid ? load_y(sd + yoff, a.ytype, lr) : 0.0;
        const double Ii = (valid && has_rowspec) ? (double)((const float *)(sd + ioff))[lr] : a.I_bar;
        const float *srow = (valid && has_rowspec) ? (const float *)(sd + soff) + lr * a.W : nullptr;
        double rh;
        if (SPLIT) {  // the row's partial sums over the group's warps, in warp order
          double hs = 0.0, Hs = 0.0;
#pragma unroll
          for (int k = 0; k < WPR; ++k) {
            hs += hb[((q + h) * WPR + k) * 2];
            if (LOSS) Hs += hb[((q + h) * WPR + k) * 2 + 1];
          }
          const double zq = valid ? zh[q >> 1] : 0.0;
          if (LOSS) {  // both halves' terms land on lane 0 (the lane whose lacc is kept)
            const double lt = (valid && w == 0) ? yv * zq - Ii * Hs : 0.0;
            const double lo = __shfl_sync(0xffffffffu, lt, 16);
            if (lane == 0) lacc += lt + lo;
          }
          rh = yv - Ii * hs;
        } else {
          rh = link_exact_pair<LOSS, DEG>(sp, a.W, a.relu, valid ? zh[q >> 1] : 0.0, yv, Ii, srow, valid && w == 0,
                                          &lacc);
        }
        const T r2[2] = {(T)__shfl_sync(0xffffffffu, rh, 0), (T)__shfl_sync(0xffffffffu, rh, 16)};
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int lu = grp + G * (q + u);
          if (lu < rows) {
            const T *rowp = tile + (size_t)lu * lda + lane_off;
#pragma unroll
            for (int v = 0; v < V; ++v) {
              T ch[VEC];
              if (KEEP) {
#pragma unroll
                for (int e = 0; e < VEC; ++e) ch[e] = av[KEEP ? q + u : 0][v][e];
              } else if (FULL) {
                unpack<T>(*reinterpret_cast<const VT *>(rowp + v * 32 * VEC), ch);
              } else {
                load_chunk<T>(rowp - lane_off, lane_off + v * 32 * VEC, a.d, ch);
              }
              if constexpr (kF2) {
                axpy4_f32x2(gacc[v], r2[u], ch);
              } else {
#pragma unroll
                for (int e = 0; e < VEC; ++e) gacc[v][e] = fma(r2[u], ch[e], gacc[v][e]);
              }
            }
          }
        }
      }
    } else
#pragma unroll
    for (int q = 0; q < RG; ++q) {
      const int lr = grp + G * q;
      if (lr < rows) {
        const double yv = load_y(sd + yoff, a.ytype, lr);
        const double Ii = has_rowspec ? (double)((const float *)(sd + ioff))[lr] : a.I_bar;
        const float *srow = has_rowspec ? (const float *)(sd + soff) + lr * a.W : nullptr;
        const double r =
            a.mode == 0
                ? link_exact<LOSS, std::is_same<T, double>::value ? 13 : POLY_EXP_DEG32>(sp, a.W, a.relu, zp[q], yv,
                                                                           Ii, srow, w == 0, &lacc)
                : row_residual<LOSS>(sp, a.W, a.relu, zp[q], yv, Ii, srow, w == 0, &lacc, a.mode);
        const T rt = (T)r;
        const T *rowp = tile + (size_t)lr * lda + lane_off;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          T ch[VEC];
          if (KEEP) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) ch[e] = av[KEEP ? q : 0][v][e];
          } else if (FULL) {
            unpack<T>(*reinterpret_cast<const VT *>(rowp + v * 32 * VEC), ch);
          } else {
            load_chunk<T>(rowp - lane_off, lane_off + v * 32 * VEC, a.d, ch);
          }
          if constexpr (kF2) {
            axpy4_f32x2(gacc[v], rt, ch);
          } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) gacc[v][e] = fma(rt, ch[e], gacc[v][e]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (++slot == S) {
      slot = 0;
      fph ^= 1u;
    }
  }

  // ------------------------------------------- per-CTA partial (fixed order)
  named_bar_sync(15, 32 * NW);  // every consumer is done with the ring
  T *gred = ring;               // [G][d]
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int c0 = w * SLAB + v * 32 * VEC + lane * VEC;
#pragma unroll
    for (int e = 0; e < VEC; ++e)
      if (c0 + e < a.d) gred[(size_t)grp * a.d + c0 + e] = gacc[v][e];
  }
  if (lane == 0) lsum[cw] = lacc;
  named_bar_sync(15, 32 * NW);
  const int t = threadIdx.x - 32;
  double *outp = a.partials + (size_t)blockIdx.x * a.d;
  for (int c = t; c < a.d; c += 32 * NW) {
    double acc = 0.0;
#pragma unroll 4
    for (int g = 0; g < G; ++g) acc += (double)gred[(size_t)g * a.d + c];
    outp[c] = acc;
  }
  if (t == 0) {
    double l = 0.0;
    for (int k = 0; k < NW; ++k) l += lsum[k];
    a.loss_partials[blockIdx.x] = l;
  }
  pdl_trigger();
}

// K8 — read-only streaming ceiling: K1's producer (the same bulk copies into
// the same ring, the same stages and grid) with consumers that only wait for
// each stage and release it.  Times the bytes K1 must move with no math;
// bench.py reports it beside K1.
__global__ void __launch_bounds__(64, 1) k_stream_probe(const void *A, int64_t row_bytes, int64_t n,
                                                        int32_t rps, int32_t stages) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int S = stages;
  const size_t stage_bytes = (size_t)rps * row_bytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)S * stage_bytes);
  uint64_t *empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t rb = n * (int64_t)blockIdx.x / gridDim.x;
  const int64_t re = n * (int64_t)(blockIdx.x + 1) / gridDim.x;
  const int nstage = (int)((re - rb + rps - 1) / rps);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      int slot = 0;
      uint32_t eph = 1;
      for (int st = 0; st < nstage; ++st) {
        if (st >= S) mbar_wait(&empty[slot], eph);
        const int64_t r0 = rb + (int64_t)st * rps;
        const uint32_t bytes = (uint32_t)(min((int64_t)rps, re - r0) * row_bytes);
        mbar_arrive_expect_tx(&full[slot], bytes);
        bulk_g2s(smem + (size_t)slot * stage_bytes, (const unsigned char *)A + r0 * row_bytes, bytes,
                 &full[slot], pol);
        if (++slot == S) {
          slot = 0;
          eph ^= 1u;
        }
      }
    }
    return;
  }
  int slot = 0;
  uint32_t fph = 0;
  for (int st = 0; st < nstage; ++st) {
    mbar_wait(&full[slot], fph);
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (++slot == S) {
      slot = 0;
      fph ^= 1u;
    }
  }
}

}  // namespace poly
