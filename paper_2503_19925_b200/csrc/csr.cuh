// K4 — CSR loss+gradient for the CT-like sparse system matrix
// (BASELINE.json configs[3]; A nonnegative), two passes:
//
//   K4f k_sell_forward  z_i = Σ_e val_e x[col_e] (fp64) from a SELL-32 copy of
//                       A (32 consecutive rows per slice, lane = row), then
//                       the W-bin link and per-row scalar with 8 lanes per
//                       row (group8_residual: the quantities of K1's
//                       row_residual), r_i stored fp32, ℓ per block.
//   K4b k_csc_backward  g_k = Σ_{i in column k} val_ik r_i  (Aᵀ r)
//                       from a SELL-32 copy of Aᵀ built once at poly_init: a
//                       slice holds 32 consecutive columns, step s of lane t is
//                       the s-th entry (ascending row) of column 32·slice + t,
//                       so each warp-step is one coalesced 256-byte load and
//                       every lane owns its column's sum in registers — no
//                       atomics, fixed summation order (deterministic).
// Both SELL copies are built once at poly_init from the caller's CSR; a
// warp-per-row CSR forward was latency-bound (dependent row_ptr -> col -> x
// loads, 2.0 TB/s in ncu).  A persistent TMA-ring variant of both passes (one
// CTA per SM, 8 consumer warps) was slower (1.5 TB/s): the x / r gathers are
// latency-bound and need the warps of many resident 128-thread CTAs.
//
// Why two passes: a one-pass fused kernel must scatter g[col] += r val for
// every nonzero (red.global at ~1 lane/1.3 cycles per SM, B300_MICROARCH.md
// "Atomics"), which caps the scatter near 140 µs for C4's 30M nonzeros; the
// gather formulation reads the values twice (≈ 2x the algorithmic bytes) but
// streams at HBM rate.
#pragma once

#include "dense.cuh"
#include "finalize.cuh"  // SolveState (the backward's optional step epilogue)

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
  const float *x;         // [d] fp32 copy of the iterate (L1-resident gathers)
  const double *spec;
  float *r;               // [n] residuals r_i (output)
  int32_t mode;
  double *loss_partials;  // [gridDim.x]
  double mu_step;         // != 0: μ_j = μ_0 + j·mu_step (K4tl's geometric bins)
};

// 4 warps per 32-column slice; warp w takes steps w, w+4, w+8, ...; the four
// warps' sums are combined in warp order.
template <typename T>
__global__ void __launch_bounds__(128) k_csc_backward(const CscEnt<T> *__restrict__ ent,
                                                      const int64_t *__restrict__ slice_off,
                                                      int32_t d, const float *__restrict__ r,
                                                      double *__restrict__ g, const int32_t *colmap) {
  __shared__ double part[4][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t s0 = slice_off[blockIdx.x], s1 = slice_off[blockIdx.x + 1];
  const CscEnt<T> *p = ent + s0 * 32 + lane;
  const int64_t len = s1 - s0;
  pdl_wait();  // r is written by the forward pass
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int64_t k = warp;
  // (a marked layout's padding entries carry row -1 and value 0)
  auto rv = [&](int32_t row) { return row >= 0 ? (double)__ldg(r + row) : 0.0; };
  for (; k + 12 < len; k += 16) {
    const CscEnt<T> q0 = p[(k) * 32], q1 = p[(k + 4) * 32], q2 = p[(k + 8) * 32],
                    q3 = p[(k + 12) * 32];
    a0 = fma((double)q0.val, rv(q0.row), a0);
    a1 = fma((double)q1.val, rv(q1.row), a1);
    a2 = fma((double)q2.val, rv(q2.row), a2);
    a3 = fma((double)q3.val, rv(q3.row), a3);
  }
  for (; k < len; k += 4) {
    const CscEnt<T> q = p[k * 32];
    a0 = fma((double)q.val, rv(q.row), a0);
  }
  part[warp][lane] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  if (warp == 0) {
    const int c = colmap ? colmap[blockIdx.x * 32 + lane] : blockIdx.x * 32 + lane;
    const double v = (part[0][lane] + part[1][lane]) + (part[2][lane] + part[3][lane]);
    if (c >= 0 && c < d) g[c] = v;
  }
  pdl_trigger();
}

// link + per-row scalar with a group of 8 lanes per row (bins j = sub, sub+8, ...)
template <bool LOSS>
__device__ __forceinline__ double group8_residual(const double *sp, int W, int relu, double z,
                                                  double yv, double Ii, const float *srow,
                                                  int sub, double *lacc, int mode) {
  const bool neg = relu && z < 0.0;
  const double zc = neg ? 0.0 : z;
  double hs = 0.0, Hs = 0.0, hp = 0.0;
  for (int j = sub; j < W; j += 8) {
    const double sj = srow ? (double)srow[j] : sp[j];
    const double e = (relu || mode == 0) ? exp_nonpos(-sp[kMaxW + j] * zc) : exp(-sp[kMaxW + j] * z);
    hs += sj * e;
    if (mode == 0) {
      if (LOSS) Hs += neg ? sj * z : sj * sp[2 * kMaxW + j] * (1.0 - e);
    } else {
      hp += sj * sp[kMaxW + j] * e;
    }
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    hs += __shfl_xor_sync(0xffffffffu, hs, o);
    if (LOSS && mode == 0) Hs += __shfl_xor_sync(0xffffffffu, Hs, o);
    if (mode != 0) hp += __shfl_xor_sync(0xffffffffu, hp, o);
  }
  double phi, l;
  if (mode == 0) {
    phi = yv - Ii * hs;
    l = yv * z - Ii * Hs;
  } else {
    hp = (relu && !(z > 0.0)) ? 0.0 : -hp;
    const double m = Ii * hs;
    if (mode == 1) {
      phi = 2.0 * (m - yv) * Ii * hp;
      l = (m - yv) * (m - yv);
    } else if (mode == 2) {
      const double rr = m - yv;
      phi = (rr > 0.0 ? 1.0 : (rr < 0.0 ? -1.0 : 0.0)) * Ii * hp;
      l = fabs(rr);
    } else {
      phi = (Ii - yv / hs) * hp;
      l = m - yv * log(m);
    }
  }
  if (LOSS && sub == 0) *lacc += l;
  return phi;
}

// K4f epilogue: z of the slice's 32 rows from the four warps' partials, then
// the link + residual with 8 lanes per row (bins across the group), warp w
// taking rows 8w .. 8w+7 in two rounds of four; every lane runs the group
// reduction (full-mask shuffles), rows past n are evaluated on dummies.
template <bool LOSS>
__device__ __forceinline__ double forward_tail(double (*part)[32], const double *sp,
                                               const CsrFwdArgs &a, int64_t slice) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane & 7;
  double lacc = 0.0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int rr = warp * 8 + h * 4 + (lane >> 3);
    const int64_t row = slice * 32 + rr;
    const bool valid = row < a.n;
    double z = (part[0][rr] + part[1][rr]) + (part[2][rr] + part[3][rr]);
    double yv = 0.0, Ii = a.I_bar;
    const float *srow = nullptr;
    if (valid) {
      if (a.ytype == 0) yv = (double)((const int32_t *)a.y)[row];
      else if (a.ytype == 1) yv = (double)((const float *)a.y)[row];
      else yv = ((const double *)a.y)[row];
      if (a.I_row) {
        Ii = (double)a.I_row[row];
        srow = a.s_row + row * a.W;
      }
    } else {
      z = 0.0;
    }
    double lrow = 0.0;
    const double phi = group8_residual<LOSS>(sp, a.W, a.relu, z, yv, Ii, srow, sub, &lrow, a.mode);
    if (valid) {
      lacc += lrow;
      if (sub == 0) a.r[row] = (float)phi;
    }
  }
  return lacc;
}

// per-block loss partial: warps combined in order (deterministic); reuses part
__device__ __forceinline__ void block_loss(double (*part)[32], double lacc, double *out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  lacc = warp_sum(lacc);
  __syncthreads();
  if (lane == 0) part[0][warp] = lacc;
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = (part[0][0] + part[0][1]) + (part[0][2] + part[0][3]);
}

// the same with nw warps (their partials summed in warp order)
__device__ __forceinline__ void block_loss_n(double (*part)[32], double lacc, double *out, int nw) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  lacc = warp_sum(lacc);
  __syncthreads();
  if (lane == 0) part[0][warp] = lacc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += part[0][w];
    out[blockIdx.x] = t;
  }
}

// K4f on a SELL-32 copy of A (rows as slices): block = 32 consecutive rows,
// warp w takes steps w, w+4, ...; z_i combined in warp order, then lane i of
// warp 0 evaluates row i's link and residual.
template <typename T, bool LOSS>
__global__ void __launch_bounds__(128) k_sell_forward(const CscEnt<T> *__restrict__ ent,
                                                      const int64_t *__restrict__ slice_off,
                                                      const CsrFwdArgs a) {
  __shared__ double sp[3 * kMaxW];
  __shared__ double part[4][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 3 * kMaxW; i += blockDim.x) sp[i] = a.spec[i];
  const int64_t s0 = slice_off[blockIdx.x], s1 = slice_off[blockIdx.x + 1];
  const CscEnt<T> *p = ent + s0 * 32 + lane;
  const int64_t len = s1 - s0;
  pdl_wait();  // x is written by the previous kernel; r is read by the previous backward
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int64_t k = warp;
  for (; k + 12 < len; k += 16) {
    const CscEnt<T> q0 = p[(k) * 32], q1 = p[(k + 4) * 32], q2 = p[(k + 8) * 32],
                    q3 = p[(k + 12) * 32];
    a0 = fma((double)q0.val, (double)__ldg(a.x + q0.row), a0);
    a1 = fma((double)q1.val, (double)__ldg(a.x + q1.row), a1);
    a2 = fma((double)q2.val, (double)__ldg(a.x + q2.row), a2);
    a3 = fma((double)q3.val, (double)__ldg(a.x + q3.row), a3);
  }
  for (; k < len; k += 4) {
    const CscEnt<T> q = p[k * 32];
    a0 = fma((double)q.val, (double)__ldg(a.x + q.row), a0);
  }
  part[warp][lane] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  block_loss(part, forward_tail<LOSS>(part, sp, a, blockIdx.x), a.loss_partials);
  pdl_trigger();
}

// ------------------------------------------------------------------------
// Compact SELL-32 ("SELL16"): the same slices, steps grouped by four; per
// group every lane holds four int16 index deltas (8 B) and four values (16 B
// for fp32), stored as two lane-contiguous arrays — 6 bytes per fp32 entry
// instead of 8, two vector loads per four entries.  Groups are dealt to the
// slice's four warps round-robin (group g to warp g % 4, as the wide form
// deals steps); each warp follows its own delta chain: the first entry of a
// group is relative to the lane's last entry in that warp's previous group,
// the chain starts at base[(slice*4 + w)*32 + lane].  Padding carries delta 0
// and value 0.  Built at poly_init when every delta fits int16 (CT: |Δ| <=
// 13 (side + 1) along a ray; Δrow within a column), else the 8-byte form.
#ifndef POLY_SELL_UNROLL
#define POLY_SELL_UNROLL 4
#endif
constexpr int kSellUnroll = POLY_SELL_UNROLL;  // groups of four steps in flight per warp
#ifndef POLY_SELL_UNROLL_F
#define POLY_SELL_UNROLL_F POLY_SELL_UNROLL
#endif
#ifndef POLY_SELL_UNROLL_B
#define POLY_SELL_UNROLL_B 8  // K4b: 8 groups (32 gathers) in flight per warp, 40 registers (C4 pass 81.4 -> 80.7 us)
#endif
#ifndef POLY_SELL_MINB_F
#define POLY_SELL_MINB_F 12  // forward: 40 registers, 12 blocks per SM (C4 pass 81.8 -> 79.8 us)
#endif
#define POLY_SELL_LB_F 128, POLY_SELL_MINB_F
#ifdef POLY_SELL_MINB_B
#define POLY_SELL_LB_B 128, POLY_SELL_MINB_B
#else
#define POLY_SELL_LB_B 128
#endif

struct Sell16 {
  const short4 *dl;        // [groups * 32]
  const void *val;         // [groups * 32] float4 / 4 doubles
  const int32_t *base;     // [nslices * 4 * 32]
  const int64_t *slice_off;  // [nslices + 1] slice start, in groups of 4 steps
};

template <typename T>
struct Val4;
template <>
struct Val4<float> {
  using type = float4;
  __device__ static float4 load(const void *p, int64_t i) { return __ldcs((const float4 *)p + i); }
};
template <>
struct Val4<double> {
  struct type {
    double x, y, z, w;
  };
  __device__ static type load(const void *p, int64_t i) {
    const double2 *q = (const double2 *)p + 2 * i;
    const double2 a = __ldcs(q), b = __ldcs(q + 1);
    return type{a.x, a.y, b.x, b.y};
  }
};

// One group of four steps: four deltas, four values, four gathers.
template <typename T>
__device__ __forceinline__ void sell16_group(const Sell16 &s, int64_t gi, int32_t &idx,
                                             const float *__restrict__ gv, double &a0, double &a1) {
  const short4 dd = __ldcs(s.dl + gi);
  const auto v = Val4<T>::load(s.val, gi);
  const int32_t i0 = idx + dd.x, i1 = i0 + dd.y, i2 = i1 + dd.z, i3 = i2 + dd.w;
  idx = i3;
  const float g0 = __ldg(gv + i0), g1 = __ldg(gv + i1), g2 = __ldg(gv + i2), g3 = __ldg(gv + i3);
  a0 = fma((double)v.x, (double)g0, a0);
  a1 = fma((double)v.y, (double)g1, a1);
  a0 = fma((double)v.z, (double)g2, a0);
  a1 = fma((double)v.w, (double)g3, a1);
}

// This warp's share of a slice: groups warp, warp+4, ..., UNR groups (4*UNR
// gathers) in flight per iteration.
template <typename T, int UNR>
__device__ __forceinline__ double sell16_dot(const Sell16 &s, int64_t slice, int warp, int lane,
                                             const float *__restrict__ gv) {
  const int64_t o0 = s.slice_off[slice], ng = s.slice_off[slice + 1] - o0;
  int32_t idx = s.base[(slice * 4 + warp) * 32 + lane];
  double a0 = 0.0, a1 = 0.0;
  int64_t g = warp;
  for (; g + 4 * (UNR - 1) < ng; g += 4 * UNR) {
    // loads of all UNR groups first (independent), then the dependent gathers
    short4 dd[UNR];
    typename Val4<T>::type vv[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      dd[u] = __ldcs(s.dl + (o0 + g + 4 * u) * 32 + lane);
      vv[u] = Val4<T>::load(s.val, (o0 + g + 4 * u) * 32 + lane);
    }
    float gg[4 * UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int32_t i0 = idx + dd[u].x, i1 = i0 + dd[u].y, i2 = i1 + dd[u].z, i3 = i2 + dd[u].w;
      idx = i3;
      gg[4 * u] = __ldg(gv + i0), gg[4 * u + 1] = __ldg(gv + i1);
      gg[4 * u + 2] = __ldg(gv + i2), gg[4 * u + 3] = __ldg(gv + i3);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      a0 = fma((double)vv[u].x, (double)gg[4 * u], a0);
      a1 = fma((double)vv[u].y, (double)gg[4 * u + 1], a1);
      a0 = fma((double)vv[u].z, (double)gg[4 * u + 2], a0);
      a1 = fma((double)vv[u].w, (double)gg[4 * u + 3], a1);
    }
  }
  for (; g < ng; g += 4) sell16_group<T>(s, (o0 + g) * 32 + lane, idx, gv, a0, a1);
  return a0 + a1;
}

template <typename T, bool LOSS>
__global__ void __launch_bounds__(POLY_SELL_LB_F) k_sell16_forward(const Sell16 s, int64_t nslices,
                                                             const CsrFwdArgs a) {
  __shared__ double sp[3 * kMaxW];
  __shared__ double part[4][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 3 * kMaxW; i += blockDim.x) sp[i] = a.spec[i];
  pdl_wait();  // x is written by the previous kernel; r is read by the previous backward
  double lacc = 0.0;
  for (int64_t sl = blockIdx.x; sl < nslices; sl += gridDim.x) {  // fixed slice -> block map
    part[warp][lane] = sell16_dot<T, POLY_SELL_UNROLL_F>(s, sl, warp, lane, a.x);
    __syncthreads();
    lacc += forward_tail<LOSS>(part, sp, a, sl);
    __syncthreads();  // part is rewritten by the next slice
  }
  block_loss(part, lacc, a.loss_partials);
  pdl_trigger();
}

// Optional epilogue of the backward for the plain EXACT step on the split
// path (d > 8192, no objective wanted, one rank): each block owns 32 columns
// of g — exactly one k_finalize block — so it forms v = anchor - γ g/n, the
// orthant clamp and the block's ||v - c||² itself, with k_finalize's
// arithmetic (same bits), and k_fin_apply follows directly.
struct StepEpi {
  int32_t on;
  int32_t set;
  double n_norm;
  const double *anchor;
  const double *center;
  SolveState *state;
  double *v_scratch;
  double *block_norm;
};

// warp 0 of a backward block: column sums of slice sl (the four warps'
// partials in warp order) to g, or — with the step epilogue on — v, the
// orthant clamp and the block's ||v - c||²
__device__ __forceinline__ void backward_column_out(double (*part)[32], const StepEpi &e, double *g, int32_t d,
                                                    int64_t sl, int lane, const int32_t *colmap = nullptr) {
  // colmap (tiled slices): the column of each slot, -1 for an empty slot
  const int64_t c = colmap ? (int64_t)colmap[sl * 32 + lane] : sl * 32 + lane;
  const double v = (part[0][lane] + part[1][lane]) + (part[2][lane] + part[3][lane]);
  const bool ok = c >= 0 && c < d;
  if (!e.on) {
    if (ok) g[c] = v;
    return;
  }
  double q = 0.0;
  if (ok) {
    const double gc = v / e.n_norm;
    double vv = e.anchor[c] - e.state->gamma * gc;
    if (e.set == 2 || e.set == 3) vv = vv > 0.0 ? vv : 0.0;
    const double df = (e.set == 1 && e.center) ? vv - e.center[c] : vv;
    q = df * df;
    e.v_scratch[c] = vv;
  }
  q = warp_sum(q);
  if (lane == 0) e.block_norm[sl] = q;
  if (sl == 0 && lane == 0) e.state->loss_cur = 0.0;  // as k_finalize without the objective
}

template <typename T>
__global__ void __launch_bounds__(POLY_SELL_LB_B) k_sell16_backward(const Sell16 s, int64_t nslices,
                                                              int32_t d, const float *__restrict__ r,
                                                              double *__restrict__ g, const StepEpi e,
                                                              const int32_t *colmap) {
  __shared__ double part[4][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  pdl_wait();  // r is written by the forward pass
  for (int64_t sl = blockIdx.x; sl < nslices; sl += gridDim.x) {
    part[warp][lane] = sell16_dot<T, POLY_SELL_UNROLL_B>(s, sl, warp, lane, r);
    __syncthreads();
    if (warp == 0) backward_column_out(part, e, g, d, sl, lane, colmap);
    __syncthreads();
  }
  pdl_trigger();
}

// (poly_init only) SELL -> SELL16.  lens: per-lane entry counts (row lengths
// from row_ptr, or column counts cnt); off16: group offsets of the slices;
// one 128-thread block per slice, warp w packs groups w, w+4, ...
template <typename T>
__global__ void k_sell16_pack(const CscEnt<T> *ent, const int64_t *slice_off, int64_t nslices,
                              const int64_t *row_ptr, const int32_t *cnt, int64_t nlanes,
                              const int64_t *off16, short4 *dl, T *val, int32_t *base,
                              int32_t *overflow) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t sl = blockIdx.x; sl < nslices; sl += gridDim.x) {
    const int64_t o0 = slice_off[sl], len = slice_off[sl + 1] - o0;
    const int64_t g0 = off16[sl], ng = off16[sl + 1] - g0;
    const int64_t li = sl * 32 + lane;
    // marked layout (row_ptr and cnt NULL): every lane spans the slice, padding
    // entries carry row -1 (they become delta 0 / value 0); the chain starts at
    // the warp's first real entry so that padding gathers stay in range
    const bool marked = !row_ptr && !cnt;
    const int64_t mylen = marked ? len : (li < nlanes ? (row_ptr ? row_ptr[li + 1] - row_ptr[li] : (int64_t)cnt[li]) : 0);
    int32_t prev = 0;
    if (marked) {
      bool found = false;
      for (int64_t g = warp; g < ng && !found; g += 4)
        for (int j = 0; j < 4 && !found; ++j) {
          const int64_t k = 4 * g + j;
          if (k < len) {
            const int32_t r = ent[(o0 + k) * 32 + lane].row;
            if (r >= 0) prev = r, found = true;
          }
        }
    } else if (4 * warp < min(mylen, len)) {
      prev = ent[(o0 + 4 * warp) * 32 + lane].row;
    }
    base[(sl * 4 + warp) * 32 + lane] = prev;
    for (int64_t g = warp; g < ng; g += 4) {
      int32_t dd[4];
      T vv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t k = 4 * g + j;
        dd[j] = 0;
        vv[j] = (T)0;
        if (k < mylen) {
          const CscEnt<T> e = ent[(o0 + k) * 32 + lane];
          if (e.row < 0) continue;  // marked padding: delta 0, value 0
          const int64_t dlt = (int64_t)e.row - prev;
          if (dlt < -32768 || dlt > 32767) atomicOr(overflow, 1);
          dd[j] = (int32_t)dlt;
          prev = e.row;
          vv[j] = e.val;
        }
      }
      dl[(g0 + g) * 32 + lane] = make_short4((short)dd[0], (short)dd[1], (short)dd[2], (short)dd[3]);
#pragma unroll
      for (int j = 0; j < 4; ++j) val[((g0 + g) * 32 + lane) * 4 + j] = vv[j];
    }
  }
}

__global__ void k_groups_of(const int64_t *slice_off, int64_t nslices, int64_t *len16) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s <= nslices;
       s += (int64_t)gridDim.x * blockDim.x)
    len16[s] = s < nslices ? (slice_off[s + 1] - slice_off[s] + 3) / 4 : 0;
}

// (poly_init only) Gather locality of a K4f slice: at step k its 32 lanes
// read x at the k-th column of 32 consecutive rows.  When d = s² (an s x s
// image, row-major) the library also keeps the transposed copy of x; for
// each slice it counts the distinct 32-byte fp32 sectors the gathers touch
// under both layouts and marks the slice for the transposed copy when that
// touches fewer (CT rays near 0° / 180° walk along image rows, so adjacent
// rays' k-th pixels are adjacent in the column-major layout).
__device__ __forceinline__ int32_t tr_index(int32_t c, int32_t s) { return (c % s) * s + c / s; }

__global__ void k_slice_layout(const int64_t *row_ptr, const int32_t *col, int64_t n, int32_t s,
                               int64_t nslices, int8_t *use_tr) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t sl = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); sl < nslices;
       sl += nw) {
    const int64_t row = sl * 32 + lane;
    const int64_t e0 = row < n ? row_ptr[row] : 0;
    const int64_t len = row < n ? row_ptr[row + 1] - e0 : 0;
    int64_t mx = len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, (int64_t)__shfl_xor_sync(0xffffffffu, mx, o));
    int64_t c_row = 0, c_tr = 0;
    for (int64_t k = 0; k < mx; ++k) {
      const bool act = k < len;
      const int32_t cc = act ? col[e0 + k] : 0;
      const int32_t a = act ? (cc >> 3) : -1 - lane;
      const int32_t b = act ? (tr_index(cc, s) >> 3) : -1 - lane;
      const unsigned ma = __match_any_sync(0xffffffffu, a), mb = __match_any_sync(0xffffffffu, b);
      c_row += act && (__ffs(ma) - 1) == lane;
      c_tr += act && (__ffs(mb) - 1) == lane;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      c_row += __shfl_xor_sync(0xffffffffu, c_row, o);
      c_tr += __shfl_xor_sync(0xffffffffu, c_tr, o);
    }
    if (lane == 0) use_tr[sl] = c_tr < c_row ? 1 : 0;
  }
}

// (poly_init only) SELL-32 copy of A itself: entry j of row i -> step j,
// lane i % 32; columns of slices marked in use_tr index the transposed copy
// of x (d + tr(col)).
template <typename T>
__global__ void k_sell_rows_fill(const int64_t *row_ptr, const int32_t *col, const T *val,
                                 int64_t n, const int64_t *slice_off, const int8_t *use_tr,
                                 int32_t s, int32_t d, CscEnt<T> *ent) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nw) {
    const int64_t e0 = row_ptr[i], e1 = row_ptr[i + 1];
    const bool tr = use_tr && use_tr[i >> 5];
    CscEnt<T> *dst = ent + slice_off[i >> 5] * 32 + (i & 31);
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      CscEnt<T> q;
      q.row = tr ? d + tr_index(col[e], s) : col[e];
      q.val = val[e];
      dst[(e - e0) * 32] = q;
    }
  }
}

// slice length for row slices: longest row of 32
__global__ void k_row_slice_len(const int64_t *row_ptr, int64_t n, int64_t nslices, int64_t *len) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslices;
       s += (int64_t)gridDim.x * blockDim.x) {
    int64_t m = 0;
    for (int64_t i = 32 * s; i < min(n, 32 * s + 32); ++i) m = max(m, row_ptr[i + 1] - row_ptr[i]);
    len[s] = m;
  }
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

// ---- tiled, block-synchronised SELL-32 of Aᵀ (square images, poly_init only)
// Slices are 4 x 8 pixel tiles (colmap: slot -> column), and the lanes' entry
// chains are re-aligned at every row block of RB rows: within block b every
// lane of slice s has boff[s][b] .. boff[s][b+1] steps (the slice's largest
// count in that block), padded with marked entries (row -1).  For the CT
// matrix a row block is ~15 views, so a warp's 32 gathers stay within a few
// views of r (4.4 instead of 18.8 sectors per request) for
// 12 % padding.
__global__ void k_colblk_count(const int32_t *rows, const int32_t *col, int64_t nnz, int32_t RB, int32_t NBK,
                               int32_t *blkcnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(blkcnt + (int64_t)col[e] * NBK + rows[e] / RB, 1);
}

// per column: exclusive prefix of its block counts (in place into bpre)
__global__ void k_colblk_prefix(const int32_t *blkcnt, int32_t d, int32_t NBK, int32_t *bpre) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < d; c += gridDim.x * blockDim.x) {
    int32_t a = 0;
    for (int b = 0; b < NBK; ++b) {
      bpre[(int64_t)c * NBK + b] = a;
      a += blkcnt[(int64_t)c * NBK + b];
    }
  }
}

// per slice: the step offset of each row block (max count over the lanes) and the length
__global__ void k_slice_blocks(const int32_t *blkcnt, const int32_t *colmap, int32_t nslices, int32_t NBK,
                               int32_t *boff, int64_t *slen) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nslices; s += gridDim.x * blockDim.x) {
    int64_t a = 0;
    for (int b = 0; b < NBK; ++b) {
      int32_t m = 0;
      for (int l = 0; l < 32; ++l) {
        const int32_t c = colmap[s * 32 + l];
        if (c >= 0) m = max(m, blkcnt[(int64_t)c * NBK + b]);
      }
      boff[(int64_t)s * NBK + b] = (int32_t)a;
      a += m;
    }
    slen[s] = a;
  }
}

template <typename T>
__global__ void k_sell_mark(CscEnt<T> *ent, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    CscEnt<T> q;
    q.row = -1;
    q.val = (T)0;
    ent[i] = q;
  }
}

template <typename T>
__global__ void k_sell_fill_sync(const int32_t *sorted_col, const int32_t *perm, const int32_t *rows, const T *val,
                                 const int64_t *colptr, const int32_t *bpre, const int32_t *boff,
                                 const int32_t *slot_of, const int64_t *slice_off, int32_t RB, int32_t NBK,
                                 int64_t nnz, CscEnt<T> *ent) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = sorted_col[k];
    const int32_t e = perm[k];
    const int32_t r = rows[e];
    const int32_t b = r / RB;
    const int64_t j = k - colptr[c] - bpre[(int64_t)c * NBK + b];
    const int32_t slot = slot_of[c];
    const int32_t s = slot >> 5;
    CscEnt<T> q;
    q.row = r;
    q.val = val[e];
    ent[(slice_off[s] + boff[(int64_t)s * NBK + b] + j) * 32 + (slot & 31)] = q;
  }
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
