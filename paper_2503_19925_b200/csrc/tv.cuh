// NEXT-2 — projection onto the paper's CT constraint set X = X1 ∩ X2,
// X1 = {||x||_TV <= τ}, X2 = R_+^d, for an s x s image
// (row-major), as the paper computes it:
//   P_X1(z): the TV prox x̄ = argmin ||x - z||^2 + λ||x||_TV (Eq.
//            TV-regularization) with λ binary-searched
//            until | ||x̄||_TV - τ | <= tv_tol (0.01 in the paper);
//   P_X:     Dykstra's algorithm (Eq. projection-intersection,
//            PAPER.md:1265-1274) until ||z_{k+1} - z_k||_2 <= tol (1e-4).
// Readings R21: anisotropic TV with forward differences; prox by
// FISTA on the dual (x = z - Dᵀu, |u| <= λ/2, step 1/8), stopped at a relative
// primal change <= rtol; λ bracketed from 1 by doubling, then bisected.
//
// B200 mapping: ONE thread-block cluster of CL CTAs runs the whole projection
// — Dykstra, bisection and every FISTA iteration — on the device.  The image
// is split into CL row bands; inside a band warp w owns image row r0 + w and
// lane t owns the PPL consecutive pixels t·PPL .. t·PPL+PPL-1 of that row.  A
// thread keeps its pixels' duals (uh, uv), momentum duals (wh, wv) and primal
// x in REGISTERS (the prox input z in its own shared-memory row); only what
// crosses a thread boundary moves:
// the left neighbour in the row by a warp shuffle, rows above/below through
// shared-memory rows (at band edges the neighbour CTA's rows over DSMEM).
// Reductions (||Δx||, ||x||, TV, the Dykstra step) are summed over the cluster
// in a fixed order, so every CTA takes the same branches.  Dykstra's state
// (z_k, p, q) lives in global memory (L2).  Two cluster barriers per FISTA
// iteration; no kernel launches inside the projection.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace poly {

namespace cg = cooperative_groups;

constexpr int kTvMaxCL = 16;
constexpr int kTvMaxRows = 16;   // image rows per band (one warp each)
constexpr int kTvMaxSide = 256;  // PPL <= 8
constexpr int kTvThreads = 32 * kTvMaxRows;

struct TvArgs {
  const double *v;     // [d] point to project
  double *out;         // [d] P_X(v) (may alias v)
  double *zk, *p, *q;  // [d] Dykstra state (global, L2-resident)
  int32_t s;           // image side, d = s*s
  int32_t nonneg;      // 1: X1 ∩ X2 by Dykstra; 0: X1 only
  double tau, tv_tol, rtol, tol;
  int32_t max_it, max_outer;
  int32_t *stats;      // optional [3]: Dykstra sweeps, bisection steps, FISTA iterations (totals)
};

__host__ __device__ __forceinline__ int band_r0(int rank, int s, int CL) { return rank * s / CL; }

// pixels per lane for a side (a warp spans a row)
__host__ __device__ inline int tv_ppl(int s) { return s <= 32 ? 1 : s <= 64 ? 2 : s <= 128 ? 4 : 8; }

// Per-CTA context: geometry, the published rows, reduction scratch.
// Shared rows are padded by one double per eight (element c at sw(c)): lane t
// touching element t*PPL + k then hits distinct banks within each half-warp.
__host__ __device__ __forceinline__ int sw(int c) { return c + (c >> 3); }
__host__ __device__ __forceinline__ int tv_row_stride(int s) { return s + (s >> 3) + 1; }

struct TvCtx {
  int s, rs, r0, nrow, rank, CL, row, c0;  // rs: padded row stride; c0 = lane * PPL
  bool active;                         // this warp owns an image row of the band
  double *pub_a, *pub_b, *pub_c;       // [kTvMaxRows][s] shared rows: xw | x, wv, uv
  double *zrow;                        // [kTvMaxRows][s] the prox input z (this CTA's rows)
  double *red, *tot, *wsum;            // [2][4], [4] (unused), [warps][4]
  int parity;
};

// Sum NV per-thread values over the CTA, then over the cluster: warp 0's lane
// r fetches rank r's partials (one DSMEM round trip) and a butterfly adds
// them — the same instruction sequence on the same inputs in every CTA, so
// all CTAs receive identical totals.  Partial slots alternate between two
// buffers, so one cluster barrier per reduction suffices: a CTA can rewrite a
// buffer only after every CTA passed the barrier of the reduction in between.
// Cluster barrier with release/acquire at cluster scope (the cooperative
// groups call also issues a GPU-scope MEMBAR, which showed up as the top
// stall of this kernel).
__device__ __forceinline__ void cluster_bar() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

template <int NV>
__device__ __forceinline__ void cluster_sum(cg::cluster_group &cl, TvCtx &t, double *v) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double *slot = t.red + 4 * t.parity;
  t.parity ^= 1;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double a = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) t.wsum[warp * 4 + k] = a;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double a = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a += t.wsum[w * 4 + threadIdx.x];
    slot[threadIdx.x] = a;
  }
  cluster_bar();
  // every warp sums the CL slots itself (lane r reads rank r): no further
  // CTA barrier; all warps of all CTAs compute the same butterfly
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double a = lane < t.CL ? cl.map_shared_rank(slot, lane)[k] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    v[k] = a;
  }
}

// The published row below / above this warp's row: the neighbour warp's row
// in this CTA, or at the band edge the neighbour CTA's row (DSMEM).
__device__ __forceinline__ const double *row_below(cg::cluster_group &cl, const TvCtx &t,
                                                   const double *pub) {
  const int w = threadIdx.x >> 5;
  if (w + 1 < t.nrow) return pub + (size_t)(w + 1) * t.rs;
  return cl.map_shared_rank(pub, t.rank + 1);
}
__device__ __forceinline__ const double *row_above(cg::cluster_group &cl, const TvCtx &t,
                                                   const double *pub) {
  const int w = threadIdx.x >> 5;
  if (w > 0) return pub + (size_t)(w - 1) * t.rs;
  const int prev_rows = t.r0 - band_r0(t.rank - 1, t.s, t.CL);
  return cl.map_shared_rank(pub, t.rank - 1) + (size_t)(prev_rows - 1) * t.rs;
}

// ||x||_TV (forward differences) of the register-resident image.
template <int PPL>
__device__ double tv_norm_x(cg::cluster_group &cl, TvCtx &t, const double (&x)[PPL]) {
  const int w = threadIdx.x >> 5;
  if (t.active) {
#pragma unroll
    for (int k = 0; k < PPL; ++k)
      if (t.c0 + k < t.s) t.pub_a[(size_t)w * t.rs + sw(t.c0 + k)] = x[k];
  }
  cluster_bar();  // rows published cluster-wide
  double acc[1] = {0.0};
  if (t.active) {
    const double *mine = t.pub_a + (size_t)w * t.rs;
    const bool has_below = t.row + 1 < t.s;
    const double *bel = has_below ? row_below(cl, t, t.pub_a) : nullptr;
#pragma unroll
    for (int k = 0; k < PPL; ++k) {
      const int c = t.c0 + k;
      if (c < t.s) {
        if (c + 1 < t.s) acc[0] += fabs(mine[sw(c + 1)] - x[k]);
        if (has_below) acc[0] += fabs(bel[sw(c)] - x[k]);
      }
    }
  }
  cluster_sum<1>(cl, t, acc);  // also orders these reads before pub_a is reused
  return acc[0];
}

// TV prox of the shared-memory rows z with parameter lam (FISTA on the dual,
// oracle_prox_tv's iteration): x = z - Dᵀu on return.  Returns the FISTA
// iterations.
template <int PPL>
__device__ int tv_prox(cg::cluster_group &cl, TvCtx &t, double (&x)[PPL], double lam, double rtol,
                       int max_it) {
  double uh[PPL], uv[PPL], wh[PPL], wv[PPL];
  const int w = threadIdx.x >> 5;
  const double *z = t.zrow + (size_t)w * t.rs;  // this warp's row of z (shared)
#pragma unroll
  for (int k = 0; k < PPL; ++k) {
    uh[k] = uv[k] = wh[k] = wv[k] = 0.0;
    x[k] = (t.active && t.c0 + k < t.s) ? z[sw(t.c0 + k)] : 0.0;
  }
  if (!(lam > 0.0)) return 0;
  const double hl = 0.5 * lam;
  const bool has_above = t.active && t.row > 0, has_below = t.active && t.row + 1 < t.s;
  double *mine_a = t.pub_a + (size_t)w * t.rs;
  double *mine_b = t.pub_b + (size_t)w * t.rs, *mine_c = t.pub_c + (size_t)w * t.rs;
  if (t.active) {  // published vertical duals start at 0
#pragma unroll
    for (int k = 0; k < PPL; ++k)
      if (t.c0 + k < t.s) mine_b[sw(t.c0 + k)] = mine_c[sw(t.c0 + k)] = 0.0;
  }
  cluster_bar();
  const double *ab_w = has_above ? row_above(cl, t, t.pub_b) : nullptr;
  const double *ab_u = has_above ? row_above(cl, t, t.pub_c) : nullptr;
  const double *bel_xw = has_below ? row_below(cl, t, t.pub_a) : nullptr;
  double tk = 1.0;
  int it = 1;
  for (;; ++it) {
    // phase A: x(u) = z - Dᵀu (the oracle's primal after iteration it-1) and
    // xw = z - Dᵀw, published for phase B (own row and the row above)
    const double whl = __shfl_up_sync(0xffffffffu, wh[PPL - 1], 1);  // left neighbour's last
    const double uhl = __shfl_up_sync(0xffffffffu, uh[PPL - 1], 1);
    double acc[2] = {0.0, 0.0};
    if (t.active) {
#pragma unroll
      for (int k = 0; k < PPL; ++k) {
        const int c = t.c0 + k;
        if (c < t.s) {
          // uh/wh at c = s-1 and uv/wv at the last image row are never set: 0
          double dw = -wh[k] - wv[k], du = -uh[k] - uv[k];
          if (c > 0) dw += (k > 0 ? wh[k - 1] : whl), du += (k > 0 ? uh[k - 1] : uhl);
          if (has_above) dw += ab_w[sw(c)], du += ab_u[sw(c)];
          const double zk = z[sw(c)];
          const double xn = zk - du;
          const double dx = xn - x[k];
          acc[0] += dx * dx;
          acc[1] += xn * xn;
          x[k] = xn;
          mine_a[sw(c)] = zk - dw;
        }
      }
    }
    cluster_sum<2>(cl, t, acc);  // its cluster barrier publishes xw
    if ((it > 1 && sqrt(acc[0]) <= rtol * sqrt(acc[1])) || it > max_it) break;
    // phase B: u+ = clip(w + D xw / 8, ±λ/2); w = u+ + ((t-1)/t+)(u+ - u);
    // the new vertical duals are published for the row below
    const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * tk * tk));
    const double beta = (tk - 1.0) / tn;
    tk = tn;
    if (t.active) {
#pragma unroll
      for (int k = 0; k < PPL; ++k) {
        const int c = t.c0 + k;
        if (c < t.s) {
          const double xc = mine_a[sw(c)];
          if (c + 1 < t.s) {
            const double un = fmin(hl, fmax(-hl, wh[k] + (mine_a[sw(c + 1)] - xc) / 8.0));
            wh[k] = un + beta * (un - uh[k]);
            uh[k] = un;
          }
          if (has_below) {
            const double un = fmin(hl, fmax(-hl, wv[k] + (bel_xw[sw(c)] - xc) / 8.0));
            wv[k] = un + beta * (un - uv[k]);
            uv[k] = un;
          }
          mine_b[sw(c)] = wv[k];
          mine_c[sw(c)] = uv[k];
        }
      }
    }
    // duals published, and every read of the xw rows done before the next
    // phase A rewrites them
    cluster_bar();
  }
  return it - 1;
}

// P_X1 of z (registers) into x (oracle_project_tv): z itself when its TV is
// <= τ, else the prox with λ bracketed and bisected.
template <int PPL>
__device__ void tv_project_ball(cg::cluster_group &cl, TvCtx &t, const TvArgs &a, double (&x)[PPL],
                                int *n_bis, int *n_fista) {
  const double *z = t.zrow + (size_t)(threadIdx.x >> 5) * t.rs;
#pragma unroll
  for (int k = 0; k < PPL; ++k) x[k] = (t.active && t.c0 + k < t.s) ? z[sw(t.c0 + k)] : 0.0;
  if (tv_norm_x<PPL>(cl, t, x) <= a.tau) return;
  double lo = 0.0, hi = 1.0;
  for (int g = 0; g < 200; ++g) {
    *n_fista += tv_prox<PPL>(cl, t, x, hi, a.rtol, a.max_it);
    if (tv_norm_x<PPL>(cl, t, x) <= a.tau) break;
    lo = hi;
    hi *= 2.0;
  }
  for (int st = 1; st <= 60; ++st) {
    const double lam = 0.5 * (lo + hi);
    *n_fista += tv_prox<PPL>(cl, t, x, lam, a.rtol, a.max_it);
    ++*n_bis;
    const double tv = tv_norm_x<PPL>(cl, t, x);
    if (fabs(tv - a.tau) <= a.tv_tol) break;
    if (tv > a.tau) lo = lam;
    else hi = lam;
  }
}

template <int PPL>
__global__ void __launch_bounds__(kTvThreads, 1) k_tv_project(const TvArgs a) {
  extern __shared__ __align__(16) double tsm[];
  cg::cluster_group cl = cg::this_cluster();
  TvCtx t;
  t.s = a.s;
  t.rs = tv_row_stride(a.s);
  t.CL = (int)cl.num_blocks();
  t.rank = (int)cl.block_rank();
  t.r0 = band_r0(t.rank, a.s, t.CL);
  t.nrow = band_r0(t.rank + 1, a.s, t.CL) - t.r0;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  t.active = w < t.nrow;
  t.row = t.r0 + w;
  t.c0 = lane * PPL;
  t.pub_a = tsm;
  t.pub_b = t.pub_a + (size_t)kTvMaxRows * t.rs;
  t.pub_c = t.pub_b + (size_t)kTvMaxRows * t.rs;
  t.zrow = t.pub_c + (size_t)kTvMaxRows * t.rs;
  t.red = t.zrow + (size_t)kTvMaxRows * t.rs;
  t.tot = t.red + 8;
  t.wsum = t.tot + 4;
  t.parity = 0;
  pdl_wait();  // v is written by the previous kernel
  pdl_trigger();
  const int64_t g0 = (int64_t)t.row * a.s + t.c0;
  bool own[PPL];
#pragma unroll
  for (int k = 0; k < PPL; ++k) own[k] = t.active && t.c0 + k < t.s;
  double x[PPL];
  double *zr = t.zrow + (size_t)w * t.rs;  // this warp's row of z (each thread writes its pixels)
  int n_bis = 0, n_fista = 0, sweeps = 0;
  if (!a.nonneg) {
#pragma unroll
    for (int k = 0; k < PPL; ++k)
      if (own[k]) zr[sw(t.c0 + k)] = a.v[g0 + k];
    tv_project_ball<PPL>(cl, t, a, x, &n_bis, &n_fista);
#pragma unroll
    for (int k = 0; k < PPL; ++k)
      if (own[k]) a.out[g0 + k] = x[k];
  } else {
    // Dykstra: z_0 = v, p_0 = q_0 = 0 (each thread touches only its pixels)
#pragma unroll
    for (int k = 0; k < PPL; ++k)
      if (own[k]) a.zk[g0 + k] = a.v[g0 + k], a.p[g0 + k] = 0.0, a.q[g0 + k] = 0.0;
    for (sweeps = 1; sweeps <= a.max_outer; ++sweeps) {
#pragma unroll
      for (int k = 0; k < PPL; ++k)
        if (own[k]) zr[sw(t.c0 + k)] = a.zk[g0 + k] + a.p[g0 + k];
      tv_project_ball<PPL>(cl, t, a, x, &n_bis, &n_fista);  // y_k in x
      double acc[1] = {0.0};
#pragma unroll
      for (int k = 0; k < PPL; ++k) {
        if (own[k]) {
          const double zk = a.zk[g0 + k], y = x[k];
          const double pn = zk + a.p[g0 + k] - y;
          const double sq = y + a.q[g0 + k];
          const double zn = sq > 0.0 ? sq : 0.0;
          a.p[g0 + k] = pn;
          a.q[g0 + k] = sq - zn;
          acc[0] += (zn - zk) * (zn - zk);
          a.zk[g0 + k] = zn;
        }
      }
      cluster_sum<1>(cl, t, acc);
      if (sqrt(acc[0]) <= a.tol) break;
    }
    if (sweeps > a.max_outer) sweeps = a.max_outer;
#pragma unroll
    for (int k = 0; k < PPL; ++k)
      if (own[k]) a.out[g0 + k] = a.zk[g0 + k];
  }
  if (t.rank == 0 && threadIdx.x == 0 && a.stats) {
    a.stats[0] += sweeps;
    a.stats[1] += n_bis;
    a.stats[2] += n_fista;
  }
  (void)lane;
}

}  // namespace poly
