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
// B200 mapping: ONE thread-block cluster of CL CTAs does the whole projection
// — Dykstra, bisection and every FISTA iteration — with the image split into
// CL row bands.  Each CTA keeps its band's prox input z, duals u (horizontal,
// vertical), momentum duals w, the primal x and the extrapolated primal xw in
// shared memory (fp64, 7 arrays); band edges are read from the neighbour
// CTAs' shared memory (DSMEM) and every reduction (||Δx||, ||x||, TV) is
// summed over the cluster in a fixed order, so all CTAs take identical branch
// decisions.  Dykstra's state (z_k, p, q) lives in global memory (L2).  Two
// cluster barriers per FISTA iteration; no kernel launches inside.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace poly {

namespace cg = cooperative_groups;

constexpr int kTvThreads = 512;
constexpr int kTvMaxCL = 16;

struct TvArgs {
  const double *v;     // [d] point to project
  double *out;         // [d] P_X(v)
  double *zk, *p, *q;  // [d] Dykstra state (global, L2-resident)
  int32_t s;           // image side, d = s*s
  int32_t nonneg;      // 1: X1 ∩ X2 by Dykstra; 0: X1 only
  double tau, tv_tol, rtol, tol;
  int32_t max_it, max_outer;
  int32_t *stats;      // optional [3]: Dykstra sweeps, bisection steps, FISTA iterations (totals)
  SolveState *state;   // optional: non-finite flag (bad = -2) for the solver
};

struct TvBand {
  int s, r0, r1, npx, rank, CL;
  double *z, *uh, *uv, *wh, *wv, *x, *xw;  // [npx] band arrays (shared)
  double *red;                             // [2][4] this CTA's cluster-reduction slots
  double *wsum;                            // [warps * 4]
  double *tot;                             // [4] reduced totals
  int parity;
};

__device__ __forceinline__ int band_r0(int rank, int s, int CL) { return rank * s / CL; }

// Sum NV per-thread values over the CTA, then over the cluster: warp 0's lane
// r fetches rank r's partials (one DSMEM round trip) and a butterfly adds
// them — the same instruction sequence on the same inputs in every CTA, so
// all CTAs receive identical totals.  The partial slots alternate between
// two buffers, so one cluster barrier per reduction suffices: a CTA can only
// rewrite a buffer after every CTA passed the barrier of the reduction in
// between, i.e. after all reads of it.
template <int NV>
__device__ __forceinline__ void cluster_sum(cg::cluster_group &cl, TvBand &b, double *v) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double *slot = b.red + 4 * b.parity;
  b.parity ^= 1;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double t = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) b.wsum[warp * 4 + k] = t;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += b.wsum[w * 4 + threadIdx.x];
    slot[threadIdx.x] = t;
  }
  cl.sync();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double t = lane < b.CL ? cl.map_shared_rank(slot, lane)[k] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0) b.tot[k] = t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = b.tot[k];
  __syncthreads();  // b.tot / b.wsum are rewritten by the next reduction
}

// ||x||_TV of the band-distributed image in b.x (forward differences; the
// vertical difference of a band's last row uses the next band's first row).
__device__ double tv_norm_x(cg::cluster_group &cl, TvBand &b) {
  const double *next_x = b.rank + 1 < b.CL ? cl.map_shared_rank(b.x, b.rank + 1) : nullptr;
  double acc[1] = {0.0};
  for (int i = threadIdx.x; i < b.npx; i += blockDim.x) {
    const int lr = i / b.s, c = i - lr * b.s;
    if (c + 1 < b.s) acc[0] += fabs(b.x[i + 1] - b.x[i]);
    if (b.r0 + lr + 1 < b.s) {
      const double below = (lr + 1 < b.r1 - b.r0) ? b.x[i + b.s] : next_x[c];
      acc[0] += fabs(below - b.x[i]);
    }
  }
  cluster_sum<1>(cl, b, acc);
  return acc[0];
}

// TV prox of b.z with parameter lam (FISTA on the dual, oracle_prox_tv's
// iteration); leaves x = z - Dᵀu in b.x.  Returns the FISTA iterations.
__device__ int tv_prox(cg::cluster_group &cl, TvBand &b, double lam, double rtol, int max_it) {
  const int s = b.s;
  for (int i = threadIdx.x; i < b.npx; i += blockDim.x) {
    b.uh[i] = b.uv[i] = b.wh[i] = b.wv[i] = 0.0;
    b.x[i] = b.z[i];
  }
  cl.sync();
  if (!(lam > 0.0)) return 0;
  const double hl = 0.5 * lam;
  const int prev_off = b.rank > 0 ? (b.r0 - band_r0(b.rank - 1, s, b.CL) - 1) * s : 0;
  const double *prev_wv = b.rank > 0 ? cl.map_shared_rank(b.wv, b.rank - 1) : nullptr;
  const double *prev_uv = b.rank > 0 ? cl.map_shared_rank(b.uv, b.rank - 1) : nullptr;
  const double *next_xw = b.rank + 1 < b.CL ? cl.map_shared_rank(b.xw, b.rank + 1) : nullptr;
  const int i0r = (int)threadIdx.x / s, i0c = (int)threadIdx.x - i0r * s;
  const int st_r = (int)blockDim.x / s, st_c = (int)blockDim.x - st_r * s;  // pixel stride as (rows, cols)
  // this thread's last pixel (pixels i = tid + k * blockDim; at most one per row
  // since s <= blockDim for every supported band)
  const int last_i = (int)threadIdx.x < b.npx
                         ? (int)threadIdx.x + ((b.npx - 1 - (int)threadIdx.x) / (int)blockDim.x) * (int)blockDim.x
                         : -1;
  const int last_r = last_i >= 0 ? last_i / s : -1, last_c = last_i >= 0 ? last_i - last_r * s : 0;
  double t = 1.0;
  int it = 1;
  for (;; ++it) {
    // phase A: x(u) = z - Dᵀu (the oracle's primal after iteration it-1) and
    // xw = z - Dᵀw; change of x against the previous primal
    double acc[2] = {0.0, 0.0};
    // the band's first row needs the previous band's last-row duals (DSMEM):
    // issued first, used last (pixels walked in reverse)
    double hwv = 0.0, huv = 0.0;
    if (i0r == 0 && b.rank > 0) hwv = prev_wv[prev_off + i0c], huv = prev_uv[prev_off + i0c];
    for (int i = last_i, lr = last_r, c = last_c; i >= (int)threadIdx.x; i -= blockDim.x) {
      const int r = b.r0 + lr;
      double dw = 0.0, du = 0.0;
      if (c + 1 < s) dw -= b.wh[i], du -= b.uh[i];
      if (c > 0) dw += b.wh[i - 1], du += b.uh[i - 1];
      if (r + 1 < s) dw -= b.wv[i], du -= b.uv[i];
      if (r > 0) {
        if (lr > 0) dw += b.wv[i - s], du += b.uv[i - s];
        else dw += hwv, du += huv;
      }
      const double xn = b.z[i] - du;
      b.xw[i] = b.z[i] - dw;
      const double dx = xn - b.x[i];
      acc[0] += dx * dx;
      acc[1] += xn * xn;
      b.x[i] = xn;
      c -= st_c, lr -= st_r;
      if (c < 0) c += s, --lr;
    }
    cluster_sum<2>(cl, b, acc);  // also publishes xw to the band above
    if ((it > 1 && sqrt(acc[0]) <= rtol * sqrt(acc[1])) || it > max_it) break;
    // phase B: u+ = clip(w + D xw / 8, ±λ/2); w = u+ + ((t-1)/t+)(u+ - u)
    const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
    const double beta = (t - 1.0) / tn;
    t = tn;
    // the band's last row needs the next band's first-row xw (DSMEM): issued
    // first, used last (pixels walked forward)
    const double hxw = (last_r == b.r1 - b.r0 - 1 && next_xw) ? next_xw[last_c] : 0.0;
    for (int i = threadIdx.x, lr = i0r, c = i0c; i < b.npx; i += blockDim.x) {
      const int r = b.r0 + lr;
      if (c + 1 < s) {
        const double un = fmin(hl, fmax(-hl, b.wh[i] + (b.xw[i + 1] - b.xw[i]) / 8.0));
        b.wh[i] = un + beta * (un - b.uh[i]);
        b.uh[i] = un;
      }
      if (r + 1 < s) {
        const double below = (lr + 1 < b.r1 - b.r0) ? b.xw[i + s] : hxw;
        const double un = fmin(hl, fmax(-hl, b.wv[i] + (below - b.xw[i]) / 8.0));
        b.wv[i] = un + beta * (un - b.uv[i]);
        b.uv[i] = un;
      }
      c += st_c, lr += st_r;
      if (c >= s) c -= s, ++lr;
    }
    cl.sync();  // duals complete before the next phase A reads the neighbours'
  }
  return it - 1;
}

// P_X1 of the band input b.z into b.x (oracle_project_tv): b.z itself when
// its TV is <= τ, else the prox with λ bracketed and bisected.
__device__ void tv_project_ball(cg::cluster_group &cl, TvBand &b, const TvArgs &a,
                                int *n_bis, int *n_fista) {
  for (int i = threadIdx.x; i < b.npx; i += blockDim.x) b.x[i] = b.z[i];
  cl.sync();
  if (tv_norm_x(cl, b) <= a.tau) return;
  double lo = 0.0, hi = 1.0;
  for (int g = 0; g < 200; ++g) {
    *n_fista += tv_prox(cl, b, hi, a.rtol, a.max_it);
    if (tv_norm_x(cl, b) <= a.tau) break;
    lo = hi;
    hi *= 2.0;
  }
  for (int st = 1; st <= 60; ++st) {
    const double lam = 0.5 * (lo + hi);
    *n_fista += tv_prox(cl, b, lam, a.rtol, a.max_it);
    ++*n_bis;
    const double tv = tv_norm_x(cl, b);
    if (fabs(tv - a.tau) <= a.tv_tol) break;
    if (tv > a.tau) lo = lam;
    else hi = lam;
  }
}

__global__ void __launch_bounds__(kTvThreads, 1) k_tv_project(const TvArgs a) {
  extern __shared__ __align__(16) double tsm[];
  cg::cluster_group cl = cg::this_cluster();
  TvBand b;
  b.s = a.s;
  b.CL = (int)cl.num_blocks();
  b.rank = (int)cl.block_rank();
  b.r0 = band_r0(b.rank, a.s, b.CL);
  b.r1 = band_r0(b.rank + 1, a.s, b.CL);
  b.npx = (b.r1 - b.r0) * a.s;
  const int cap = ((a.s + b.CL - 1) / b.CL) * a.s;  // largest band
  b.z = tsm;
  b.uh = b.z + cap;
  b.uv = b.uh + cap;
  b.wh = b.uv + cap;
  b.wv = b.wh + cap;
  b.x = b.wv + cap;
  b.xw = b.x + cap;
  b.red = b.xw + cap;
  b.tot = b.red + 8;
  b.wsum = b.tot + 4;
  b.parity = 0;
  pdl_wait();  // v is written by the previous kernel
  pdl_trigger();
  const int64_t g0 = (int64_t)b.r0 * a.s;
  int n_bis = 0, n_fista = 0, sweeps = 0;
  if (!a.nonneg) {
    for (int i = threadIdx.x; i < b.npx; i += blockDim.x) b.z[i] = a.v[g0 + i];
    tv_project_ball(cl, b, a, &n_bis, &n_fista);
    for (int i = threadIdx.x; i < b.npx; i += blockDim.x) a.out[g0 + i] = b.x[i];
  } else {
    // Dykstra: z_0 = v, p_0 = q_0 = 0
    for (int i = threadIdx.x; i < b.npx; i += blockDim.x) {
      a.zk[g0 + i] = a.v[g0 + i];
      a.p[g0 + i] = 0.0;
      a.q[g0 + i] = 0.0;
    }
    for (sweeps = 1; sweeps <= a.max_outer; ++sweeps) {
      for (int i = threadIdx.x; i < b.npx; i += blockDim.x) b.z[i] = a.zk[g0 + i] + a.p[g0 + i];
      tv_project_ball(cl, b, a, &n_bis, &n_fista);  // y_k in b.x
      double acc[1] = {0.0};
      for (int i = threadIdx.x; i < b.npx; i += blockDim.x) {
        const double zk = a.zk[g0 + i], y = b.x[i];
        const double pn = zk + a.p[g0 + i] - y;
        const double sq = y + a.q[g0 + i];
        const double zn = sq > 0.0 ? sq : 0.0;
        a.p[g0 + i] = pn;
        a.q[g0 + i] = sq - zn;
        acc[0] += (zn - zk) * (zn - zk);
        a.zk[g0 + i] = zn;
      }
      cluster_sum<1>(cl, b, acc);
      if (sqrt(acc[0]) <= a.tol) break;
    }
    if (sweeps > a.max_outer) sweeps = a.max_outer;
    for (int i = threadIdx.x; i < b.npx; i += blockDim.x) a.out[g0 + i] = a.zk[g0 + i];
  }
  if (b.rank == 0 && threadIdx.x == 0) {
    if (a.stats) {
      a.stats[0] += sweeps;
      a.stats[1] += n_bis;
      a.stats[2] += n_fista;
    }
  }
}

}  // namespace poly
