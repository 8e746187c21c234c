// Matrix-free parallel-beam projector for the CT workload (SURVEY.md §8(f)
// NEXT-4: "a matrix-free Siddon/Joseph projector for CT, which removes the
// 243 MB CSR stream and moves the bound from HBM to ALU").
//
// Geometry (reading R12, gen/ct.py): an N x N image with pixel
// pitch Δ = 1/N, pixel (r, c) centred at (X_c, Y_r) = ((c - N/2)Δ, (r - N/2)Δ);
// ray (k, b), k < V views, b < B bins, is the line {p : p·n_k = t_b} with
// n_k = (cos θ_k, sin θ_k), θ_k = kπ/V and t_b = (b - (B-1)/2)Δ; row i = kB + b
// (axis-aligned views take exact 0/±1 for cos/sin).
// A[i, rN + c] is the length of that line inside pixel (r, c) — the
// Siddon segment length ("fractional contribution of pixel k to
// the line integral") — which for a square pixel is the closed-form chord
//   L(δ) = Δ/max(a,b)          |δ| <= Δ|a-b|/2
//        = (Δ(a+b)/2 - |δ|)/(ab)  Δ|a-b|/2 < |δ| < Δ(a+b)/2
//        = 0                    otherwise,
// with a = |cos θ|, b = |sin θ| and δ the signed distance of the pixel centre
// from the line.  The kernels evaluate it on the fly instead of streaming A:
//   K5f k_pb_forward   one block per view, one thread per ray: image rows are
//                      staged through shared memory (for views with
//                      |sin θ| > |cos θ| the rows of the transposed image, in
//                      which the ray is again "steep"); each ray adds the at
//                      most 3 pixels per row its footprint covers; then the
//                      link and residual per ray (fp64) as K1, r stored fp32.
//   K5b k_pb_backward  one thread per (pixel, half of the views): for every
//                      view the at most 2 bins whose rays cross the pixel,
//                      residuals staged per view chunk in shared memory; the
//                      two halves are added in order (deterministic).
#pragma once

#include "dense.cuh"

namespace poly {

struct PbGeom {
  int32_t N, V, B;
  int32_t v0;          // first view of this handle's rows (row_offset / B)
  int32_t nv;          // views held (n_local / B)
  const double *trig;  // [2V]: cos θ_k, sin θ_k (host libm, θ_k = kπ/V)
};

// chord length / Δ for a pixel whose centre is u pixels (along the frame's
// columns) from the ray's crossing point, a = |cos| >= b = |sin| of the frame:
// plateau 1/a for u a <= p1, ramp (p2 - u a)/(a b) up to p2, 0 beyond —
// written as selects (no branches in the inner loops).
__device__ __forceinline__ float chord(float u, float a, float p1, float p2, float inv_a, float inv_ab) {
  const float da = u * a;
  const float ramp = fmaxf(0.0f, (p2 - da) * inv_ab);
  return da <= p1 ? inv_a : ramp;
}

constexpr int kPbRows = 32;  // image rows staged per chunk in the forward

// z_i for the rays of one view, then the residual (mode EXACT).  x32 holds
// x (row-major) at [0, d) and its transpose at [d, 2d).
template <bool LOSS>
__global__ void __launch_bounds__(512) k_pb_forward(const PbGeom g, const float *__restrict__ x32,
                                                    const CsrFwdArgs a) {
  extern __shared__ __align__(16) float xs[];  // [kPbRows][N]
  __shared__ double sp[3 * kMaxW];
  __shared__ double wl[16];
  const int N = g.N, B = g.B;
  const int kl = blockIdx.x, k = g.v0 + kl;
  const int b = threadIdx.x;
  for (int i = threadIdx.x; i < 3 * kMaxW; i += blockDim.x) sp[i] = a.spec[i];
  const double cth = g.trig[2 * k], sth = g.trig[2 * k + 1];
  const bool steep = fabs(cth) >= fabs(sth);
  const double cf = steep ? cth : sth, sf = steep ? sth : cth;  // frame cos / sin
  const float *xsrc = steep ? x32 : x32 + (size_t)N * N;
  // axis-aligned views (|sin| below 1e-12, as gen/ct.py's 1e-15 direction test):
  // a ray on a pixel edge belongs to the pixel on its positive side
  const bool axis = fabs(sf) < 1e-12;
  const float a_ = axis ? 1.0f : (float)fabs(cf), b_ = axis ? 0.0f : (float)fabs(sf);
  const float inv_a = 1.0f / a_, inv_ab = b_ > 0.0f ? 1.0f / (a_ * b_) : 0.0f;
  const float w = 0.5f * (a_ + b_) * inv_a;  // footprint half-width in columns
  // crossing column in frame row r: c*(r) = C0 - r tan
  const double tb = ((double)b - 0.5 * (double)(B - 1)) / (double)N;
  const double tanf_ = sf / cf;
  const double c0 = (double)(N / 2);  // centre pixel index (integer N/2, as gen/ct.py)
  const double C0 = c0 + tb * N / cf + c0 * tanf_;
  pdl_wait();  // x is written by the previous kernel; r is read by the previous backward
  float zf = 0.0f;
  double z = 0.0;
  for (int r0 = 0; r0 < N; r0 += kPbRows) {
    __syncthreads();  // previous chunk consumed
    const int nr = min(kPbRows, N - r0);
    // stage the chunk with async copies (many in flight; a load->store loop
    // serialises on L2 latency): 16-byte pieces when the rows allow it
    if ((N & 3) == 0) {
      const float4 *src = reinterpret_cast<const float4 *>(xsrc + (size_t)r0 * N);
      for (int i = threadIdx.x; i < nr * N / 4; i += blockDim.x) cp_async16(xs + 4 * i, src + i);
    } else {
      for (int i = threadIdx.x; i < nr * N; i += blockDim.x) cp_async4(xs + i, xsrc + (size_t)r0 * N + i);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    if (b < B) {
      // crossing column at the chunk's first row in fp64, split into an
      // integer and an fp32 fraction; within the chunk the fraction steps by
      // -tan in fp32 (|rr tan| < 32: error ~2e-6 columns)
      const double csd = C0 - (double)r0 * tanf_;
      const double cfl = floor(csd);
      const float fr0 = (float)(csd - cfl);
      const int ci0 = (int)cfl;
      const float tn = (float)tanf_;
      if (axis) {  // uniform per view: a ray on a pixel edge goes to the positive side
        for (int rr = 0; rr < nr; ++rr) {
          const float u = fmaf(-(float)rr, tn, fr0);
          const float kf = floorf(u + 0.5f);       // the one pixel with -1/2 <= c* - cc < 1/2
          const int cc = ci0 + (int)kf;
          if (cc >= 0 && cc < N) zf += xs[rr * N + cc];
        }
      } else {
        const float p1 = 0.5f * (a_ - b_), p2 = 0.5f * (a_ + b_);
        for (int rr = 0; rr < nr; ++rr) {
          const float u = fmaf(-(float)rr, tn, fr0);
          const float kf = floorf(u);
          const float fr = u - kf;
          const int j_lo = (int)ceilf(fr - w);  // candidates ci + j_lo .. ci + j_lo + 2
          const int cc0 = ci0 + (int)kf + j_lo;
          const float sd0 = fr - (float)j_lo;    // c* - cc0
          const float *xr = xs + rr * N;
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const int cc = cc0 + j;
            const float l = chord(fabsf(sd0 - (float)j), a_, p1, p2, inv_a, inv_ab);
            if (cc >= 0 && cc < N) zf = fmaf(l, xr[cc], zf);
          }
        }
      }
      z += (double)zf;  // fp32 partial per chunk, fp64 across chunks
      zf = 0.0f;
    }
  }
  z /= (double)N;  // chord lengths in units of Δ
  double lacc = 0.0;
  if (b < B) {
    const int64_t row = (int64_t)kl * B + b;
    const double yv = load_y_global(a.y, a.ytype, row);
    // link in-lane (W bins), the quantities of K1's link_exact
    const bool neg = a.relu && z < 0.0;
    const double zc = neg ? 0.0 : z;
    double hs = 0.0, Hs = 0.0;
    for (int j = 0; j < a.W; ++j) {
      const double e = exp_nonpos<9>(-sp[kMaxW + j] * zc);
      hs = fma(sp[j], e, hs);
      if (LOSS) Hs += neg ? sp[j] * z : sp[j] * sp[2 * kMaxW + j] * (1.0 - e);
    }
    a.r[row] = (float)(yv - a.I_bar * hs);
    if (LOSS) lacc = yv * z - a.I_bar * Hs;
  }
  // per-block loss partial, warps in order
  lacc = warp_sum(lacc);
  if ((threadIdx.x & 31) == 0) wl[threadIdx.x >> 5] = lacc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double l = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) l += wl[i];
    a.loss_partials[blockIdx.x] = l;
  }
  pdl_trigger();
}

constexpr int kPbViews = 32;  // residual views staged per chunk in the backward
constexpr int kPbTile = 16;   // backward blocks cover 16 x 16 pixel tiles

// Per-view record of the backward, built once per chunk: the bin coordinate
// of the tile's corner pixel in fp64 split into an integer and an fp32
// fraction, so that a pixel's own coordinate is base_f + dc cos + dr sin with
// |dc|, |dr| < 16 (fp32 error ~1e-6 bins).
struct PbView {
  float cs, sn, base_f, wb;   // cos, sin, fraction at the tile corner, footprint half-width
  float p1, inv_max, inv_ab;  // plateau half-width, plateau and ramp scales
  int base_i;                 // integer part at the tile corner
};

// g_pixel = Σ_views Σ_bins L r: one thread per (pixel, half of the views).
// Block = one 16 x 16 tile; half h covers views [h*ceil(nv/2), ...);
// out2[h*d + pixel] (fp64).
__global__ void __launch_bounds__(256) k_pb_backward(const PbGeom g, const float *__restrict__ r,
                                                     double *__restrict__ out2) {
  extern __shared__ __align__(16) float rs[];  // [kPbViews][B]
  __shared__ PbView vw[kPbViews];
  const int N = g.N, B = g.B;
  const int64_t d = (int64_t)N * N;
  const int half = blockIdx.y;
  const int vh = (g.nv + 1) / 2;
  const int va = half * vh, vb = min(g.nv, va + vh);
  const int tiles_c = (N + kPbTile - 1) / kPbTile;
  const int tr0 = (blockIdx.x / tiles_c) * kPbTile, tc0 = (blockIdx.x % tiles_c) * kPbTile;
  const int dr = threadIdx.x / kPbTile, dc = threadIdx.x % kPbTile;
  const int pr = tr0 + dr, pc = tc0 + dc;
  const bool own = pr < N && pc < N;
  pdl_wait();  // r is written by the forward pass
  double acc = 0.0;
  for (int v0 = va; v0 < vb; v0 += kPbViews) {
    const int nv = min(kPbViews, vb - v0);
    __syncthreads();
    for (int i = threadIdx.x; i < nv * B; i += blockDim.x) cp_async4(rs + i, r + (int64_t)v0 * B + i);
    if (threadIdx.x < nv) {
      const int k = g.v0 + v0 + threadIdx.x;
      const double cs = g.trig[2 * k], sn = g.trig[2 * k + 1];
      const bool axis = fabs(cs) < 1e-12 || fabs(sn) < 1e-12;
      const float a_ = axis ? (fabs(cs) < 1e-12 ? 0.0f : 1.0f) : (float)fabs(cs);
      const float b_ = axis ? (fabs(sn) < 1e-12 ? 0.0f : 1.0f) : (float)fabs(sn);
      const float amax = fmaxf(a_, b_), amin = fminf(a_, b_);
      // b* of the tile corner: (X cos + Y sin) N + (B-1)/2, X N = tc0 - N/2
      const double bsd = fma((double)(tc0 - N / 2), cs, (double)(tr0 - N / 2) * sn) + 0.5 * (B - 1);
      const double bfl = floor(bsd);
      PbView v;
      v.cs = axis ? (fabs(cs) < 1e-12 ? 0.0f : (float)cs) : (float)cs;
      v.sn = axis ? (fabs(sn) < 1e-12 ? 0.0f : (float)sn) : (float)sn;
      v.base_f = (float)(bsd - bfl);
      v.wb = 0.5f * (a_ + b_);
      v.p1 = 0.5f * (amax - amin);
      v.inv_max = 1.0f / amax;
      v.inv_ab = amin > 0.0f ? 1.0f / (a_ * b_) : 0.0f;
      v.base_i = (int)bfl;  // may be negative; axis views are the ones with inv_ab == 0
      vw[threadIdx.x] = v;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    if (own) {
      float accf = 0.0f;
      for (int vv = 0; vv < nv; ++vv) {
        const PbView v = vw[vv];
        const bool axis = v.inv_ab == 0.0f;
        const int base_i = v.base_i;
        const float u = fmaf((float)dc, v.cs, fmaf((float)dr, v.sn, v.base_f));
        const float *rv = rs + vv * B;
        if (axis) {  // the one bin with -1/2 < b* - b <= 1/2
          const int bb = base_i + (int)ceilf(u - 0.5f);
          if (bb >= 0 && bb < B) accf += rv[bb];
        } else {
          const float kf = floorf(u);
          const float fr = u - kf;
          const int j_lo = (int)ceilf(fr - v.wb);
          const int bb0 = base_i + (int)kf + j_lo;
          const float sd0 = fr - (float)j_lo;  // b* - bb0
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int bb = bb0 + j;
            const float dd = fabsf(sd0 - (float)j);
            const float l = dd <= v.p1 ? v.inv_max : fmaxf(0.0f, (v.wb - dd) * v.inv_ab);
            if (bb >= 0 && bb < B) accf = fmaf(l, rv[bb], accf);
          }
        }
      }
      acc += (double)accf;
    }
  }
  if (own) out2[half * d + (int64_t)pr * N + pc] = acc / (double)N;
  pdl_trigger();
}

// g = out2[0] + out2[1] (the two view halves, in order) into the partial row
__global__ void k_pb_combine(const double *__restrict__ out2, int64_t d, double *__restrict__ g) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d;
       i += (int64_t)gridDim.x * blockDim.x)
    g[i] = out2[i] + out2[d + i];
}

}  // namespace poly
