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
//                      most 2 pixels per row its footprint covers; then the
//                      link and residual per ray (fp64) as K1, r stored fp32.
//   K5b k_pb_backward  one thread per 2 pixels of a 16 x 16 tile row and a
//                      16th of the views: for every view the at most 2
//                      bins whose rays cross each pixel, from the 32-bin
//                      window of residuals the tile can reach (staged per
//                      view chunk in shared memory); the last of a tile's
//                      16 view-range blocks adds their partials in order
//                      (deterministic).
#pragma once

#include "dense.cuh"

namespace poly {

#ifndef POLY_PB_ROWSPLIT
#define POLY_PB_ROWSPLIT 2
#endif
constexpr int kPbRowSplit = POLY_PB_ROWSPLIT;  // forward blocks per view (row ranges)

struct PbGeom {
  int32_t N, V, B;
  int32_t v0;          // first view of this handle's rows (row_offset / B)
  int32_t nv;          // views held (n_local / B)
  const double *trig;  // [2V]: cos θ_k, sin θ_k (host libm, θ_k = kπ/V)
  double *zpart;       // [kPbRowSplit][n_local] forward partial sums per row range
  int32_t *ticket;     // [nv] forward blocks finished per view (reset by the last)
  int32_t *tticket;    // [tiles] backward blocks finished per tile (reset by the last)
};

// chord length / Δ for a pixel whose centre is dd (>= 0) pixel widths from
// the ray, measured along the axis the scales refer to:
//   min(plateau, max(0, kp - dd * kd))
// equals the plateau 1/max(a,b) for dd <= Δ|a-b|/2, the ramp beyond it and 0
// past the footprint (the ramp reaches the plateau value exactly at the
// plateau's edge) — three instructions, no branches.
__device__ __forceinline__ float chord(float dd, float plateau, float kd, float kp) {
  return fminf(plateau, fmaxf(0.0f, fmaf(-dd, kd, kp)));
}

#ifndef POLY_PB_MAGIC
#define POLY_PB_MAGIC 1   // floor/ceil through fp32 adds instead of F2I/I2F conversions (same results)
#endif
// floor(u) for |u| < 2^22 as a float and an int: u + 1.5·2^23 rounded towards -inf has unit ulp, so its
// mantissa holds floor(u) — two adds on the fp32 pipe instead of F2I + I2F
__device__ __forceinline__ void floor_fi(float u, float &kf, int &ki) {
#if POLY_PB_MAGIC
  const float t = __fadd_rd(u, 12582912.0f);
  kf = t - 12582912.0f;
  ki = __float_as_int(t) - 0x4B400000;
#else
  ki = __float2int_rd(u);
  kf = (float)ki;
#endif
}
// ceil(fr - w) for fr in [0, 1), w in (0, 1): 1 when fr > w, else 0 (fr - w > -1 and is never rounded to zero)
__device__ __forceinline__ void ceil01_fi(float fr, float w, float &jf, int &ji) {
#if POLY_PB_MAGIC
  const bool up = fr > w;
  jf = up ? 1.0f : 0.0f;
  ji = up ? 1 : 0;
#else
  ji = __float2int_ru(fr - w);
  jf = (float)ji;
#endif
}

#ifndef POLY_PB_ROWS
#define POLY_PB_ROWS 32
#endif
constexpr int kPbRows = POLY_PB_ROWS;  // image rows per staged chunk in the forward
#ifndef POLY_PB_NBUF
#define POLY_PB_NBUF 1
#endif
constexpr int kPbBufs = POLY_PB_NBUF;  // stage buffers (1: no prefetch, more resident blocks)
constexpr int kPbPad = 4;    // zero columns on either side of a staged row (no bounds checks)

// z_i for the rays of one view, then the residual (mode EXACT).  x32 holds
// x (row-major) at [0, d) and its transpose at [d, 2d).
template <bool LOSS>
__global__ void __launch_bounds__(512) k_pb_forward(const PbGeom g, const float *__restrict__ x32,
                                                    const CsrFwdArgs a) {
  extern __shared__ __align__(16) float xs[];  // [kPbBufs][kPbRows][N + 2 kPbPad], image columns at kPbPad
  __shared__ __align__(8) uint64_t mbar[2];
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
  // chord in column units: distance dd columns = dd a perpendicular
  const float kd = a_ * inv_ab, kp = 0.5f * (a_ + b_) * inv_ab, kp1 = kp - kd;
  const int NP = N + 2 * kPbPad;
  for (int i = threadIdx.x; i < kPbBufs * kPbRows * 2 * kPbPad; i += blockDim.x) {
    const int rr = i / (2 * kPbPad), q = i - rr * 2 * kPbPad;
    xs[rr * NP + (q < kPbPad ? q : N + q)] = 0.0f;
  }
  // crossing column in frame row r: c*(r) = C0 - r tan
  const double tb = ((double)b - 0.5 * (double)(B - 1)) / (double)N;
  const double tanf_ = sf / cf;
  const double c0 = (double)(N / 2);  // centre pixel index (integer N/2, as gen/ct.py)
  const double C0 = c0 + tb * N / cf + c0 * tanf_;
  // frame rows where the ray's footprint can touch the image: c*(r) within
  // [-2, N + 1] (half-width <= 1 column); other rows add exact zeros, so the
  // loops skip them (a ray outside the image skips everything)
  int r_lo = 0, r_hi = N;
  if (tanf_ == 0.0) {
    if (!(C0 >= -2.0 && C0 <= N + 1.0)) r_lo = r_hi = 0;
  } else {
    const double ra = (C0 + 2.0) / tanf_, rb2 = (C0 - N - 1.0) / tanf_;
    r_lo = (int)fmax(0.0, floor(fmin(ra, rb2)) - 1.0);
    r_hi = (int)fmin((double)N, ceil(fmax(ra, rb2)) + 2.0);
    if (r_hi < r_lo) r_hi = r_lo;
  }
  // this block's row range (blockIdx.y of kPbRowSplit): the view's rays are
  // split by rows so that the grid is several waves of blocks, not 2.4
  const int rs = blockIdx.y;
  const int rb = (int)((int64_t)N * rs / kPbRowSplit), re = (int)((int64_t)N * (rs + 1) / kPbRowSplit);
  if (threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();  // x is written by the previous kernel; r is read by the previous backward
  // Rows are staged in chunks of kPbRows through kPbBufs buffers: chunk
  // c + kPbBufs is requested as soon as chunk c is consumed.  Rows of 16-byte multiples go through the TMA engine (one bulk
  // copy per row, lanes of warp 0, completion on the buffer's mbarrier); other
  // widths through per-thread cp.async completing on the same mbarrier.
  const bool tma = (N & 3) == 0;
  const int nchunks = (re - rb + kPbRows - 1) / kPbRows;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  auto issue = [&](int c) {
    const int buf = c % kPbBufs, r0 = rb + c * kPbRows, nr = min(kPbRows, re - r0);
    float *dst = xs + buf * kPbRows * NP + kPbPad;
    if (tma) {
      if (threadIdx.x < 32) {
        if (threadIdx.x == 0) mbar_arrive_expect_tx(&mbar[buf], (uint32_t)(nr * N * 4));
        __syncwarp();
        for (int rr = threadIdx.x; rr < nr; rr += 32)
          bulk_g2s(dst + rr * NP, xsrc + (size_t)(r0 + rr) * N, (uint32_t)(N * 4), &mbar[buf], pol);
      }
    } else {
      for (int i = threadIdx.x; i < nr * N; i += blockDim.x) {
        const int rr = i / N, q = i - rr * N;
        cp_async4(dst + rr * NP + q, xsrc + (size_t)r0 * N + i);
      }
      cp_async_mbar_arrive(&mbar[buf]);  // (.noinc) one arrival per thread, counted below
    }
  };
  if (!tma && threadIdx.x == 0) {  // per-thread arrivals: re-init with the thread count
    mbar_init(&mbar[0], blockDim.x);
    mbar_init(&mbar[1], blockDim.x);
    fence_mbar_init();
  }
  __syncthreads();
  for (int c = 0; c < kPbBufs && c < nchunks; ++c) issue(c);
  float zf = 0.0f;
  double z = 0.0;
  for (int c = 0; c < nchunks; ++c) {
    const int buf = c % kPbBufs, r0 = rb + c * kPbRows, nr = min(kPbRows, re - r0);
    mbar_wait(&mbar[buf], (uint32_t)((c / kPbBufs) & 1));
    const float *xsb = xs + buf * kPbRows * NP;
    if (b < B) {
      // crossing column at the chunk's first row in fp64, split into an
      // integer and an fp32 fraction; within the chunk the fraction steps by
      // -tan in fp32 (|rr tan| < 32: error ~2e-6 columns)
      const double csd = C0 - (double)r0 * tanf_;
      const double cfl = floor(csd);
      const float fr0 = (float)(csd - cfl);
      const int ci0 = (int)cfl;
      const float tn = (float)tanf_;
      // candidate columns are clamped into the zero padding once the ray
      // has left the image (their chord weights then multiply zeros)
      if (axis) {  // uniform per view: a ray on a pixel edge goes to the positive side
        const int ra = max(0, r_lo - r0), rz = min(nr, r_hi - r0);
#pragma unroll 4
        for (int rr = ra; rr < rz; ++rr) {
          const float u = fmaf(-(float)rr, tn, fr0);
          const int cc = min(max(ci0 + __float2int_rd(u + 0.5f), -1), N);  // -1/2 <= c* - cc < 1/2
          zf += xsb[rr * NP + kPbPad + cc];
        }
      } else {
        const int ra = max(0, r_lo - r0), rz = min(nr, r_hi - r0);
        // EXACT01: w < 1, so ceil(fr - w) is 0 or 1 (a comparison); the 45-degree view (w = 1, where
        // fr = 0 gives -1) keeps the conversions.  Uniform per block.
        auto rows = [&](auto EXACT01) {
#pragma unroll 4
          for (int rr = ra; rr < rz; ++rr) {
            const float u = fmaf(-(float)rr, tn, fr0);
            int ki, j_lo;
            float kf, jf;
            floor_fi(u, kf, ki);
            const float fr = u - kf;
            // the footprint [c* - w, c* + w] (w <= 1) holds at most two pixel
            // centres with a nonzero chord: cc0 = ceil(c* - w) and cc0 + 1
            if (decltype(EXACT01)::value) {
              ceil01_fi(fr, w, jf, j_lo);
            } else {
              j_lo = __float2int_ru(fr - w);
              jf = (float)j_lo;
            }
            const int cc0 = min(max(ci0 + ki + j_lo, -2), N);
            const float sd0 = fr - jf;  // c* - cc0 (unclamped), in (w - 1, w]
            const float *xr = xsb + rr * NP + kPbPad + cc0;
            // |sd0 - 1| = 1 - sd0: the second chord's argument folds into one FMA
            zf = fmaf(chord(fabsf(sd0), inv_a, kd, kp), xr[0], zf);
            zf = fmaf(fminf(inv_a, fmaxf(0.0f, fmaf(sd0, kd, kp1))), xr[1], zf);
          }
        };
        if (w < 1.0f)
          rows(std::true_type{});
        else
          rows(std::false_type{});
      }
      z += (double)zf;  // fp32 partial per chunk, fp64 across chunks
      zf = 0.0f;
    }
    __syncthreads();  // buffer consumed: request chunk c + kPbBufs into it
    if (c + kPbBufs < nchunks) issue(c + kPbBufs);
  }
  // partial sums of the row ranges; the view's last block adds them in order
  __shared__ int last;
  const int64_t nloc = (int64_t)g.nv * B;
  if (b < B) g.zpart[rs * nloc + (int64_t)kl * B + b] = z;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(g.ticket + kl, 1) == kPbRowSplit - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) g.ticket[kl] = 0;  // ready for the next launch
  if (b < B) {
    z = 0.0;
    for (int q = 0; q < kPbRowSplit; ++q) z += __ldcg(g.zpart + q * nloc + (int64_t)kl * B + b);
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

constexpr int kPbViews = 32;  // views staged per chunk in the backward
constexpr int kPbTile = 16;   // backward blocks cover 16 x 16 pixel tiles
#ifndef POLY_PB_PX
#define POLY_PB_PX 2
#endif
#ifndef POLY_PB_PARTS
#define POLY_PB_PARTS 16
#endif
constexpr int kPbPx = POLY_PB_PX;  // consecutive pixels of a tile row per thread
constexpr int kPbWin = 32;    // bins staged per view: every bin a tile's pixels can reach
constexpr int kPbParts = POLY_PB_PARTS;  // view ranges, one block each (partials added in order)

// Per-view record of the backward, built once per chunk: the bin coordinate
// b* of the tile's corner pixel relative to the start wlo of the view's
// staged bin window (fp64 arithmetic, fp32 result in [1, 24)), so that a
// pixel's own coordinate is base_f + dc cos + dr sin with dc, dr < 16.
struct PbView {
  float cs, sn, base_f, wb;     // cos, sin, corner b* - wlo, footprint half-width
  float inv_max, kd, kp;        // chord scales (chord(); kd = 0: axis-aligned view)
  int wlo;                      // first staged bin
};

// g_pixel = Σ_views Σ_bins L r: one thread per kPbPx pixels of a tile row and
// one range of views (blockIdx.y of kPbParts); out[part*d + pixel] (fp64).
// Per chunk of views a tile stages only the 32-bin window of r each view's
// rays can reach inside the tile (zeros outside [0, B): no bounds checks).
__global__ void __launch_bounds__(kPbTile * kPbTile / kPbPx) k_pb_backward(const PbGeom g,
                                                                          const float *__restrict__ r,
                                                                          double *__restrict__ out,
                                                                          double *__restrict__ gout) {
  __shared__ __align__(16) float rs[kPbViews][kPbWin];
  __shared__ PbView vw[kPbViews];
  __shared__ int last;
  constexpr int TPR = kPbTile / kPbPx;  // threads per tile row
  const int N = g.N, B = g.B;
  const int64_t d = (int64_t)N * N;
  const int part = blockIdx.y;
  const int vh = (g.nv + kPbParts - 1) / kPbParts;
  const int va = part * vh, vb = min(g.nv, va + vh);
  const int tiles_c = (N + kPbTile - 1) / kPbTile;
  const int tr0 = (blockIdx.x / tiles_c) * kPbTile, tc0 = (blockIdx.x % tiles_c) * kPbTile;
  const int dr = threadIdx.x / TPR, dc0 = (threadIdx.x % TPR) * kPbPx;
  const int pr = tr0 + dr;
  pdl_wait();  // r is written by the forward pass
  float accf[kPbPx];
  double acc[kPbPx];
#pragma unroll
  for (int q = 0; q < kPbPx; ++q) acc[q] = 0.0;
  for (int v0 = va; v0 < vb; v0 += kPbViews) {
    const int nv = min(kPbViews, vb - v0);
    __syncthreads();  // previous chunk consumed
    if ((int)threadIdx.x < nv) {
      const int k = g.v0 + v0 + threadIdx.x;
      const double cs = g.trig[2 * k], sn = g.trig[2 * k + 1];
      const bool axis = fabs(cs) < 1e-12 || fabs(sn) < 1e-12;
      const float a_ = axis ? (fabs(cs) < 1e-12 ? 0.0f : 1.0f) : (float)fabs(cs);
      const float b_ = axis ? (fabs(sn) < 1e-12 ? 0.0f : 1.0f) : (float)fabs(sn);
      const float amax = fmaxf(a_, b_), amin = fminf(a_, b_);
      const double csr = axis ? (fabs(cs) < 1e-12 ? 0.0 : cs) : cs, snr = axis ? (fabs(sn) < 1e-12 ? 0.0 : sn) : sn;
      // b* of the tile corner: (X cos + Y sin) N + (B-1)/2, X N = tc0 - N/2;
      // the tile's b* span [lo, hi] sets the window (candidates floor(b*) - 1 .. + 1)
      const double bsd = fma((double)(tc0 - N / 2), csr, (double)(tr0 - N / 2) * snr) + 0.5 * (B - 1);
      const double e = (double)(kPbTile - 1);
      const double lo = bsd + fmin(0.0, e * csr) + fmin(0.0, e * snr);
      const int wlo = (int)floor(lo) - 1;
      PbView v;
      v.cs = (float)csr;
      v.sn = (float)snr;
      v.base_f = (float)(bsd - (double)wlo);
      v.wb = 0.5f * (a_ + b_);
      v.inv_max = 1.0f / amax;
      v.kd = amin > 0.0f ? 1.0f / (a_ * b_) : 0.0f;
      v.kp = v.wb * v.kd;
      v.wlo = wlo;
      vw[threadIdx.x] = v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nv * kPbWin; i += blockDim.x) {
      const int vv = i / kPbWin, j = i - vv * kPbWin;
      const int bb = vw[vv].wlo + j;
      rs[vv][j] = (bb >= 0 && bb < B) ? __ldg(r + (int64_t)(v0 + vv) * B + bb) : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kPbPx; ++q) accf[q] = 0.0f;
    for (int vv = 0; vv < nv; ++vv) {
      const PbView v = vw[vv];
      const float *rv = rs[vv];
      const float u0 = fmaf((float)dc0, v.cs, fmaf((float)dr, v.sn, v.base_f));
      if (v.kd == 0.0f) {  // axis-aligned (uniform): the one bin with -1/2 < b* - b <= 1/2
#pragma unroll
        for (int q = 0; q < kPbPx; ++q) {
          const float u = fmaf((float)q, v.cs, u0);
          accf[q] += rv[__float2int_ru(u - 0.5f)];
        }
      } else {
#pragma unroll
        for (int q = 0; q < kPbPx; ++q) {
          const float u = fmaf((float)q, v.cs, u0);
          int ki, j_lo;
          float kf, jf;
          floor_fi(u, kf, ki);
          const float fr = u - kf;
          ceil01_fi(fr, v.wb, jf, j_lo);
          const float sd0 = fr - jf;  // b* - (bin ki + j_lo)
          const float *rb = rv + ki + j_lo;
          // sd0 <= wb < 1, so |sd0 - 1| = 1 - sd0 folds into one FMA
          accf[q] = fmaf(chord(fabsf(sd0), v.inv_max, v.kd, v.kp), rb[0], accf[q]);
          accf[q] = fmaf(fminf(v.inv_max, fmaxf(0.0f, fmaf(sd0, v.kd, v.kp - v.kd))), rb[1], accf[q]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < kPbPx; ++q) acc[q] += (double)accf[q];  // fp32 per chunk, fp64 across chunks
  }
#pragma unroll
  for (int q = 0; q < kPbPx; ++q) {
    const int pc = tc0 + dc0 + q;
    if (pr < N && pc < N) out[part * d + (int64_t)pr * N + pc] = acc[q] / (double)N;
  }
  // the tile's last block adds the kPbParts partials in order into g
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(g.tticket + blockIdx.x, 1) == kPbParts - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) g.tticket[blockIdx.x] = 0;  // ready for the next launch
#pragma unroll
  for (int q = 0; q < kPbPx; ++q) {
    const int pc = tc0 + dc0 + q;
    if (pr < N && pc < N) {
      const int64_t i = (int64_t)pr * N + pc;
      double v = __ldcg(out + i);
      for (int p = 1; p < kPbParts; ++p) v += __ldcg(out + p * d + i);
      gout[i] = v;
    }
  }
  pdl_trigger();
}

}  // namespace poly
