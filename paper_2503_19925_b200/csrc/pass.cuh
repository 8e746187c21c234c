// K4p — the whole K4t pass (strip forward, link, tile backward) as one
// persistent kernel: one CTA per SM, two grid-wide barriers.
//
// The three K4t kernels each stream a few hundred KB per CTA, so every CTA's
// start (barrier set-up, strip or ray-list staging, ring fill) and drain, and
// the two kernel boundaries of a pass, are a tenth of the pass.
// Here the CTAs stay resident for the whole pass:
//   phase F   warps 0-11 consume the strip units, warp 12 produces them (as
//             k_strip_forward); the other warps help stage the iterate strip;
//   (local)   warp 15 starts streaming this CTA's backward tiles into the
//             backward ring (static records) — it fills during phases L;
//             warps 0-14 copy the ray-list rows of the CTA's first two tiles;
//   barrier   every CTA's pz written;
//   phase L   warps 0-14 run the link of a contiguous row range (2 rows per
//             thread in flight), r_i and the CTA's objective partial;
//   barrier   every r_i written;
//   phase B   per tile: r gathered into the tile's list buffer (double
//             buffered: warp 14 prepares the next tile while consumers
//             stream), 2·TH consumer warps walk the records (as
//             k_tile_backward), halves combined, column output or the step
//             epilogue.
// The grid barriers need every CTA resident: the grid is the SM count, one
// CTA per SM (shared memory), and the kernel triggers its dependents only at
// its end; the waits are bounded (2 s) and a timeout sets SolveState::comm_err
// = 2, which poly_solve reports.
#pragma once

#include "tiled.cuh"

namespace poly {

constexpr int kPassWarps = 16;
constexpr int kPassFwdStages = 7;
constexpr int kPassMaxBwdStages = 16;
constexpr int kPassProdF = kFwdWarps;  // forward producer warp (12)
constexpr int kPassProdB = 15;         // backward producer warp
constexpr int kPassGroup = 15 * 32;    // warps 0-14: staging, link, list preparation

struct PassSync {
  uint32_t *gbar;  // [2] grid barrier: arrivals, generation
  int32_t *err;    // SolveState::comm_err
  int32_t nstb;    // backward ring stages
  int32_t abytes;  // region A (strip | two ray-list buffers), 128-byte multiple
  int32_t lcap;    // one ray-list buffer, floats
};

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// grid-wide barrier of the threads in named barrier `id` (count `nthr`, which
// include thread 0) across all CTAs; bounded wait
__device__ __forceinline__ void pass_grid_barrier(const PassSync &ps, int id, int nthr) {
  named_bar(id, nthr);
  if (threadIdx.x == 0) {
    const uint32_t gen = ld_acquire_u32(ps.gbar + 1);
    __threadfence();
    if (atomicAdd(ps.gbar, 1u) == gridDim.x - 1) {
      atomicExch(ps.gbar, 0u);
      __threadfence();
      atomicAdd(ps.gbar + 1, 1u);
    } else {
      unsigned long long t0, t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      while (ld_acquire_u32(ps.gbar + 1) == gen) {
        __nanosleep(32);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t0 > 2000000000ull) {
          atomicExch(ps.err, 2);
          break;
        }
      }
    }
    __threadfence();
  }
  named_bar(id, nthr);
}

#ifdef POLY_PASS_TRACE
#define PASS_T(i)                                                             \
  do {                                                                        \
    if ((blockIdx.x == 0 || blockIdx.x == 100) && threadIdx.x == 0) {         \
      unsigned long long tt;                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));                  \
      tr[i] = tt;                                                             \
    }                                                                         \
  } while (0)
#else
#define PASS_T(i) \
  do {            \
  } while (0)
#endif

template <bool LOSS>
__global__ void __launch_bounds__(kPassWarps * 32, 1)
    k_ct_pass(const StripFwd f, const TileBwd t, const CsrFwdArgs a, const float *__restrict__ x,
              double *__restrict__ g, int32_t d, const StepEpi e, const PassSync ps) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ double sp[3 * kMaxW];
  __shared__ double part[8 * 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#ifdef POLY_PASS_TRACE
  unsigned long long tr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  PASS_T(0);
  // region A: the strip (phase F) | two ray-list buffers (phase B)
  float *sx = (float *)smem;
  // region B: the forward ring (phase F) | the backward ring (phase B)
  uint8_t *ringB = smem + ps.abytes;
  uint64_t *bar = (uint64_t *)(ringB + kPassFwdStages * kFwdStageBytes);
  uint64_t *ffull = bar, *fempty = bar + kPassFwdStages;
  uint64_t *bfull = bar + 2 * kPassFwdStages, *bempty = bfull + kPassMaxBwdStages;
  int4 *desc = (int4 *)(bempty + kPassMaxBwdStages);
  const int ncw = 2 * t.npw;                    // backward consumer warps (<= 14)
  const int sbytes = kBwdCG * ncw * kRecBytes;  // one backward stage
  const int strip = blockIdx.x % f.NS;
  const int u0 = f.unit_start[strip], nu = f.unit_start[strip + 1] - u0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPassFwdStages; ++s) {
      mbar_init(ffull + s, 1);
      mbar_init(fempty + s, kFwdWarps);
    }
    for (int s = 0; s < ps.nstb; ++s) {
      mbar_init(bfull + s, 1);
      mbar_init(bempty + s, ncw);
    }
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 3 * kMaxW; i += blockDim.x) sp[i] = a.spec[i];
  __syncthreads();

  // ------------------------------------------------------------ phase F
  if (warp == kPassProdF) {
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      pdl_wait();  // the counter was reset in the previous pass
      int it = 0, st = 0;
      uint32_t eph = 0;
      int u = atomicAdd(f.ctr + strip, 1);
      for (;;) {
        const bool done = u >= nu;
        const int un = done ? nu : atomicAdd(f.ctr + strip, 1);
        const int64_t U = (int64_t)u0 + u;
        const int64_t g0 = done ? 0 : f.unit_off[U], ng = done ? 1 : f.unit_off[U + 1] - g0;
        for (int64_t k = 0; k < ng; k += kFwdCG) {
          if (it >= kPassFwdStages) mbar_wait(fempty + st, eph ^ 1);
          const int c = done ? 0 : kFwdCG;
          desc[st] = make_int4(done ? -1 : u, (int)k, c, (k == 0 ? 1 : 0) | (k + c >= ng ? 2 : 0));
          uint8_t *sb = ringB + st * kFwdStageBytes;
          if (done) {
            mbar_arrive(ffull + st);
          } else {
            const uint32_t data = (uint32_t)c * kFwdWarps * kRecBytes;
            mbar_arrive_expect_tx(ffull + st, data + (k == 0 ? kFwdHdr : 0));
            if (k == 0) bulk_g2s(sb, f.hdr + U * kFwdHdr, kFwdHdr, ffull + st, pol);
            bulk_g2s(sb + kFwdHdr, f.rec + (g0 + k) * kFwdWarps * kRecBytes, data, ffull + st, pol);
          }
          ++it;
          if (++st == kPassFwdStages) st = 0, eph ^= 1;
        }
        if (done) break;
        u = un;
      }
    }
    __syncwarp();
  } else {
    // every other warp stages the strip (rows_img x P floats, columns >= ws zero)
    const int c0 = strip * f.W;
    const int ws = min(f.W, f.cols_img - c0);
    const int sw = warp < kPassProdF ? warp : warp - 1;  // 0..14
    pdl_wait();  // x is written by the previous step kernel
    for (int r = sw; r < f.rows_img; r += kPassWarps - 1) {
      const float *xr = x + (int64_t)r * f.cols_img + c0;
      float *srw = sx + r * f.P;
      for (int c = lane; c < f.P; c += 32) {
        if (c < ws) cp_async4(srw + c, xr + c);
        else srw[c] = 0.f;
      }
    }
    cp_async_wait_all();
    named_bar(1, kPassWarps * 32 - 32);
    if (warp < kFwdWarps) {
      int idx = 0, row = -1;
      double a0 = 0.0, a1 = 0.0;
      int st = 0;
      uint32_t ph = 0;
      for (;; st = st + 1 == kPassFwdStages ? 0 : st + 1, ph ^= st == 0 ? 1u : 0u) {
        mbar_wait(ffull + st, ph);
        const int4 dsc = desc[st];
        if (dsc.x < 0) break;
        const uint8_t *sb = ringB + st * kFwdStageBytes;
        if (dsc.w & 1) {
          idx = ((const uint16_t *)sb)[warp * 32 + lane];
          row = ((const int32_t *)(sb + kFwdWarps * 32 * 2))[warp * 32 + lane];
          a0 = a1 = 0.0;
        }
        const uint8_t *rb = sb + kFwdHdr + warp * kRecBytes;
#pragma unroll
        for (int k = 0; k < kFwdCG; ++k) rec_group(rb + k * kFwdWarps * kRecBytes, lane, idx, sx, (k & 1) ? a1 : a0);
        __syncwarp();
        if (lane == 0) mbar_arrive(fempty + st);
        if ((dsc.w & 2) && row >= 0) f.pz[(int64_t)strip * f.n + row] = a0 + a1;
      }
    }
  }
  __syncthreads();  // the forward ring and the strip are free; this CTA's pz are written
  PASS_T(1);

  // tiles of this CTA: blockIdx.x, +gridDim.x, ...
  const int ntl = blockIdx.x < t.ntiles ? (t.ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  float *lbuf[2] = {(float *)smem, (float *)smem + ps.lcap};
  if (warp == kPassProdB) {
    // the backward producer: every tile's stages, in order, into the ring
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      int st = 0;
      uint32_t eph = 0;
      int64_t it = 0;
      for (int jj = 0; jj < ntl; ++jj) {
        const int tile = blockIdx.x + jj * gridDim.x;
        const int64_t G0 = t.tile_off[tile], ns = (t.tile_off[tile + 1] - G0) / kBwdCG;
        for (int64_t k = 0; k < ns; ++k) {
          if (it >= ps.nstb) mbar_wait(bempty + st, eph ^ 1);
          mbar_arrive_expect_tx(bfull + st, sbytes);
          bulk_g2s(ringB + st * sbytes, t.rec + bwd_stage_off(t, tile, G0, k), sbytes, bfull + st, pol);
          ++it;
          if (++st == ps.nstb) st = 0, eph ^= 1;
        }
      }
    }
    return;  // warp 15 takes no part in what follows
  }
  const int gt = threadIdx.x;  // 0 .. kPassGroup-1
  // the ray-list rows of the first two tiles (static)
  for (int jj = 0; jj < min(ntl, 2); ++jj) {
    const int tile = blockIdx.x + jj * gridDim.x;
    const int64_t L0 = t.list_off[tile];
    const int L = (int)(t.list_off[tile + 1] - L0);
    for (int i = 4 * gt; i < L; i += 4 * kPassGroup) cp_async16((int32_t *)lbuf[jj] + i, t.list + L0 + i);
  }
  pass_grid_barrier(ps, 2, kPassGroup);  // every CTA's pz
  PASS_T(2);
  if (blockIdx.x == 0 && gt < f.NS) f.ctr[gt] = 0;  // for the next pass's forward

  // ------------------------------------------------------------ phase L
  {
    const int64_t per = (a.n + gridDim.x - 1) / gridDim.x, r0 = per * blockIdx.x, r1 = min(a.n, r0 + per);
    double lacc = 0.0;
    for (int64_t base = r0; base < r1; base += 2 * kPassGroup) {
      double z[2] = {0.0, 0.0}, yv[2] = {0.0, 0.0}, Ii[2] = {a.I_bar, a.I_bar};
      const float *srow[2] = {nullptr, nullptr};
      int64_t row[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        row[q] = base + gt + q * kPassGroup;
        if (row[q] < r1) {
          for (int s = 0; s < f.NS; ++s) z[q] += __ldcg(f.pz + (int64_t)s * a.n + row[q]);
          if (a.ytype == 0) yv[q] = (double)((const int32_t *)a.y)[row[q]];
          else if (a.ytype == 1) yv[q] = (double)((const float *)a.y)[row[q]];
          else yv[q] = ((const double *)a.y)[row[q]];
          if (a.I_row) {
            Ii[q] = (double)a.I_row[row[q]];
            srow[q] = a.s_row + row[q] * a.W;
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (row[q] < r1) {
          double l;
          a.r[row[q]] = (float)row_residual_serial<LOSS>(sp, a.W, a.relu, z[q], yv[q], Ii[q], srow[q], &l, a.mode,
                                                         a.mu_step);
          lacc += l;
        }
      }
    }
    if (LOSS) {
      lacc = warp_sum(lacc);
      if (lane == 0) part[warp] = lacc;
      named_bar(2, kPassGroup);
      if (gt == 0) {
        double tl = 0.0;
        for (int w = 0; w < kPassGroup / 32; ++w) tl += part[w];
        a.loss_partials[blockIdx.x] = tl;
      }
    }
  }
  cp_async_wait_all();                   // (the list rows)
  PASS_T(3);
  pass_grid_barrier(ps, 2, kPassGroup);  // every r_i
  PASS_T(4);

  // ------------------------------------------------------------ phase B
  // r of tile 0 into buffer 0 by the whole group; later tiles are prepared by
  // warp 14 while the consumers stream the current one
  auto gather = [&](int jj, int t0, int nt) {
    const int tile = blockIdx.x + jj * gridDim.x;
    const int64_t L0 = t.list_off[tile];
    const int L = (int)(t.list_off[tile + 1] - L0);
    float *b = lbuf[jj & 1];
    if (jj >= 2) {  // the rows themselves first
      for (int i = 4 * t0; i < L; i += 4 * nt) cp_async16((int32_t *)b + i, t.list + L0 + i);
      cp_async_wait_all();
      __syncwarp();
    }
    for (int i = t0; i < L; i += nt) cp_async4(b + i, a.r + ((const int32_t *)b)[i]);
    cp_async_wait_all();
  };
  if (ntl > 0) gather(0, gt, kPassGroup);
  named_bar(2, kPassGroup);
  PASS_T(5);
  int st = 0;
  uint32_t ph = 0;
  for (int jj = 0; jj < ntl; ++jj) {
    const int tile = blockIdx.x + jj * gridDim.x;
    if (warp == 14) {
      if (jj + 1 < ntl) gather(jj + 1, lane, 32);
    } else if (warp < ncw) {
      const float *sr = lbuf[jj & 1];
      const int pw = warp % t.npw, h = warp / t.npw;
      const int64_t G0 = t.tile_off[tile];
      const int nst = (int)((t.tile_off[tile + 1] - G0) / kBwdCG);
      const int slot = tile * kTileSlots + pw * 32 + lane;
      int idx = (int)t.base[(int64_t)slot * 2 + h];
      double a0 = 0.0, a1 = 0.0;
      for (int k = 0; k < nst; ++k, st = st + 1 == ps.nstb ? 0 : st + 1, ph ^= st == 0 ? 1u : 0u) {
        mbar_wait(bfull + st, ph);
#pragma unroll
        for (int q = 0; q < kBwdCG; ++q)
          rec_group(ringB + st * sbytes + (q * ncw + warp) * kRecBytes, lane, idx, sr, (q & 1) ? a1 : a0);
        __syncwarp();
        if (lane == 0) mbar_arrive(bempty + st);
      }
      const double v = a0 + a1;
      if (h > 0) part[pw * 32 + lane] = v;
      named_bar(3, ncw * 32);
      if (h == 0) {
        const double acc = v + part[pw * 32 + lane];
        const int32_t c = t.tcol[slot];
        if (!e.on) {
          if (c >= 0) g[c] = acc;
        } else {
          const int32_t c_first = __shfl_sync(0xffffffffu, c, 0);
          double q = 0.0;
          if (c >= 0 && c < d) {
            const double gc = acc / e.n_norm;
            double vv = e.anchor[c] - e.state->gamma * gc;
            if (e.set == 2 || e.set == 3) vv = vv > 0.0 ? vv : 0.0;
            const double df = (e.set == 1 && e.center) ? vv - e.center[c] : vv;
            q = df * df;
            e.v_scratch[c] = vv;
          }
          q = warp_sum(q);
          if (lane == 0 && c_first >= 0) {
            e.block_norm[c_first >> 5] = q;
            if (c_first == 0) e.state->loss_cur = 0.0;
          }
        }
      }
      named_bar(3, ncw * 32);  // part is rewritten by the next tile
    }
    named_bar(2, kPassGroup);  // the next tile's list buffer is ready; this one is free
    if (jj == 0) PASS_T(6);
  }
  PASS_T(7);
#ifdef POLY_PASS_TRACE
  if ((blockIdx.x == 0 || blockIdx.x == 100) && threadIdx.x == 0)
    printf("cta %d: F %.2f | bar1 %.2f | L %.2f | bar2 %.2f | gather0 %.2f | tile0 %.2f | tile1 %.2f us\n", blockIdx.x,
           (tr[1] - tr[0]) * 1e-3, (tr[2] - tr[1]) * 1e-3, (tr[3] - tr[2]) * 1e-3, (tr[4] - tr[3]) * 1e-3,
           (tr[5] - tr[4]) * 1e-3, (tr[6] - tr[5]) * 1e-3, (tr[7] - tr[6]) * 1e-3);
#endif
  pdl_trigger();
}

template <bool LOSS>
__global__ void __launch_bounds__(kPassWarps * 32, 1)
    k_ct_linkbwd(const StripFwd f, const TileBwd t, const CsrFwdArgs a, double *__restrict__ g, int32_t d,
                 const StepEpi e, const PassSync ps) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ double sp[3 * kMaxW];
  __shared__ double part[8 * 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#ifdef POLY_PASS_TRACE
  unsigned long long tr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  PASS_T(0);
  // region A: the strip (phase F) | two ray-list buffers (phase B)
  float *sx = (float *)smem;
  // region B: the forward ring (phase F) | the backward ring (phase B)
  uint8_t *ringB = smem + ps.abytes;
  uint64_t *bar = (uint64_t *)(ringB + ps.nstb * (kBwdCG * 2 * t.npw * kRecBytes));
  uint64_t *ffull = bar, *fempty = bar + kPassFwdStages;
  uint64_t *bfull = bar + 2 * kPassFwdStages, *bempty = bfull + kPassMaxBwdStages;
  int4 *desc = (int4 *)(bempty + kPassMaxBwdStages);
  const int ncw = 2 * t.npw;                    // backward consumer warps (<= 14)
  const int sbytes = kBwdCG * ncw * kRecBytes;  // one backward stage
  const int strip = blockIdx.x % f.NS;
  const int u0 = f.unit_start[strip], nu = f.unit_start[strip + 1] - u0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPassFwdStages; ++s) {
      mbar_init(ffull + s, 1);
      mbar_init(fempty + s, kFwdWarps);
    }
    for (int s = 0; s < ps.nstb; ++s) {
      mbar_init(bfull + s, 1);
      mbar_init(bempty + s, ncw);
    }
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 3 * kMaxW; i += blockDim.x) sp[i] = a.spec[i];
  __syncthreads();


  // tiles of this CTA: blockIdx.x, +gridDim.x, ...
  const int ntl = blockIdx.x < t.ntiles ? (t.ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  float *lbuf[2] = {(float *)smem, (float *)smem + ps.lcap};
  if (warp == kPassProdB) {
    // the backward producer: every tile's stages, in order, into the ring
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      int st = 0;
      uint32_t eph = 0;
      int64_t it = 0;
      for (int jj = 0; jj < ntl; ++jj) {
        const int tile = blockIdx.x + jj * gridDim.x;
        const int64_t G0 = t.tile_off[tile], ns = (t.tile_off[tile + 1] - G0) / kBwdCG;
        for (int64_t k = 0; k < ns; ++k) {
          if (it >= ps.nstb) mbar_wait(bempty + st, eph ^ 1);
          mbar_arrive_expect_tx(bfull + st, sbytes);
          bulk_g2s(ringB + st * sbytes, t.rec + bwd_stage_off(t, tile, G0, k), sbytes, bfull + st, pol);
          ++it;
          if (++st == ps.nstb) st = 0, eph ^= 1;
        }
      }
    }
    return;  // warp 15 takes no part in what follows
  }
  const int gt = threadIdx.x;  // 0 .. kPassGroup-1
  // the ray-list rows of the first two tiles (static)
  for (int jj = 0; jj < min(ntl, 2); ++jj) {
    const int tile = blockIdx.x + jj * gridDim.x;
    const int64_t L0 = t.list_off[tile];
    const int L = (int)(t.list_off[tile + 1] - L0);
    for (int i = 4 * gt; i < L; i += 4 * kPassGroup) cp_async16((int32_t *)lbuf[jj] + i, t.list + L0 + i);
  }
  pdl_wait();  // the forward kernel's pz
  PASS_T(2);
  if (blockIdx.x == 0 && gt < f.NS) f.ctr[gt] = 0;  // for the next pass's forward

  // ------------------------------------------------------------ phase L
  {
    const int64_t per = (a.n + gridDim.x - 1) / gridDim.x, r0 = per * blockIdx.x, r1 = min(a.n, r0 + per);
    double lacc = 0.0;
    for (int64_t base = r0; base < r1; base += 2 * kPassGroup) {
      double z[2] = {0.0, 0.0}, yv[2] = {0.0, 0.0}, Ii[2] = {a.I_bar, a.I_bar};
      const float *srow[2] = {nullptr, nullptr};
      int64_t row[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        row[q] = base + gt + q * kPassGroup;
        if (row[q] < r1) {
          for (int s = 0; s < f.NS; ++s) z[q] += __ldcg(f.pz + (int64_t)s * a.n + row[q]);
          if (a.ytype == 0) yv[q] = (double)((const int32_t *)a.y)[row[q]];
          else if (a.ytype == 1) yv[q] = (double)((const float *)a.y)[row[q]];
          else yv[q] = ((const double *)a.y)[row[q]];
          if (a.I_row) {
            Ii[q] = (double)a.I_row[row[q]];
            srow[q] = a.s_row + row[q] * a.W;
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (row[q] < r1) {
          double l;
          a.r[row[q]] = (float)row_residual_serial<LOSS>(sp, a.W, a.relu, z[q], yv[q], Ii[q], srow[q], &l, a.mode,
                                                         a.mu_step);
          lacc += l;
        }
      }
    }
    if (LOSS) {
      lacc = warp_sum(lacc);
      if (lane == 0) part[warp] = lacc;
      named_bar(2, kPassGroup);
      if (gt == 0) {
        double tl = 0.0;
        for (int w = 0; w < kPassGroup / 32; ++w) tl += part[w];
        a.loss_partials[blockIdx.x] = tl;
      }
    }
  }
  cp_async_wait_all();                   // (the list rows)
  PASS_T(3);
  pass_grid_barrier(ps, 2, kPassGroup);  // every r_i
  PASS_T(4);

  // ------------------------------------------------------------ phase B
  // r of tile 0 into buffer 0 by the whole group; later tiles are prepared by
  // warp 14 while the consumers stream the current one
  auto gather = [&](int jj, int t0, int nt) {
    const int tile = blockIdx.x + jj * gridDim.x;
    const int64_t L0 = t.list_off[tile];
    const int L = (int)(t.list_off[tile + 1] - L0);
    float *b = lbuf[jj & 1];
    if (jj >= 2) {  // the rows themselves first
      for (int i = 4 * t0; i < L; i += 4 * nt) cp_async16((int32_t *)b + i, t.list + L0 + i);
      cp_async_wait_all();
      __syncwarp();
    }
    for (int i = t0; i < L; i += nt) cp_async4(b + i, a.r + ((const int32_t *)b)[i]);
    cp_async_wait_all();
  };
  if (ntl > 0) gather(0, gt, kPassGroup);
  named_bar(2, kPassGroup);
  PASS_T(5);
  int st = 0;
  uint32_t ph = 0;
  for (int jj = 0; jj < ntl; ++jj) {
    const int tile = blockIdx.x + jj * gridDim.x;
    if (warp == 14) {
      if (jj + 1 < ntl) gather(jj + 1, lane, 32);
    } else if (warp < ncw) {
      const float *sr = lbuf[jj & 1];
      const int pw = warp % t.npw, h = warp / t.npw;
      const int64_t G0 = t.tile_off[tile];
      const int nst = (int)((t.tile_off[tile + 1] - G0) / kBwdCG);
      const int slot = tile * kTileSlots + pw * 32 + lane;
      int idx = (int)t.base[(int64_t)slot * 2 + h];
      double a0 = 0.0, a1 = 0.0;
      for (int k = 0; k < nst; ++k, st = st + 1 == ps.nstb ? 0 : st + 1, ph ^= st == 0 ? 1u : 0u) {
        mbar_wait(bfull + st, ph);
#pragma unroll
        for (int q = 0; q < kBwdCG; ++q)
          rec_group(ringB + st * sbytes + (q * ncw + warp) * kRecBytes, lane, idx, sr, (q & 1) ? a1 : a0);
        __syncwarp();
        if (lane == 0) mbar_arrive(bempty + st);
      }
      const double v = a0 + a1;
      if (h > 0) part[pw * 32 + lane] = v;
      named_bar(3, ncw * 32);
      if (h == 0) {
        const double acc = v + part[pw * 32 + lane];
        const int32_t c = t.tcol[slot];
        if (!e.on) {
          if (c >= 0) g[c] = acc;
        } else {
          const int32_t c_first = __shfl_sync(0xffffffffu, c, 0);
          double q = 0.0;
          if (c >= 0 && c < d) {
            const double gc = acc / e.n_norm;
            double vv = e.anchor[c] - e.state->gamma * gc;
            if (e.set == 2 || e.set == 3) vv = vv > 0.0 ? vv : 0.0;
            const double df = (e.set == 1 && e.center) ? vv - e.center[c] : vv;
            q = df * df;
            e.v_scratch[c] = vv;
          }
          q = warp_sum(q);
          if (lane == 0 && c_first >= 0) {
            e.block_norm[c_first >> 5] = q;
            if (c_first == 0) e.state->loss_cur = 0.0;
          }
        }
      }
      named_bar(3, ncw * 32);  // part is rewritten by the next tile
    }
    named_bar(2, kPassGroup);  // the next tile's list buffer is ready; this one is free
    if (jj == 0) PASS_T(6);
  }
  PASS_T(7);
#ifdef POLY_PASS_TRACE
  if ((blockIdx.x == 0 || blockIdx.x == 100) && threadIdx.x == 0)
    printf("cta %d: F %.2f | bar1 %.2f | L %.2f | bar2 %.2f | gather0 %.2f | tile0 %.2f | tile1 %.2f us\n", blockIdx.x,
           (tr[1] - tr[0]) * 1e-3, (tr[2] - tr[1]) * 1e-3, (tr[3] - tr[2]) * 1e-3, (tr[4] - tr[3]) * 1e-3,
           (tr[5] - tr[4]) * 1e-3, (tr[6] - tr[5]) * 1e-3, (tr[7] - tr[6]) * 1e-3);
#endif
  pdl_trigger();
}

}  // namespace poly
