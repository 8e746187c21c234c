// K4t — tiled CSR loss+gradient (fp32 A): both gathers from shared memory,
// both streams through TMA bulk copies.
//
// The compact SELL pair (csr.cuh, K4f/K4b) gathers x and r through L1/L2,
// and its dependent delta-load -> gather chains hold it at ~4.5 TB/s
// (DESIGN.md §7).  K4t re-blocks the caller's CSR once at poly_init so that
// every gather hits shared memory and the matrix is read as large contiguous
// bulk copies (plain per-warp LDG streams of the same bytes measured 3.7-5.0
// TB/s even with the gathers removed: too many short concurrent streams):
//
//   K4tf k_strip_forward   the image's columns are cut into NS strips of W
//                          columns; a CTA (one per SM) stages the fp32
//                          iterate of one strip (rows x P floats, P odd so
//                          that vertically adjacent pixels fall in different
//                          banks).  A producer lane takes units of 8 x 32 row
//                          segments (a row's entries inside the strip; lane =
//                          segment) off the strip's work counter and streams
//                          them into a 5-stage shared-memory ring with
//                          cp.async.bulk; 8 consumer warps walk their
//                          segments: entries ascending in the strip-local
//                          index as 8-bit deltas + fp32 values, 5 bytes per
//                          entry, one 640-byte record per warp-group (32
//                          delta words, then 32 float4).  Each segment's
//                          partial ⟨a_i, x⟩ goes to pz[strip][i].  Segments
//                          are sorted by length within a strip (~3 % padding
//                          instead of 16 %).
//   K4tl k_strip_link      z_i = Σ_strip pz[strip][i] (strip order), then the
//                          W-bin link and per-row scalar φ_i (one lane per
//                          row, four bins in flight), r_i (fp32), ℓ per block.
//   K4tb k_tile_backward   g_k = Σ_i a_ik r_i (Aᵀ r) over pixel
//                          tiles of 32 x 8 (one image row of 32 pixels per
//                          warp = one k_finalize block): the CTA stages r of
//                          the tile's sorted ray list in shared memory; a
//                          producer lane streams the tile's records (16 warps
//                          x 640 bytes per stage, 6 stages) while 16 consumer
//                          warps — two per pixel row, each a contiguous half
//                          of the row's entries — walk ascending rows as
//                          8-bit deltas into the list.  No atomics; fixed
//                          summation order (deterministic).
//
// Generic CSR: a non-square d is treated as one image row of d pixels (strips
// and tiles of consecutive columns).  poly_init falls back to the SELL pair
// when a delta does not fit 8 bits, a strip or ray list does not fit shared
// memory, or A is fp64.
#pragma once

#include "csr.cuh"

namespace poly {

constexpr int kTileSlots = 256;      // pixels per backward tile (32 x 8)
constexpr int kChunkRegs = 8;        // r chunks per backward thread held in registers across the wait
constexpr int kMaxStrips = 64;
constexpr int kRecBytes = 640;       // one warp-group: 32 x 4 B deltas + 32 x 16 B values
#ifndef POLY_FWD_WARPS
#define POLY_FWD_WARPS 12
#endif
#ifndef POLY_FWD_CG
#define POLY_FWD_CG 2
#endif
#ifndef POLY_BWD_CG
#define POLY_BWD_CG 1
#endif
constexpr int kFwdWarps = POLY_FWD_WARPS;  // forward consumer warps (+1 producer warp)
constexpr int kFwdCG = POLY_FWD_CG;        // group-rows per forward stage (units padded to a multiple)
#ifndef POLY_FWD_STAGES
#define POLY_FWD_STAGES 8             // 141 KB of the forward's records in flight per SM
#endif
#ifndef POLY_BWD_STAGES
#define POLY_BWD_STAGES 6
#endif
#ifndef POLY_FWD_PF
#define POLY_FWD_PF 0                 // L2 prefetch of the next unit
#endif
#ifndef POLY_BWD_PF
#define POLY_BWD_PF 0                // L2 prefetch this many stages ahead (<= stages: off)
#endif
#ifndef POLY_STRIP_KB
#define POLY_STRIP_KB 100              // largest iterate strip (shared memory), KB
#endif
// Records read with L2 evict-last (POLY_L2_KEEP_MB="fwd,bwd" overrides; experiments only).  Off: at C4 the
// gain was 0.4 us per pass at best, and with part of the backward's records evict-last 1-2 % of
// graph-replayed solves differed in their bits from run to run (0 of 2999 without; cause not found — see
// DESIGN.md §7), which breaks the path's determinism guarantee.
constexpr double kTiledKeepFwdMB = 0.0;
constexpr double kTiledKeepBwdMB = 0.0;
constexpr int kFwdStages = POLY_FWD_STAGES;
constexpr int kFwdHdr = kFwdWarps * 32 * 6;  // per unit: uint16 base[256], then int32 row[256]
constexpr int kFwdStageBytes = kFwdHdr + kFwdCG * kFwdWarps * kRecBytes;
constexpr int kBwdWarps = 16;        // backward consumer warps: 8 pixel rows x 2 halves (+1 producer)
constexpr int kBwdStages = POLY_BWD_STAGES;
constexpr int kBwdCG = POLY_BWD_CG;        // group-rows per backward stage (tiles padded to a multiple)
constexpr int kBwdStageBytes = kBwdCG * kBwdWarps * kRecBytes;
#ifndef POLY_TILE_CHAIN
#define POLY_TILE_CHAIN 4             // entries summed in fp32 before the fp64 accumulator (1: exact fp64 products)
#endif

struct StripFwd {
  const uint8_t *rec;        // unit U's group-row k of warp w: record ((unit_off[U] + k) * kFwdWarps + w)
  const uint8_t *hdr;        // [units][kFwdHdr]: strip-local index of each lane's first entry (uint16),
                             // then each lane's row (int32, -1: no segment)
  const int64_t *unit_off;   // [units + 1] first group-row of each unit
  const int32_t *unit_start; // [NS + 1] first unit of each strip
  int32_t *ctr;              // [NS] work counters (zeroed by the link kernel after every forward)
  double *pz;                // [NS][n] partial z (rows a strip does not touch stay 0)
  int64_t n;
  int32_t NS, rows_img, cols_img, W, P;
  int64_t xs_off;            // the fp32 iterate's strip copies: strip s at x[xs_off + s * SP] (finalize.cuh X32Strip)
  int32_t SP;                // floats per strip copy (rows_img * P rounded up to 4)
  int32_t keep;              // of every 1024 units of a strip, the first `keep` are read with L2 evict-last
                             // (they stay in L2 across passes: the solver re-reads the same A every pass)
};

struct TileBwd {
  const uint8_t *rec;        // tile t's group-row k of warp w (= half * 8 + pixel row): record
                             // ((tile_off[t] + k) * 2 * npw + w); zero records pad the shorter halves
  const int64_t *tile_off;   // [ntiles + 1] first group-row of each tile
  const uint16_t *base;      // [ntiles * 256][2] list position before each half's first entry
  const int32_t *list;       // per tile, the aligned float4 chunks of r its rays touch (r's float4 index,
                             // ascending); an entry's position = 4 * chunk + (row & 3)
  const int64_t *list_off;   // [ntiles + 1]
  const int32_t *tcol;       // [ntiles * 256] column of each slot, -1: none
  int32_t ntiles;
  int32_t npw;               // pixel warps per tile (TW * TH / 32); 2 * npw consumer warps
  int32_t interleave;        // 1: stage k of every tile stored together ([k][tile]: the CTAs' bulk
                             // copies walk one contiguous region), 0: tile-major
  int32_t keep;              // of every 1024 stages of a tile, the first `keep` are read with L2 evict-last
};

// byte offset of stage k of tile t (first group-row G0 in the tile-major form)
__device__ __forceinline__ int64_t bwd_stage_off(const TileBwd &t, int tile, int64_t G0, int64_t k) {
  return (t.interleave ? k * t.ntiles + tile : G0 / kBwdCG + k) * ((int64_t)kBwdCG * 2 * t.npw * kRecBytes);
}

// L2 prefetch of a contiguous range through the TMA engine (no shared memory):
// the ring's bulk copies then find their bytes in L2
__device__ __forceinline__ void bulk_prefetch_l2(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_all;" ::: "memory");
}

__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// one 640-byte record in shared memory: this lane's four deltas and values,
// gathered against s[] from idx (advanced)
__device__ __forceinline__ void rec_group(const uint8_t *rec, int lane, int &idx, const float *__restrict__ s,
                                          double &acc) {
  const uint32_t dd = *(const uint32_t *)(rec + lane * 4);
  const float4 v = *(const float4 *)(rec + 128 + lane * 16);
  const int i0 = idx + (int)(dd & 0xffu), i1 = i0 + (int)((dd >> 8) & 0xffu);
  const int i2 = i1 + (int)((dd >> 16) & 0xffu), i3 = i2 + (int)(dd >> 24);
  idx = i3;
#if POLY_TILE_CHAIN == 4
  float q = v.x * s[i0];
  q = fmaf(v.y, s[i1], q);
  q = fmaf(v.z, s[i2], q);
  q = fmaf(v.w, s[i3], q);
  acc += (double)q;
#else
  acc = fma((double)v.x, (double)s[i0], acc);
  acc = fma((double)v.y, (double)s[i1], acc);
  acc = fma((double)v.z, (double)s[i2], acc);
  acc = fma((double)v.w, (double)s[i3], acc);
#endif
}

// the link and per-row scalar of one row in this lane (group8_residual's
// quantities), four bins in flight, partial sums combined in a fixed order
// mu_step != 0: μ_j = μ_0 + j·mu_step (an arithmetic progression, checked at
// poly_init): e^{-μ_j z} from the smallest-μ bin by a ratio e^{-|mu_step| z}
// (exact algebra; rounding grows by one ulp per bin), two exponentials per
// row instead of W.
template <bool LOSS>
__device__ __forceinline__ double row_residual_serial(const double *sp, int W, int relu, double z, double yv,
                                                      double Ii, const float *srow, double *l_out, int mode,
                                                      double mu_step = 0.0) {
  const bool neg = relu && z < 0.0;
  const double zc = neg ? 0.0 : z;
  double hs[4] = {0.0, 0.0, 0.0, 0.0}, Hs[4] = {0.0, 0.0, 0.0, 0.0}, hp[4] = {0.0, 0.0, 0.0, 0.0};
  const bool geo = mu_step != 0.0 && (relu || mode == 0);
  double eg = 0.0, rg = 1.0;  // geometric: the current bin's exponential and the ratio
  if (geo) {
    const int j0 = mu_step < 0.0 ? W - 1 : 0;  // the smallest μ
    eg = exp_nonpos<POLY_EXP_DEG32>(-sp[kMaxW + j0] * zc);
    rg = exp_nonpos<POLY_EXP_DEG32>(-fabs(mu_step) * zc);
  }
  auto bin = [&](int j, int q) {
    const double sj = srow ? (double)srow[j] : sp[j];
    double e;
    if (geo) {
      e = eg;
      eg *= rg;
    } else {
      e = (relu || mode == 0) ? exp_nonpos<POLY_EXP_DEG32>(-sp[kMaxW + j] * zc) : exp(-sp[kMaxW + j] * z);
    }
    hs[q] = fma(sj, e, hs[q]);
    if (mode == 0) {
      if (LOSS) Hs[q] += neg ? sj * z : sj * sp[2 * kMaxW + j] * (1.0 - e);
    } else {
      hp[q] = fma(sj * sp[kMaxW + j], e, hp[q]);
    }
  };
  if (geo && mu_step < 0.0) {
    // smallest μ last: walk the bins downwards (accumulators as in the upward walk)
    int j = W - 1;
    for (; j >= 3; j -= 4) {
#pragma unroll
      for (int q = 0; q < 4; ++q) bin(j - q, q);
    }
    for (; j >= 0; --j) bin(j, 0);
  } else {
    int j = 0;
    for (; j + 4 <= W; j += 4) {
#pragma unroll
      for (int q = 0; q < 4; ++q) bin(j + q, q);
    }
    for (; j < W; ++j) bin(j, 0);
  }
  const double hst = (hs[0] + hs[1]) + (hs[2] + hs[3]);
  const double Hst = (Hs[0] + Hs[1]) + (Hs[2] + Hs[3]);
  double hpt = (hp[0] + hp[1]) + (hp[2] + hp[3]);
  double phi, l;
  if (mode == 0) {
    phi = yv - Ii * hst;
    l = yv * z - Ii * Hst;
  } else {
    hpt = (relu && !(z > 0.0)) ? 0.0 : -hpt;
    const double m = Ii * hst;
    if (mode == 1) {
      phi = 2.0 * (m - yv) * Ii * hpt;
      l = (m - yv) * (m - yv);
    } else if (mode == 2) {
      const double rr = m - yv;
      phi = (rr > 0.0 ? 1.0 : (rr < 0.0 ? -1.0 : 0.0)) * Ii * hpt;
      l = fabs(rr);
    } else {
      phi = (Ii - yv / hst) * hpt;
      l = m - yv * log(m);
    }
  }
  *l_out = LOSS ? l : 0.0;
  return phi;
}

// K4tf: grid = one CTA per SM (rounded to a multiple of NS), CTA b serves strip b % NS.
__global__ void __launch_bounds__((kFwdWarps + 1) * 32, 1) k_strip_forward(const StripFwd f,
                                                                           const float *__restrict__ x) {
  extern __shared__ __align__(128) uint8_t smem[];
  float *sx = (float *)smem;
  uint8_t *stg = smem + ((f.SP * 4 + 127) & ~127);
  uint64_t *full = (uint64_t *)(stg + kFwdStages * kFwdStageBytes);
  uint64_t *empty = full + kFwdStages;
  int4 *desc = (int4 *)(empty + kFwdStages);
  uint64_t *xbar = (uint64_t *)(desc + kFwdStages);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int strip = blockIdx.x % f.NS;
  const int u0 = f.unit_start[strip], nu = f.unit_start[strip + 1] - u0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kFwdStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kFwdWarps);
    }
    mbar_init(xbar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == kFwdWarps) {
    // producer: units off the strip's counter, their header + records into the ring
    if (lane == 0) {
      const uint64_t pol_first = l2_evict_first_policy(), pol_last = l2_evict_last_policy();
      // (starting the ring before the wait — records are static — measured
      // slower in the graph: 126 vs 118 us per C4 step)
      pdl_wait();  // the counter is reset by the previous link kernel, x written by the step kernel
      // the strip's iterate: one bulk copy of its strip-layout fp32 copy (the
      // strip's other CTAs read the same bytes: kept in L2)
      pdl_proxy_fence();
      mbar_arrive_expect_tx(xbar, (uint32_t)f.SP * 4);
      bulk_g2s(sx, x + f.xs_off + (int64_t)strip * f.SP, (uint32_t)f.SP * 4, xbar, l2_evict_last_policy());
      int it = 0, st = 0;
      uint32_t eph = 0;  // stage index and the ring's pass parity (incremental: no division)
      int u = atomicAdd(f.ctr + strip, 1);
      auto prefetch_unit = [&](int uu) {
        if (POLY_FWD_PF && uu < nu) {
          const int64_t UU = (int64_t)u0 + uu, a0 = f.unit_off[UU], a1 = f.unit_off[UU + 1];
          bulk_prefetch_l2(f.hdr + UU * kFwdHdr, kFwdHdr);
          bulk_prefetch_l2(f.rec + a0 * kFwdWarps * kRecBytes, (uint32_t)((a1 - a0) * kFwdWarps * kRecBytes));
        }
      };
      prefetch_unit(u);
      for (;;) {
        const bool done = u >= nu;
        const int un = done ? nu : atomicAdd(f.ctr + strip, 1);  // the next unit, prefetched while this one streams
        const int64_t U = (int64_t)u0 + u;
        const int64_t g0 = done ? 0 : f.unit_off[U], ng = done ? 1 : f.unit_off[U + 1] - g0;
        const uint64_t pol = (int64_t)u * 1024 < (int64_t)f.keep * nu ? pol_last : pol_first;
        for (int64_t k = 0; k < ng; k += kFwdCG) {
          if (k == kFwdCG) prefetch_unit(un);
          if (it >= kFwdStages) mbar_wait(empty + st, eph ^ 1);
          const int c = done ? 0 : kFwdCG;  // units are padded to a multiple of kFwdCG group-rows
          desc[st] = make_int4(done ? -1 : u, (int)k, c, (k == 0 ? 1 : 0) | (k + c >= ng ? 2 : 0));
          uint8_t *sb = stg + st * kFwdStageBytes;
          if (done) {
            mbar_arrive(full + st);
          } else {
            const uint32_t data = (uint32_t)c * kFwdWarps * kRecBytes;
            mbar_arrive_expect_tx(full + st, data + (k == 0 ? kFwdHdr : 0));
            if (k == 0) bulk_g2s(sb, f.hdr + U * kFwdHdr, kFwdHdr, full + st, pol);
            bulk_g2s(sb + kFwdHdr, f.rec + (g0 + k) * kFwdWarps * kRecBytes, data, full + st, pol);
          }
          ++it;
          if (++st == kFwdStages) st = 0, eph ^= 1;
        }
        if (done) break;
        if (ng <= kFwdCG) prefetch_unit(un);
        u = un;
      }
    }
    return;
  }
  // consumers: the strip (rows_img x P floats, columns >= W zero) arrives on xbar
  mbar_wait(xbar, 0);
  pdl_trigger();
  int idx = 0, row = -1;
  double a0 = 0.0, a1 = 0.0;
  int st = 0;
  uint32_t ph = 0;
  for (;; st = st + 1 == kFwdStages ? 0 : st + 1, ph ^= st == 0 ? 1u : 0u) {
    mbar_wait(full + st, ph);
    const int4 dsc = desc[st];
    if (dsc.x < 0) break;
    const uint8_t *sb = stg + st * kFwdStageBytes;
    if (dsc.w & 1) {
      idx = ((const uint16_t *)sb)[warp * 32 + lane];
      row = ((const int32_t *)(sb + kFwdWarps * 32 * 2))[warp * 32 + lane];
      a0 = a1 = 0.0;
    }
    const uint8_t *rb = sb + kFwdHdr + warp * kRecBytes;
#pragma unroll
    for (int k = 0; k < kFwdCG; ++k) rec_group(rb + k * kFwdWarps * kRecBytes, lane, idx, sx, (k & 1) ? a1 : a0);
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);
    if ((dsc.w & 2) && row >= 0) f.pz[(int64_t)strip * f.n + row] = a0 + a1;
  }
}

// K4tl: z_i from the strips' partials (strip order), the link and φ_i; one
// lane per row; ℓ per block (fixed grid: deterministic).
template <bool LOSS>
__global__ void __launch_bounds__(256, 4) k_strip_link(const CsrFwdArgs a, const double *__restrict__ pz, int32_t NS,
                                                       int32_t *ctr) {
  __shared__ double sp[3 * kMaxW];
  __shared__ double part[4][32];
  for (int i = threadIdx.x; i < 3 * kMaxW; i += blockDim.x) sp[i] = a.spec[i];
  __syncthreads();
  pdl_wait();  // the forward's partials
  if (blockIdx.x == 0 && threadIdx.x < NS) ctr[threadIdx.x] = 0;  // for the next forward
  // The backward is launched when this kernel's CTAs exit, not earlier: with the trigger here (so that the
  // backward's prologue and ring fill overlap the link, ~0.8 us per pass) 1-2 % of graph-replayed solves
  // differed in their bits once the backward's first stages came from L2 (POLY_L2_KEEP_MB), and none in
  // 1499 without the overlap; -DPOLY_LINK_EARLY=1 restores the early trigger.
#if defined(POLY_LINK_EARLY) && POLY_LINK_EARLY
  pdl_trigger();
#endif
  double lacc = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < a.n;
       row += (int64_t)gridDim.x * blockDim.x) {
    double z = 0.0, yv, Ii = a.I_bar;
    for (int s = 0; s < NS; ++s) z += ld_prev(pz + (int64_t)s * a.n + row);
    if (a.ytype == 0) yv = (double)((const int32_t *)a.y)[row];
    else if (a.ytype == 1) yv = (double)((const float *)a.y)[row];
    else yv = ((const double *)a.y)[row];
    const float *srow = nullptr;
    if (a.I_row) {
      Ii = (double)a.I_row[row];
      srow = a.s_row + row * a.W;
    }
    double l;
    a.r[row] = (float)row_residual_serial<LOSS>(sp, a.W, a.relu, z, yv, Ii, srow, &l, a.mode, a.mu_step);
    lacc += l;
  }
  block_loss_n(part, lacc, a.loss_partials, blockDim.x >> 5);
}

// K4tb: one CTA per tile.  Dynamic shared memory: the ring, the ray list
// (staged as row indices, then overwritten in place by r), the barriers.
__global__ void __launch_bounds__((kBwdWarps + 1) * 32, 1)
    k_tile_backward(const TileBwd t, const float *__restrict__ r, double *__restrict__ g, int32_t d,
                    const StepEpi e, int32_t lcap) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ double part[8 * 32];
  const int ncw = 2 * t.npw;                       // consumer warps
  const int sbytes = kBwdCG * ncw * kRecBytes;     // one stage
  uint8_t *stg = smem;
  float *sr = (float *)(smem + kBwdStages * sbytes);
  uint64_t *full = (uint64_t *)(sr + lcap);
  uint64_t *empty = full + kBwdStages;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x;
  const int64_t G0 = t.tile_off[tile], ng = t.tile_off[tile + 1] - G0;
  if (tid == 0) {
    for (int s = 0; s < kBwdStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, ncw);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == ncw) {
    // producer: the tile's records are static — streaming starts before the wait
    if (lane == 0) {
      const uint64_t pol_first = l2_evict_first_policy(), pol_last = l2_evict_last_policy();
#ifdef POLY_BWD_LATE
      pdl_wait();  // (experiment) no streaming before the link kernel has completed
#endif
      const int64_t ns = ng / kBwdCG;
      const int64_t nkeep = (ns * t.keep + 1023) >> 10;
      if (POLY_BWD_PF > kBwdStages && ns > kBwdStages)
        for (int64_t q = kBwdStages; q < min(ns, (int64_t)POLY_BWD_PF); ++q)
          bulk_prefetch_l2(t.rec + bwd_stage_off(t, tile, G0, q), sbytes);
      int st = 0;
      uint32_t eph = 0;
      for (int64_t k = 0; k < ns; ++k, st = st + 1 == kBwdStages ? 0 : st + 1, eph ^= st == 0 ? 1u : 0u) {
        if (POLY_BWD_PF > kBwdStages && k + POLY_BWD_PF < ns)
          bulk_prefetch_l2(t.rec + bwd_stage_off(t, tile, G0, k + POLY_BWD_PF), sbytes);
        if (k >= kBwdStages) mbar_wait(empty + st, eph ^ 1);
        mbar_arrive_expect_tx(full + st, sbytes);
        bulk_g2s(stg + st * sbytes, t.rec + bwd_stage_off(t, tile, G0, k), sbytes, full + st,
                 k < nkeep ? pol_last : pol_first);
      }
    }
    return;
  }
  const int pw = warp % t.npw, h = warp / t.npw;
  // r of the tile's rays, staged as whole aligned float4 chunks of r (the
  // rays through a tile are runs of consecutive rows, one per view): the
  // chunk table is static, read before the wait; after it one 16-byte load
  // and store per chunk (per-element cp.async gathers cost 8 LSU cycles each)
  const int nthr = ncw * 32;
  const int64_t C0 = t.list_off[tile];
  const int nc = (int)(t.list_off[tile + 1] - C0);
  int32_t csrc[kChunkRegs];
#pragma unroll
  for (int q = 0; q < kChunkRegs; ++q) {
    const int c = tid + q * nthr;
    csrc[q] = c < nc ? t.list[C0 + c] : 0;
  }
  const int slot = tile * kTileSlots + pw * 32 + lane;
  int idx = (int)t.base[(int64_t)slot * 2 + h];
  pdl_wait();  // r is written by the link kernel
  const float4 *r4 = (const float4 *)r;
  float4 *sr4 = (float4 *)sr;
#pragma unroll
  for (int q = 0; q < kChunkRegs; ++q) {
    const int c = tid + q * nthr;
    if (c < nc) sr4[c] = __ldcg(r4 + csrc[q]);
  }
  for (int c = tid + kChunkRegs * nthr; c < nc; c += nthr) sr4[c] = __ldcg(r4 + t.list[C0 + c]);
  named_bar(1, nthr);
  double a0 = 0.0, a1 = 0.0;
  const int nst = (int)(ng / kBwdCG);
  int st = 0;
  uint32_t ph = 0;
  for (int k = 0; k < nst; ++k, st = st + 1 == kBwdStages ? 0 : st + 1, ph ^= st == 0 ? 1u : 0u) {
    mbar_wait(full + st, ph);
#pragma unroll
    for (int q = 0; q < kBwdCG; ++q)
      rec_group(stg + st * sbytes + (q * ncw + warp) * kRecBytes, lane, idx, sr, (q & 1) ? a1 : a0);
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);
  }
  const double v = a0 + a1;
  if (h > 0) part[pw * 32 + lane] = v;
  named_bar(1, ncw * 32);
  if (h > 0) {
    pdl_trigger();
    return;
  }
  const double acc = v + part[pw * 32 + lane];
  const int32_t c = t.tcol[slot];
  if (!e.on) {
    if (c >= 0) g[c] = acc;
  } else {
    // the plain-step epilogue (csr.cuh StepEpi): this warp's 32 columns are
    // one k_finalize block (poly_init checks), same arithmetic, same bits
    const int32_t c_first = __shfl_sync(0xffffffffu, c, 0);
    double q = 0.0;
    if (c >= 0 && c < d) {
      const double gc = acc / e.n_norm;
      double vv = ld_prev(e.anchor + c) - e.state->gamma * gc;
      if (e.set == 2 || e.set == 3) vv = vv > 0.0 ? vv : 0.0;
      const double df = (e.set == 1 && e.center) ? vv - e.center[c] : vv;
      q = df * df;
      e.v_scratch[c] = vv;
    }
    q = warp_sum(q);
    if (lane == 0 && c_first >= 0) {
      e.block_norm[c_first >> 5] = q;
      if (c_first == 0) e.state->loss_cur = 0.0;  // as k_finalize without the objective
    }
  }
  pdl_trigger();
}

// ------------------------------------------------------------ build (poly_init)
// Image geometry shared by the build kernels: d = rows_img x cols_img
// (row-major pixels; rows_img = 1 for a non-square d).
struct TiledGeom {
  int32_t rows_img, cols_img;
  int32_t NS, W, P;          // strips
  int32_t TW, TH, tiles_x;   // tiles: TW x TH pixels (32 x 8, or 256 x 1 for one image row)
  int32_t lb, rb, pb;        // sort-key field widths: strip-local index, row, ray-list position
};

__device__ __forceinline__ void strip_of(const TiledGeom &m, int32_t col, int32_t &strip, int32_t &loc) {
  const int32_t r = col / m.cols_img, c = col - r * m.cols_img;
  strip = c / m.W;
  loc = r * m.P + (c - strip * m.W);
}

__device__ __forceinline__ void tile_of(const TiledGeom &m, int32_t col, int32_t &tile, int32_t &slot) {
  const int32_t r = col / m.cols_img, c = col - r * m.cols_img;
  tile = (r / m.TH) * m.tiles_x + c / m.TW;
  slot = (r % m.TH) * m.TW + c % m.TW;
}

// forward sort keys (strip | row | local index) and the segment lengths
__global__ void k_tf_keys(const int32_t *rows, const int32_t *col, int64_t nnz, int64_t n, TiledGeom m,
                          uint64_t *key, int32_t *perm, int32_t *seglen) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t s, loc;
    strip_of(m, col[e], s, loc);
    const uint32_t r = (uint32_t)rows[e];
    key[e] = ((uint64_t)s << (m.rb + m.lb)) | ((uint64_t)r << m.lb) | (uint64_t)loc;
    perm[e] = (int32_t)e;
    // one atomic per (warp, segment): a row's entries are adjacent in the CSR
    const int64_t sg = (int64_t)s * n + r;
    const unsigned peers = __match_any_sync(__activemask(), sg);
    if ((__ffs(peers) - 1) == (int)(threadIdx.x & 31)) atomicAdd(seglen + sg, __popc(peers));
  }
}

// first sorted position of every segment
__global__ void k_tf_segstart(const uint64_t *ks, int64_t nnz, int64_t n, TiledGeom m, int64_t *segstart) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t q = ks[k] >> m.lb;
    if (k == 0 || (ks[k - 1] >> m.lb) != q)
      segstart[(int64_t)(q >> m.rb) * n + (int64_t)(q & ((1ull << m.rb) - 1))] = k;
  }
}

// per strip: segments longest first (a unit's first lane holds its longest
// segment; ties by row), rows the strip does not touch last; segments per strip
__global__ void k_tf_order_keys(const int32_t *seglen, int64_t n, int32_t NS, uint64_t *key, int32_t *rowv,
                                int32_t *nz) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)NS * n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = (int32_t)(i / n);
    const int32_t len = seglen[i];
    key[i] = ((uint64_t)s << 32) | (uint64_t)(len > 0 ? (uint32_t)(0x7fffffff - len) : 0xffffffffu);
    rowv[i] = (int32_t)(i - (int64_t)s * n);
    if (len > 0) atomicAdd(nz + s, 1);
  }
}

// groups of every unit (its first lane holds the longest segment)
__global__ void k_tf_unitlen(const int32_t *unit_start, int32_t NS, const int32_t *srow, const int32_t *seglen,
                             int64_t n, int64_t units, int64_t *ulen) {
  for (int64_t U = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; U <= units; U += (int64_t)gridDim.x * blockDim.x) {
    if (U == units) {
      ulen[U] = 0;
      continue;
    }
    int s = 0;
    while (s + 1 < NS && unit_start[s + 1] <= U) ++s;
    const int64_t i = (int64_t)s * n + (U - unit_start[s]) * (kFwdWarps * 32);
    const int64_t g = (seglen[(int64_t)s * n + srow[i]] + 3) / 4;
    ulen[U] = (g + kFwdCG - 1) / kFwdCG * kFwdCG;
  }
}

// one warp per (unit, warp), lane = segment: header and records
__global__ void k_tf_pack(const int32_t *unit_start, int32_t NS, const int32_t *srow, const int32_t *seglen,
                          const int32_t *nz, const int64_t *segstart, const uint64_t *ks, const int32_t *perm,
                          const float *val, int64_t n, int64_t units, const int64_t *unit_off, TiledGeom m,
                          uint8_t *rec, uint8_t *hdr, int32_t *overflow) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < units * kFwdWarps; q += nw) {
    const int64_t U = q / kFwdWarps;
    const int w = (int)(q % kFwdWarps);
    int s = 0;
    while (s + 1 < NS && unit_start[s + 1] <= U) ++s;
    const int64_t j = (U - unit_start[s]) * (kFwdWarps * 32) + w * 32 + lane;
    int32_t row = -1, len = 0;
    int64_t st = 0;
    if (j < nz[s]) {
      row = srow[(int64_t)s * n + j];
      len = seglen[(int64_t)s * n + row];
      st = segstart[(int64_t)s * n + row];
    }
    const uint64_t lmask = (1ull << m.lb) - 1;
    int32_t prev = len > 0 ? (int32_t)(ks[st] & lmask) : 0;
    ((uint16_t *)(hdr + U * kFwdHdr))[w * 32 + lane] = (uint16_t)prev;
    ((int32_t *)(hdr + U * kFwdHdr + kFwdWarps * 32 * 2))[w * 32 + lane] = row;
    const int64_t g0 = unit_off[U], ng = unit_off[U + 1] - g0;
    for (int64_t g = 0; g < ng; ++g) {
      uint32_t dd = 0;
      float v4[4];
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) {
        const int64_t k = 4 * g + qq;
        v4[qq] = 0.f;
        if (k < len) {
          const int32_t loc = (int32_t)(ks[st + k] & lmask);
          const int32_t dlt = loc - prev;
          if (dlt < 0 || dlt > 255) atomicOr(overflow, 1);
          dd |= (uint32_t)(dlt & 0xff) << (8 * qq);
          prev = loc;
          v4[qq] = val[perm[st + k]];
        }
      }
      uint8_t *rp = rec + ((g0 + g) * kFwdWarps + w) * kRecBytes;
      ((uint32_t *)rp)[lane] = dd;
      ((float4 *)(rp + 128))[lane] = make_float4(v4[0], v4[1], v4[2], v4[3]);
    }
  }
}

// backward sort keys (tile | row | slot)
__global__ void k_tb_keys(const int32_t *rows, const int32_t *col, int64_t nnz, TiledGeom m, uint64_t *key,
                          int32_t *perm) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t t, sl;
    tile_of(m, col[e], t, sl);
    key[e] = ((uint64_t)t << (m.rb + 8)) | ((uint64_t)(uint32_t)rows[e] << 8) | (uint64_t)sl;
    perm[e] = (int32_t)e;
  }
}

// first entry of every (tile, r chunk) pair — a chunk = 4 rows i with the
// same i >> 2 (one aligned float4 of r); chunks per tile
__global__ void k_tb_pairs(const uint64_t *ks, int64_t nnz, TiledGeom m, int32_t *flag, int32_t *tcnt) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const int sh = 8 + min(2, m.rb);  // (tile, row >> 2)
    const bool f = k == 0 || (ks[k - 1] >> sh) != (ks[k] >> sh);
    flag[k] = f ? 1 : 0;
    // one atomic per (warp, tile): sorted neighbours share the tile
    const int64_t t = (int64_t)(ks[k] >> (m.rb + 8));
    const unsigned act = __activemask();
    const unsigned peers = __match_any_sync(act, f ? t : (int64_t)-1);
    const int c = __popc(peers & __ballot_sync(act, f));
    if (f && (__ffs(peers & __ballot_sync(act, f)) - 1) == (int)(threadIdx.x & 31)) atomicAdd(tcnt + t, c);
  }
}

// chunk tables (r's float4 index of each chunk a tile's rays touch, ascending)
// and the second sort's keys (tile*256 + slot | position of the row in the
// tile's staged r: 4 * chunk + (row & 3))
__global__ void k_tb_list(const uint64_t *ks, const int32_t *pidx, const int32_t *flag, const int64_t *pstart,
                          const int64_t *list_off, int64_t nnz, TiledGeom m, int32_t *list, uint64_t *key2) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t q = ks[k];
    const int64_t t = (int64_t)(q >> (m.rb + 8));
    const int64_t ci = (int64_t)pidx[k] - 1 - pstart[t];  // inclusive scan of flag: chunk within the tile
    const int32_t row = (int32_t)((q >> 8) & ((1ull << m.rb) - 1));
    if (flag[k]) list[list_off[t] + ci] = row >> 2;
    key2[k] = ((uint64_t)(t * kTileSlots + (int64_t)(q & 0xffu)) << m.pb) | (uint64_t)(4 * ci + (row & 3));
  }
}

// entries and first position per (tile, slot)
__global__ void k_tb_slots(const uint64_t *ks2, int64_t nnz, TiledGeom m, int32_t *cnt, int64_t *start) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t q = ks2[k] >> m.pb;
    atomicAdd(cnt + q, 1);
    if (k == 0 || (ks2[k - 1] >> m.pb) != q) start[q] = k;
  }
}

// groups per pixel row = longest of its 32 slots
__global__ void k_tb_warplen(const int32_t *cnt, int64_t nwarps, int64_t *wlen) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nwarps; w += (int64_t)gridDim.x * blockDim.x) {
    int32_t m = 0;
    for (int l = 0; l < 32; ++l) m = max(m, cnt[w * 32 + l]);
    wlen[w] = (m + 3) / 4;
  }
}

// group-rows per tile: the longest half of its 8 pixel rows
__global__ void k_tb_tilelen(const int64_t *wlen, int64_t ntiles, int64_t *tlen) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= ntiles; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t m = 0;
    if (t < ntiles)
      for (int w = 0; w < 8; ++w) m = max(m, (wlen[t * 8 + w] + 1) / 2);
    tlen[t] = (m + kBwdCG - 1) / kBwdCG * kBwdCG;
  }
}

// one warp per (tile, pixel row), lane = slot: records of both halves, the
// halves' bases; also the slot -> column map
__global__ void k_tb_pack(const uint64_t *ks2, const int32_t *perm2, const float *val, const int32_t *cnt,
                          const int64_t *start, const int64_t *wlen, const int64_t *tile_off, int64_t nwarps,
                          TiledGeom m, int32_t d, uint8_t *rec, uint16_t *base, int32_t *tcol, int32_t *overflow,
                          int32_t interleave, int32_t npw) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < nwarps; w += nw) {
    const int64_t q = w * 32 + lane;  // tile * 256 + slot
    const int64_t t = q / kTileSlots;
    const int pw = (int)(w % 8);
    const int32_t sl = (int32_t)(q % kTileSlots);
    const int64_t r = (t / m.tiles_x) * m.TH + sl / m.TW, c = (t % m.tiles_x) * m.TW + sl % m.TW;
    const int64_t col = r * m.cols_img + c;
    tcol[q] = (r < m.rows_img && c < m.cols_img && col < d) ? (int32_t)col : -1;
    const int32_t len = cnt[q];
    const int64_t st = len > 0 ? start[q] : 0;
    const uint64_t pmask = (1ull << m.pb) - 1;
    int32_t prev = len > 0 ? (int32_t)(ks2[st] & pmask) : 0;
    if (prev > 65535) atomicOr(overflow, 4);
    const int64_t ng = wlen[w], per = (ng + 1) / 2;  // half 0: groups [0, per), half 1: [per, ng)
    base[q * 2] = (uint16_t)prev;
    base[q * 2 + 1] = (uint16_t)prev;  // (ng <= per: the second half is all padding)
    for (int64_t g = 0; g < ng; ++g) {
      if (g == per) base[q * 2 + 1] = (uint16_t)prev;
      const int64_t hh = g < per ? 0 : 1, k = g - hh * per;
      uint32_t dd = 0;
      float v4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t e = 4 * g + j;
        v4[j] = 0.f;
        if (e < len) {
          const int32_t pos = (int32_t)(ks2[st + e] & pmask);
          const int32_t dlt = pos - prev;
          if (dlt < 0 || dlt > 255) atomicOr(overflow, 2);
          dd |= (uint32_t)(dlt & 0xff) << (8 * j);
          prev = pos;
          v4[j] = val[perm2[st + e]];
        }
      }
      const int64_t ntl = nwarps / 8;
      const int64_t ncw = 2 * npw;
      const int64_t ri = interleave ? ((k / kBwdCG) * ntl + t) * (kBwdCG * ncw) + (k % kBwdCG) * ncw
                                    : (tile_off[t] + k) * ncw;
      uint8_t *rp = rec + (ri + hh * npw + pw) * kRecBytes;
      ((uint32_t *)rp)[lane] = dd;
      ((float4 *)(rp + 128))[lane] = make_float4(v4[0], v4[1], v4[2], v4[3]);
    }
  }
}

}  // namespace poly
