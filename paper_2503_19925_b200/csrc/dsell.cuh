// K4 on "DSELL": SELL-32 slices with a per-slice dictionary of the vector
// entries they touch, staged in shared memory, and one-byte local deltas.
//
// Both passes of K4 (forward z = A x, backward g = Aᵀ r; Eq. operator,
// PAPER.md:893-896, Aᵀ form PAPER.md:57) gather one fp32 vector entry per
// nonzero.  On the SELL16 form (csr.cuh) a warp's 32 gathers touch 10-17
// different 32-byte sectors (ncu: 9.6 / 16.9 sectors per request), so the
// L1 sector pipe, not HBM, bounds both passes (55-58 % of DRAM peak).  Here
// every slice — 32 consecutive rows (forward) or columns (backward), lanes =
// rows / columns — carries the sorted set F_s of vector indices its nonzeros
// touch, as runs (global start, local base).  A block first stages F_s of x
// (forward) or r (backward) into shared memory with coalesced cp.async
// copies out of L2, then streams the slice's nonzeros and gathers from
// shared memory.  With the targets replaced by local indices into F_s, the
// steps of a lane (ascending target) advance by small amounts — for the CT
// matrix by 1 along a ray within an image row or within a view, by a run
// length between rows / views — so a step is one byte of delta plus the fp32
// value: 5 bytes per nonzero instead of 6.
//
// Stream layout per slice (G groups of 4 steps): dl[(goff + g)*32 + lane]
// (uchar4: the deltas of steps 4g..4g+3) and val[...] (float4).  Warp w of the
// 12-warp block takes the contiguous groups [w G/12, (w+1) G/12) and starts
// its chain at base[(slice*12 + w)*32 + lane] (uint16: the running local index
// before its first step).  Blocks are persistent (two per SM) and stage the
// next slice's dictionary (cp.async, double-buffered) while they stream the
// current one, so the L2 latency of the staging stays off the critical path.  A gap > 255 is bridged by filler steps (delta 255, value
// 0); padding steps after a lane's last nonzero carry (0, 0).  A lane's local
// index always stays inside [0, |F_s|), so every gather is a valid read and
// padding adds exact zeros.
#pragma once

#include "csr.cuh"  // CscEnt, CsrFwdArgs, forward_tail, block_loss, StepEpi

namespace poly {

struct DSell {
  const uchar4 *dl;          // [groups * 32]
  const float4 *val;         // [groups * 32]
  const uint16_t *base;      // [nslices * kDsWarps * 32]
  const int64_t *goff;       // [nslices + 1] slice start, in groups
  const int2 *runs;          // per slice nruns + 1 entries {global start, local base}; last = {0, |F_s|}
  const int64_t *run_off;    // [nslices + 1]
};

constexpr int kDsWarps = 12;   // warps per block = chunks of a slice (2 blocks per SM: <= 85 registers)
constexpr int kDsThreads = 32 * kDsWarps;
constexpr int kDsPackThreads = 256;
constexpr int kDsMaxWords = 16384;  // bitmap words per slice in the pack kernel (target span <= 524288)
constexpr size_t kDsPackSmem = (size_t)2 * kDsMaxWords * 4;  // dynamic: bits + word prefixes

// ------------------------------------------------------------------ staging
// Issue the copies of F_s of src (global fp32 vector) into fp[0, |F_s|)
// (cp.async, not waited for here): warp w takes runs w*32 .. w*32+31, then
// every 12*32-th block of runs; each lane reads one run entry (coalesced), the
// warp walks the 32 runs through shuffles and its lanes copy run elements.
__device__ __forceinline__ void ds_stage_async(const DSell &s, int64_t sl, const float *__restrict__ src,
                                               float *fp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = s.run_off[sl], r1 = s.run_off[sl + 1] - 1;  // the last entry is the sentinel
  for (int64_t rb = r0 + warp * 32; rb < r1; rb += kDsWarps * 32) {
    int2 R = make_int2(0, 0);
    int len = 0;
    if (rb + lane < r1) {
      R = s.runs[rb + lane];
      len = s.runs[rb + lane + 1].y - R.y;
    }
    const int m = (int)(r1 - rb < 32 ? r1 - rb : 32);
    for (int j = 0; j < m; ++j) {
      const int st = __shfl_sync(0xffffffffu, R.x, j), bs = __shfl_sync(0xffffffffu, R.y, j);
      const int ln = __shfl_sync(0xffffffffu, len, j);
      for (int l = lane; l < ln; l += 32) cp_async4(fp + bs + l, src + st + l);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// this warp's chunk of the slice, loaded into registers in batches of up to
// kDsBatch groups (all loads of a batch issued before any use), then
// Σ val * fp[idx] in fp64 from the staged dictionary.  ds_load issues the
// first batch; ds_dot consumes it (and loads further batches if the chunk is
// longer), so the HBM latency of the stream overlaps the dictionary staging.
constexpr int kDsBatch = 8;
struct DsRegs {
  uchar4 dd[kDsBatch];
  float4 vv[kDsBatch];
};

__device__ __forceinline__ void ds_load(const DSell &s, int64_t g0, int64_t g, int64_t qb, int lane, DsRegs &r) {
#pragma unroll
  for (int u = 0; u < kDsBatch; ++u) {
    const int64_t gi = (g0 + g + u) * 32 + lane;
    if (g + u < qb) {
      r.dd[u] = __ldcs(s.dl + gi);
      r.vv[u] = __ldcs(s.val + gi);
    } else {
      r.dd[u] = make_uchar4(0, 0, 0, 0);
      r.vv[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

__device__ __forceinline__ void ds_chunk(const DSell &s, int64_t sl, int warp, int64_t *g0, int64_t *qa,
                                         int64_t *qb) {
  *g0 = s.goff[sl];
  const int64_t G = s.goff[sl + 1] - *g0;
  *qa = warp * G / kDsWarps;
  *qb = (warp + 1) * G / kDsWarps;
}

__device__ __forceinline__ double ds_dot(const DSell &s, int64_t sl, int warp, int lane, const float *fp,
                                         DsRegs &r) {
  int64_t g0, qa, qb;
  ds_chunk(s, sl, warp, &g0, &qa, &qb);
  int32_t idx = s.base[(sl * kDsWarps + warp) * 32 + lane];
  double a0 = 0.0, a1 = 0.0;
  for (int64_t g = qa; g < qb; g += kDsBatch) {
    if (g != qa) ds_load(s, g0, g, qb, lane, r);
#pragma unroll
    for (int u = 0; u < kDsBatch; ++u) {
      const int32_t i0 = idx + r.dd[u].x, i1 = i0 + r.dd[u].y, i2 = i1 + r.dd[u].z, i3 = i2 + r.dd[u].w;
      idx = i3;
      a0 = fma((double)r.vv[u].x, (double)fp[i0], a0);
      a1 = fma((double)r.vv[u].y, (double)fp[i1], a1);
      a0 = fma((double)r.vv[u].z, (double)fp[i2], a0);
      a1 = fma((double)r.vv[u].w, (double)fp[i3], a1);
    }
  }
  return a0 + a1;
}

// the kDsWarps chunk partials of lane `lane`, in warp order
__device__ __forceinline__ double ds_sum(double (*part)[32], int lane) {
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < kDsWarps; ++w) t += part[w][lane];
  return t;
}

// ------------------------------------------------------------------ build (poly_init)
// One block per slice (grid-stride).  Inputs: the padded SELL-32 copy ent
// (step-major, lane-minor; entries of a lane ascending in target), the lane
// lengths (row_ptr differences, or the column counts cnt).  COUNT mode writes
// |F_s|, nruns and the group count G per slice; WRITE mode (given the scanned
// offsets) writes runs, deltas, values and bases.  *bad != 0: a slice's
// target span exceeds the bitmap (the caller keeps the SELL16 form).
template <bool WRITE>
__global__ void __launch_bounds__(kDsPackThreads) k_dsell_pack(
    const CscEnt<float> *ent, const int64_t *slice_off, int64_t nslices, const int64_t *row_ptr,
    const int32_t *cnt, int64_t nlanes, int64_t *fp_len, int64_t *nruns, int64_t *ngroups,
    const int64_t *goff, const int64_t *run_off, uchar4 *dl, float4 *val, uint16_t *base, int2 *runs,
    int32_t *bad) {
  extern __shared__ uint32_t ds_pack_smem[];
  uint32_t *bits = ds_pack_smem, *pre = ds_pack_smem + kDsMaxWords;
  __shared__ int32_t s_min, s_max;
  __shared__ uint32_t s_tot[2][kDsPackThreads];
  __shared__ int32_t s_lmax;
  const int tid = threadIdx.x;
  for (int64_t sl = blockIdx.x; sl < nslices; sl += gridDim.x) {
    const int64_t o0 = slice_off[sl], len = slice_off[sl + 1] - o0;
    auto lane_len = [&](int lane) -> int64_t {
      const int64_t li = sl * 32 + lane;
      if (li >= nlanes) return 0;
      return row_ptr ? row_ptr[li + 1] - row_ptr[li] : (int64_t)cnt[li];
    };
    if (tid == 0) {
      s_min = INT32_MAX;
      s_max = -1;
      s_lmax = 0;
    }
    __syncthreads();
    // a) target span
    int32_t mn = INT32_MAX, mx = -1;
    for (int64_t f = tid; f < len * 32; f += blockDim.x) {
      const int64_t k = f >> 5;
      const int lane = (int)(f & 31);
      if (k < lane_len(lane)) {
        const int32_t t = ent[(o0 + k) * 32 + lane].row;
        mn = min(mn, t);
        mx = max(mx, t);
      }
    }
    atomicMin(&s_min, mn);
    atomicMax(&s_max, mx);
    __syncthreads();
    const int32_t tmin = s_min, tmax = s_max;
    const bool empty = tmax < 0;
    const int nwords = empty ? 0 : (int)((tmax - tmin) / 32 + 1);
    if (nwords > kDsMaxWords) {
      if (tid == 0) atomicOr(bad, 1);
      __syncthreads();
      continue;
    }
    // b) bitmap of the targets
    for (int w = tid; w < nwords; w += blockDim.x) bits[w] = 0u;
    __syncthreads();
    for (int64_t f = tid; f < len * 32; f += blockDim.x) {
      const int64_t k = f >> 5;
      const int lane = (int)(f & 31);
      if (k < lane_len(lane)) {
        const int32_t t = ent[(o0 + k) * 32 + lane].row - tmin;
        atomicOr(&bits[t >> 5], 1u << (t & 31));
      }
    }
    __syncthreads();
    // c) per-word exclusive prefix of the popcounts (rank), and run starts
    const int cw = (nwords + blockDim.x - 1) / blockDim.x;
    const int wa = min(nwords, tid * cw), wb = min(nwords, wa + cw);
    uint32_t pc = 0, rc = 0;
    for (int w = wa; w < wb; ++w) {
      const uint32_t x = bits[w];
      const uint32_t carry = w > 0 ? (bits[w - 1] >> 31) : 0u;
      pc += __popc(x);
      rc += __popc(x & ~((x << 1) | carry));
    }
    s_tot[0][tid] = pc;
    s_tot[1][tid] = rc;
    __syncthreads();
    if (tid == 0) {  // serial scan of 256 chunk sums (build time only)
      uint32_t a = 0, b = 0;
      for (int i = 0; i < (int)blockDim.x; ++i) {
        const uint32_t x = s_tot[0][i], y = s_tot[1][i];
        s_tot[0][i] = a;
        s_tot[1][i] = b;
        a += x;
        b += y;
      }
      if (!WRITE) {
        fp_len[sl] = a;
        nruns[sl] = b;
      }
    }
    __syncthreads();
    {
      uint32_t a = s_tot[0][tid], b = s_tot[1][tid];
      for (int w = wa; w < wb; ++w) {
        const uint32_t x = bits[w];
        pre[w] = a;
        if (WRITE) {
          const uint32_t carry = w > 0 ? (bits[w - 1] >> 31) : 0u;
          uint32_t st = x & ~((x << 1) | carry);
          while (st) {
            const int bpos = __ffs(st) - 1;
            st &= st - 1;
            const uint32_t loc = a + __popc(x & ((1u << bpos) - 1u));
            runs[run_off[sl] + b] = make_int2(tmin + w * 32 + bpos, (int)loc);
            ++b;
          }
        }
        a += __popc(x);
      }
    }
    __syncthreads();
    auto rank = [&](int32_t t) -> int32_t {
      const int32_t u = t - tmin;
      return (int32_t)(pre[u >> 5] + __popc(bits[u >> 5] & ((1u << (u & 31)) - 1u)));
    };
    // d) the lanes' delta chains (warp 0, one lane per row / column)
    if (tid < 32) {
      const int lane = tid;
      const int64_t ll = lane_len(lane);
      if (!WRITE) {
        int64_t steps = 0;
        int32_t prev = 0;
        for (int64_t k = 0; k < ll; ++k) {
          const int32_t li = rank(ent[(o0 + k) * 32 + lane].row);
          const int32_t dlt = li - prev;
          steps += 1 + (dlt > 255 ? (dlt - 1) / 255 : 0);
          prev = li;
        }
        atomicMax(&s_lmax, (int32_t)steps);
      } else {
        const int64_t g0 = goff[sl], G = goff[sl + 1] - g0;
        unsigned char *db = reinterpret_cast<unsigned char *>(dl);
        float *vb = reinterpret_cast<float *>(val);
        int64_t st = 0;
        int32_t run_idx = 0;
        int w_next = 0;
        auto emit = [&](int32_t delta, float v) {
          while (w_next < kDsWarps && st == (w_next * G / kDsWarps) * 4) {  // chunk start: the chain's state
            base[(sl * kDsWarps + w_next) * 32 + lane] = (uint16_t)run_idx;
            ++w_next;
          }
          const int64_t gi = (g0 + st / 4) * 32 + lane;
          db[gi * 4 + (st & 3)] = (unsigned char)delta;
          vb[gi * 4 + (st & 3)] = v;
          run_idx += delta;
          ++st;
        };
        for (int64_t k = 0; k < ll; ++k) {
          const CscEnt<float> e = ent[(o0 + k) * 32 + lane];
          int32_t dlt = rank(e.row) - run_idx;
          while (dlt > 255) {
            emit(255, 0.0f);
            dlt -= 255;
          }
          emit(dlt, e.val);
        }
        while (st < 4 * G) emit(0, 0.0f);
        while (w_next < kDsWarps) base[(sl * kDsWarps + w_next++) * 32 + lane] = (uint16_t)run_idx;
      }
    }
    __syncthreads();
    if (!WRITE && tid == 0) ngroups[sl] = (s_lmax + 3) / 4;
    if (WRITE && tid == 0) {
      const int64_t nrun = run_off[sl + 1] - run_off[sl] - 1;
      uint32_t tot = 0;
      for (int w = 0; w < nwords; ++w) tot += __popc(bits[w]);
      runs[run_off[sl] + nrun] = make_int2(0, (int)tot);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ K4f / K4b on DSELL
// Persistent blocks of 12 warps (two per SM), slices sl = blockIdx.x +
// k * gridDim.x; shared memory holds two dictionary buffers of fp_cap floats:
// slice k+1 is staged into one while slice k is streamed from the other.
template <bool LOSS>
__global__ void __launch_bounds__(kDsThreads, 2) k_dsell_forward(const DSell s, int64_t nslices, int32_t fp_cap,
                                                                 const CsrFwdArgs a) {
  extern __shared__ __align__(16) float ds_buf[];
  __shared__ double sp[3 * kMaxW];
  __shared__ double part[kDsWarps][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cap = (fp_cap + 3) & ~3;
  for (int i = threadIdx.x; i < 3 * kMaxW; i += blockDim.x) sp[i] = a.spec[i];
  pdl_wait();  // x is written by the previous kernel; r is read by the previous backward
  double lacc = 0.0;
  int k = 0;
  if ((int64_t)blockIdx.x < nslices) ds_stage_async(s, blockIdx.x, a.x, ds_buf);
  for (int64_t sl = blockIdx.x; sl < nslices; sl += gridDim.x, ++k) {
    const int64_t nx = sl + gridDim.x;
    if (nx < nslices) ds_stage_async(s, nx, a.x, ds_buf + ((k + 1) & 1) * cap);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    DsRegs rg;
    {
      int64_t g0, qa, qb;
      ds_chunk(s, sl, warp, &g0, &qa, &qb);
      ds_load(s, g0, qa, qb, lane, rg);  // the stream does not depend on the dictionary
    }
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // this slice's copies (own); barrier: everyone's
    __syncthreads();
    part[warp][lane] = ds_dot(s, sl, warp, lane, ds_buf + (k & 1) * cap, rg);
    __syncthreads();
    if (warp == 0) {  // z_i = the chunk sums in warp order; forward_tail adds part[0..3][row]
      const double z = ds_sum(part, lane);
      part[0][lane] = z;
      part[1][lane] = part[2][lane] = part[3][lane] = 0.0;
    }
    __syncthreads();
    if (warp < 4) lacc += forward_tail<LOSS>(part, sp, a, sl);
    __syncthreads();  // part and this buffer are reused
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  block_loss_n(part, lacc, a.loss_partials, kDsWarps);
  pdl_trigger();
}

__global__ void __launch_bounds__(kDsThreads, 2) k_dsell_backward(const DSell s, int64_t nslices, int32_t fp_cap,
                                                                  int32_t d, const float *__restrict__ r,
                                                                  double *__restrict__ g, const StepEpi e) {
  extern __shared__ __align__(16) float ds_buf[];
  __shared__ double part[kDsWarps][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cap = (fp_cap + 3) & ~3;
  pdl_wait();  // r is written by the forward pass
  int k = 0;
  if ((int64_t)blockIdx.x < nslices) ds_stage_async(s, blockIdx.x, r, ds_buf);
  for (int64_t sl = blockIdx.x; sl < nslices; sl += gridDim.x, ++k) {
    const int64_t nx = sl + gridDim.x;
    if (nx < nslices) ds_stage_async(s, nx, r, ds_buf + ((k + 1) & 1) * cap);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    DsRegs rg;
    {
      int64_t g0, qa, qb;
      ds_chunk(s, sl, warp, &g0, &qa, &qb);
      ds_load(s, g0, qa, qb, lane, rg);
    }
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    part[warp][lane] = ds_dot(s, sl, warp, lane, ds_buf + (k & 1) * cap, rg);
    __syncthreads();
    if (warp == 0) {
      const double v = ds_sum(part, lane);
      part[0][lane] = v;
      part[1][lane] = part[2][lane] = part[3][lane] = 0.0;
      backward_column_out(part, e, g, d, sl, lane);
    }
    __syncthreads();
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  pdl_trigger();
}

}  // namespace poly
