// Whole-solve kernel for small dense problems (C1-sized: n·d up to ~50k
// elements per CTA): EXACT, Eq.(extragrad-method), runs all
// T iterations inside ONE thread-block cluster with A resident in shared
// memory.  A C1 iteration through the general path is four kernel launches
// (two K1 passes + two step kernels, ~17 µs even graph-replayed with PDL);
// here an F evaluation costs one cluster barrier.
//
// Each of the CL CTAs holds a contiguous block of rows of A (and y) in shared
// memory for the whole solve.  Per F evaluation at the point x:
//   warps take rows round-robin: z_i = <a_i, x> (fp64 lane partials, warp
//   sum), the link and per-row scalar (row_residual: the same quantities as
//   K1), g_warp += r_i a_i in fp64 registers; the CTA's warps are combined in
//   order into this CTA's partial, which is pushed (st.async) into slot row
//   `rank` of every CTA, completing on that CTA's mbarrier; every CTA then
//   sums the CL rows in rank order (identical bits in every CTA), scales by
//   1/n and applies the step and projection itself, so the iterate is
//   replicated without another exchange.  Slots are double-buffered by
//   evaluation parity (see the loop).
#pragma once

#include <cooperative_groups.h>

#include <type_traits>

#include "dense.cuh"
#include "tv.cuh"  // st.async / cluster mbarrier helpers

namespace poly {

constexpr int kSmallThreads = 512;
constexpr int kSmallMaxD = 256;   // fp64 g accumulators per lane: d / 32 <= 8
constexpr int kSmallMaxCL = 16;

struct SmallArgs {
  const void *A;        // [n][lda] global
  int64_t lda;
  int32_t n, d, W, ytype, relu, mode, set;
  const void *y;
  double I_bar, R, gamma;
  int64_t n_norm;       // the n of Eq.(operator)
  const double *spec;   // [3*kMaxW]
  const double *center; // [d] or null
  double *x;            // [d] in: x_in, out: x_{T+1}
  int32_t T;
  double *trace;        // [2T] or null: ℓ at each evaluation point
  SolveState *state;    // bad flag
};

__device__ __forceinline__ void cl_bar() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// x_out = P_X(v) on the block (every thread of the CTA participates); returns ||v - c||.
__device__ double small_project(const SmallArgs &a, double *v, double *x_out, double *red) {
  const int d = a.d;
  double q = 0.0;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    double vc = v[c];
    if (a.set == 2 || a.set == 3) vc = vc > 0.0 ? vc : 0.0;
    v[c] = vc;
    const double df = (a.set == 1 && a.center) ? vc - a.center[c] : vc;
    q += df * df;
  }
  q = warp_sum(q);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = q;
  __syncthreads();
  double nr = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) nr += red[w];
  const double nrm = sqrt(nr);
  double scale = 1.0;
  if ((a.set == 1 || a.set == 3) && nrm > a.R) scale = a.R / nrm;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    const double vc = v[c];
    if (a.set == 1) {
      const double ck = a.center ? a.center[c] : 0.0;
      x_out[c] = scale == 1.0 ? vc : ck + (vc - ck) * scale;
    } else {
      x_out[c] = vc * scale;
    }
  }
  __syncthreads();  // red and x_out complete
  return nrm;
}

template <typename T, bool LOSS>
__global__ void __launch_bounds__(kSmallThreads, 1) k_small_solve(const SmallArgs a) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) unsigned char ssm[];
  cg::cluster_group cl = cg::this_cluster();
  const int CL = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NWp = kSmallThreads / 32;
  const int d = a.d;
  const int r0 = (int)((int64_t)a.n * rank / CL), r1 = (int)((int64_t)a.n * (rank + 1) / CL);
  const int rows = r1 - r0;
  const int ldd = (d + 1) & ~1;  // smem row pitch (elements), 8-byte aligned rows for double
  // every CTA lays out its shared memory for the largest block, ceil(n / CL)
  // rows, so that the arrays sit at the same offsets in every CTA: remote
  // pushes address the receiver's slots and mbarriers by the sender's offsets
  const int rows_cap = (a.n + CL - 1) / CL;
  T *As = reinterpret_cast<T *>(ssm);
  double *ys = reinterpret_cast<double *>(As + (size_t)rows_cap * ldd + ((size_t)rows_cap * ldd & 1));
  double *sp = ys + rows_cap;                    // [3*kMaxW]
  double *xa = sp + 3 * kMaxW;                   // [d] anchor x_t
  double *xe = xa + kSmallMaxD;                  // [d] evaluation point
  double *vv = xe + kSmallMaxD;                  // [d] step vector
  double *part = vv + kSmallMaxD;                // [2][d + 1] partial g and loss (double-buffered)
  double *wp = part + 2 * (kSmallMaxD + 1);      // [NWp][d + 1]
  double *red = wp + NWp * (kSmallMaxD + 1);     // [NWp]
  uint64_t *mbar = reinterpret_cast<uint64_t *>(red + NWp);  // [2]
  double *slots = reinterpret_cast<double *>(mbar + 2);       // [2][CL][d + 1] pushed partials
  // A block, y, spectrum, x_1 = P_X(x_in)
  for (int i = threadIdx.x; i < rows * d; i += blockDim.x) {
    const int r = i / d, c = i - r * d;
    As[(size_t)r * ldd + c] = ((const T *)a.A)[(int64_t)(r0 + r) * a.lda + c];
  }
  for (int i = threadIdx.x; i < rows; i += blockDim.x) ys[i] = load_y_global(a.y, a.ytype, r0 + i);
  for (int i = threadIdx.x; i < 3 * kMaxW; i += blockDim.x) sp[i] = a.spec[i];
  for (int c = threadIdx.x; c < d; c += blockDim.x) vv[c] = a.x[c];
  if (threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_mbar_init();
  }
  cl_bar();  // every CTA's mbarriers exist before the first push
  small_project(a, vv, xa, red);
  for (int c = threadIdx.x; c < d; c += blockDim.x) xe[c] = xa[c];
  __syncthreads();
  const double inv_n = 1.0 / (double)a.n_norm;
  int bad = 0;
  for (int e = 0; e < 2 * a.T; ++e) {
    // ---- one F evaluation at xe (this CTA's rows)
    double gacc[kSmallMaxD / 32];
#pragma unroll
    for (int k = 0; k < kSmallMaxD / 32; ++k) gacc[k] = 0.0;
    double lacc = 0.0;
    constexpr int DEG = std::is_same<T, double>::value ? 13 : 9;
    const bool pairs = a.mode == 0 && a.W <= 32;
    int r = warp;
    if (pairs) {
      // two rows per pass: one butterfly for both dots, one 16-lane link each
      for (; r + NWp < rows; r += 2 * NWp) {
        const T *ar0 = As + (size_t)r * ldd, *ar1 = As + (size_t)(r + NWp) * ldd;
        double p0 = 0.0, p1 = 0.0;
#pragma unroll
        for (int k = 0; k < kSmallMaxD / 32; ++k) {
          const int c = lane + 32 * k;
          if (c < d) {
            const double xc = xe[c];
            p0 = fma((double)ar0[c], xc, p0);
            p1 = fma((double)ar1[c], xc, p1);
          }
        }
        const double zh = pair_sum(p0, p1);
        const int hr = (lane & 16) ? r + NWp : r;
        const double rh = link_exact_pair<LOSS, DEG>(sp, a.W, a.relu, zh, ys[hr], a.I_bar, nullptr,
                                                      true, &lacc);
        const double phi0 = __shfl_sync(0xffffffffu, rh, 0), phi1 = __shfl_sync(0xffffffffu, rh, 16);
#pragma unroll
        for (int k = 0; k < kSmallMaxD / 32; ++k) {
          const int c = lane + 32 * k;
          if (c < d) gacc[k] = fma(phi1, (double)ar1[c], fma(phi0, (double)ar0[c], gacc[k]));
        }
      }
    }
    for (; r < rows; r += NWp) {
      const T *ar = As + (size_t)r * ldd;
      double p = 0.0;
#pragma unroll
      for (int k = 0; k < kSmallMaxD / 32; ++k) {
        const int c = lane + 32 * k;
        if (c < d) p = fma((double)ar[c], xe[c], p);
      }
      const double z = warp_sum(p);
      const double phi = a.mode == 0
                             ? link_exact<LOSS, DEG>(sp, a.W, a.relu, z, ys[r], a.I_bar, nullptr, true, &lacc)
                             : row_residual<LOSS>(sp, a.W, a.relu, z, ys[r], a.I_bar, nullptr, true, &lacc,
                                                  a.mode);
#pragma unroll
      for (int k = 0; k < kSmallMaxD / 32; ++k) {
        const int c = lane + 32 * k;
        if (c < d) gacc[k] = fma(phi, (double)ar[c], gacc[k]);
      }
    }
    double *wrow = wp + (size_t)warp * (kSmallMaxD + 1);
#pragma unroll
    for (int k = 0; k < kSmallMaxD / 32; ++k) {
      const int c = lane + 32 * k;
      if (c < d) wrow[c] = gacc[k];
    }
    if (lane == 0) wrow[kSmallMaxD] = lacc;
    __syncthreads();
    // ---- this CTA's partial (warps in order), pushed to every CTA's slot row
    // `rank` with st.async completing on the receiver's mbarrier (no cluster
    // barrier); slots alternate by evaluation parity — a CTA can only push
    // evaluation e+2 after every CTA pushed e+1, i.e. after it finished
    // reading the slots of e
    const int q = e & 1, D1 = d + 1;
    const uint32_t sb = smem_u32(slots) + 8u * (uint32_t)((q * CL + rank) * D1), mb = smem_u32(&mbar[q]);
    for (int c = threadIdx.x; c <= kSmallMaxD; c += blockDim.x) {
      if (c < d || c == kSmallMaxD) {
        double s = 0.0;
        for (int w = 0; w < NWp; ++w) s += wp[(size_t)w * (kSmallMaxD + 1) + c];
        const uint32_t off = 8u * (uint32_t)(c < d ? c : d);
        for (int r = 0; r < CL; ++r) st_async_f64(mapa_u32(sb + off, r), s, mapa_u32(mb, r));
      }
    }
    if (threadIdx.x == 0) mbar_expect_tx(mb, (uint32_t)(CL * D1 * 8));
    mbar_wait_cluster(mb, (uint32_t)((e >> 1) & 1));
    // ---- sum over the cluster in rank order, step from the anchor, project
    const double *sq = slots + (size_t)q * CL * D1;
    for (int c = threadIdx.x; c <= d; c += blockDim.x) {
      double s = 0.0;
      for (int r = 0; r < CL; ++r) s += sq[(size_t)r * D1 + c];
      if (c < d) vv[c] = xa[c] - a.gamma * (s * inv_n);
      else if (LOSS && rank == 0 && a.trace) a.trace[e] = s * inv_n;
    }
    __syncthreads();
    const bool half = (e & 1) == 0;  // x_{t+1/2} from x_t, then x_{t+1} from x_t
    const double nrm = small_project(a, vv, half ? xe : xa, red);
    if (!isfinite(nrm) && !bad) bad = e + 1;
    if (!half) {
      for (int c = threadIdx.x; c < d; c += blockDim.x) xe[c] = xa[c];
      __syncthreads();
    }
  }
  if (rank == 0) {
    for (int c = threadIdx.x; c < d; c += blockDim.x) a.x[c] = xa[c];
    if (threadIdx.x == 0 && bad && a.state->bad == 0) a.state->bad = bad;
  }
  cl_bar();  // no CTA exits while others may still read its partials
}

}  // namespace poly
