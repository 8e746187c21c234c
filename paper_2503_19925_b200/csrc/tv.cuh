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
// B200 mapping: a thread-block cluster of CL CTAs does the whole projection
// — Dykstra, the λ search and every FISTA iteration — with the image split into
// CL row bands (s <= 256).  Each CTA keeps its band's prox input z, primal x,
// extrapolated primal xw and momentum duals w in shared memory (rows of pitch
// SC) and the duals u in registers (tv_prox); inside the FISTA loop the band
// edges and the reductions (||Δx||, ||x||) travel as st.async pushes that
// complete on the receiver's mbarrier — no cluster barrier per iteration —
// and every sum is a fixed tree, so all CTAs take identical branch decisions.
// Outside the loop (TV norms, Dykstra) the reductions use cluster_sum.
// Dykstra's state (z_k, p, q) lives in global memory (L2).  No kernel
// launches inside.  K such clusters (one grid) run the λ search K values at a
// time (reading R22: round of K evaluations, K = 1 the paper's bisection):
// cluster c computes the prox at the c-th λ of the round, the clusters meet
// at a global-memory barrier, read the K TV values in order and all take the
// same decision; the selected cluster broadcasts its prox through global
// memory.  Every cluster keeps its own copy of the Dykstra state and runs the
// identical (deterministic) sweep, so no other exchange is needed.
#pragma once

#include <cooperative_groups.h>

#include <type_traits>

#include "common.cuh"

namespace poly {

namespace cg = cooperative_groups;

constexpr int kTvThreads = 512;
constexpr int kTvMaxCL = 16;
constexpr int kTvMaxK = 16;  // λ values per search round (clusters)

struct TvArgs {
  const double *v;     // [d] point to project
  double *out;         // [d] P_X(v)
  double *zk, *p, *q;  // [d] Dykstra state (global, L2-resident)
  int32_t s;           // image side, d = s*s
  int32_t nonneg;      // 1: X1 ∩ X2 by Dykstra; 0: X1 only
  double tau, tv_tol, rtol, tol;
  int32_t max_it, max_outer;
  int32_t *stats;      // optional [4]: Dykstra sweeps, search rounds, FISTA iterations (totals),
                       // [3] set to 1 if the clusters failed to meet (not co-resident)
  SolveState *state;   // optional: non-finite flag (bad = -2) for the solver
  // k-ary λ search (reading R22): K clusters evaluate K values of λ per round
  int32_t K;
  double *tv_vals;     // [2][K] TV of each cluster's prox, by round parity (global)
  unsigned int *gbar;  // cross-cluster barrier counter (zeroed before every launch)
  double *xsel;        // [d] the selected prox, broadcast to the other clusters
  unsigned long long timeout_ns;  // bound on every cross-cluster wait
  int32_t warm;        // 1: each prox starts FISTA from the previous prox's duals (reading R23)
  double *u_state;     // [K][2][d] duals (horizontal, vertical) per pixel, per cluster (warm starts)
};

constexpr int kTvMaxRpt = 8;
#ifndef POLY_TV_CHUNK
#define POLY_TV_CHUNK 1
#endif
constexpr int kTvChunk = POLY_TV_CHUNK;  // rows whose loads tv_prox issues together  // band rows per thread (s <= 256: at most 16 rows over >= 2 row groups)

// shared doubles of tv_prox's edge buffers
__host__ __device__ inline int tv_edge_doubles(int s) {
  const int SC = (s + 31) & ~31, H = kTvThreads / SC;
  return H * SC + H * kTvMaxRpt * (SC / 32);
}

struct TvBand {
  int s, r0, r1, npx, rank, CL;
  int SC, H, RPT;                          // row pitch of the band arrays (s rounded up to 32) and
                                           // tv_prox's thread map (row groups, rows each)
  double *z, *x, *xw, *wh, *wv;            // [rows][SC] band arrays (shared; padding columns 0)
  double *edge;                            // tv_prox's edge buffers
  double *red;                             // [2][4] this CTA's cluster-reduction slots
  double *wsum;                            // [warps * 4]
  double *tot;                             // [4] reduced totals
  int parity;
  // tv_prox's point-to-point exchange (shared): mbarriers red[2], up[2], dn[2];
  // red_slots[2][kTvMaxCL][2], halo_up[2][SC][2] (u_v, w_v of the previous
  // band's last row), halo_dn[2][SC] (xw of the next band's first row); the
  // buffer and phase of each use follow from counts every CTA shares
  uint64_t *mbar;
  double *xs;
  uint32_t n_red, n_a, n_b;  // reductions, phase-A and phase-B executions (same in every CTA)
  double *ush, *usv;         // warm starts: this cluster's duals per global pixel (NULL: cold)
};

// shared bytes of tv_prox's exchange area (after the reduction scratch)
__host__ __device__ inline int tv_xchg_bytes(int s) {
  const int SC = (s + 31) & ~31;
  return 6 * 8 + 8 + (2 * kTvMaxCL * 2 + 2 * SC * 2 + 2 * SC) * 8;  // (+8: 16-byte alignment)
}

__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// remote (cluster) shared-memory stores completing on the target CTA's mbarrier
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr), "d"(v),
               "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async_v2f64(uint32_t raddr, double a, double b, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "d"(a), "d"(b), "r"(rbar)
               : "memory");
}
// wait for phase `parity` of a local mbarrier completed by remote st.async
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAITC_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

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
  const int R = b.r1 - b.r0;
  for (int i = threadIdx.x; i < R * b.SC; i += blockDim.x) {
    const int lr = i / b.SC, c = i - lr * b.SC;
    if (c >= b.s) continue;
    if (c + 1 < b.s) acc[0] += fabs(b.x[i + 1] - b.x[i]);
    if (b.r0 + lr + 1 < b.s) {
      const double below = (lr + 1 < R) ? b.x[i + b.SC] : next_x[c];
      acc[0] += fabs(below - b.x[i]);
    }
  }
  cluster_sum<1>(cl, b, acc);
  return acc[0];
}

// TV prox of b.z with parameter lam (FISTA on the dual, oracle_prox_tv's
// iteration); leaves x = z - Dᵀu in b.x.  Returns the FISTA iterations.
//
// Thread map: thread t owns column c = t % SC (SC = s rounded up to 32) of
// RPT consecutive band rows starting at h*RPT (h = t / SC) and keeps its
// duals u (horizontal, vertical) in registers; w, z, x and xw are band arrays
// in shared memory (row pitch SC, lanes on consecutive columns:
// conflict-free).  Horizontal neighbours of u and xw come from shuffles (the
// warp-edge columns through small shared buffers), vertical ones from the
// thread's own next row, the row group above/below or — for the band's edge
// rows — the halo the neighbouring CTA pushed.  The boundary rules are data
// (no per-pixel branches); see the loop.
// the dynamic shared memory of k_tv_project
extern __shared__ __align__(16) double tv_smem[];

// fp64 shared-memory array addressed from tv_smem by an element offset, so
// the compiler knows the address space inside tv_prox (not inlined; generic
// pointers would make every access a 64-bit generic load).
struct SmemF64 {
  double *p;
  __device__ explicit SmemF64(int off) : p(tv_smem + off) {}
  __device__ __forceinline__ double ld(int i) const { return p[i]; }
  __device__ __forceinline__ void st(int i, double v) const { p[i] = v; }
};

// clip to [-h, h] (h >= 0); fmin/fmax cost ~12 instructions each for fp64
__device__ __forceinline__ double tv_clip(double v, double h) {
  v = v > h ? h : v;
  return v < -h ? -h : v;
}

// rows per thread for pitch SC: bands of at most ceil(SC/16) rows over 512/SC row groups
__host__ __device__ constexpr int tv_mr(int SC) { return ((SC + 15) / 16 + kTvThreads / SC - 1) / (kTvThreads / SC); }

template <int SC, bool WARM>
__device__ int tv_prox(cg::cluster_group &cl, TvBand &bref, double lam, double rtol, int max_it) {
  // a private copy of the band (registers): tv_prox is not inlined, and the
  // reductions' parity flips on the caller's (local-memory) copy would put a
  // local store in front of every cluster barrier's release fence
  TvBand b = bref;
  constexpr int MR = tv_mr(SC);
  static_assert(MR <= kTvMaxRpt, "rows per thread");
  constexpr int NCW = SC >> 5;
  const int s = b.s, R = b.r1 - b.r0;
  const int h = (int)threadIdx.x / SC, c = (int)threadIdx.x - h * SC;
  const int lane = threadIdx.x & 31, cw = c >> 5;
  const int lr0 = h * b.RPT;
  const int nr = max(0, min(b.RPT, R - lr0));
  const bool col_ok = c < s;
  // shared: z, x, xw and the momentum duals wh, wv as [rows][SC] band arrays;
  // edge buffers bot_uv[h][c] (last row of row group h) and e_uh[h][k][cw]
  // (warp-edge u_h, lane 31)
  // (32-bit shared addresses: this function is not inlined, and generic
  // pointers would turn every access into a 64-bit generic load)
  const int e_o = (int)(b.edge - b.z);  // (b.z is tv_smem)
  const SmemF64 Z(0), X((int)(b.x - b.z)), XW((int)(b.xw - b.z)), WH((int)(b.wh - b.z)), WV((int)(b.wv - b.z)),
      BU(e_o), EU(e_o + b.H * SC);
  const int eb = (h * MR) * NCW + cw;  // e_uh[h][k][cw] = e_uh[eb + k*NCW]
  for (int i = threadIdx.x; i < R * SC; i += blockDim.x) {
    X.st(i, Z.ld(i));
    XW.st(i, 0.0), WH.st(i, 0.0), WV.st(i, 0.0);
  }
  for (int i = threadIdx.x; i < b.H * SC; i += blockDim.x) BU.st(i, 0.0);
  for (int i = threadIdx.x; i < b.H * MR * NCW; i += blockDim.x) EU.st(i, 0.0);
  cl.sync();
  if (!(lam > 0.0)) {  // x = z (no reductions yet: bref.parity unchanged); the duals become 0
    if (bref.ush) {
      for (int i = threadIdx.x; i < R * s; i += blockDim.x) {
        bref.ush[(int64_t)b.r0 * s + i] = 0.0;
        bref.usv[(int64_t)b.r0 * s + i] = 0.0;
      }
      cl.sync();
    }
    return 0;
  }
  const double hl = 0.5 * lam;
  // Boundary rules as data, so the per-pixel code has no branches: a dual
  // that the oracle never updates (no right / lower neighbour, or a padding
  // row or column) is clipped to [-0, 0] and stays 0, and a 0 term adds
  // exactly nothing to the divergence sums.  pm: rows with pixels; vm: rows
  // with a lower neighbour (bit k = row lr0 + k).
  const double hlh = (c + 1 < s) ? hl : 0.0;
  unsigned pm = 0, vm = 0;
#pragma unroll
  for (int k = 0; k < MR; ++k) {
    if (k < nr && col_ok) pm |= 1u << k;
    if (k < nr && col_ok && b.r0 + lr0 + k + 1 < s) vm |= 1u << k;
  }
  const bool left_edge = lane == 0 && cw > 0, right_edge = lane == 31 && cw + 1 < NCW;
  // Exchanges without cluster barriers: every CTA pushes (st.async) its
  // reduction partials to all CTAs, its first row of xw to the band above and
  // its last row of (u_v, w_v) to the band below, each completing on the
  // receiver's mbarrier; buffers alternate, and a producer can be at most one
  // use ahead (its next push of a buffer needs a reduction the receiver only
  // joins after reading it).
  const bool has_up = b.rank > 0, has_dn = b.rank + 1 < b.CL;
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(b.mbar);  // red[2], up[2], dn[2]
  const uint32_t xs = (uint32_t)__cvta_generic_to_shared(b.xs);
  const uint32_t red_o = xs, up_o = xs + 2 * kTvMaxCL * 2 * 8, dn_o = up_o + 2 * SC * 2 * 8;
  const double *red_slots = b.xs, *halo_up = b.xs + 2 * kTvMaxCL * 2, *halo_dn = halo_up + 2 * SC * 2;
  const bool up_local = lr0 > 0 && col_ok, up_halo = lr0 == 0 && has_up && col_ok;
  const bool dn_local = lr0 + nr < R && col_ok, dn_halo = lr0 + nr == R && nr > 0 && has_dn && col_ok;
  const bool push_up = lr0 == 0 && nr > 0 && has_up && col_ok;   // xw row 0 -> band above
  const bool push_dn = lr0 + nr == R && nr > 0 && has_dn && col_ok;  // (u_v, w_v) last row -> band below
  const int i0 = lr0 * SC + c;
  // every lane of the warp has all MR rows (the common case; no per-row predicates)
  const bool full_rows = __all_sync(0xffffffffu, nr == MR && col_ok);
  double uh[MR], uv[MR];
#pragma unroll
  for (int k = 0; k < MR; ++k) uh[k] = uv[k] = 0.0;
  // warm start (reading R23): u0 = the previous prox's duals clipped to this
  // λ's box (a dual with no neighbour has the box [-0, 0]), w0 = u0; the
  // edge buffers and the row above the band get the same starting values
#ifndef POLY_TV_WARM_CODE
#define POLY_TV_WARM_CODE 1
#endif
  constexpr bool warm = POLY_TV_WARM_CODE && WARM;
  if (warm) {
    const int64_t g0 = (int64_t)b.r0 * s;
    const double *ush = bref.ush, *usv = bref.usv;
#pragma unroll
    for (int k = 0; k < MR; ++k) {
      if (!((pm >> k) & 1)) continue;
      const int64_t pix = g0 + (int64_t)(lr0 + k) * s + c;
      const double hlv = (vm >> k) & 1 ? hl : 0.0;
      uh[k] = tv_clip(ush[pix], hlh);
      uv[k] = tv_clip(usv[pix], hlv);
      WH.st(i0 + k * SC, uh[k]);
      WV.st(i0 + k * SC, uv[k]);
      if (lane == 31 && k < nr) EU.st(eb + k * NCW, uh[k]);
      if (k == nr - 1) BU.st(h * SC + c, uv[k]);
    }
    cl.sync();
  }
  // the row above the band at iteration 1: (u_v, w_v) of its starting duals
  // (0 cold, u0 warm) placed in the halo slot iteration 1 reads — the slot the
  // band above last pushed into, consumed by the previous prox; its next push
  // goes to the other slot, and the one after can only come after this CTA's
  // iteration-1 phase A (it waits on a reduction this CTA joins after it)
  if (up_halo) {
    const uint32_t q = (b.n_b - 1) & 1;
    const double v0 = warm ? tv_clip(bref.usv[(int64_t)(b.r0 - 1) * s + c], hl) : 0.0;
    double *hu = const_cast<double *>(halo_up) + (q * SC + c) * 2;
    hu[0] = v0;
    hu[1] = v0;
  }
  double t = 1.0;
  int it = 1;
  for (;; ++it) {
    // this iteration's xw halo from the band below (pushed in its phase A)
    if (threadIdx.x == 0 && has_dn) mbar_expect_tx(mb + 8 * (4 + (b.n_a & 1)), (uint32_t)s * 8u);
    // phase A: x(u) = z - Dᵀu (the oracle's primal after iteration it-1) and
    // xw = z - Dᵀw; change of x against the previous primal
    double acc[2] = {0.0, 0.0};
    if (nr > 0) {  // warp-uniform
      double a_uv = 0.0, a_wv = 0.0;  // row above
      if (up_local) a_uv = BU.ld((h - 1) * SC + c), a_wv = WV.ld(i0 - SC);
      if (lr0 == 0 && has_up) {  // (u_v, w_v) halo pushed by the band above in its last phase B
        const uint32_t q = (b.n_b - 1) & 1;
        if (it > 1) mbar_wait_cluster(mb + 8 * (2 + q), ((b.n_b - 1) >> 1) & 1);
        if (up_halo) a_uv = halo_up[(q * SC + c) * 2], a_wv = halo_up[(q * SC + c) * 2 + 1];
      }
      auto phase_a = [&](auto full_t) {
        constexpr bool full = decltype(full_t)::value;
        // rows in chunks of CH: a chunk's loads are issued before its
        // arithmetic and stores (the compiler cannot move a load above a
        // shared store it cannot disambiguate)
#pragma unroll
        for (int kk = 0; kk < MR; kk += kTvChunk) {
          constexpr int CH = kTvChunk;
          double l_uh[CH], wh_i[CH], wh_l[CH], wv_i[CH], zi[CH], xo[CH];
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const int k = kk + j;
            if (k >= MR) break;
            const int i = i0 + k * SC;
            l_uh[j] = __shfl_up_sync(0xffffffffu, uh[k], 1);
            if (lane == 0) l_uh[j] = 0.0;
            if (left_edge) l_uh[j] = EU.ld(eb + k * NCW - 1);
            const bool on = full ? true : (pm >> k) & 1;
            wh_i[j] = wh_l[j] = wv_i[j] = zi[j] = xo[j] = 0.0;
            if (on) {
              wh_i[j] = WH.ld(i), wv_i[j] = WV.ld(i), zi[j] = Z.ld(i), xo[j] = X.ld(i);
              if (c > 0) wh_l[j] = WH.ld(i - 1);
            }
          }
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const int k = kk + j;
            if (k >= MR) break;
            const int i = i0 + k * SC;
            const bool on = full ? true : (pm >> k) & 1;
            // the oracle's sums with its zero terms kept: -w_h(c) + w_h(c-1) - w_v(r) + w_v(r-1)
            const double dw = ((wh_l[j] - wh_i[j]) - wv_i[j]) + a_wv;
            const double du = ((l_uh[j] - uh[k]) - uv[k]) + a_uv;
            const double xn = zi[j] - du;
            const double dx = xn - xo[j];
            if (on) {  // (rows past the band or padding columns contribute nothing)
              acc[0] = fma(dx, dx, acc[0]);
              acc[1] = fma(xn, xn, acc[1]);
              const double xwn = zi[j] - dw;
              X.st(i, xn), XW.st(i, xwn);
              if (k == 0 && push_up)
                st_async_f64(mapa_u32(dn_o + 8u * (uint32_t)((b.n_a & 1) * SC + c), b.rank - 1), xwn,
                             mapa_u32(mb + 8 * (4 + (b.n_a & 1)), b.rank - 1));
            }
            a_uv = uv[k], a_wv = wv_i[j];
          }
        }
      };
      if (full_rows) phase_a(std::true_type());
      else phase_a(std::false_type());
    }
    // ||Δx||², ||x||² over the cluster: lanes, then the CTA's warps, then the
    // CL ranks, each by the same xor butterfly (a fixed pairwise tree, so every
    // lane of every CTA ends with identical bits); every CTA pushes its pair to
    // every rank and sums the CL pairs itself
    {
      const uint32_t q = b.n_red & 1;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        double v = acc[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) b.wsum[(threadIdx.x >> 5) * 4 + k] = v;
      }
      __syncthreads();  // also: xw, x of every row group written
      if (threadIdx.x < 32) {
        const int NWp = (int)(blockDim.x >> 5);
        double p0 = lane < NWp ? b.wsum[lane * 4] : 0.0, p1 = lane < NWp ? b.wsum[lane * 4 + 1] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          p0 += __shfl_xor_sync(0xffffffffu, p0, o);
          p1 += __shfl_xor_sync(0xffffffffu, p1, o);
        }
        if (lane < b.CL)
          st_async_v2f64(mapa_u32(red_o + 16u * (uint32_t)(q * kTvMaxCL + b.rank), lane), p0, p1,
                         mapa_u32(mb + 8 * q, lane));
      }
      if (threadIdx.x == 0) mbar_expect_tx(mb + 8 * q, (uint32_t)b.CL * 16u);
      mbar_wait_cluster(mb + 8 * q, (b.n_red >> 1) & 1);
      acc[0] = lane < b.CL ? red_slots[(q * kTvMaxCL + lane) * 2] : 0.0;
      acc[1] = lane < b.CL ? red_slots[(q * kTvMaxCL + lane) * 2 + 1] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], o);
        acc[1] += __shfl_xor_sync(0xffffffffu, acc[1], o);
      }
      ++b.n_red;
    }
    if ((it > 1 && sqrt(acc[0]) <= rtol * sqrt(acc[1])) || it > max_it) break;
    // phase B: u+ = clip(w + D xw / 8, ±λ/2); w = u+ + ((t-1)/t+)(u+ - u)
    const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
    const double beta = (t - 1.0) / tn;
    t = tn;
    // the (u_v, w_v) halo the band above will push in its phase B
    if (threadIdx.x == 0 && has_up) mbar_expect_tx(mb + 8 * (2 + (b.n_b & 1)), (uint32_t)s * 16u);
    if (nr > 0) {
      double dn_xw = 0.0;  // row below the thread's last row
      if (dn_local) dn_xw = XW.ld(i0 + nr * SC);
      if (lr0 + nr == R && has_dn) {
        const uint32_t q = b.n_a & 1;
        mbar_wait_cluster(mb + 8 * (4 + q), (b.n_a >> 1) & 1);
        if (dn_halo) dn_xw = halo_dn[q * SC + c];
      }
      auto phase_b = [&](auto full_t) {
        constexpr bool full = decltype(full_t)::value;
#pragma unroll
        for (int kk = 0; kk < MR; kk += kTvChunk) {
          constexpr int CH = kTvChunk;
          double xr[CH + 1], r_xw[CH], wh_i[CH], wv_i[CH];
#pragma unroll
          for (int j = 0; j <= CH; ++j) {  // xw of rows kk .. kk+CH (the last: next chunk / row below)
            const int k = kk + j;
            if (k > MR) break;
            xr[j] = dn_xw;
            if (k < MR && (full || ((pm >> k) & 1))) xr[j] = XW.ld(i0 + k * SC);
          }
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const int k = kk + j;
            if (k >= MR) break;
            const int i = i0 + k * SC;
            const bool on = full ? true : (pm >> k) & 1;
            r_xw[j] = __shfl_down_sync(0xffffffffu, xr[j], 1);
            wh_i[j] = wv_i[j] = 0.0;
            if (on) {
              wh_i[j] = WH.ld(i), wv_i[j] = WV.ld(i);
              if (right_edge) r_xw[j] = XW.ld(i + 1);
            }
          }
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const int k = kk + j;
            if (k >= MR) break;
            const int i = i0 + k * SC;
            const bool on = full ? true : (pm >> k) & 1;
            const double cur = xr[j], nxt = xr[j + 1];
            const double hlv = (vm >> k) & 1 ? hl : 0.0;
            const double unh = tv_clip(wh_i[j] + (r_xw[j] - cur) / 8.0, on ? hlh : 0.0);  // u_h stays 0 off the band
            const double unv = tv_clip(wv_i[j] + (nxt - cur) / 8.0, hlv);
            const double wvn = unv + beta * (unv - uv[k]);
            if (on) {
              WH.st(i, unh + beta * (unh - uh[k]));
              WV.st(i, wvn);
            }
            uh[k] = unh;
            uv[k] = unv;
            if (lane == 31 && k < nr) EU.st(eb + k * NCW, unh);
            if (k == nr - 1) {
              BU.st(h * SC + c, unv);
              if (push_dn)
                st_async_v2f64(mapa_u32(up_o + 16u * (uint32_t)((b.n_b & 1) * SC + c), b.rank + 1), unv, wvn,
                               mapa_u32(mb + 8 * (2 + (b.n_b & 1)), b.rank + 1));
            }
          }
        }
      };
      if (full_rows) phase_b(std::true_type());
      else phase_b(std::false_type());
    }
    ++b.n_a, ++b.n_b;
    __syncthreads();  // duals of every row group written before the next phase A
  }
  // the band below pushed this (last) iteration's xw halo: consume its phase
  if (has_dn) mbar_wait_cluster(mb + 8 * (4 + (b.n_a & 1)), (b.n_a >> 1) & 1);
  ++b.n_a;
  // this prox's duals: the next prox's starting point (the pointers are
  // re-read here, volatile, so that they are not kept live through the loop)
  if (warm) {
    double *ush = *(double *volatile *)&bref.ush, *usv = *(double *volatile *)&bref.usv;
    const int64_t g0 = (int64_t)b.r0 * s;
#pragma unroll
    for (int k = 0; k < MR; ++k) {
      if (!((pm >> k) & 1)) continue;
      const int64_t pix = g0 + (int64_t)(lr0 + k) * s + c;
      ush[pix] = uh[k];
      usv[pix] = uv[k];
    }
  }
  cl.sync();  // x final everywhere (callers read the neighbours' x); duals stored
  bref.parity = b.parity;
  bref.n_red = b.n_red, bref.n_a = b.n_a, bref.n_b = b.n_b;
  return it - 1;
}

#ifndef POLY_TV_INLINE
__noinline__
#endif
__device__ int tv_prox_any(cg::cluster_group &cl, TvBand &b, double lam, double rtol, int max_it) {
  const bool w = b.ush != nullptr;
  switch (b.SC) {
    case 32: return w ? tv_prox<32, true>(cl, b, lam, rtol, max_it) : tv_prox<32, false>(cl, b, lam, rtol, max_it);
    case 64: return w ? tv_prox<64, true>(cl, b, lam, rtol, max_it) : tv_prox<64, false>(cl, b, lam, rtol, max_it);
    case 96: return w ? tv_prox<96, true>(cl, b, lam, rtol, max_it) : tv_prox<96, false>(cl, b, lam, rtol, max_it);
    case 128: return w ? tv_prox<128, true>(cl, b, lam, rtol, max_it) : tv_prox<128, false>(cl, b, lam, rtol, max_it);
    case 160: return w ? tv_prox<160, true>(cl, b, lam, rtol, max_it) : tv_prox<160, false>(cl, b, lam, rtol, max_it);
    case 192: return w ? tv_prox<192, true>(cl, b, lam, rtol, max_it) : tv_prox<192, false>(cl, b, lam, rtol, max_it);
    case 224: return w ? tv_prox<224, true>(cl, b, lam, rtol, max_it) : tv_prox<224, false>(cl, b, lam, rtol, max_it);
    default: return w ? tv_prox<256, true>(cl, b, lam, rtol, max_it) : tv_prox<256, false>(cl, b, lam, rtol, max_it);
  }
}

__device__ __forceinline__ unsigned tv_ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long tv_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// The K clusters meet (every thread of every CTA calls it; epoch counts the
// meetings of this launch, the same in all CTAs).  A cluster that waits past
// timeout_ns flags stats[3] and from then on no barrier waits again.
__device__ void tv_grid_sync(cg::cluster_group &cl, const TvArgs &a, unsigned &epoch) {
  ++epoch;
  if (a.K <= 1) return;
  __threadfence();  // this CTA's global writes (TV values, the selected prox) before the arrival
  cl.sync();
  if (cl.block_rank() == 0 && threadIdx.x == 0) {
    atomicAdd(a.gbar, 1u);
    const unsigned target = (unsigned)a.K * epoch;
    const unsigned long long t0 = tv_clock();
    while (tv_ld_acquire(a.gbar) < target) {
      if (*(volatile int32_t *)(a.stats + 3) || tv_clock() - t0 > a.timeout_ns) {
        atomicExch(a.stats + 3, 1);
        break;
      }
    }
    __threadfence();
  }
  cl.sync();
}

// P_X1(b.z) into b.x: the λ search of reading R22 (oracle_project_tv_k), this
// cluster evaluating value c of every round.  *n_bis counts rounds.
__device__ void tv_project_ball(cg::cluster_group &cl, TvBand &b, const TvArgs &a, int c, unsigned &epoch,
                                unsigned &round, int *n_bis, int *n_fista) {
  const int K = a.K > 1 ? a.K : 1;
  const int nb = (b.r1 - b.r0) * b.SC;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) b.x[i] = b.z[i];
  cl.sync();
  if (tv_norm_x(cl, b) <= a.tau) return;
  // every cluster publishes its TV for the round and reads all K in order
  auto exchange = [&](double tv, double *all) {
    const int slot = (int)(round & 1u) * K;
    ++round;
    if (K > 1 && cl.block_rank() == 0 && threadIdx.x == 0) a.tv_vals[slot + c] = tv;
    tv_grid_sync(cl, a, epoch);
    for (int k = 0; k < K; ++k) all[k] = (K == 1) ? tv : __ldcg(a.tv_vals + slot + k);
  };
  double all[kTvMaxK], lam[kTvMaxK];
  double lo = 0.0, hi = 1.0;
  bool found = false;
  for (int g = 0; g * K < 200 && !found; ++g) {
    const int e = g * K + c;
    double tv = INFINITY;
    if (e < 200) {
      *n_fista += tv_prox_any(cl, b, ldexp(1.0, e), a.rtol, a.max_it);
      tv = tv_norm_x(cl, b);
    }
    exchange(tv, all);
    for (int k = 0; k < K; ++k) {
      const int ek = g * K + k;
      if (ek < 200 && all[k] <= a.tau) {
        hi = ldexp(1.0, ek);
        lo = ek == 0 ? 0.0 : ldexp(1.0, ek - 1);
        found = true;
        break;
      }
    }
    if (!found) {
      const int ek = (g + 1) * K - 1 < 199 ? (g + 1) * K - 1 : 199;
      lo = ldexp(1.0, ek);
      hi = 2.0 * lo;
    }
  }
  int sel = K - 1;
  for (int st = 1; st <= 60; ++st) {
    for (int k = 0; k < K; ++k)
      lam[k] = K == 1 ? 0.5 * (lo + hi) : lo + (hi - lo) * (double)(k + 1) / (double)(K + 1);
    *n_fista += tv_prox_any(cl, b, lam[c], a.rtol, a.max_it);
    ++*n_bis;
    exchange(tv_norm_x(cl, b), all);
    int hit = -1, ks = -1;
    for (int k = 0; k < K && hit < 0; ++k)
      if (fabs(all[k] - a.tau) <= a.tv_tol) hit = k;
    for (int k = 0; k < K && ks < 0; ++k)
      if (all[k] <= a.tau) ks = k;
    if (hit >= 0) {
      sel = hit;
      break;
    }
    sel = ks >= 0 ? ks : K - 1;
    if (ks >= 0) {
      const double nlo = ks > 0 ? lam[ks - 1] : lo;
      hi = lam[ks];
      lo = nlo;
    } else {
      lo = lam[K - 1];
    }
  }
  if (K > 1) {  // the selected cluster's prox becomes everyone's b.x
    const int64_t g0 = (int64_t)b.r0 * b.s;
    if (c == sel)
      for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        const int lr = i / b.SC, cc = i - lr * b.SC;
        if (cc < b.s) a.xsel[g0 + (int64_t)lr * b.s + cc] = b.x[i];
      }
    tv_grid_sync(cl, a, epoch);
    if (c != sel)
      for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        const int lr = i / b.SC, cc = i - lr * b.SC;
        if (cc < b.s) b.x[i] = __ldcg(a.xsel + g0 + (int64_t)lr * b.s + cc);
      }
    __syncthreads();
    tv_grid_sync(cl, a, epoch);  // xsel is rewritten by the next selection only after everyone read it
  }
}

__global__ void __launch_bounds__(kTvThreads, 1) k_tv_project(const TvArgs a) {
  double *tsm = tv_smem;
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)(blockIdx.x / cl.num_blocks());  // this cluster's λ slot of each round
  const int64_t dd = (int64_t)a.s * a.s;
  double *zk = a.zk + c * dd, *pp = a.p + c * dd, *qq = a.q + c * dd;  // private Dykstra state
  unsigned epoch = 0, round = 0;
  TvBand b;
  b.s = a.s;
  b.CL = (int)cl.num_blocks();
  b.rank = (int)cl.block_rank();
  b.r0 = band_r0(b.rank, a.s, b.CL);
  b.r1 = band_r0(b.rank + 1, a.s, b.CL);
  b.npx = (b.r1 - b.r0) * a.s;
  b.SC = (a.s + 31) & ~31;
  const int cap_r = (a.s + b.CL - 1) / b.CL, cap = cap_r * b.SC;  // largest band
  b.H = kTvThreads / b.SC;
  b.RPT = (cap_r + b.H - 1) / b.H;
  b.z = tsm;
  b.x = b.z + cap;
  b.xw = b.x + cap;
  b.wh = b.xw + cap;
  b.wv = b.wh + cap;
  b.edge = b.wv + cap;
  b.red = b.edge + tv_edge_doubles(a.s);
  b.tot = b.red + 8;
  b.wsum = b.tot + 4;
  b.parity = 0;
  b.mbar = reinterpret_cast<uint64_t *>(b.wsum + (kTvThreads / 32) * 4);
  b.xs = reinterpret_cast<double *>((reinterpret_cast<uintptr_t>(b.mbar + 6) + 15) & ~(uintptr_t)15);
  b.n_red = b.n_a = b.n_b = 0;
  b.ush = b.usv = nullptr;
  if (a.warm && a.u_state) {  // this cluster's duals start at 0 for every projection
    b.ush = a.u_state + (int64_t)c * 2 * dd;
    b.usv = b.ush + dd;
    for (int64_t i = (int64_t)b.r0 * a.s + threadIdx.x; i < (int64_t)b.r1 * a.s; i += blockDim.x)
      b.ush[i] = b.usv[i] = 0.0;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 6; ++i) mbar_init(b.mbar + i, 1);
    fence_mbar_init();
  }
  cl.sync();
  pdl_wait();  // v is written by the previous kernel
  // with K > 1 the clusters wait for one another: a dependent launched early
  // could hold the SMs a not-yet-placed cluster needs, so trigger at the end
  if (a.K <= 1) pdl_trigger();
  const int64_t g0 = (int64_t)b.r0 * a.s;
  const int nb = (b.r1 - b.r0) * b.SC;  // band arrays incl. padding columns
  // band element i (pitch SC) <-> global pixel g0 + gi(i); padding columns have gi < 0
  auto gi = [&](int i) -> int64_t {
    const int lr = i / b.SC, c = i - lr * b.SC;
    return c < a.s ? (int64_t)lr * a.s + c : -1;
  };
  int n_bis = 0, n_fista = 0, sweeps = 0;
  if (!a.nonneg) {
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
      const int64_t j = gi(i);
      b.z[i] = j >= 0 ? a.v[g0 + j] : 0.0;
    }
    tv_project_ball(cl, b, a, c, epoch, round, &n_bis, &n_fista);
    if (c == 0)
      for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        const int64_t j = gi(i);
        if (j >= 0) a.out[g0 + j] = b.x[i];
      }
  } else {
    // Dykstra: z_0 = v, p_0 = q_0 = 0
    for (int i = threadIdx.x; i < b.npx; i += blockDim.x) {
      zk[g0 + i] = a.v[g0 + i];
      pp[g0 + i] = 0.0;
      qq[g0 + i] = 0.0;
    }
    for (sweeps = 1; sweeps <= a.max_outer; ++sweeps) {
      for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        const int64_t j = gi(i);
        b.z[i] = j >= 0 ? zk[g0 + j] + pp[g0 + j] : 0.0;
      }
      tv_project_ball(cl, b, a, c, epoch, round, &n_bis, &n_fista);  // y_k in b.x
      double acc[1] = {0.0};
      for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        const int64_t j = gi(i);
        if (j < 0) continue;
        const double z0 = zk[g0 + j], y = b.x[i];
        const double pn = z0 + pp[g0 + j] - y;
        const double sq = y + qq[g0 + j];
        const double zn = sq > 0.0 ? sq : 0.0;
        pp[g0 + j] = pn;
        qq[g0 + j] = sq - zn;
        acc[0] += (zn - z0) * (zn - z0);
        zk[g0 + j] = zn;
      }
      cluster_sum<1>(cl, b, acc);
      if (sqrt(acc[0]) <= a.tol) break;
    }
    if (sweeps > a.max_outer) sweeps = a.max_outer;
    if (c == 0)
      for (int i = threadIdx.x; i < b.npx; i += blockDim.x) a.out[g0 + i] = zk[g0 + i];
  }
  if (c == 0 && b.rank == 0 && threadIdx.x == 0) {
    if (a.stats) {
      a.stats[0] += sweeps;
      a.stats[1] += n_bis;
      a.stats[2] += n_fista;
    }
  }
  if (a.K > 1) pdl_trigger();
}

}  // namespace poly
