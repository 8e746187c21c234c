// K2/K3 — fixed-order reduction of the per-CTA partial gradients, the 1/n
// scale of Eq.(operator), and the extragradient step + projection
//   x_out = P_X(x_anchor - γ g)
// onto X = B(R; c), R_+^d or R_+^d ∩ B(R).
//
// Grid: ceil(d/32) blocks of 256 threads; thread (cl, sl) = (tid % 32,
// tid / 32) sums partial rows i = sl, sl+8, ... of column blockIdx.x*32+cl,
// and the 8 slices are combined in order — deterministic for a fixed grid.
// The projection needs ||v - c||: each block writes its share, and the last
// block to arrive (atomic ticket) forms the norm in fixed order and applies
// the scale to all d entries.
#pragma once

#include "common.cuh"

namespace poly {

enum FinMode : int32_t {
  FIN_GRAD = 0,       // g = Σ partials / n, loss
  FIN_STEP = 1,       // x_out = P_X(anchor - γ Σ partials / n)
  FIN_REDUCE = 2,     // comm[0..d) = Σ partials, comm[d] = Σ loss partials (unnormalised)
  FIN_GRAD_COMM = 3,  // g = comm / n, loss = comm[d] / n
  FIN_STEP_COMM = 4,  // x_out = P_X(anchor - γ comm / n)
  FIN_PROJECT = 5,    // x_out = P_X(anchor)
};

struct SolveState {
  double gamma;
  double loss_cur;     // ℓ at the last evaluation
  double *trace;       // [trace_cap] or null
  int32_t trace_cap;
  int32_t counter;     // F evaluations folded into a step so far
  int32_t bad;         // 0 or first (1-based) step counter whose iterate was non-finite
  uint32_t ticket;
  // averaged iterate (poly_solve_ex): x̄_k over iterates ⌈k/2⌉..k
  int32_t k;           // index of the last iterate folded into the window sum
  int32_t stopped;     // 1 once ||x̄_k - x̄_{k-1}|| <= tol (k >= 2)
  int32_t k_stop;
  int32_t comm_err;    // K9: a peer did not publish within the wait bound (set on the device)
  double tol;
  double move;
};

// K4t strip copies of the fp32 iterate (tiled.cuh): strip s of W image
// columns stored as rows x P floats (the forward's shared-memory layout,
// padding columns zero) at x32[off + s * SP], so the forward stages a strip
// with one bulk copy.  W == 0: none.
struct X32Strip {
  int32_t W, P, rows, cols, SP;
  int64_t off;
};

// the fp32 copies of x_k: row-major, the transposed image at [d, 2d)
// (tr_side > 0), the strip copies (xs.W > 0)
__device__ __forceinline__ void x32_store(float *o, int64_t d, int32_t tr_side, const X32Strip &xs, int64_t k,
                                          float v) {
  o[k] = v;
  if (tr_side) o[d + (k % tr_side) * tr_side + k / tr_side] = v;
  if (xs.W) {
    const int64_t r = k / xs.cols, c = k - r * xs.cols, s = c / xs.W;
    o[xs.off + s * xs.SP + r * xs.P + (c - s * xs.W)] = v;
  }
}

struct FinArgs {
  int32_t mode;
  int32_t d;
  int32_t G;                 // number of partial rows
  int32_t GL;                // number of loss partials
  int32_t split;             // 1: skip the last-block tail; k_fin_apply finishes the step
  int32_t need_loss;         // 0: the objective is not wanted (its partials are not summed)
  int32_t set;
  int64_t n_norm;            // the n of Eq.(operator)
  const double *partials;    // [G][d]
  const double *loss_partials;  // [G]
  double *comm;              // [d+1]
  double *g_out;             // optional [d]
  const double *anchor;      // [d]
  double *x_out;             // [d] (may alias anchor)
  float *x32_out;            // optional [d]: fp32 copy of x_out (gathered by the CSR pass)
  int32_t tr_side;           // > 0: x32_out is [2d] and x32_out[d + tr(k)] holds the transposed copy
  X32Strip xs;               // K4t strip copies in x32_out (xs.W > 0)
  double *v_scratch;         // [d]
  double *block_norm;        // [gridDim.x]
  const double *center;      // [d] or null
  double R;
  SolveState *state;
};

__global__ void __launch_bounds__(256) k_finalize(const FinArgs a) {
  __shared__ double sm[8][33];
  __shared__ double s_loss;
  __shared__ int s_last;
  pdl_wait();
  pdl_trigger();
  const int tid = threadIdx.x, cl = tid & 31, sl = tid >> 5;
  const int NWf = (int)(blockDim.x >> 5);  // 8, or 2 when there is at most one partial row
  const int c = blockIdx.x * 32 + cl;
  const int mode = a.mode;
  const bool from_comm = (mode == FIN_GRAD_COMM || mode == FIN_STEP_COMM);
  const bool needs_g = (mode != FIN_PROJECT);

  // ---- gradient column sums (a5), fixed order
  double tot = 0.0;
  if (needs_g) {
    double acc = 0.0;
    if (c < a.d) {
      if (from_comm) {
        if (sl == 0) acc = ld_prev(a.comm + c);
      } else {
        // four independent accumulators (loads in flight together), combined
        // in a fixed order: deterministic for a fixed G
        double q0 = 0.0, q1 = 0.0, q2 = 0.0, q3 = 0.0;
        const double *col = a.partials + c;
        const size_t st = (size_t)NWf * a.d;
        int i = sl;
        for (; i + 3 * NWf < a.G; i += 4 * NWf) {
          q0 += ld_prev(col + (size_t)i * a.d);
          q1 += ld_prev(col + (size_t)i * a.d + st);
          q2 += ld_prev(col + (size_t)i * a.d + 2 * st);
          q3 += ld_prev(col + (size_t)i * a.d + 3 * st);
        }
        for (; i < a.G; i += NWf) q0 += ld_prev(col + (size_t)i * a.d);
        acc = (q0 + q1) + (q2 + q3);
      }
    }
    sm[sl][cl] = acc;
  }
  // ---- loss (block 0, warp 1; only block 0 uses s_loss), fixed order — the
  // partial sums only when the objective is wanted: with one partial per
  // forward block (CSR: 4129) they are a long serial tail
  if (blockIdx.x == 0 && sl == 1 && needs_g) {
    double l = 0.0;
    if (from_comm) {
      l = (cl == 0) ? ld_prev(a.comm + a.d) : 0.0;
    } else if (a.need_loss) {
      for (int i = cl; i < a.GL; i += 32) l += ld_prev(a.loss_partials + i);
    }
    l = warp_sum(l);
    if (cl == 0) s_loss = l;
  }
  __syncthreads();
  if (sl != 0) {
    if (mode == FIN_GRAD || mode == FIN_GRAD_COMM || mode == FIN_REDUCE) return;
  }
  if (sl == 0 && needs_g) {
    for (int k = 0; k < NWf; ++k) tot += sm[k][cl];
  }
  if (mode == FIN_REDUCE) {
    if (c < a.d) a.comm[c] = tot;
    if (blockIdx.x == 0 && cl == 0) a.comm[a.d] = s_loss;
    return;
  }
  const double nn = (double)a.n_norm;
  if (mode == FIN_GRAD || mode == FIN_GRAD_COMM) {
    if (c < a.d && a.g_out) a.g_out[c] = tot / nn;
    if (blockIdx.x == 0 && cl == 0) a.state->loss_cur = s_loss / nn;
    return;
  }

  // ---- step + projection (a7)
  double q = 0.0;
  if (sl == 0) {
    if (c < a.d) {
      double v = ld_prev(a.anchor + c);
      if (needs_g) {
        const double g = tot / nn;
        if (a.g_out) a.g_out[c] = g;
        v = v - a.state->gamma * g;
      }
      if (a.set == 2 || a.set == 3) v = v > 0.0 ? v : 0.0;
      const double df = (a.set == 1 && a.center) ? v - a.center[c] : v;
      q = df * df;
      a.v_scratch[c] = v;
    }
    q = warp_sum(q);
    if (cl == 0) {
      a.block_norm[blockIdx.x] = q;
      if (blockIdx.x == 0 && needs_g) a.state->loss_cur = s_loss / nn;
    }
  }
  if (a.split) return;  // k_fin_apply (next kernel) forms the norm and writes x_out
  if (sl == 0) {
    if (cl == 0) {
      __threadfence();
      const uint32_t prev = atomicAdd(&a.state->ticket, 1u);
      s_last = (prev == gridDim.x - 1);
    }
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // last block: ||v - c||² in fixed order, then the scale
  if (sl == 0) {
    double nr = 0.0;
    for (int b = cl; b < (int)gridDim.x; b += 32) nr += ((volatile double *)a.block_norm)[b];
    nr = warp_sum(nr);
    if (cl == 0) sm[0][0] = nr;
  }
  __syncthreads();
  const double nrm = sqrt(sm[0][0]);
  double scale = 1.0;
  if ((a.set == 1 || a.set == 3) && nrm > a.R) scale = a.R / nrm;
  for (int k = tid; k < a.d; k += blockDim.x) {
    const double v = ((volatile double *)a.v_scratch)[k];
    double xo;
    if (a.set == 1) {
      const double ck = a.center ? a.center[k] : 0.0;
      xo = scale == 1.0 ? v : ck + (v - ck) * scale;
    } else {
      xo = v * scale;
    }
    a.x_out[k] = xo;
    if (a.x32_out) x32_store(a.x32_out, a.d, a.tr_side, a.xs, k, (float)xo);
  }
  if (tid == 0) {
    SolveState *s = a.state;
    s->ticket = 0;
    if (needs_g) {
      const int k = s->counter;
      if (s->trace && k < s->trace_cap) s->trace[k] = *(volatile double *)&s->loss_cur;
      s->counter = k + 1;
      if (!isfinite(nrm) && s->bad == 0) s->bad = k + 1;
    } else if (!isfinite(nrm) && s->bad == 0) {
      s->bad = -1;
    }
  }
}

// Tail of the step for large d (FinArgs.split = 1): every block forms
// ||v - c||² from the block partials of k_finalize in the same fixed order
// (identical bits in every block), then scales its slice of v into x_out.
// Replaces the single-block tail, which serialised d/256 dependent loads.
__global__ void k_to_f32(const double *x, int64_t d, int32_t tr_side, const X32Strip xs, float *out) {
  pdl_wait();
  pdl_trigger();
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < d;
       k += (int64_t)gridDim.x * blockDim.x) {
    x32_store(out, d, tr_side, xs, k, (float)x[k]);
  }
}

__global__ void __launch_bounds__(256) k_fin_apply(const FinArgs a) {
  __shared__ double s_w[8];
  pdl_wait();
#ifndef POLY_FIN_LATE
  pdl_trigger();
#endif
  const int tid = threadIdx.x;
  const int nb = (a.d + 31) / 32;  // k_finalize blocks
  // all 256 threads read the block norms (loads in flight together), then a
  // fixed tree: per-thread strided sums, warp butterflies, warps in order —
  // the same bits in every block
  double nr = 0.0;
  for (int b = tid; b < nb; b += 256) nr += ld_prev(a.block_norm + b);
  nr = warp_sum(nr);
  if ((tid & 31) == 0) s_w[tid >> 5] = nr;
  __syncthreads();
  const double nrm = sqrt(((s_w[0] + s_w[1]) + (s_w[2] + s_w[3])) + ((s_w[4] + s_w[5]) + (s_w[6] + s_w[7])));
  double scale = 1.0;
  if ((a.set == 1 || a.set == 3) && nrm > a.R) scale = a.R / nrm;
  for (int k = blockIdx.x * blockDim.x + tid; k < a.d; k += gridDim.x * blockDim.x) {
    const double v = ld_prev(a.v_scratch + k);
    double xo;
    if (a.set == 1) {
      const double ck = a.center ? a.center[k] : 0.0;
      xo = scale == 1.0 ? v : ck + (v - ck) * scale;
    } else {
      xo = v * scale;
    }
    a.x_out[k] = xo;
    if (a.x32_out) x32_store(a.x32_out, a.d, a.tr_side, a.xs, k, (float)xo);
  }
  if (blockIdx.x == 0 && tid == 0) {
    SolveState *s = a.state;
    const bool needs_g = (a.mode != FIN_PROJECT);
    if (needs_g) {
      const int k = s->counter;
      if (s->trace && k < s->trace_cap) s->trace[k] = s->loss_cur;
      s->counter = k + 1;
      if (!isfinite(nrm) && s->bad == 0) s->bad = k + 1;
    } else if (!isfinite(nrm) && s->bad == 0) {
      s->bad = -1;
    }
  }
}

// ------------------------------------------------------------ averaged iterate
// x̄_k = mean of iterates x_{⌈k/2⌉..k} (SPEC.md:357 window,
// reading R15), maintained as a window sum S: after x_k arrives,
//   S += x_k,  and for odd k (⌈k/2⌉ grows by one) S -= x_{(k-1)/2},
// with the iterates kept in a ring hist[cap][d], cap > k/2 + 1.  The stop rule
// ||x̄_k - x̄_{k-1}||_2 <= tol is decided in k_avg_b.  Once
// stopped, both kernels are no-ops, so iterations the host launched past the
// stop leave x̄, the ring and the state untouched.
struct AvgArgs {
  const double *x;      // [d] the new iterate x_k
  double *hist;         // [cap][d]
  double *S;            // [d] window sum
  double *xbar;         // [d] x̄_{k-1} in, x̄_k out
  double *block_norm;   // [ceil(d/256)]
  int32_t d;
  int32_t cap;
  SolveState *state;
};

__global__ void __launch_bounds__(256) k_avg_a(const AvgArgs a) {
  __shared__ double wsum[8];
  pdl_wait();
  pdl_trigger();
  if (a.state->stopped) return;
  const int k = a.state->k + 1;
  const int lo = (k + 1) / 2;  // ⌈k/2⌉
  const double cnt = (double)(k - lo + 1);
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  double q = 0.0;
  if (c < a.d) {
    const double xk = a.x[c];
    double s = a.S[c] + xk;
    if (k & 1) s -= a.hist[(size_t)(((k - 1) / 2) % a.cap) * a.d + c];
    a.hist[(size_t)(k % a.cap) * a.d + c] = xk;
    a.S[c] = s;
    const double xb = s / cnt;
    const double df = xb - a.xbar[c];
    a.xbar[c] = xb;
    q = df * df;
  }
  q = warp_sum(q);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = q;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += wsum[w];
    a.block_norm[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(32) k_avg_b(const AvgArgs a, int32_t nblocks) {
  pdl_wait();
  pdl_trigger();
  SolveState *s = a.state;
  if (s->stopped) return;
  double q = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += 32) q += a.block_norm[b];
  q = warp_sum(q);
  if (threadIdx.x == 0) {
    const int k = s->k + 1;
    const double mv = sqrt(q);
    s->k = k;
    s->move = mv;
    if (k >= 2 && mv <= s->tol) {
      s->stopped = 1;
      s->k_stop = k;
    }
  }
}

}  // namespace poly
