/*
 * poly.h — C ABI of the B200-native (sm_100a) hot path of EXACT, the
 * projected-extragradient estimator of arXiv 2503.19925.
 *
 * The library evaluates, on the GPU,
 *
 *   h(t)  = Σ_j s_j exp(-μ_j t_+)                     Eq.(function-h-plus)
 *   F(x)  = (1/n) Σ_i [y_i - Ī h(<a_i, x>)] a_i       Eq.(operator),
 *   ℓ(x)  = (1/n) Σ_i [y_i <a_i,x> - Ī H(<a_i,x>)],   H' = h                (reading R2;
 *                                                      ∇ℓ = F, so EXACT's VI is min_X ℓ)
 *   x_{t+1/2} = P_X(x_t - γ F(x_t)),
 *   x_{t+1}   = P_X(x_t - γ F(x_{t+1/2}))              Eq.(extragrad-method)
 *
 * with P_X the ℓ2 projection onto X = B(R; c), the
 * nonnegative orthant or R_+^d ∩ B(R) (reading R14).
 * Per-row spectra (s'_ij, Ī'_i) implement the known-materials reduction of
 * Appendix A.1.
 *
 * Conventions (all entry points):
 *  - Return value: POLY_OK (0) or one of the POLY_E* codes below; on error
 *    poly_last_error() returns a thread-local, NUL-terminated message.
 *  - "device" pointers are CUDA device (or managed) memory of the current
 *    device; "host" pointers are ordinary or pinned host memory.  Vectors
 *    marked "device or host" are classified with cudaPointerGetAttributes.
 *  - Work is enqueued on the cudaStream_t given in poly_problem.stream and is
 *    asynchronous, except where a host output is requested (then the call
 *    synchronises that stream before returning).
 *  - The handle BORROWS every device array of poly_problem until poly_free;
 *    the caller must keep them alive and unmodified.  Host arrays (s, mu,
 *    center) are copied during poly_init.  With POLY_FLAG_HOST_INPUTS the
 *    matrix/measurement arrays are host pointers and are copied into
 *    library-owned device memory during poly_init.
 *  - Multi-GPU (world > 1): one process per GPU; every rank calls every
 *    entry point in lockstep (NCCL semantics).  Each rank holds a contiguous
 *    block of rows; F is the allreduce(sum) over ranks of the local
 *    unnormalised sums, scaled by 1/n_global, so every rank sees identical
 *    bits and applies the identical projection.  On an NCCL error the rank
 *    aborts its communicator (ncclCommAbort) and returns POLY_ENCCL.
 *  - Not thread-safe per handle; distinct handles may be used concurrently.
 */
#ifndef POLY_H_
#define POLY_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define POLY_ABI_VERSION 5

/* status codes */
#define POLY_OK 0
#define POLY_EINVAL 1        /* bad argument: dims, spectrum, alignment, set, ... */
#define POLY_ECUDA 2         /* CUDA runtime / launch failure (message has the CUDA error) */
#define POLY_ENCCL 3         /* NCCL failure or NCCL unavailable when world > 1 */
#define POLY_ENONFINITE 4    /* poly_solve produced a non-finite iterate */
#define POLY_ENOMEM 5        /* device allocation failed */
#define POLY_EUNSUPPORTED 6  /* valid request outside what this build implements */

/* poly_problem.layout */
#define POLY_DENSE 0         /* A row-major n_local x d, row pitch lda elements */
#define POLY_CSR 1           /* row_ptr[n_local+1] (int64), col[nnz] (int32), val[nnz] */
#define POLY_PARALLEL_BEAM 2 /* matrix-free CT projector: A[kB+b, rN+c] = length of the line
                                {p : p·(cos θ_k, sin θ_k) = t_b} inside pixel (r, c) of an N x N
                                image with pitch 1/N centred on pixel (N/2, N/2), θ_k = kπ/V,
                                t_b = (b - (B-1)/2)/N (R12); A is never stored */
/* poly_problem.dtype: element type of A (dense) or val (CSR) */
#define POLY_F32 0
#define POLY_F64 1
/* poly_problem.ytype: element type of y */
#define POLY_Y_I32 0         /* Poisson counts (Eq. Poisson-model), must be >= 0 */
#define POLY_Y_F32 1         /* counts + electronic noise, may be negative */
#define POLY_Y_F64 2         /* e.g. noiseless expected counts in tests */
/* poly_problem.set: the constraint set X */
#define POLY_SET_NONE 0      /* X = R^d (P_X = identity) */
#define POLY_SET_BALL 1      /* X = B(R; center), center NULL = 0 */
#define POLY_SET_NONNEG 2    /* X = R_+^d */
#define POLY_SET_NONNEG_BALL 3 /* X = R_+^d ∩ B(R), center must be NULL (P_B ∘ P_+ is exact) */
#define POLY_SET_TV_NONNEG 4 /* X = {||x||_TV <= tv_tau} ∩ R_+^d for an s x s image (d = s^2),
                                the paper's CT set: Dykstra (Eq.
                                projection-intersection) over the TV ball, approximated by the TV
                                prox with λ bisected to |TV - tau| <= tv_tol, and the orthant */
#define POLY_SET_TV 5        /* X = {||x||_TV <= tv_tau} alone (same approximate projection)   */
/* poly_problem.flags */
#define POLY_FLAG_HOST_INPUTS 1u /* A/row_ptr/col/val/y/s_row/I_row are HOST pointers; copied at init */
#define POLY_FLAG_NO_GRAPH 2u    /* poly_solve launches kernels directly instead of via a CUDA graph */
#define POLY_FLAG_NO_PDL 4u      /* disable programmatic dependent launch between kernels */
#define POLY_FLAG_NO_SMALL 16u   /* never use the cluster-resident whole-solve kernel for small
                                    dense problems (poly_solve then replays the general graph) */
#define POLY_FLAG_COMM 8u        /* use the NCCL path (reduce -> ncclAllReduce -> step) even when
                                    world == 1; needs nccl_id.  Exercises the collective path on one GPU */
#define POLY_FLAG_P2P 32u        /* allocate a peer-reduce window (with world > 1 or POLY_FLAG_COMM);
                                    after poly_p2p_open the cross-rank sum runs as one kernel over
                                    NVLink peer memory (K9) instead of ncclAllReduce */

#define POLY_FLAG_NVLS 64u       /* allocate for K9-NVLS (with world > 1 or POLY_FLAG_COMM): after
                                    poly_nvls_open the cross-rank sum runs as one kernel over an
                                    NVLink multicast object — the NVSwitch adds the ranks' vectors
                                    (multimem.ld_reduce) and broadcasts the sums (multimem.st) —
                                    instead of ncclAllReduce.  Exclusive with POLY_FLAG_P2P. */

/* poly_problem.mode: which per-row scalar the fused pass evaluates.  Every mode
 * streams A once and returns g = (1/n) Σ_i φ_i a_i and a scalar objective.   */
#define POLY_MODE_EXACT 0    /* φ_i = y_i - Ī h(z_i): g = F(x), Eq.(operator); ℓ of reading R2 */
#define POLY_MODE_L2 1       /* MSE-GD baseline: L2 = (1/n) Σ (Ī h - y)^2,
                                φ_i = 2 (Ī h - y_i) Ī h'(z_i)                               */
#define POLY_MODE_L1 2       /* PolyakSGM baseline: L1 = (1/n) Σ |Ī h - y|,
                                φ_i = sign(Ī h - y_i) Ī h'(z_i), sign(0) = 0                 */
#define POLY_MODE_NLL 3      /* Poisson NLL scaled by 1/n:
                                (1/n) Σ [Ī h - y log(Ī h)], φ_i = (Ī - y_i/h) h'(z_i)        */
/* h'(t) = -Σ_j s_j μ_j e^{-μ_j t} for t > 0; 0 for t <= 0 when relu = 1. */

/* poly_solve flags */
#define POLY_SOLVE_PROFILE 1u    /* time every kernel with CUDA events (implies no graph);
                                    read with poly_kernel_times */

typedef struct poly_handle poly_handle; /* opaque, library-owned */

typedef struct poly_problem {
  int64_t n_local;     /* rows held by this rank (>= 0)                                  */
  int64_t n_global;    /* n of the 1/n in Eq.(operator): total rows over all ranks (>= 1) */
  int64_t row_offset;  /* global index of this rank's first row (bookkeeping only)       */
  int64_t d;           /* columns = length of x (>= 1)                                   */
  int32_t layout;      /* POLY_DENSE | POLY_CSR                                          */
  int32_t dtype;       /* POLY_F32 | POLY_F64                                            */
  const void *A;       /* dense: device, row-major, 16-byte aligned, lda*elsize % 16 == 0 */
  int64_t lda;         /* dense: row pitch in elements, lda >= d                         */
  const int64_t *row_ptr; /* CSR: device [n_local+1], row_ptr[0] = 0, nondecreasing      */
  const int32_t *col;  /* CSR: device [nnz], 0 <= col < d                                */
  const void *val;     /* CSR: device [nnz], dtype elements                              */
  int64_t nnz;         /* CSR: number of stored entries = row_ptr[n_local]               */
  int32_t ytype;       /* POLY_Y_I32 | POLY_Y_F32 | POLY_Y_F64                           */
  int32_t W;           /* spectral bins, 1 <= W <= 64                                    */
  const void *y;       /* device [n_local] measurements                                  */
  const double *s;     /* host [W]: s_j in (0,1], |Σ s_j - 1| <= 1e-12 */
  const double *mu;    /* host [W]: μ_j > 0                                              */
  double I_bar;        /* Ī > 0                                                          */
  const float *s_row;  /* optional device [n_local*W]: per-row spectrum s'_ij (A.1)      */
  const float *I_row;  /* optional device [n_local]: per-row intensity Ī'_i (A.1); both or neither */
  int32_t relu;        /* 1: h uses t_+ (Eq. function-h-plus); 0: Eq.(eq:model-orig)     */
  int32_t set;         /* POLY_SET_*                                                     */
  double R;            /* ball radius (> 0) for POLY_SET_BALL / POLY_SET_NONNEG_BALL     */
  const double *center;/* host [d] ball centre or NULL (= 0)                             */
  int32_t rank;        /* 0 <= rank < world                                              */
  int32_t world;       /* number of ranks (>= 1); world > 1 needs nccl_id                */
  const void *nccl_id; /* host, 128-byte ncclUniqueId from poly_nccl_unique_id on rank 0 */
  void *stream;        /* cudaStream_t (NULL = legacy default stream)                    */
  uint32_t flags;      /* POLY_FLAG_*                                                    */
  int32_t mode;        /* POLY_MODE_* (0 = EXACT's operator F)                           */
  /* Multiple detector windows (footnote PAPER.md:842; Eq. model:multi-material
   * PAPER.md:782-799 with M = 1): windows = Ω > 1 stacks Ω measurements of
   * every ray.  Then s is host [Ω*W] (window-major, each window a spectrum
   * with the invariants above), mu is host [W] (per wavelength, shared),
   * I_win is host [Ω] (Ī_ω > 0; I_bar is ignored), y is device [Ω*n_local]
   * (window-major, same ytype for all windows), and
   *   F(x) = (1/(Ω n_global)) Σ_ω Σ_i [y_ωi - Ī_ω h_ω(<a_i,x>)] a_i.
   * Needs mode = EXACT and no per-row spectra (POLY_EUNSUPPORTED otherwise).
   * windows = 0 or 1: a single window as above. */
  int32_t windows;
  const double *I_win;
  /* TV sets (POLY_SET_TV_NONNEG, POLY_SET_TV): anisotropic TV of the s x s image
   * (forward differences, R21), 2 <= s <= 256 (the projection runs in
   * one thread-block cluster; larger images return POLY_EUNSUPPORTED).  Zero
   * selects the default in brackets. */
  double tv_tau;         /* TV radius τ >= 0 (the paper: the truth's TV)          */
  double tv_tol;         /* [0.01] bisection stop |TV(x̄) - τ| <= tv_tol          */
  double tv_rtol;        /* [1e-6] prox: FISTA stops at relative primal change <= tv_rtol         */
  double tv_dykstra_tol; /* [1e-4] Dykstra stops at ||z_{k+1} - z_k|| <= tol    */
  int32_t tv_max_it;     /* [5000] FISTA iterations per prox                                    */
  int32_t tv_max_outer;  /* [1000] Dykstra sweeps                                              */
  /* POLY_PARALLEL_BEAM geometry: N = pb_side (d = N*N, 2 <= N <= 4096; the
   * forward's 32-row shared stage limits N to 1768 on sm_100a: larger sides
   * return POLY_EUNSUPPORTED), V = pb_views, B = pb_bins <= 1024; this rank
   * holds rows [row_offset, row_offset + n_local), both multiples of B (whole
   * views).  fp32 chord lengths; mode EXACT, no per-row spectra.  A, row_ptr,
   * col, val are unused. */
  int32_t pb_side, pb_views, pb_bins, pb_reserved;
  /* TV sets: λ values evaluated per round of the TV-prox search, one
   * thread-block cluster each (reading R22); 0 or 1 = the paper's bisection
   * (the default), up to 16.  More than can be resident: POLY_EUNSUPPORTED. */
  int32_t tv_k;
  /* TV sets: 0 (default) = each TV prox of one projection starts FISTA from
   * the dual solution of the previous prox (same cluster; the first from 0),
   * clipped to the new λ's box (reading R23); 1 = every prox from 0. */
  int32_t tv_cold;
} poly_problem;

/* Validate *p, copy host parameters, pick the kernel configuration for
 * (layout, dtype, d), allocate the workspaces (per-CTA partial gradients,
 * solver state, communicator) and, when world > 1, create the NCCL
 * communicator.  *out receives the handle (NULL on error).
 * Errors: POLY_EINVAL (dimension mismatch SPEC.md:63,311; spectrum invariants
 * SPEC.md:24-28; R <= 0 for a ball set; misaligned A; NONNEG_BALL with a
 * centre), POLY_EUNSUPPORTED (dense d above the largest tile, W > 64),
 * POLY_ENOMEM, POLY_ECUDA, POLY_ENCCL. */
int poly_init(const poly_problem *p, poly_handle **out);

/* One evaluation of the operator, Eq.(operator):
 *   g[k]  = F(x)_k,  k < d        (device or host [d] fp64; may be NULL)
 *   *loss = ℓ(x)                  (host double; may be NULL — then no sync)
 * x: device or host [d] fp64.  One pass over A (the fused row-tile kernel),
 * the fixed-order partial reduction and, for world > 1, one allreduce. */
int poly_loss_grad(poly_handle *h, const double *x, double *g, double *loss);

/* EXACT, Eq.(extragrad-method), T iterations with constant step γ > 0.
 * Small dense problems (single rank, A in fp32/fp64 fitting the shared memory
 * of one 16-CTA cluster, d <= 256, no per-row spectra, ball/orthant sets) run
 * all T iterations in one cluster-resident kernel; POLY_FLAG_NO_SMALL opts out.
 *   x_1 = P_X(x_in);  x_{t+1/2} = P_X(x_t - γ F(x_t));  x_{t+1} = P_X(x_t - γ F(x_{t+1/2})).
 * x: device or host [d] fp64; in: x_in, out: x_{T+1} (always in X).
 * trace: host [2T] fp64 or NULL; receives ℓ at each of the 2T points where F
 * was evaluated.  flags: POLY_SOLVE_*.  On a non-finite iterate returns
 * POLY_ENONFINITE with *bad_iter = the 1-based iteration t (bad_iter may be
 * NULL).  Synchronises the stream before returning. */
int poly_solve(poly_handle *h, double *x, int T, double gamma, uint32_t flags,
               double *trace, int *bad_iter);

/* Options of poly_solve_ex. */
#define POLY_METHOD_EXTRAGRADIENT 0 /* EXACT, Eq.(extragrad-method): 2 passes per iteration        */
#define POLY_METHOD_GD 1            /* projected gradient x_{t+1} = P_X(x_t - γ g(x_t)): the MSE-GD
                                       baseline's iteration (§3.1); 1 pass per iteration            */
typedef struct poly_solve_opts {
  int32_t T_max;       /* >= 0 iterations at most                                               */
  int32_t method;      /* POLY_METHOD_*                                                         */
  double gamma;        /* > 0 constant step                                                     */
  double tol;          /* averaging: stop at the first k >= 2 with ||x̄_k - x̄_{k-1}||_2 <= tol
                          (1e-5); 0 = never stop early                            */
  int32_t average;     /* 1: x̄_k = mean of iterates ⌈k/2⌉..k (reading R15)        */
  uint32_t flags;      /* POLY_SOLVE_* (PROFILE)                                                */
} poly_solve_opts;

typedef struct poly_solve_info {
  int32_t iters;       /* iterations run up to the stop (k - 1 for the stopping iterate x_k)    */
  int32_t stopped;     /* 1 if the tolerance was met                                            */
  int32_t bad_iter;    /* 1-based iteration of a non-finite iterate, else 0                     */
  int32_t reserved;
  double move;         /* ||x̄_k - x̄_{k-1}||_2 at the stop / last iterate (averaging), else 0    */
} poly_solve_info;

/* Iterative solve with the options above (Eq. extragrad-method or projected
 * GD, optional averaged iterate and stopping rule of PAPER.md:1277-1280).
 * x: device or host [d] fp64; in: x_in (x_1 = P_X(x_in)); out: x̄_k when
 * opts->average, else the last iterate.  x_last: NULL or device/host [d]
 * receiving the last iterate x_k at the stop.  info: host, may be NULL.
 * Iterations run as CUDA-graph replays; the stop is detected on the device
 * and polled by the host one graph behind, so a few iterations past the stop
 * may execute — they change neither the returned x̄_k nor x_last nor info.
 * Errors: as poly_solve; POLY_ENONFINITE sets info->bad_iter. */
int poly_solve_ex(poly_handle *h, const poly_solve_opts *opts, double *x, double *x_last,
                  poly_solve_info *info);

/* Forward projection z_i = <a_i, x> for the local rows, accumulated in fp64
 * (fp32 A values promoted exactly), fixed reduction order.
 * x: device [d] fp64; z: device [n_local] fp64. */
int poly_forward(poly_handle *h, const double *x, double *z);

/* Expected counts λ_i = Ī_i h_i(<a_i, x>) (Eq. model),
 * fp64 throughout.  x: device [d] fp64; lam: device [n_local] fp64. */
int poly_expected_counts(poly_handle *h, const double *x, double *lam);

/* Known-materials reparameterisation of Appendix A.1:
 *   Ī'_i = Ī Σ_j s_j e^{-μ_j b_i},  s'_ij = s_j e^{-μ_j b_i} / Σ_k s_k e^{-μ_k b_i},
 * with b_i the known-material line integral, replaced by max(b_i, 0) when
 * clamp = 1 (reading R7).  b: device [n] fp64; s_row: device [n*W] fp32;
 * I_row: device [n] fp32; s, mu: host [W].  Enqueued on `stream`. */
int poly_reparameterize(int32_t W, const double *s, const double *mu, double I_bar, int64_t n,
                        const double *b, int32_t clamp, float *s_row, float *I_row, void *stream);

/* x = P_X(v) for the handle's constraint set (the projection step a7 alone).
 * v, x: device [d] fp64 (may alias).  For the TV sets also returns, in
 * stats (host [3], may be NULL), the Dykstra sweeps, bisection steps and
 * FISTA iterations that projection used.  Synchronises the stream. */
int poly_project(poly_handle *h, const double *v, double *x, int64_t *stats);

/* K8, the read-only streaming ceiling of a dense handle: streams the
 * handle's A through K1's ring (same grid, stages, bulk copies) with no
 * arithmetic, `reps` times back to back; *ms = average device time per pass.
 * POLY_EUNSUPPORTED for CSR handles.  Synchronises the stream. */
int poly_stream_probe(poly_handle *h, int32_t reps, double *ms);

/* Average device time (ms) of each kernel class over the last poly_solve
 * called with POLY_SOLVE_PROFILE: out[0] loss+grad pass (the fused A-stream
 * kernel), out[1] reduce/project kernel(s), out[2] allreduce (0 if world==1),
 * out[3] loss+grad launches, out[4] all kernel launches.  nout <= 5. */
int poly_kernel_times(poly_handle *h, double *out, int32_t nout);

/* Static description of the chosen configuration, for reports:
 * out[0] grid CTAs, out[1] threads/CTA, out[2] rows per stage, out[3] stages,
 * out[4] dynamic smem bytes, out[5] SM count; dense handles also report the K1
 * instantiation k_dense_loss_grad<T, V, WPR, NW, RPS, LOSS, FULL>: out[6] V,
 * out[7] WPR, out[8] NW, out[9] FULL (1: d fills the tile exactly, no column
 * masks); 0 for CSR / matrix-free handles.  out[10] ranks of the handle's
 * NCCL communicator (ncclCommCount; 0 without one), out[11] 1 when the
 * cross-rank sum runs as K9 (poly_p2p_open), out[12] the CSR layout poly_init
 * built: 3 K4t (strip forward + tile backward, the default for fp32 A when
 * every local index delta fits 8 bits; then out[0] forward CTAs, out[1] its
 * threads, out[2] column strips, out[3] backward tiles, out[4] forward smem),
 * 1 SELL16, 2 DSELL, 0 the 8-byte SELL; -1 for dense / matrix-free handles.
 * out[13] bytes of A (dense) or of its K4t copies that every pass reads with
 * the L2 evict-last policy, so that they stay in L2 from one pass to the next
 * (the rest streams evict-first); 0 otherwise.  nout <= 14. */
int poly_describe(poly_handle *h, int64_t *out, int32_t nout);

/* Write a fresh 128-byte ncclUniqueId into out (host).  Call on rank 0 and
 * broadcast the bytes to all ranks before poly_init.  POLY_ENCCL if NCCL
 * cannot be loaded. */
int poly_nccl_unique_id(void *out128);

/* K9 peer reduce (step a6 without NCCL).  With
 * POLY_FLAG_P2P every rank exports its window with poly_p2p_handle (64 bytes,
 * a cudaIpcMemHandle_t), the caller all-gathers the world*64 bytes in rank
 * order (e.g. torch.distributed.all_gather_object) and every rank calls
 * poly_p2p_open with them; from then on each F evaluation's sum over ranks is
 * one kernel that publishes this rank's unnormalised sums, waits for every
 * rank's flag (system-scope acquire) and adds the ranks' windows in rank order
 * over NVLink — identical bits on every rank.  All ranks must call
 * poly_p2p_open before their next evaluation.  Errors: POLY_EINVAL (no
 * POLY_FLAG_P2P, called twice), POLY_ECUDA (no peer access; the handle keeps
 * the NCCL path). */
int poly_p2p_handle(poly_handle *h, void *out64);
int poly_p2p_open(poly_handle *h, const void *handles);

/* K9-NVLS setup (step a6 through the switch).
 * Collective, in two calls on every rank of a handle made with POLY_FLAG_NVLS:
 *   1. poly_nvls_handle: rank 0 creates an NVLink multicast object sized for
 *      flags + 4 slots of d+1 doubles (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED
 *      required, else POLY_EUNSUPPORTED) and writes a 64-byte descriptor to
 *      out64 (host); other ranks' output is unused.  The caller broadcasts rank
 *      0's 64 bytes (e.g. torch.distributed.broadcast_object_list).
 *   2. poly_nvls_open(desc64 = rank 0's descriptor, host): every rank receives
 *      the object's file descriptor from rank 0 over an abstract unix socket
 *      (poly_share_fd; the ranks must share a node), adds its device, binds a
 *      physical copy of the window and maps the unicast and multicast views;
 *      two barriers over the handle's communicator order the steps.  From the
 *      next F evaluation on, every cross-rank sum is k_nvls_reduce.
 * Every wait inside the kernel is bounded (POLY_COMM_TIMEOUT_S, default 300 s);
 * on a timeout the solve returns POLY_ENCCL and the communicator is aborted.
 * Errors: POLY_EINVAL (no flag, wrong order, foreign descriptor),
 * POLY_EUNSUPPORTED (no multicast support), POLY_ECUDA / POLY_ENOMEM (driver
 * calls), POLY_ENCCL (a rank did not join within the timeout). */
int poly_nvls_handle(poly_handle *h, void *out64);
int poly_nvls_open(poly_handle *h, const void *desc64);

/* Same-node file-descriptor hand-off used by poly_nvls_open: rank 0 listens
 * on the abstract unix socket `name` and passes fd_in (SCM_RIGHTS) to the
 * world-1 other ranks, which connect (retrying up to timeout_s seconds) and
 * receive a duplicate in *fd_out; on rank 0 *fd_out = fd_in.  Collective over
 * the ranks of one node.  Errors: POLY_EINVAL, POLY_ENCCL (timeout). */
int poly_share_fd(int32_t rank, int32_t world, const char *name, int fd_in, int *fd_out, double timeout_s);

/* Release everything the handle owns (workspaces, graphs, communicator,
 * peer / multicast windows).  With K9 or K9-NVLS every rank must have
 * finished its last evaluation before any rank frees (e.g. a barrier). */
void poly_free(poly_handle *h);

/* Thread-local message for the last error of this thread ("" if none). */
const char *poly_last_error(void);

/* POLY_ABI_VERSION of the loaded library. */
int poly_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* POLY_H_ */
