// Host implementation of the C ABI in include/poly.h.
//
// Per F evaluation the library enqueues, on its own work
// stream (ordered after the caller's stream with events):
//   K1 k_dense_loss_grad, or K4f/K4b k_sell16_forward/backward (CSR), or
//   K5f/K5b k_pb_forward/backward (matrix-free parallel beam)   one pass over A
//   K2/K3 k_finalize (+ k_fin_apply)                fixed-order reduce, 1/n,
//                                                   step + projection
//   (k_tv_project for the TV sets, between the step and k_fin_apply)
//   (world > 1: k_finalize(REDUCE) -> ncclAllReduce(d+1 doubles), or K9
//    k_peer_reduce after poly_p2p_open -> k_finalize)
// and poly_solve replays one CUDA graph per U EXACT iterations
// (Eq. extragrad-method) with programmatic dependent launch
// between the kernels so the next A stream starts while the step finishes.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <poll.h>
#include <unistd.h>
#include <nccl.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <thread>
#include <type_traits>
#include <vector>

#include "../../include/poly.h"
#include "aux.cuh"
#include "csr.cuh"
#include "dense.cuh"
#include "finalize.cuh"
#include "tv.cuh"
#include "small.cuh"
#include "ctproj.cuh"
#include "p2p.cuh"
#include "nvls.cuh"
#include "dsell.cuh"
#include "tiled.cuh"

using namespace poly;

namespace {

thread_local char g_err[1024] = "";

int fail(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

#define CK(call)                                                                               \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess)                                                                     \
      return fail(POLY_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                                   \
  } while (0)

#define TRY(call)           \
  do {                      \
    int r_ = (call);        \
    if (r_ != POLY_OK) return r_; \
  } while (0)

// ------------------------------------------------------------------ NCCL
struct NcclApi {
  void *lib = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclCommAbort) commAbort = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
  decltype(&ncclCommGetAsyncError) asyncErr = nullptr;
  decltype(&ncclCommCount) count = nullptr;
};

NcclApi *nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api.lib ? &api : nullptr;
  tried = true;
  const char *names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char *nm : names) {
    api.lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (api.lib) break;
  }
  if (!api.lib) return nullptr;
  api.getUniqueId = (decltype(api.getUniqueId))dlsym(api.lib, "ncclGetUniqueId");
  api.commInitRank = (decltype(api.commInitRank))dlsym(api.lib, "ncclCommInitRank");
  api.allReduce = (decltype(api.allReduce))dlsym(api.lib, "ncclAllReduce");
  api.commDestroy = (decltype(api.commDestroy))dlsym(api.lib, "ncclCommDestroy");
  api.commAbort = (decltype(api.commAbort))dlsym(api.lib, "ncclCommAbort");
  api.errStr = (decltype(api.errStr))dlsym(api.lib, "ncclGetErrorString");
  api.asyncErr = (decltype(api.asyncErr))dlsym(api.lib, "ncclCommGetAsyncError");
  api.count = (decltype(api.count))dlsym(api.lib, "ncclCommCount");
  if (!api.getUniqueId || !api.commInitRank || !api.allReduce || !api.commDestroy ||
      !api.commAbort || !api.errStr || !api.asyncErr || !api.count) {
    api.lib = nullptr;
    return nullptr;
  }
  return &api;
}

// ------------------------------------------------------- kernel variants
struct DenseVariant {
  int V, WPR, NW, RPS;
  const void *fn[2][2];  // [FULL][LOSS]
};

#define DV(T, V, WPR, NW, RPS)                                                          \
  DenseVariant {                                                                        \
    V, WPR, NW, RPS, {                                                                  \
      {(const void *)&k_dense_loss_grad<T, V, WPR, NW, RPS, false, false>,              \
       (const void *)&k_dense_loss_grad<T, V, WPR, NW, RPS, true, false>},              \
          {(const void *)&k_dense_loss_grad<T, V, WPR, NW, RPS, false, true>,           \
           (const void *)&k_dense_loss_grad<T, V, WPR, NW, RPS, true, true>}            \
    }                                                                                   \
  }

// columns per slab: 32 lanes x (16 B / elsize) x V
const DenseVariant kDenseF32[] = {
    DV(float, 1, 1, 16, 64), DV(float, 2, 1, 16, 32), DV(float, 4, 1, 16, 32),
    DV(float, 8, 1, 12, 24), DV(float, 8, 2, 12, 12), DV(float, 8, 4, 12, 6),
    DV(float, 8, 8, 8, 1),
};
// alternative tiles, selectable with POLY_K1_TUNE=<index> (tuning runs only)
const DenseVariant kDenseTuneF32[] = {
    DV(float, 8, 1, 12, 12), DV(float, 8, 1, 16, 16), DV(float, 8, 4, 12, 3),  DV(float, 4, 1, 16, 16),
    DV(float, 8, 2, 12, 12), DV(float, 4, 1, 16, 48), DV(float, 8, 1, 8, 16),  DV(float, 8, 4, 8, 4),
};
const DenseVariant kDenseF64[] = {
    DV(double, 1, 1, 16, 64), DV(double, 2, 1, 16, 32), DV(double, 4, 1, 16, 16),
    DV(double, 8, 1, 12, 12), DV(double, 8, 2, 12, 6),  DV(double, 8, 4, 12, 3),
    DV(double, 8, 8, 8, 1),
};

const void *kCsrFwd[2][2] = {
    {(const void *)&k_sell_forward<float, false>, (const void *)&k_sell_forward<float, true>},
    {(const void *)&k_sell_forward<double, false>, (const void *)&k_sell_forward<double, true>},
};
const void *kCscBwd[2] = {(const void *)&k_csc_backward<float>,
                          (const void *)&k_csc_backward<double>};
const void *kSell16Fwd[2][2] = {
    {(const void *)&k_sell16_forward<float, false>, (const void *)&k_sell16_forward<float, true>},
    {(const void *)&k_sell16_forward<double, false>, (const void *)&k_sell16_forward<double, true>},
};
const void *kSell16Bwd[2] = {(const void *)&k_sell16_backward<float>,
                             (const void *)&k_sell16_backward<double>};
constexpr int kSplitFinD = 8192;  // d above which the step tail runs as k_fin_apply

constexpr size_t kSmemLimit = 227 * 1024;
constexpr size_t kRingBudget = 200 * 1024;

__global__ void k_min_i32(const int32_t *y, int64_t n, int32_t *out) {
  int32_t m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = min(m, y[i]);
  if (m < 0) atomicMin(out, m);
}

__global__ void k_sum_windows(const void *y, int ytype, int Om, int64_t n, void *out,
                              int32_t *overflow) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (ytype == POLY_Y_I32) {
      int64_t t = 0;
      for (int w = 0; w < Om; ++w) t += ((const int32_t *)y)[(size_t)w * n + i];
      if (t > INT32_MAX) atomicOr(overflow, 1);
      ((int32_t *)out)[i] = (int32_t)t;
    } else {
      double t = 0.0;
      for (int w = 0; w < Om; ++w)
        t += ytype == POLY_Y_F32 ? (double)((const float *)y)[(size_t)w * n + i]
                                 : ((const double *)y)[(size_t)w * n + i];
      ((double *)out)[i] = t;
    }
  }
}

__global__ void k_iota(int32_t *v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int32_t)i;
}

__global__ void k_widen(const int32_t *c, int64_t d, int64_t *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= d;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i < d ? c[i] : 0;
}

__global__ void k_check_csr(const int64_t *rp, const int32_t *col, int64_t n, int64_t nnz, int d,
                            int32_t *bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i == 0 && rp[0] != 0) atomicOr(bad, 1);
    if (i == n && rp[n] != nnz) atomicOr(bad, 2);
    if (i < n && rp[i + 1] < rp[i]) atomicOr(bad, 4);
  }
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    if (col[e] < 0 || col[e] >= d) atomicOr(bad, 8);
}

bool is_device_ptr(const void *p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

}  // namespace

struct poly_handle {
  poly_problem p{};
  int dev = 0, sms = 0;
  int elsize = 4, ysz = 4;
  int Om = 1;          // detector windows (folded into one spectrum at init)
  int64_t n_norm = 1;  // the n of Eq.(operator): Ω n_global
  cudaStream_t user = nullptr, work = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  std::vector<void *> owned;  // library-owned device buffers
  double *spec = nullptr, *center = nullptr;
  // K1
  const DenseVariant *dv = nullptr;
  int full = 0;
  int k1_grid = 0, k1_threads = 0, k1_stages = 0, k1_side = 0, k1_keep = 0;
  int64_t keep_bytes = 0;        // bytes of A (or its K4t copies) read with L2 evict-last per pass
  size_t k1_smem = 0;
  int k4_grid = 0;                     // K4f blocks (= loss partials)
  int nrslices = 0;                    // 32-row SELL slices of A
  void *sell_rows = nullptr;           // CscEnt<T>[row_slice_off[k4_grid] * 32]: {col, val}
  int64_t *row_slice_off = nullptr;    // [k4_grid + 1]
  int nslices = 0;                     // K4b blocks: 32-column SELL slices of A^T
  void *sell = nullptr;                // CscEnt<T>[slice_off[nslices] * 32]
  int64_t *slice_off = nullptr;        // [nslices + 1] slice start, in 32-entry steps
  int32_t *colmap = nullptr;           // tiled K4b slices: column of each slot (-1 empty), NULL = identity
  float *rbuf = nullptr;               // [n_local] residuals between K4f and K4b
  float *xa32 = nullptr, *xh32 = nullptr, *xin32 = nullptr;  // CSR: fp32 copies of xa, xh, a caller's x
  int tr_side = 0;                     // CSR, d = s²: fp32 copies also hold x transposed at [d, 2d)
  X32Strip xs{};                       // K4t: fp32 copies also hold the forward's strips
  int64_t tr_slices = 0;               // K4f slices that gather from the transposed copy
  bool sell16 = false;                 // both SELL copies in the 6-byte delta form
  bool dsell = false;                  // fp32: both copies in the dictionary-staged 5-byte form (dsell.cuh)
  DSell dfwd{}, dbwd{};
  int32_t dfwd_cap = 0, dbwd_cap = 0;  // largest |F_s| per direction (shared-memory staging)
  size_t dfwd_smem = 0, dbwd_smem = 0;
  int dbwd_grid = 0;                   // persistent backward blocks (forward: k4_grid)
  // POLY_PARALLEL_BEAM
  PbGeom pb{};
  double *pb_trig = nullptr, *pb_out2 = nullptr, *pb_zpart = nullptr;
  int32_t *pb_ticket = nullptr, *pb_tticket = nullptr;
  int k4f16_grid = 0, k4b16_grid = 0;  // resident-slot grids (slices dealt grid-stride)
  // K4t (tiled.cuh): strip forward + link + tile backward, the default for fp32 CSR
  bool tiled = false;
  StripFwd tfwd{};
  TileBwd tbwd{};
  int tf_grid = 0, tb_grid = 0;        // forward CTAs (2 per SM), backward CTAs (one per tile)
  size_t tf_smem = 0, tb_smem = 0;
  bool tile_epi = false;               // every warp of K4tb covers one k_finalize block
  int32_t tb_lcap = 0;                 // K4tb ray-list capacity (floats, multiple of 4)
  double mu_step = 0.0;                // != 0: μ is an arithmetic progression (geometric bins in K4tl)
  int64_t tf_groups = 0, tb_groups = 0;
  StepEpi epi{};                        // K4b's step epilogue for the next pass (on = 0: write g)
  // TV sets: Dykstra state, statistics, cluster launch shape
  double *tv_zk = nullptr, *tv_p = nullptr, *tv_q = nullptr;  // [tv_k][d] each
  int32_t *tv_stats = nullptr;         // [4]
  int tv_cl = 0;
  int tv_k = 1;                        // clusters = λ values per search round (reading R22)
  double *tv_vals = nullptr, *tv_xsel = nullptr;
  double *tv_ustate = nullptr;         // [tv_k][2][d] warm-start duals (reading R23), NULL when cold
  unsigned int *tv_gbar = nullptr;
  size_t tv_smem = 0;
  Sell16 fwd16{}, bwd16{};
  int64_t sell_steps = 0;              // slice_off[nslices]
  int64_t sell_row_steps = 0;          // row_slice_off[k4_grid]
  int fin_split = 0;
  // workspaces
  int G = 0;  // partial rows
  double *partials = nullptr, *loss_partials = nullptr, *comm = nullptr;
  double *xa = nullptr, *xh = nullptr, *xin = nullptr, *gbuf = nullptr;
  double *vscratch = nullptr, *block_norm = nullptr, *trace = nullptr;
  int trace_cap = 0;
  SolveState *state = nullptr, *hstate = nullptr;
  int fin_grid = 0;
  bool pdl = true, use_graph = true;
  cudaGraphExec_t gexec[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [loss][U>1]
  cudaGraphExec_t gexec_ex[2][2][2] = {};  // poly_solve_ex: [method][average][U>1]
  // averaged iterate workspaces (allocated on first use)
  double *hist = nullptr, *Ssum = nullptr, *xbar = nullptr, *avg_norm = nullptr;
  int avg_cap = 0;
  int graph_U = 8;
  ncclComm_t nccl = nullptr;
  bool comm_path = false;  // world > 1 or POLY_FLAG_COMM: reduce -> allreduce -> step
  double comm_timeout_s = 300.0;  // POLY_COMM_TIMEOUT_S: host watchdog on waits with a communicator
  bool no_epi = false;            // POLY_NO_EPI (read once at init): no K4b step epilogue
  cudaEvent_t ev_poll[2] = {nullptr, nullptr}, ev_sync = nullptr;
  // K9 peer reduce (POLY_FLAG_P2P + poly_p2p_open): this rank's window, the
  // peers' IPC mappings, the per-block evaluation counters
  char *p2p_win = nullptr;
  char *p2p_peer[kP2PMaxRanks] = {};
  unsigned long long *p2p_epoch = nullptr;
  bool p2p = false;
  // K9-NVLS (POLY_FLAG_NVLS + poly_nvls_open): the multicast window
  struct {
    bool on = false;
    CUmemGenericAllocationHandle mc = 0, mem = 0;
    bool have_mc = false, have_mem = false, bound = false;
    CUdeviceptr uc_va = 0, mc_va = 0;
    bool uc_mapped = false, mc_mapped = false;
    size_t size = 0;
    int fd = -1, listen_fd = -1;
    unsigned long long *epoch = nullptr;
  } nv;
  // profiling
  bool prof = false;
  std::vector<cudaEvent_t> evpool;
  size_t evused = 0;
  struct Rec { int kind; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  double ktimes[5] = {0, 0, 0, 0, 0};
};

namespace {

template <typename... Args>
int launch(poly_handle *h, const void *fn, dim3 grid, dim3 block, size_t smem, bool pdl,
           Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = h->work;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl && h->pdl) ? 1 : 0;
  void *argv[] = {(void *)&args...};
  CK(cudaLaunchKernelExC(&cfg, fn, argv));
  return POLY_OK;
}

cudaEvent_t prof_event(poly_handle *h) {
  if (h->evused == h->evpool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    h->evpool.push_back(e);
  }
  return h->evpool[h->evused++];
}

struct ProfScope {
  poly_handle *h;
  int kind;
  cudaEvent_t a = nullptr;
  ProfScope(poly_handle *h_, int k) : h(h_), kind(k) {
    if (h->prof) {
      a = prof_event(h);
      cudaEventRecord(a, h->work);
    }
  }
  ~ProfScope() {
    if (h->prof) {
      cudaEvent_t b = prof_event(h);
      cudaEventRecord(b, h->work);
      h->recs.push_back({kind, a, b});
    }
  }
};

// K1 / K4: one pass over A at x (fp64, device)
int enqueue_pass(poly_handle *h, const double *x, bool loss) {
  ProfScope ps(h, 0);
  const poly_problem &p = h->p;
  if (p.layout == POLY_DENSE) {
    DenseArgs a{};
    a.A = p.A;
    a.lda = p.lda;
    a.n = p.n_local;
    a.d = (int32_t)p.d;
    a.W = p.W;
    a.y = p.y;
    a.ytype = p.ytype;
    a.relu = p.relu;
    a.s_row = p.s_row;
    a.I_row = p.I_row;
    a.I_bar = p.I_bar;
    a.x = x;
    a.spec = h->spec;
    a.partials = h->partials;
    a.loss_partials = h->loss_partials;
    a.stages = h->k1_stages;
    a.mode = p.mode;
    a.side_stride = h->k1_side;
    a.keep_stages = h->k1_keep;
    return launch(h, h->dv->fn[h->full][loss ? 1 : 0], dim3(h->k1_grid), dim3(h->k1_threads), h->k1_smem,
                  true, a);
  }
  CsrFwdArgs a{};
  a.row_ptr = p.row_ptr;
  a.col = p.col;
  a.val = p.val;
  a.n = p.n_local;
  a.W = p.W;
  a.y = p.y;
  a.ytype = p.ytype;
  a.relu = p.relu;
  a.s_row = p.s_row;
  a.I_row = p.I_row;
  a.I_bar = p.I_bar;
  if (p.layout == POLY_PARALLEL_BEAM) {
    const float *x32 = x == h->xa ? h->xa32 : (x == h->xh ? h->xh32 : nullptr);
    if (!x32) {
      TRY(launch(h, (const void *)&k_to_f32, dim3((unsigned)std::min<int64_t>(1024, (p.d + 255) / 256)),
                 dim3(256), 0, true, x, (int64_t)p.d, (int32_t)h->tr_side, h->xs, h->xin32));
      x32 = h->xin32;
    }
    CsrFwdArgs a{};
    a.n = p.n_local;
    a.W = p.W;
    a.y = p.y;
    a.ytype = p.ytype;
    a.relu = p.relu;
    a.I_bar = p.I_bar;
    a.spec = h->spec;
    a.r = h->rbuf;
    a.loss_partials = h->loss_partials;
    a.mode = p.mode;
    const int thr = std::max(32, (p.pb_bins + 31) / 32 * 32);
    TRY(launch(h, loss ? (const void *)&k_pb_forward<true> : (const void *)&k_pb_forward<false>,
               dim3(h->pb.nv, kPbRowSplit), dim3(thr), (size_t)kPbBufs * kPbRows * (p.pb_side + 2 * kPbPad) * 4, true, h->pb,
               x32, a));
    const unsigned tiles = (unsigned)(((p.pb_side + kPbTile - 1) / kPbTile) * ((p.pb_side + kPbTile - 1) / kPbTile));
    return launch(h, (const void *)&k_pb_backward, dim3(tiles, kPbParts), dim3(kPbTile * kPbTile / kPbPx), 0, true,
                  h->pb, (const float *)h->rbuf, h->pb_out2, h->partials);
  }
  // fp32 copy of x for the gathers: written by the step kernel for the
  // internal iterates, converted here for a caller's x
  const float *x32 = x == h->xa ? h->xa32 : (x == h->xh ? h->xh32 : nullptr);
  if (!x32) {
    TRY(launch(h, (const void *)&k_to_f32, dim3((unsigned)std::min<int64_t>(1024, (p.d + 255) / 256)),
               dim3(256), 0, true, x, (int64_t)p.d, (int32_t)h->tr_side, h->xs, h->xin32));
    x32 = h->xin32;
  }
  a.x = x32;
  a.spec = h->spec;
  a.r = h->rbuf;
  a.mode = p.mode;
  a.loss_partials = h->loss_partials;
  a.mu_step = h->mu_step;
  if (h->tiled) {
    TRY(launch(h, (const void *)&k_strip_forward, dim3(h->tf_grid), dim3((kFwdWarps + 1) * 32), h->tf_smem, true,
               h->tfwd, x32));
    TRY(launch(h, loss ? (const void *)&k_strip_link<true> : (const void *)&k_strip_link<false>, dim3(h->k4_grid),
               dim3(256), 0, true, a, (const double *)h->tfwd.pz, h->tfwd.NS, h->tfwd.ctr));
    return launch(h, (const void *)&k_tile_backward, dim3(h->tb_grid), dim3((2 * h->tbwd.npw + 1) * 32), h->tb_smem, true,
                  h->tbwd, (const float *)h->rbuf, h->partials, (int32_t)p.d, h->epi, h->tb_lcap);
  }
  if (h->dsell) {
    TRY(launch(h, loss ? (const void *)&k_dsell_forward<true> : (const void *)&k_dsell_forward<false>,
               dim3(h->k4_grid), dim3(kDsThreads), h->dfwd_smem, true, h->dfwd, (int64_t)h->nrslices,
               h->dfwd_cap, a));
    return launch(h, (const void *)&k_dsell_backward, dim3(h->dbwd_grid), dim3(kDsThreads), h->dbwd_smem, true,
                  h->dbwd, (int64_t)h->nslices, h->dbwd_cap, (int32_t)p.d, (const float *)h->rbuf, h->partials,
                  h->epi);
  }
  if (h->sell16) {
    TRY(launch(h, kSell16Fwd[p.dtype][loss ? 1 : 0], dim3(h->k4f16_grid), dim3(128), 0, true,
               h->fwd16, (int64_t)h->nrslices, a));
    return launch(h, kSell16Bwd[p.dtype], dim3(h->k4b16_grid), dim3(128), 0, true, h->bwd16,
                  (int64_t)h->nslices, (int32_t)p.d, (const float *)h->rbuf, h->partials, h->epi,
                  (const int32_t *)h->colmap);
  }
  TRY(launch(h, kCsrFwd[p.dtype][loss ? 1 : 0], dim3(h->k4_grid), dim3(128), 0, true,
             (const void *)h->sell_rows, (const int64_t *)h->row_slice_off, a));
  int32_t d32 = (int32_t)p.d;
  const float *rb = h->rbuf;
  double *gp = h->partials;
  const int32_t *cmap = h->colmap;
  if (p.dtype == POLY_F32)
    return launch(h, kCscBwd[0], dim3(h->nslices), dim3(128), 0, true,
                  (const CscEnt<float> *)h->sell, (const int64_t *)h->slice_off, d32, rb, gp, cmap);
  return launch(h, kCscBwd[1], dim3(h->nslices), dim3(128), 0, true,
                (const CscEnt<double> *)h->sell, (const int64_t *)h->slice_off, d32, rb, gp, cmap);
}

float *x32_of(poly_handle *h, const double *x) {
  return x == h->xa ? h->xa32 : (x == h->xh ? h->xh32 : nullptr);
}

FinArgs fin_base(poly_handle *h, int mode) {
  FinArgs f{};
  f.mode = mode;
  f.d = (int32_t)h->p.d;
  f.G = h->G;
  f.GL = h->p.layout == POLY_CSR ? h->k4_grid : (h->p.layout == POLY_PARALLEL_BEAM ? h->pb.nv : h->G);
  f.split = h->fin_split;
  f.need_loss = 1;
  f.set = h->p.set;
  f.n_norm = h->n_norm;
  f.partials = h->partials;
  f.loss_partials = h->loss_partials;
  f.comm = h->comm;
  f.v_scratch = h->vscratch;
  f.block_norm = h->block_norm;
  f.center = h->center;
  f.R = h->p.R;
  f.state = h->state;
  f.xs = h->xs;
  return f;
}

// P_X onto a TV set: one cluster of tv_cl CTAs (k_tv_project), in place allowed
int enqueue_tv(poly_handle *h, const double *v, double *out) {
  TvArgs a{};
  a.v = v;
  a.out = out;
  a.zk = h->tv_zk;
  a.p = h->tv_p;
  a.q = h->tv_q;
  a.s = (int32_t)llround(std::sqrt((double)h->p.d));
  a.nonneg = h->p.set == POLY_SET_TV_NONNEG ? 1 : 0;
  a.tau = h->p.tv_tau;
  a.tv_tol = h->p.tv_tol > 0.0 ? h->p.tv_tol : 0.01;
  a.rtol = h->p.tv_rtol > 0.0 ? h->p.tv_rtol : 1e-6;
  a.tol = h->p.tv_dykstra_tol > 0.0 ? h->p.tv_dykstra_tol : 1e-4;
  a.max_it = h->p.tv_max_it > 0 ? h->p.tv_max_it : 5000;
  a.max_outer = h->p.tv_max_outer > 0 ? h->p.tv_max_outer : 1000;
  a.stats = h->tv_stats;
  a.K = h->tv_k;
  a.tv_vals = h->tv_vals;
  a.gbar = h->tv_gbar;
  a.xsel = h->tv_xsel;
  a.timeout_ns = 20ull * 1000000000ull;
  a.warm = h->tv_ustate ? 1 : 0;
  a.u_state = h->tv_ustate;
  if (h->tv_k > 1) CK(cudaMemsetAsync(h->tv_gbar, 0, 4, h->work));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(h->tv_cl * h->tv_k);
  cfg.blockDim = dim3(kTvThreads);
  cfg.dynamicSmemBytes = h->tv_smem;
  cfg.stream = h->work;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = h->tv_cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = h->pdl ? 2 : 1;
  void *argv[] = {(void *)&a};
  CK(cudaLaunchKernelExC(&cfg, (const void *)&k_tv_project, argv));
  return POLY_OK;
}

// Cluster-resident whole solve for small dense problems (csrc/small.cuh).
// Returns POLY_EUNSUPPORTED (no error message) when the problem does not fit.
int small_solve_config(poly_handle *h, int *cl, size_t *smem) {
  const poly_problem &p = h->p;
  if (p.layout != POLY_DENSE || h->comm_path || p.s_row || p.d > kSmallMaxD || p.n_local < 1 ||
      p.set > POLY_SET_NONNEG_BALL || (p.flags & POLY_FLAG_NO_SMALL))
    return POLY_EUNSUPPORTED;
  const int C = (int)std::min<int64_t>(kSmallMaxCL, p.n_local);
  const int64_t rows = (p.n_local + C - 1) / C;
  const int64_t ldd = (p.d + 1) & ~1;
  const size_t s = (size_t)rows * ldd * h->elsize + 8 + (size_t)rows * 8 + 3 * kMaxW * 8 +
                   3 * kSmallMaxD * 8 + 2 * (kSmallMaxD + 1) * 8 +
                   (kSmallThreads / 32) * (kSmallMaxD + 1) * 8 + (kSmallThreads / 32) * 8 +
                   2 * 8 + (size_t)2 * C * (p.d + 1) * 8;  // mbarriers + pushed partials
  if (s > 200 * 1024) return POLY_EUNSUPPORTED;
  // a non-portable cluster of C CTAs with this much shared memory must be
  // schedulable on this part (MIG slices, smaller GPCs): else the general path
  {
    const void *fn = p.dtype == POLY_F32 ? (const void *)&k_small_solve<float, false>
                                         : (const void *)&k_small_solve<double, false>;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s) != cudaSuccess ||
        cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
      cudaGetLastError();
      return POLY_EUNSUPPORTED;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(kSmallThreads);
    cfg.dynamicSmemBytes = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg) != cudaSuccess || nclusters < 1) {
      cudaGetLastError();
      return POLY_EUNSUPPORTED;
    }
  }
  *cl = C;
  *smem = s;
  return POLY_OK;
}

int launch_small_solve(poly_handle *h, double *x_dev, int T, bool loss, int C, size_t smem) {
  const poly_problem &p = h->p;
  SmallArgs a{};
  a.A = p.A;
  a.lda = p.lda;
  a.n = (int32_t)p.n_local;
  a.d = (int32_t)p.d;
  a.W = p.W;
  a.ytype = p.ytype;
  a.relu = p.relu;
  a.mode = p.mode;
  a.set = p.set;
  a.y = p.y;
  a.I_bar = p.I_bar;
  a.R = p.R;
  a.gamma = h->hstate->gamma;
  a.n_norm = h->n_norm;
  a.spec = h->spec;
  a.center = h->center;
  a.x = x_dev;
  a.T = T;
  a.trace = loss ? h->trace : nullptr;
  a.state = h->state;
  const void *fn = p.dtype == POLY_F32
                       ? (loss ? (const void *)&k_small_solve<float, true> : (const void *)&k_small_solve<float, false>)
                       : (loss ? (const void *)&k_small_solve<double, true> : (const void *)&k_small_solve<double, false>);
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kSmallThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = h->work;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void *argv[] = {(void *)&a};
  CK(cudaLaunchKernelExC(&cfg, fn, argv));
  return POLY_OK;
}

int enqueue_fin(poly_handle *h, const FinArgs &f) {
  ProfScope ps(h, 1);
  // one partial row (CSR / matrix-free backward) or the comm buffer: warp 0
  // sums the columns and warp 1 of block 0 the loss — two warps suffice
  const bool one_row = f.G <= 1 || f.mode == FIN_GRAD_COMM || f.mode == FIN_STEP_COMM || f.mode == FIN_PROJECT;
  TRY(launch(h, (const void *)&k_finalize, dim3(h->fin_grid), dim3(one_row ? 64 : 256), 0, true, f));
  const bool steps = f.mode == FIN_STEP || f.mode == FIN_STEP_COMM || f.mode == FIN_PROJECT;
  if (h->tv_cl && steps) TRY(enqueue_tv(h, f.v_scratch, f.v_scratch));
  if (f.split && steps) {
    const int grid = (int)std::min<int64_t>(h->sms, (h->p.d + 255) / 256);
    TRY(launch(h, (const void *)&k_fin_apply, dim3(grid), dim3(256), 0, true, f));
  }
  return POLY_OK;
}

// the part of enqueue_fin after k_finalize, for a pass whose epilogue already
// wrote v and the block norms (FIN_STEP on the split path)
int enqueue_fin_tail(poly_handle *h, const FinArgs &f) {
  ProfScope ps(h, 1);
  if (h->tv_cl) TRY(enqueue_tv(h, f.v_scratch, f.v_scratch));
  const int grid = (int)std::min<int64_t>(h->sms, (h->p.d + 255) / 256);
  return launch(h, (const void *)&k_fin_apply, dim3(grid), dim3(256), 0, true, f);
}

int enqueue_allreduce(poly_handle *h) {
  ProfScope ps(h, 2);
  NcclApi *api = nccl_api();
  ncclResult_t r = api->allReduce(h->comm, h->comm, (size_t)h->p.d + 1, ncclFloat64, ncclSum,
                                  h->nccl, h->work);
  if (r != ncclSuccess) {
    api->commAbort(h->nccl);
    h->nccl = nullptr;
    return fail(POLY_ENCCL, "ncclAllReduce failed: %s", api->errStr(r));
  }
  return POLY_OK;
}

// K9: the cross-rank sum over NVLink peer memory (csrc/p2p.cuh)
int enqueue_peer_reduce(poly_handle *h) {
  ProfScope ps(h, 2);
  PeerArgs a{};
  a.comm = h->comm;
  a.n = h->p.d + 1;
  a.world = (int32_t)h->p.world;
  a.rank = (int32_t)h->p.rank;
  for (int r = 0; r < a.world; ++r) a.win[r] = h->p2p_peer[r];
  a.epoch = h->p2p_epoch;
  a.err = &h->state->comm_err;
  a.timeout_ns = (unsigned long long)(h->comm_timeout_s * 1e9);
  // the same grid on every rank (same d; the SM count of the GPU model)
  const int grid = (int)std::min<int64_t>(std::min(h->sms, kP2PMaxBlocks), (a.n + 255) / 256);
  // with PDL the blocks start while the reduce kernel drains and wait for it
  // (griddepcontrol.wait); K9 never triggers early, so its dependents start
  // after it exits and never compete with its waiting blocks for SMs
  return launch(h, (const void *)&k_peer_reduce, dim3(grid), dim3(256), 0, true, a);
}

int enqueue_nvls_reduce(poly_handle *h);

// F at x, then either g/loss (step == false) or x_out = P_X(anchor - γ F(x)).
int enqueue_eval(poly_handle *h, const double *x, bool loss, bool step, const double *anchor,
                 double *x_out, double *g_out) {
  FinArgs f = fin_base(h, 0);
  f.need_loss = loss ? 1 : 0;
  f.anchor = anchor;
  f.x_out = x_out;
  f.x32_out = x32_of(h, x_out);
  f.tr_side = h->tr_side;
  f.g_out = g_out;
  // compact-SELL CSR on the split path, plain step, no objective, one rank:
  // K4b's epilogue does k_finalize's work (same bits) and k_fin_apply follows
  const bool fuse = (h->sell16 || h->dsell || (h->tiled && h->tile_epi)) && h->p.layout == POLY_CSR && !h->comm_path && step && !loss && !g_out &&
                    f.split && !h->no_epi;
  h->epi = StepEpi{};
  if (fuse) {
    h->epi.on = 1;
    h->epi.set = f.set;
    h->epi.n_norm = (double)f.n_norm;
    h->epi.anchor = anchor;
    h->epi.center = f.center;
    h->epi.state = f.state;
    h->epi.v_scratch = f.v_scratch;
    h->epi.block_norm = f.block_norm;
  }
  const int prc = enqueue_pass(h, x, loss);
  h->epi = StepEpi{};
  TRY(prc);
  if (!h->comm_path) {
    f.mode = step ? FIN_STEP : FIN_GRAD;
    if (fuse) return enqueue_fin_tail(h, f);
    return enqueue_fin(h, f);
  }
  FinArgs r = f;
  r.mode = FIN_REDUCE;
  TRY(enqueue_fin(h, r));
  TRY(h->nv.on ? enqueue_nvls_reduce(h) : (h->p2p ? enqueue_peer_reduce(h) : enqueue_allreduce(h)));
  f.mode = step ? FIN_STEP_COMM : FIN_GRAD_COMM;
  return enqueue_fin(h, f);
}

// one EXACT iteration on the internal iterate xa (anchor), half-step in xh
int enqueue_iteration(poly_handle *h, bool loss) {
  TRY(enqueue_eval(h, h->xa, loss, true, h->xa, h->xh, nullptr));
  return enqueue_eval(h, h->xh, loss, true, h->xa, h->xa, nullptr);
}

AvgArgs avg_args(poly_handle *h) {
  AvgArgs a{};
  a.x = h->xa;
  a.hist = h->hist;
  a.S = h->Ssum;
  a.xbar = h->xbar;
  a.block_norm = h->avg_norm;
  a.d = (int32_t)h->p.d;
  a.cap = h->avg_cap;
  a.state = h->state;
  return a;
}

int enqueue_avg(poly_handle *h) {
  ProfScope ps(h, 1);
  const AvgArgs a = avg_args(h);
  const int nb = (int)((h->p.d + 255) / 256);
  TRY(launch(h, (const void *)&k_avg_a, dim3(nb), dim3(256), 0, true, a));
  return launch(h, (const void *)&k_avg_b, dim3(1), dim3(32), 0, true, a, (int32_t)nb);
}

// one iteration of poly_solve_ex: EXACT (2 passes) or projected GD (1 pass)
// on the internal iterate xa, then the averaged-iterate update
int enqueue_iteration_ex(poly_handle *h, int method, bool average) {
  if (method == POLY_METHOD_EXTRAGRADIENT)
    TRY(enqueue_iteration(h, false));
  else
    TRY(enqueue_eval(h, h->xa, false, true, h->xa, h->xa, nullptr));
  if (average) TRY(enqueue_avg(h));
  return POLY_OK;
}

int build_graph_ex(poly_handle *h, int method, bool average, int U, cudaGraphExec_t *out) {
  cudaGraph_t g = nullptr;
  CK(cudaStreamBeginCapture(h->work, cudaStreamCaptureModeThreadLocal));
  int rc = POLY_OK;
  for (int u = 0; u < U && rc == POLY_OK; ++u) rc = enqueue_iteration_ex(h, method, average);
  cudaError_t e = cudaStreamEndCapture(h->work, &g);
  if (rc != POLY_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (e != cudaSuccess) return fail(POLY_ECUDA, "graph capture: %s", cudaGetErrorString(e));
  e = cudaGraphInstantiate(out, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return fail(POLY_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
  // upload now, not at the first launch (which would then carry the upload)
  if (cudaGraphUpload(*out, h->work) != cudaSuccess)
    return fail(POLY_ECUDA, "graph upload: %s", cudaGetErrorString(cudaGetLastError()));
  return POLY_OK;
}

int build_graph(poly_handle *h, bool loss, int U, cudaGraphExec_t *out) {
  cudaGraph_t g = nullptr;
  CK(cudaStreamBeginCapture(h->work, cudaStreamCaptureModeThreadLocal));
  int rc = POLY_OK;
  for (int u = 0; u < U && rc == POLY_OK; ++u) rc = enqueue_iteration(h, loss);
  cudaError_t e = cudaStreamEndCapture(h->work, &g);
  if (rc != POLY_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (e != cudaSuccess) return fail(POLY_ECUDA, "graph capture: %s", cudaGetErrorString(e));
  e = cudaGraphInstantiate(out, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return fail(POLY_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
  // upload now, not at the first launch (which would then carry the upload)
  if (cudaGraphUpload(*out, h->work) != cudaSuccess)
    return fail(POLY_ECUDA, "graph upload: %s", cudaGetErrorString(cudaGetLastError()));
  return POLY_OK;
}

int sync_in(poly_handle *h) {
  CK(cudaEventRecord(h->ev_in, h->user));
  CK(cudaStreamWaitEvent(h->work, h->ev_in, 0));
  return POLY_OK;
}
int sync_out(poly_handle *h) {
  CK(cudaEventRecord(h->ev_out, h->work));
  CK(cudaStreamWaitEvent(h->user, h->ev_out, 0));
  return POLY_OK;
}

// Poll the communicator for an asynchronous error (a failed peer, a network
// error).  On one the communicator is aborted so that this rank returns
// instead of hanging (poly.h: "a rank aborts its communicator").
int check_comm(poly_handle *h) {
  if (!h->comm_path) return POLY_OK;
  if (!h->nccl) return fail(POLY_ENCCL, "the communicator was aborted by an earlier error");
  NcclApi *api = nccl_api();
  ncclResult_t st = ncclSuccess;
  const ncclResult_t q = api->asyncErr(h->nccl, &st);
  if (q != ncclSuccess || (st != ncclSuccess && st != ncclInProgress)) {
    api->commAbort(h->nccl);
    h->nccl = nullptr;
    return fail(POLY_ENCCL, "NCCL asynchronous error: %s; communicator aborted",
                api->errStr(q != ncclSuccess ? q : st));
  }
  return POLY_OK;
}

// Host wait for ev.  Without a communicator: cudaEventSynchronize.  With one,
// the wait polls NCCL's asynchronous error state and gives up after
// comm_timeout_s: the communicator is aborted (which also releases NCCL
// kernels waiting on a dead peer) and POLY_ENCCL returned.
int wait_event(poly_handle *h, cudaEvent_t ev) {
  if (!h->comm_path) {
    CK(cudaEventSynchronize(ev));
    return POLY_OK;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaEventQuery(ev);
    if (q == cudaSuccess) return POLY_OK;
    if (q != cudaErrorNotReady) return fail(POLY_ECUDA, "stream failed: %s", cudaGetErrorString(q));
    TRY(check_comm(h));
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el > h->comm_timeout_s) {
      NcclApi *api = nccl_api();
      if (h->nccl) api->commAbort(h->nccl);
      h->nccl = nullptr;
      return fail(POLY_ENCCL, "no progress for %.0f s with a communicator (a peer stopped?); aborted",
                  h->comm_timeout_s);
    }
    std::this_thread::sleep_for(std::chrono::microseconds(el < 0.01 ? 2 : 50));
  }
}

// The TV projection's clusters flag stats[3] when they failed to meet.
int check_tv_meet(poly_handle *h) {
  if (!h->tv_stats || h->tv_k <= 1) return POLY_OK;
  int32_t f = 0;
  CK(cudaMemcpy(&f, h->tv_stats + 3, 4, cudaMemcpyDeviceToHost));
  if (f) return fail(POLY_ECUDA, "TV projection: the %d clusters did not meet (not co-resident)", h->tv_k);
  return POLY_OK;
}

// Drain the work stream (through wait_event, so a hung collective cannot
// block the host forever).
int sync_work(poly_handle *h) {
  CK(cudaEventRecord(h->ev_sync, h->work));
  return wait_event(h, h->ev_sync);
}

template <typename T>
int dev_alloc(poly_handle *h, T **ptr, size_t count) {
  void *p = nullptr;
  cudaError_t e = cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(POLY_ENOMEM, "cudaMalloc(%zu bytes): %s", count * sizeof(T), cudaGetErrorString(e));
  }
  h->owned.push_back(p);
  *ptr = (T *)p;
  return POLY_OK;
}

void dev_release(poly_handle *h, void *ptr) {
  for (auto it = h->owned.begin(); it != h->owned.end(); ++it)
    if (*it == ptr) {
      cudaFree(ptr);
      h->owned.erase(it);
      return;
    }
}

int copy_in(poly_handle *h, const void **field, size_t bytes) {
  if (!*field || bytes == 0) return POLY_OK;
  void *d = nullptr;
  TRY(dev_alloc(h, (unsigned char **)&d, bytes));
  CK(cudaMemcpyAsync(d, *field, bytes, cudaMemcpyHostToDevice, h->work));
  *field = d;
  return POLY_OK;
}

int validate(const poly_problem *p) {
  if (!p) return fail(POLY_EINVAL, "problem is NULL");
  if (p->n_local < 0) return fail(POLY_EINVAL, "n_local < 0");
  if (p->n_global < 1 || p->n_global < p->n_local) return fail(POLY_EINVAL, "n_global must be >= max(1, n_local)");
  if (p->d < 1 || p->d > (1 << 30)) return fail(POLY_EINVAL, "d out of range");
  if (p->layout != POLY_DENSE && p->layout != POLY_CSR && p->layout != POLY_PARALLEL_BEAM)
    return fail(POLY_EINVAL, "bad layout");
  if (p->layout == POLY_PARALLEL_BEAM) {
    if (p->pb_side < 2 || p->pb_side > 4096 || (int64_t)p->pb_side * p->pb_side != p->d)
      return fail(POLY_EINVAL, "parallel beam: d must be pb_side^2, 2 <= pb_side <= 4096");
    if (p->pb_views < 1 || p->pb_bins < 1 || p->pb_bins > 1024)
      return fail(POLY_EINVAL, "parallel beam: need pb_views >= 1 and 1 <= pb_bins <= 1024");
    if (p->n_local % p->pb_bins || p->row_offset % p->pb_bins ||
        p->row_offset + p->n_local > (int64_t)p->pb_views * p->pb_bins)
      return fail(POLY_EINVAL, "parallel beam: rows must be whole views of the V*B rays");
    if (p->mode != POLY_MODE_EXACT || p->s_row)
      return fail(POLY_EUNSUPPORTED, "parallel beam: mode EXACT without per-row spectra only");
  }
  if (p->dtype != POLY_F32 && p->dtype != POLY_F64) return fail(POLY_EINVAL, "bad dtype");
  if (p->ytype < POLY_Y_I32 || p->ytype > POLY_Y_F64) return fail(POLY_EINVAL, "bad ytype");
  if (p->W < 1) return fail(POLY_EINVAL, "W < 1 (SPEC.md:28)");
  if (p->W > kMaxW) return fail(POLY_EUNSUPPORTED, "W > %d", kMaxW);
  if (!p->s || !p->mu) return fail(POLY_EINVAL, "spectrum pointers are NULL");
  if (p->windows < 0) return fail(POLY_EINVAL, "windows < 0");
  const int Om = p->windows > 1 ? p->windows : 1;
  if (Om > 1 && !p->I_win) return fail(POLY_EINVAL, "windows > 1 needs I_win");
  for (int w = 0; w < Om; ++w) {
    double tot = 0.0;
    for (int j = 0; j < p->W; ++j) {
      const double sj = p->s[(size_t)w * p->W + j];
      if (!(sj > 0.0 && sj <= 1.0)) return fail(POLY_EINVAL, "s[%d] of window %d not in (0,1] (SPEC.md:25)", j, w);
      tot += sj;
    }
    if (std::fabs(tot - 1.0) > 1e-12) return fail(POLY_EINVAL, "window %d: sum_j s_j = %.17g != 1 (SPEC.md:25)", w, tot);
    if (Om > 1 && (!(p->I_win[w] > 0.0) || !std::isfinite(p->I_win[w])))
      return fail(POLY_EINVAL, "I_win[%d] must be > 0", w);
  }
  for (int j = 0; j < p->W; ++j)
    if (!(p->mu[j] > 0.0) || !std::isfinite(p->mu[j])) return fail(POLY_EINVAL, "mu[%d] must be > 0 (SPEC.md:26)", j);
  if (Om == 1 && (!(p->I_bar > 0.0) || !std::isfinite(p->I_bar))) return fail(POLY_EINVAL, "I_bar must be > 0 (SPEC.md:27)");
  if (p->mode < POLY_MODE_EXACT || p->mode > POLY_MODE_NLL) return fail(POLY_EINVAL, "bad mode");
  if (Om > 1 && (p->mode != POLY_MODE_EXACT || p->s_row))
    return fail(POLY_EUNSUPPORTED, "windows > 1 needs mode EXACT and no per-row spectra");
  if ((p->s_row == nullptr) != (p->I_row == nullptr)) return fail(POLY_EINVAL, "s_row and I_row must both be given or both NULL");
  if (p->relu != 0 && p->relu != 1) return fail(POLY_EINVAL, "relu must be 0 or 1");
  if (p->set < POLY_SET_NONE || p->set > POLY_SET_TV) return fail(POLY_EINVAL, "bad set");
  if (p->set == POLY_SET_TV_NONNEG || p->set == POLY_SET_TV) {
    const int64_t s = (int64_t)llround(std::sqrt((double)p->d));
    if (s * s != p->d || s < 2) return fail(POLY_EINVAL, "TV sets need d = s*s (an s x s image), s >= 2");
    if (!(p->tv_tau >= 0.0) || p->tv_tol < 0.0 || p->tv_rtol < 0.0 || p->tv_dykstra_tol < 0.0 ||
        p->tv_max_it < 0 || p->tv_max_outer < 0)
      return fail(POLY_EINVAL, "TV parameters must be >= 0");
    if (p->center) return fail(POLY_EINVAL, "TV sets take no center");
  }
  if ((p->set == POLY_SET_BALL || p->set == POLY_SET_NONNEG_BALL) && !(p->R > 0.0))
    return fail(POLY_EINVAL, "ball radius must be > 0");
  if (p->set == POLY_SET_NONNEG_BALL && p->center) return fail(POLY_EINVAL, "NONNEG_BALL requires center = NULL");
  if (p->world < 1 || p->rank < 0 || p->rank >= p->world) return fail(POLY_EINVAL, "bad rank/world");
  if ((p->world > 1 || (p->flags & POLY_FLAG_COMM)) && !p->nccl_id)
    return fail(POLY_EINVAL, "world > 1 (or POLY_FLAG_COMM) needs nccl_id");
  if (p->n_local > 0) {
    if (!p->y) return fail(POLY_EINVAL, "y is NULL");
    if (p->layout == POLY_DENSE) {
      if (!p->A) return fail(POLY_EINVAL, "A is NULL");
      if (p->lda < p->d) return fail(POLY_EINVAL, "lda < d");
      const int es = p->dtype == POLY_F32 ? 4 : 8;
      if ((p->lda * es) % 16 != 0) return fail(POLY_EINVAL, "lda*elsize must be a multiple of 16 bytes");
      if (!(p->flags & POLY_FLAG_HOST_INPUTS) && ((uintptr_t)p->A % 16) != 0)
        return fail(POLY_EINVAL, "A must be 16-byte aligned");
    } else if (p->layout == POLY_CSR) {
      if (!p->row_ptr || (p->nnz > 0 && (!p->col || !p->val))) return fail(POLY_EINVAL, "CSR arrays are NULL");
      if (p->nnz < 0) return fail(POLY_EINVAL, "nnz < 0");
    }
  }
  return POLY_OK;
}

int setup_dense(poly_handle *h) {
  const poly_problem &p = h->p;
  const int vec = 16 / h->elsize;
  const DenseVariant *tab = p.dtype == POLY_F32 ? kDenseF32 : kDenseF64;
  const DenseVariant *dv = nullptr;
  for (int i = 0; i < 7; ++i) {
    const int64_t cols = (int64_t)32 * vec * tab[i].V * tab[i].WPR;
    if (p.d <= cols) {
      dv = &tab[i];
      break;
    }
  }
  if (!dv) return fail(POLY_EUNSUPPORTED, "dense d = %lld exceeds the largest tile (%d columns)",
                       (long long)p.d, 32 * vec * 8 * 8);
  if (const char *tv = getenv("POLY_K1_TUNE")) {
    const int i = atoi(tv);
    const int nt = (int)(sizeof(kDenseTuneF32) / sizeof(kDenseTuneF32[0]));
    if (p.dtype == POLY_F32 && i >= 0 && i < nt &&
        p.d <= (int64_t)32 * vec * kDenseTuneF32[i].V * kDenseTuneF32[i].WPR)
      dv = &kDenseTuneF32[i];
  }
  h->dv = dv;
  h->full = (p.d == (int64_t)32 * vec * dv->V * dv->WPR) ? 1 : 0;
  h->k1_threads = 32 * (dv->NW + 1);
  const int G = dv->NW / dv->WPR;
  const int RG = dv->RPS / G;
  const size_t stage = (size_t)dv->RPS * p.lda * h->elsize;
  h->k1_side = (int)(((size_t)dv->RPS * (12 + 4 * p.W) + 15) / 16 * 16);
  // z exchange [2][G][RG][WPR] + link partials [2][G][RG][WPR][2] + spectrum + mbarriers + loss
  const size_t fixed = (size_t)6 * G * RG * dv->WPR * 8 + 3 * kMaxW * 8 + 2 * 8 * 8 + dv->NW * 8 + 256;
  int S = (int)(kRingBudget / (stage + h->k1_side));
  S = std::max(2, std::min(8, S));
  size_t ring = (size_t)S * stage;
  const size_t gred = (size_t)G * p.d * h->elsize;
  while (ring < gred && S < 8) ring = (size_t)(++S) * stage;
  if (ring < gred) return fail(POLY_EUNSUPPORTED, "tile configuration does not fit (ring < reduction)");
  h->k1_stages = S;
  h->k1_smem = ring + (size_t)S * h->k1_side + fixed;
  if (h->k1_smem > kSmemLimit) {
    S = 2;
    h->k1_stages = S;
    h->k1_smem = (size_t)S * (stage + h->k1_side) + fixed;
    if (h->k1_smem > kSmemLimit || (size_t)S * stage < gred)
      return fail(POLY_EUNSUPPORTED, "row of %lld elements too large for the smem ring", (long long)p.lda);
  }
  for (int l = 0; l < 2; ++l)
    CK(cudaFuncSetAttribute(dv->fn[h->full][l], cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)h->k1_smem));
  const int64_t tiles = (p.n_local + dv->RPS - 1) / dv->RPS;
  h->k1_grid = (int)std::max<int64_t>(1, std::min<int64_t>(h->sms, tiles));
  h->G = h->k1_grid;
  {
    // each CTA's first stages kept in L2 across passes (evict-last); POLY_K1_KEEP_MB overrides
    double keep_mb = kK1KeepMB;
    if (const char *e = getenv("POLY_K1_KEEP_MB")) keep_mb = atof(e);
    h->k1_keep = (int)(keep_mb * 1e6 / ((double)stage * h->k1_grid));
    h->keep_bytes = std::min<int64_t>((int64_t)h->k1_keep * (int64_t)stage * h->k1_grid,
                                      (int64_t)p.n_local * p.lda * (int64_t)h->elsize);
  }
  return POLY_OK;
}

// DSELL (dsell.cuh) of one direction from its padded SELL-32 copy: count
// pass (|F_s|, runs, groups per slice), offsets on the host, write pass.
// POLY_EUNSUPPORTED (no message) when a slice's target span exceeds the pack
// kernel's bitmap or the staged dictionary would not fit shared memory.
int build_dsell_dir(poly_handle *h, const CscEnt<float> *ent, const int64_t *slice_off, int64_t nslices,
                    const int64_t *row_ptr, const int32_t *cnt, int64_t nlanes, DSell *out, int32_t *cap,
                    size_t *smem) {
  cudaStream_t st = h->work;
  std::vector<void *> tmp;
  auto done = [&](int code) {
    cudaStreamSynchronize(st);
    for (void *q : tmp) cudaFree(q);
    return code;
  };
  auto talloc = [&](size_t bytes, void **ptr) -> int {
    if (cudaMalloc(ptr, std::max<size_t>(bytes, 16)) != cudaSuccess) {
      cudaGetLastError();
      return fail(POLY_ENOMEM, "DSELL build: cudaMalloc(%zu) failed", bytes);
    }
    tmp.push_back(*ptr);
    return POLY_OK;
  };
  int64_t *fpl = nullptr, *nrun = nullptr, *ngr = nullptr;
  int32_t *bad = nullptr;
  int rc;
  if ((rc = talloc((size_t)nslices * 8, (void **)&fpl)) || (rc = talloc((size_t)nslices * 8, (void **)&nrun)) ||
      (rc = talloc((size_t)nslices * 8, (void **)&ngr)) || (rc = talloc(4, (void **)&bad)))
    return done(rc);
  CK(cudaFuncSetAttribute((const void *)&k_dsell_pack<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)kDsPackSmem));
  CK(cudaFuncSetAttribute((const void *)&k_dsell_pack<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)kDsPackSmem));
  cudaMemsetAsync(bad, 0, 4, st);
  const int grid = (int)std::min<int64_t>(std::max<int64_t>(1, nslices), (int64_t)h->sms * 2);
  k_dsell_pack<false><<<grid, kDsPackThreads, kDsPackSmem, st>>>(ent, slice_off, nslices, row_ptr, cnt, nlanes, fpl,
                                                                 nrun, ngr, nullptr, nullptr, nullptr, nullptr,
                                                                 nullptr, nullptr, bad);
  std::vector<int64_t> hf((size_t)nslices), hr((size_t)nslices), hg((size_t)nslices);
  int32_t hbad = 0;
  cudaMemcpyAsync(hf.data(), fpl, (size_t)nslices * 8, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(hr.data(), nrun, (size_t)nslices * 8, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(hg.data(), ngr, (size_t)nslices * 8, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess)
    return done(fail(POLY_ECUDA, "DSELL count: %s", cudaGetErrorString(cudaGetLastError())));
  if (hbad) return done(POLY_EUNSUPPORTED);
  std::vector<int64_t> goff((size_t)nslices + 1, 0), roff((size_t)nslices + 1, 0);
  int64_t fmax = 0, rmax = 0;
  for (int64_t i = 0; i < nslices; ++i) {
    goff[i + 1] = goff[i] + hg[i];
    roff[i + 1] = roff[i] + hr[i] + 1;
    fmax = std::max(fmax, hf[i]);
    rmax = std::max(rmax, hr[i] + 1);
  }
  // two dictionary buffers (double-buffered staging); local indices fit uint16
  const size_t sm = (size_t)2 * (((size_t)fmax + 3) & ~(size_t)3) * 4;
  if (sm > (size_t)110 * 1024 || fmax >= 65536) return done(POLY_EUNSUPPORTED);
  (void)rmax;
  const int64_t groups = goff[nslices];
  int64_t *dgoff = nullptr, *droff = nullptr;
  uchar4 *dl = nullptr;
  float4 *val = nullptr;
  uint16_t *base = nullptr;
  int2 *runs = nullptr;
  if ((rc = dev_alloc(h, &dgoff, (size_t)nslices + 1)) || (rc = dev_alloc(h, &droff, (size_t)nslices + 1)) ||
      (rc = dev_alloc(h, &dl, (size_t)std::max<int64_t>(1, groups) * 32)) ||
      (rc = dev_alloc(h, &val, (size_t)std::max<int64_t>(1, groups) * 32)) ||
      (rc = dev_alloc(h, &base, (size_t)nslices * kDsWarps * 32)) ||
      (rc = dev_alloc(h, &runs, (size_t)std::max<int64_t>(1, roff[nslices]))))
    return done(rc);
  cudaMemcpyAsync(dgoff, goff.data(), goff.size() * 8, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(droff, roff.data(), roff.size() * 8, cudaMemcpyHostToDevice, st);
  k_dsell_pack<true><<<grid, kDsPackThreads, kDsPackSmem, st>>>(ent, slice_off, nslices, row_ptr, cnt, nlanes,
                                                                nullptr, nullptr, nullptr, dgoff, droff, dl, val,
                                                                base, runs, bad);
  if (cudaStreamSynchronize(st) != cudaSuccess)
    return done(fail(POLY_ECUDA, "DSELL write: %s", cudaGetErrorString(cudaGetLastError())));
  *out = DSell{dl, val, base, dgoff, runs, droff};
  *cap = (int32_t)fmax;
  *smem = sm;
  return done(POLY_OK);
}

// SELL-32 copy of Aᵀ for K4b (poly_init only): stable radix sort of the
// entries by column (ties keep CSR order = ascending row), column pointers by
// histogram + scan, slice length = longest column of 32, zero padding.
template <typename T>
int build_sell_t(poly_handle *h) {
  const poly_problem &p = h->p;
  const int64_t nnz = p.nnz, d = p.d;
  if (nnz >= (int64_t)1 << 31) return fail(POLY_EUNSUPPORTED, "nnz >= 2^31");
  h->nslices = (int)((d + 31) / 32);
  TRY(dev_alloc(h, &h->slice_off, (size_t)h->nslices + 1));
  cudaStream_t st = h->work;
  std::vector<void *> tmp;
  auto talloc = [&](size_t bytes, void **ptr) -> int {
    if (cudaMalloc(ptr, std::max<size_t>(bytes, 16)) != cudaSuccess) {
      cudaGetLastError();
      return fail(POLY_ENOMEM, "SELL build: cudaMalloc(%zu) failed", bytes);
    }
    tmp.push_back(*ptr);
    return POLY_OK;
  };
  auto done = [&](int code) {
    cudaStreamSynchronize(st);
    for (void *q : tmp) cudaFree(q);
    return code;
  };
  int32_t *rows = nullptr, *perm_in = nullptr, *perm = nullptr, *keys = nullptr, *cnt = nullptr;
  int64_t *cnt64 = nullptr, *colptr = nullptr, *slen = nullptr;
  int rc;
  if ((rc = talloc(nnz * 4, (void **)&rows)) || (rc = talloc(nnz * 4, (void **)&perm_in)) ||
      (rc = talloc(nnz * 4, (void **)&perm)) || (rc = talloc(nnz * 4, (void **)&keys)) ||
      (rc = talloc(d * 4, (void **)&cnt)) || (rc = talloc((d + 1) * 8, (void **)&cnt64)) ||
      (rc = talloc((d + 1) * 8, (void **)&colptr)) ||
      (rc = talloc((size_t)(h->nslices + 1) * 8, (void **)&slen)))
    return done(rc);
  const int g = 148 * 8;
  if (nnz > 0) {
    k_entry_rows<<<g, 256, 0, st>>>(p.row_ptr, p.n_local, rows);
    k_iota<<<g, 256, 0, st>>>(perm_in, nnz);
  }
  cudaMemsetAsync(cnt, 0, d * 4, st);
  if (nnz > 0) k_col_count<<<g, 256, 0, st>>>(p.col, nnz, cnt);
  size_t tb = 0, tb2 = 0, tb3 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, p.col, keys, perm_in, perm, (int)nnz, 0,
                                  32 - __builtin_clz((unsigned)std::max<int64_t>(1, d)), st);
  cub::DeviceScan::ExclusiveSum(nullptr, tb2, cnt64, colptr, (int)d + 1, st);
  cub::DeviceScan::ExclusiveSum(nullptr, tb3, slen, h->slice_off, h->nslices + 1, st);
  void *tstore = nullptr;
  if ((rc = talloc(std::max(tb, std::max(tb2, tb3)), &tstore))) return done(rc);
  if (nnz > 0) {
    size_t t = tb;
    if (cub::DeviceRadixSort::SortPairs(tstore, t, p.col, keys, perm_in, perm, (int)nnz, 0,
                                        32 - __builtin_clz((unsigned)std::max<int64_t>(1, d)),
                                        st) != cudaSuccess)
      return done(fail(POLY_ECUDA, "SELL build: radix sort failed"));
  }
  k_widen<<<(int)std::min<int64_t>(4096, (d + 256) / 256), 256, 0, st>>>(cnt, d, cnt64);
  size_t t2 = tb2;
  cub::DeviceScan::ExclusiveSum(tstore, t2, cnt64, colptr, (int)d + 1, st);
  // opt-in (POLY_K4B_SYNC=1), square images (d = side², side % 8 == 0): 4 x 8
  // pixel tiles as slices and lane chains re-aligned every row block (csr.cuh
  // k_sell_fill_sync).  On C4 it cuts K4b's gather sectors per request from
  // 16.9 to 7.2 but adds 9 % padding and runs slower (46 vs 40 us): the pass
  // is latency-bound, not sector-bound
  const int side = h->tr_side;
  const bool synced = side > 0 && side % 8 == 0 && (int64_t)side * side == d && nnz > 0 &&
                      getenv("POLY_K4B_SYNC") && !getenv("POLY_DSELL");
  int32_t NBK = 24;
  if (const char *e = getenv("POLY_K4B_BLOCKS")) NBK = std::max(1, atoi(e));
  const int32_t RB = (int32_t)std::max<int64_t>(1, (p.n_local + NBK - 1) / NBK);
  int32_t *blkoff = nullptr, *bpre = nullptr, *blkcnt = nullptr, *slot_of = nullptr;
  if (synced) {
    std::vector<int32_t> cm((size_t)h->nslices * 32, -1), so((size_t)d, -1);
    const int tw = 8, th = 4, tpr = side / tw;
    for (int t = 0; t < h->nslices; ++t) {
      const int r0 = (t / tpr) * th, c0 = (t % tpr) * tw;
      for (int l = 0; l < 32; ++l) {
        const int r = r0 + l / tw, c = c0 + l % tw;
        if (r < side) {
          cm[(size_t)t * 32 + l] = r * side + c;
          so[(size_t)r * side + c] = t * 32 + l;
        }
      }
    }
    if ((rc = dev_alloc(h, &h->colmap, cm.size())) || (rc = talloc((size_t)d * 4, (void **)&slot_of)) ||
        (rc = talloc((size_t)d * NBK * 4, (void **)&blkcnt)) || (rc = talloc((size_t)d * NBK * 4, (void **)&bpre)) ||
        (rc = talloc((size_t)h->nslices * NBK * 4, (void **)&blkoff)))
      return done(rc);
    cudaMemcpyAsync(h->colmap, cm.data(), cm.size() * 4, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(slot_of, so.data(), so.size() * 4, cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(blkcnt, 0, (size_t)d * NBK * 4, st);
    k_colblk_count<<<g, 256, 0, st>>>(rows, p.col, nnz, RB, NBK, blkcnt);
    k_colblk_prefix<<<(int)((d + 255) / 256), 256, 0, st>>>(blkcnt, (int32_t)d, NBK, bpre);
    k_slice_blocks<<<(h->nslices + 127) / 128, 128, 0, st>>>(blkcnt, h->colmap, h->nslices, NBK, blkoff, slen);
  } else {
    k_slice_len<<<(h->nslices + 255) / 256, 256, 0, st>>>(cnt, (int32_t)d, h->nslices, slen);
  }
  cudaMemsetAsync(slen + h->nslices, 0, 8, st);
  size_t t3 = tb3;
  cub::DeviceScan::ExclusiveSum(tstore, t3, slen, h->slice_off, h->nslices + 1, st);
  int64_t steps = 0;
  cudaMemcpyAsync(&steps, h->slice_off + h->nslices, 8, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess)
    return done(fail(POLY_ECUDA, "SELL build: %s", cudaGetErrorString(cudaGetLastError())));
  CscEnt<T> *ent = nullptr;
  if ((rc = dev_alloc(h, &ent, (size_t)std::max<int64_t>(1, steps) * 32))) return done(rc);
  if (synced) {
    k_sell_mark<T><<<g, 256, 0, st>>>(ent, std::max<int64_t>(1, steps) * 32);
    k_sell_fill_sync<T><<<g, 256, 0, st>>>(keys, perm, rows, (const T *)p.val, colptr, bpre, blkoff, slot_of,
                                           h->slice_off, RB, NBK, nnz, ent);
  } else {
    cudaMemsetAsync(ent, 0, (size_t)std::max<int64_t>(1, steps) * 32 * sizeof(CscEnt<T>), st);
    if (nnz > 0)
      k_sell_fill<T><<<g, 256, 0, st>>>(keys, perm, rows, (const T *)p.val, colptr, h->slice_off,
                                        nnz, ent);
  }
  h->sell = ent;
  h->sell_steps = steps;
  // DSELL (fp32, dsell.cuh): the forward copy needs every row's entries ascending in
  // column (a segmented sort of the caller's CSR; the summation order of z_i
  // then follows the sorted columns) and no transposed-x layout
  // opt-in (POLY_DSELL=1): on C4 it streams 13 % fewer bytes than SELL16 but
  // spends them on per-slice staging instructions and barriers
  const bool want_ds = std::is_same<T, float>::value && getenv("POLY_DSELL") && p.n_local > 0 && nnz > 0 &&
                       nnz < ((int64_t)1 << 31) && p.n_local < ((int64_t)1 << 31);
  const int32_t *rcol = p.col;
  const T *rval = (const T *)p.val;
  if (want_ds) {
    int32_t *cs = nullptr;
    T *vs = nullptr;
    if ((rc = talloc((size_t)nnz * 4, (void **)&cs)) || (rc = talloc((size_t)nnz * sizeof(T), (void **)&vs)))
      return done(rc);
    size_t tbs = 0;
    cub::DeviceSegmentedSort::StableSortPairs(nullptr, tbs, p.col, cs, (const T *)p.val, vs, (int)nnz,
                                              (int)p.n_local, p.row_ptr, p.row_ptr + 1, st);
    void *tss = nullptr;
    if ((rc = talloc(tbs, &tss))) return done(rc);
    if (cub::DeviceSegmentedSort::StableSortPairs(tss, tbs, p.col, cs, (const T *)p.val, vs, (int)nnz,
                                                  (int)p.n_local, p.row_ptr, p.row_ptr + 1, st) != cudaSuccess)
      return done(fail(POLY_ECUDA, "DSELL build: segmented sort failed"));
    rcol = cs;
    rval = vs;
  }
  // SELL-32 of A (row slices) for K4f
  const int64_t nrs = h->nrslices;
  TRY(dev_alloc(h, &h->row_slice_off, (size_t)nrs + 1));
  int64_t *rlen = nullptr;
  if ((rc = talloc((size_t)(nrs + 1) * 8, (void **)&rlen))) return done(rc);
  size_t tb4 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb4, rlen, h->row_slice_off, (int)nrs + 1, st);
  void *tstore2 = nullptr;
  if ((rc = talloc(tb4, &tstore2))) return done(rc);
  cudaMemsetAsync(rlen, 0, (size_t)(nrs + 1) * 8, st);
  if (p.n_local > 0) k_row_slice_len<<<(int)std::min<int64_t>(4096, (nrs + 255) / 256), 256, 0, st>>>(
      p.row_ptr, p.n_local, nrs, rlen);
  cub::DeviceScan::ExclusiveSum(tstore2, tb4, rlen, h->row_slice_off, (int)nrs + 1, st);
  int64_t rsteps = 0;
  cudaMemcpyAsync(&rsteps, h->row_slice_off + nrs, 8, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess)
    return done(fail(POLY_ECUDA, "SELL build: %s", cudaGetErrorString(cudaGetLastError())));
  CscEnt<T> *rent = nullptr;
  if ((rc = dev_alloc(h, &rent, (size_t)std::max<int64_t>(1, rsteps) * 32))) return done(rc);
  cudaMemsetAsync(rent, 0, (size_t)std::max<int64_t>(1, rsteps) * 32 * sizeof(CscEnt<T>), st);
  int8_t *use_tr = nullptr;
  if (h->tr_side && p.n_local > 0 && !want_ds) {
    if ((rc = talloc((size_t)nrs, (void **)&use_tr))) return done(rc);
    k_slice_layout<<<(int)std::min<int64_t>(4096, (nrs + 7) / 8), 256, 0, st>>>(
        p.row_ptr, p.col, p.n_local, h->tr_side, nrs, use_tr);
    std::vector<int8_t> ut((size_t)nrs);
    if (cudaMemcpyAsync(ut.data(), use_tr, (size_t)nrs, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return done(fail(POLY_ECUDA, "SELL layout: %s", cudaGetErrorString(cudaGetLastError())));
    h->tr_slices = 0;
    for (int8_t v : ut) h->tr_slices += v;
  }
  const int fill_side = h->tr_side;
  if (!h->tr_slices) h->tr_side = 0;  // no slice gains: no transposed copy is maintained
  if (p.n_local > 0)
    k_sell_rows_fill<T><<<g, 256, 0, st>>>(p.row_ptr, rcol, rval, p.n_local,
                                           h->row_slice_off, h->tr_slices ? use_tr : nullptr,
                                           fill_side, (int32_t)p.d, rent);
  h->sell_rows = rent;
  h->sell_row_steps = rsteps;
  if (want_ds) {
    if (cudaStreamSynchronize(st) != cudaSuccess)
      return done(fail(POLY_ECUDA, "SELL build: %s", cudaGetErrorString(cudaGetLastError())));
    int r1 = build_dsell_dir(h, (const CscEnt<float> *)ent, h->slice_off, h->nslices, nullptr, cnt, d, &h->dbwd,
                             &h->dbwd_cap, &h->dbwd_smem);
    int r2 = r1 == POLY_OK ? build_dsell_dir(h, (const CscEnt<float> *)rent, h->row_slice_off, nrs, p.row_ptr,
                                             nullptr, p.n_local, &h->dfwd, &h->dfwd_cap, &h->dfwd_smem)
                           : r1;
    if (r2 == POLY_OK) {
      const void *fns[3] = {(const void *)&k_dsell_forward<false>, (const void *)&k_dsell_forward<true>,
                            (const void *)&k_dsell_backward};
      const size_t sms[3] = {h->dfwd_smem, h->dfwd_smem, h->dbwd_smem};
      for (int i = 0; i < 3; ++i)
        CK(cudaFuncSetAttribute(fns[i], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sms[i]));
      h->dsell = true;
      h->tr_side = 0;  // the forward stages x itself: no transposed copy
      h->tr_slices = 0;
      // persistent grids, two 16-warp blocks per SM; one loss partial per forward block
      h->k4_grid = (int)std::min<int64_t>(nrs, (int64_t)h->sms * 2);
      h->dbwd_grid = (int)std::min<int64_t>(h->nslices, (int64_t)h->sms * 2);
      dev_release(h, rent);
      dev_release(h, ent);
      h->sell_rows = h->sell = nullptr;
      return done(POLY_OK);
    }
    if (r2 != POLY_EUNSUPPORTED) return done(r2);
    g_err[0] = 0;  // fall back to the SELL16 / SELL forms below
  }
  // compact delta form of both copies, when every delta fits int16
  if (!getenv("POLY_NO_SELL16") && p.n_local > 0) {
    int32_t *ovf = nullptr;
    int64_t *len16 = nullptr, *foff = nullptr, *boff = nullptr;
    const int64_t nmax = std::max<int64_t>(nrs, h->nslices) + 1;
    if ((rc = talloc(4, (void **)&ovf)) || (rc = talloc((size_t)nmax * 8, (void **)&len16)))
      return done(rc);
    if ((rc = dev_alloc(h, &foff, (size_t)nrs + 1)) || (rc = dev_alloc(h, &boff, (size_t)h->nslices + 1)))
      return done(rc);
    size_t tb5 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb5, len16, foff, (int)nmax, st);
    void *ts5 = nullptr;
    if ((rc = talloc(tb5, &ts5))) return done(rc);
    int64_t fgroups = 0, bgroups = 0;
    k_groups_of<<<64, 256, 0, st>>>(h->row_slice_off, nrs, len16);
    cub::DeviceScan::ExclusiveSum(ts5, tb5, len16, foff, (int)nrs + 1, st);
    cudaMemcpyAsync(&fgroups, foff + nrs, 8, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return done(fail(POLY_ECUDA, "SELL16 scan"));
    k_groups_of<<<64, 256, 0, st>>>(h->slice_off, h->nslices, len16);
    cub::DeviceScan::ExclusiveSum(ts5, tb5, len16, boff, (int)h->nslices + 1, st);
    cudaMemcpyAsync(&bgroups, boff + h->nslices, 8, cudaMemcpyDeviceToHost, st);
    cudaMemsetAsync(ovf, 0, 4, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return done(fail(POLY_ECUDA, "SELL16 scan"));
    short4 *fdl = nullptr, *bdl = nullptr;
    T *fval = nullptr, *bval = nullptr;
    int32_t *fbase = nullptr, *bbase = nullptr;
    const size_t fe = (size_t)std::max<int64_t>(1, fgroups) * 32, be = (size_t)std::max<int64_t>(1, bgroups) * 32;
    if ((rc = dev_alloc(h, &fdl, fe)) || (rc = dev_alloc(h, &fval, fe * 4)) ||
        (rc = dev_alloc(h, &fbase, (size_t)nrs * 128)) || (rc = dev_alloc(h, &bdl, be)) ||
        (rc = dev_alloc(h, &bval, be * 4)) || (rc = dev_alloc(h, &bbase, (size_t)h->nslices * 128)))
      return done(rc);
    k_sell16_pack<T><<<(int)std::min<int64_t>(65535, nrs), 128, 0, st>>>(
        rent, h->row_slice_off, nrs, p.row_ptr, nullptr, p.n_local, foff, fdl, fval, fbase, ovf);
    k_sell16_pack<T><<<(int)std::min<int64_t>(65535, h->nslices), 128, 0, st>>>(
        ent, h->slice_off, h->nslices, nullptr, h->colmap ? nullptr : cnt, d, boff, bdl, bval, bbase, ovf);
    int32_t hov = 0;
    cudaMemcpyAsync(&hov, ovf, 4, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess)
      return done(fail(POLY_ECUDA, "SELL16 pack: %s", cudaGetErrorString(cudaGetLastError())));
    if (!hov) {
      h->sell16 = true;
      // one block per slice: the block scheduler balances the uneven slices
      // (a grid-stride deal over the resident slots measured 12 % slower)
      h->k4f16_grid = (int)nrs;
      h->k4b16_grid = h->nslices;
      // the loss partials are per forward block
      if (h->k4f16_grid > h->k4_grid) return done(fail(POLY_ECUDA, "SELL16 grid"));
      h->k4_grid = h->k4f16_grid;
      h->fwd16 = Sell16{fdl, fval, fbase, foff};
      h->bwd16 = Sell16{bdl, bval, bbase, boff};
      dev_release(h, rent);  // the 8-byte copies are no longer needed
      dev_release(h, ent);
      h->sell_rows = h->sell = nullptr;
    } else {
      for (void *q : {(void *)fdl, (void *)fval, (void *)fbase, (void *)bdl, (void *)bval,
                      (void *)bbase, (void *)foff, (void *)boff})
        dev_release(h, q);
    }
  }
  return done(POLY_OK);
}

// K4t (tiled.cuh) from the caller's fp32 CSR (poly_init only): the strip
// forward copy and the tile backward copy, both as 8-bit deltas + fp32
// values.  Returns POLY_EUNSUPPORTED (message cleared) when the matrix does
// not fit the format; build_sell then builds the SELL pair.
int build_tiled(poly_handle *h) {
  const poly_problem &p = h->p;
  const int64_t nnz = p.nnz, d = p.d, n = p.n_local;
  if (p.dtype != POLY_F32 || nnz < 1 || n < 1 || nnz >= ((int64_t)1 << 31) || n >= ((int64_t)1 << 31) ||
      getenv("POLY_NO_TILED") || getenv("POLY_DSELL") || getenv("POLY_K4B_SYNC"))
    return POLY_EUNSUPPORTED;
  TiledGeom m{};
  {
    const int64_t s = (int64_t)llround(std::sqrt((double)d));
    if (s * s == d && s > 1) m.rows_img = m.cols_img = (int32_t)s;
    else m.rows_img = 1, m.cols_img = (int32_t)d;
  }
  // strips: the fewest with a strip of <= POLY_STRIP_KB (the rest of the SM holds the ring)
  // and every ascending delta (< P + W) within 8 bits
  // (and the strip plus the forward's ring within one SM's 227 KB)
  const size_t kStripBytes = std::min<size_t>((size_t)POLY_STRIP_KB * 1024,
                                              227 * 1024 - (size_t)kFwdStages * kFwdStageBytes - 512);
  for (m.NS = 1; m.NS <= kMaxStrips; ++m.NS) {
    m.W = (m.cols_img + m.NS - 1) / m.NS;
    m.P = m.rows_img > 1 ? (m.W | 1) : m.W;
    if ((size_t)m.rows_img * m.P * 4 <= kStripBytes && (m.rows_img == 1 || m.P + m.W <= 256)) break;
  }
  if (m.NS > kMaxStrips || (int64_t)m.rows_img * m.P > 65535) return POLY_EUNSUPPORTED;
  m.NS = (m.cols_img + m.W - 1) / m.W;
  if (m.rows_img > 1) {
    // 32 x TH tiles, TH in 4..8 chosen so that the busiest SM (two backward
    // CTAs each) holds the fewest pixel rows: C4 (256 rows) takes TH = 7,
    // 296 tiles = 2 per SM, instead of 256 tiles of 8 rows (two on 108 SMs,
    // one on 40)
    m.TW = 32;
    int64_t best = INT64_MAX;
    for (int th = 8; th >= 4; --th) {
      const int64_t nt = (int64_t)((m.rows_img + th - 1) / th) * ((m.cols_img + 31) / 32);
      const int64_t cost = (nt + 2 * h->sms - 1) / (2 * h->sms) * th;
      if (cost < best) best = cost, m.TH = th;
    }
    if (getenv("POLY_TILE_TH")) m.TH = std::max(1, std::min(8, atoi(getenv("POLY_TILE_TH"))));
  } else {
    m.TW = kTileSlots, m.TH = 1;
  }
  const int32_t npw = m.TW * m.TH / 32;
  m.tiles_x = (m.cols_img + m.TW - 1) / m.TW;
  const int64_t ntiles = (int64_t)((m.rows_img + m.TH - 1) / m.TH) * m.tiles_x;
  if (ntiles >= ((int64_t)1 << 23)) return POLY_EUNSUPPORTED;
  const int64_t nwarps = ntiles * 8;
  cudaStream_t st = h->work;
  // POLY_BUILD_TIMING=1: per-phase build times on stderr (syncs the stream)
  static const bool btime = getenv("POLY_BUILD_TIMING") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto mark = [&](const char *what) {
    if (!btime) return;
    cudaStreamSynchronize(st);
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[tiled build] %-28s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t_last).count());
    t_last = t;
  };
  std::vector<void *> tmp;
  std::vector<void *> mine;  // persistent buffers, released on failure
  // temporaries come from one arena (one cudaMalloc / cudaFree instead of ~25:
  // poly_init is inside the end-to-end measurement), overflow from cudaMalloc
  const int64_t nsn_est = (int64_t)m.NS * n;
  size_t arena_cap = (size_t)nnz * 40 + (size_t)nsn_est * 40 + (size_t)ntiles * kTileSlots * 16 + ((size_t)64 << 20);
  char *arena = nullptr;
  size_t arena_used = 0;
  if (cudaMalloc((void **)&arena, arena_cap) != cudaSuccess) {
    cudaGetLastError();
    arena = nullptr;
    arena_cap = 0;
  } else {
    tmp.push_back(arena);
  }
  auto talloc = [&](size_t bytes, void **ptr) -> int {
    const size_t need = (std::max<size_t>(bytes, 16) + 255) & ~(size_t)255;
    if (arena && arena_used + need <= arena_cap) {
      *ptr = arena + arena_used;
      arena_used += need;
      return POLY_OK;
    }
    if (cudaMalloc(ptr, std::max<size_t>(bytes, 16)) != cudaSuccess) {
      cudaGetLastError();
      return fail(POLY_ENOMEM, "tiled build: cudaMalloc(%zu) failed", bytes);
    }
    tmp.push_back(*ptr);
    return POLY_OK;
  };
  auto palloc = [&](size_t bytes, void **ptr) -> int {
    unsigned char *q = nullptr;
    TRY(dev_alloc(h, &q, bytes));
    mine.push_back(q);
    *ptr = q;
    return POLY_OK;
  };
  auto done = [&](int code) {
    cudaStreamSynchronize(st);
    for (void *q : tmp) cudaFree(q);
    if (code != POLY_OK)
      for (void *q : mine) dev_release(h, q);
    if (code == POLY_EUNSUPPORTED) g_err[0] = 0;
    return code;
  };
  const int g = 148 * 8;
  int rc;
  // ---- forward: sort by (strip, row, local index)
  int32_t *rows = nullptr, *perm_in = nullptr, *perm = nullptr, *seglen = nullptr, *nz = nullptr, *ovf = nullptr;
  uint64_t *kin = nullptr, *ks = nullptr;
  int64_t *segstart = nullptr;
  const int64_t nsn = (int64_t)m.NS * n;
  if ((rc = talloc(nnz * 4, (void **)&rows)) || (rc = talloc(nnz * 4, (void **)&perm_in)) ||
      (rc = talloc(nnz * 4, (void **)&perm)) || (rc = talloc(nnz * 8, (void **)&kin)) ||
      (rc = talloc(nnz * 8, (void **)&ks)) || (rc = talloc(nsn * 4, (void **)&seglen)) ||
      (rc = talloc(nsn * 8, (void **)&segstart)) || (rc = talloc(kMaxStrips * 4, (void **)&nz)) ||
      (rc = talloc(4, (void **)&ovf)))
    return done(rc);
  cudaMemsetAsync(seglen, 0, nsn * 4, st);
  cudaMemsetAsync(nz, 0, kMaxStrips * 4, st);
  cudaMemsetAsync(ovf, 0, 4, st);
  mark("alloc fwd temps (before rows)");
  k_entry_rows<<<g, 256, 0, st>>>(p.row_ptr, n, rows);
  const int sbits = 32 - __builtin_clz((unsigned)std::max(1, m.NS - 1));
  auto nbits = [](int64_t v) { int b = 1; while (b < 62 && ((int64_t)1 << b) <= v) ++b; return b; };  // bits of v >= 0
  m.lb = nbits((int64_t)m.rows_img * m.P - 1);
  m.rb = nbits(n - 1);
  k_tf_keys<<<g, 256, 0, st>>>(rows, p.col, nnz, n, m, kin, perm_in, seglen);
  // 64-bit key radix sorts (temporary storage sized per call)
  auto sort64 = [&](const uint64_t *ki, uint64_t *ko, const int32_t *vi, int32_t *vo, int64_t items, int bits) -> int {
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, ki, ko, vi, vo, (int)items, 0, bits, st);
    void *ts = nullptr;
    TRY(talloc(tb, &ts));
    if (cub::DeviceRadixSort::SortPairs(ts, tb, ki, ko, vi, vo, (int)items, 0, bits, st) != cudaSuccess)
      return fail(POLY_ECUDA, "tiled build: radix sort failed");
    return POLY_OK;
  };
  if ((rc = sort64(kin, ks, perm_in, perm, nnz, sbits + m.rb + m.lb))) return done(rc);
  mark("fwd keys + sort");
  k_tf_segstart<<<g, 256, 0, st>>>(ks, nnz, n, m, segstart);
  // segments of each strip longest first
  uint64_t *okin = nullptr, *oks = nullptr;
  int32_t *orin = nullptr, *srow = nullptr;
  if ((rc = talloc(nsn * 8, (void **)&okin)) || (rc = talloc(nsn * 8, (void **)&oks)) ||
      (rc = talloc(nsn * 4, (void **)&orin)) || (rc = talloc(nsn * 4, (void **)&srow)))
    return done(rc);
  mark("segstart/order alloc");
  k_tf_order_keys<<<g, 256, 0, st>>>(seglen, n, m.NS, okin, orin, nz);
  if ((rc = sort64(okin, oks, orin, srow, nsn, 32 + sbits))) return done(rc);
  std::vector<int32_t> hnz(m.NS);
  cudaMemcpyAsync(hnz.data(), nz, m.NS * 4, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess)
    return done(fail(POLY_ECUDA, "tiled build: %s", cudaGetErrorString(cudaGetLastError())));
  std::vector<int32_t> ustart(m.NS + 1, 0);
  for (int s = 0; s < m.NS; ++s) ustart[s + 1] = ustart[s] + (hnz[s] + kFwdWarps * 32 - 1) / (kFwdWarps * 32);
  const int64_t units = ustart[m.NS];
  int32_t *d_ustart = nullptr, *d_ctr = nullptr;
  int64_t *ulen = nullptr, *uoff = nullptr;
  uint8_t *fhdr = nullptr;
  double *pz = nullptr;
  if ((rc = palloc((m.NS + 1) * 4, (void **)&d_ustart)) || (rc = palloc(m.NS * 4, (void **)&d_ctr)) ||
      (rc = palloc((units + 1) * 8, (void **)&uoff)) || (rc = palloc(std::max<int64_t>(1, units) * kFwdHdr, (void **)&fhdr)) ||
      (rc = palloc(nsn * 8, (void **)&pz)) || (rc = talloc((units + 1) * 8, (void **)&ulen)))
    return done(rc);
  cudaMemcpyAsync(d_ustart, ustart.data(), (m.NS + 1) * 4, cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(d_ctr, 0, m.NS * 4, st);
  cudaMemsetAsync(pz, 0, nsn * 8, st);
  k_tf_unitlen<<<(int)std::min<int64_t>(4096, (units + 256) / 256), 256, 0, st>>>(d_ustart, m.NS, srow, seglen, n,
                                                                                 units, ulen);
  size_t tb3 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb3, ulen, uoff, (int)units + 1, st);
  void *ts3 = nullptr;
  if ((rc = talloc(tb3, &ts3))) return done(rc);
  cub::DeviceScan::ExclusiveSum(ts3, tb3, ulen, uoff, (int)units + 1, st);
  int64_t frows = 0;
  cudaMemcpyAsync(&frows, uoff + units, 8, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess)
    return done(fail(POLY_ECUDA, "tiled build: %s", cudaGetErrorString(cudaGetLastError())));
  uint8_t *frec = nullptr;
  if ((rc = palloc((size_t)std::max<int64_t>(1, frows) * kFwdWarps * kRecBytes, (void **)&frec))) return done(rc);
  k_tf_pack<<<(int)std::min<int64_t>(65535, (units * kFwdWarps + 7) / 8), 256, 0, st>>>(
      d_ustart, m.NS, srow, seglen, nz, segstart, ks, perm, (const float *)p.val, n, units, uoff, m, frec, fhdr, ovf);
  mark("fwd order sort + units + pack");
  // ---- backward: sort by (tile, row, slot), ray lists, then by (tile, slot, list position)
  int32_t *flag = nullptr, *pidx = nullptr, *tcnt = nullptr, *list = nullptr;
  int64_t *tcnt64 = nullptr, *pstart = nullptr, *loff = nullptr;
  if ((rc = talloc(nnz * 4, (void **)&flag)) || (rc = talloc(nnz * 4, (void **)&pidx)) ||
      (rc = talloc(ntiles * 4, (void **)&tcnt)) || (rc = talloc((ntiles + 1) * 8, (void **)&tcnt64)) ||
      (rc = talloc((ntiles + 1) * 8, (void **)&pstart)) || (rc = palloc((ntiles + 1) * 8, (void **)&loff)))
    return done(rc);
  cudaMemsetAsync(tcnt, 0, ntiles * 4, st);
  k_tb_keys<<<g, 256, 0, st>>>(rows, p.col, nnz, m, kin, perm_in);
  const int tbits = 32 - __builtin_clz((unsigned)std::max<int64_t>(1, ntiles - 1));
  if ((rc = sort64(kin, ks, perm_in, perm, nnz, tbits + m.rb + 8))) return done(rc);
  mark("bwd keys + sort");
  k_tb_pairs<<<g, 256, 0, st>>>(ks, nnz, m, flag, tcnt);
  size_t tb4 = 0, tb5 = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tb4, flag, pidx, (int)nnz, st);
  cub::DeviceScan::ExclusiveSum(nullptr, tb5, tcnt64, loff, (int)ntiles + 1, st);
  void *ts4 = nullptr;
  if ((rc = talloc(std::max(tb4, tb5), &ts4))) return done(rc);
  cub::DeviceScan::InclusiveSum(ts4, tb4, flag, pidx, (int)nnz, st);
  // first chunk of every tile: the chunk tables' offsets
  k_widen<<<(int)std::min<int64_t>(4096, (ntiles + 256) / 256), 256, 0, st>>>(tcnt, ntiles, tcnt64);
  cub::DeviceScan::ExclusiveSum(ts4, tb5, tcnt64, pstart, (int)ntiles + 1, st);
  cub::DeviceScan::ExclusiveSum(ts4, tb5, tcnt64, loff, (int)ntiles + 1, st);
  int64_t nlist = 0;
  cudaMemcpyAsync(&nlist, loff + ntiles, 8, cudaMemcpyDeviceToHost, st);
  std::vector<int32_t> htc(ntiles);
  cudaMemcpyAsync(htc.data(), tcnt, ntiles * 4, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess)
    return done(fail(POLY_ECUDA, "tiled build: %s", cudaGetErrorString(cudaGetLastError())));
  int32_t lmax = 0;  // most r chunks of a tile
  for (int32_t v : htc) lmax = std::max(lmax, v);
  lmax *= 4;         // floats
  const int32_t lcap = std::max(4, lmax);
  const size_t bwd_smem = (size_t)kBwdStages * kBwdCG * 2 * npw * kRecBytes + (size_t)lcap * 4 + 2 * kBwdStages * 8;
  const size_t fwd_smem = (((((size_t)m.rows_img * m.P + 3) & ~(size_t)3) * 4 + 127) & ~(size_t)127) +
                          (size_t)kFwdStages * kFwdStageBytes + 2 * kFwdStages * 8 + kFwdStages * 16 + 8;
  if (bwd_smem + 2048 > 227 * 1024 || fwd_smem > 227 * 1024) {
    if (btime) fprintf(stderr, "[tiled build] unsupported: smem fwd %zu bwd %zu\n", fwd_smem, bwd_smem);
    return done(POLY_EUNSUPPORTED);
  }
  if ((rc = palloc((size_t)(nlist + 4) * 4, (void **)&list))) return done(rc);
  cudaMemsetAsync(list, 0, (size_t)(nlist + 4) * 4, st);
  mark("bwd pairs/scans/list alloc");
  m.pb = nbits(std::max(1, lmax) - 1);
  k_tb_list<<<g, 256, 0, st>>>(ks, pidx, flag, pstart, loff, nnz, m, list, kin);
  const int qbits = m.pb + 32 - __builtin_clz((unsigned)std::max<int64_t>(1, ntiles * kTileSlots - 1));
  if ((rc = sort64(kin, ks, perm, perm_in, nnz, qbits))) return done(rc);
  // perm_in now maps the (tile, slot, position) order to the caller's entries
  int32_t *scnt = nullptr, *tcol = nullptr;
  int64_t *sstart = nullptr, *wlen = nullptr, *tlen = nullptr, *toff = nullptr;
  uint16_t *bbase = nullptr;
  const int64_t nslot = ntiles * kTileSlots;
  if ((rc = talloc(nslot * 4, (void **)&scnt)) || (rc = talloc(nslot * 8, (void **)&sstart)) ||
      (rc = talloc(nwarps * 8, (void **)&wlen)) || (rc = talloc((ntiles + 1) * 8, (void **)&tlen)) ||
      (rc = palloc((ntiles + 1) * 8, (void **)&toff)) || (rc = palloc(nslot * 2 * 2, (void **)&bbase)) ||
      (rc = palloc(nslot * 4, (void **)&tcol)))
    return done(rc);
  mark("bwd list + sort2 + allocs");
  cudaMemsetAsync(scnt, 0, nslot * 4, st);
  k_tb_slots<<<g, 256, 0, st>>>(ks, nnz, m, scnt, sstart);
  k_tb_warplen<<<(int)std::min<int64_t>(4096, (nwarps + 255) / 256), 256, 0, st>>>(scnt, nwarps, wlen);
  k_tb_tilelen<<<(int)std::min<int64_t>(4096, (ntiles + 256) / 256), 256, 0, st>>>(wlen, ntiles, tlen);
  size_t tb6 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb6, tlen, toff, (int)ntiles + 1, st);
  void *ts6 = nullptr;
  if ((rc = talloc(tb6, &ts6))) return done(rc);
  cub::DeviceScan::ExclusiveSum(ts6, tb6, tlen, toff, (int)ntiles + 1, st);
  int64_t brows = 0;
  cudaMemcpyAsync(&brows, toff + ntiles, 8, cudaMemcpyDeviceToHost, st);
  std::vector<int64_t> htl(ntiles);
  cudaMemcpyAsync(htl.data(), tlen, ntiles * 8, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess)
    return done(fail(POLY_ECUDA, "tiled build: %s", cudaGetErrorString(cudaGetLastError())));
  int64_t tmax = 0;
  for (int64_t v : htl) tmax = std::max(tmax, v);
  // stage-interleaved tiles ([stage][tile]) unless the tiles' lengths differ by more than 1/8
  const int32_t inter = getenv("POLY_BWD_TILE_MAJOR") ? 0 : (tmax * ntiles <= brows + brows / 8 ? 1 : 0);
  uint8_t *brec = nullptr;
  const size_t bbytes = (size_t)std::max<int64_t>(1, inter ? tmax * ntiles : brows) * 2 * npw * kRecBytes;
  if ((rc = palloc(bbytes, (void **)&brec))) return done(rc);
  cudaMemsetAsync(brec, 0, bbytes, st);  // the shorter halves' padding records
  k_tb_pack<<<(int)std::min<int64_t>(65535, (nwarps + 7) / 8), 256, 0, st>>>(
      ks, perm_in, (const float *)p.val, scnt, sstart, wlen, toff, nwarps, m, (int32_t)d, brec, bbase, tcol, ovf,
      inter, npw);
  mark("bwd slots/scan/pack");
  int32_t hov = 0;
  cudaMemcpyAsync(&hov, ovf, 4, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess)
    return done(fail(POLY_ECUDA, "tiled build: %s", cudaGetErrorString(cudaGetLastError())));
  if (hov) {
    if (btime) fprintf(stderr, "[tiled build] unsupported: a local delta does not fit 8 bits (code %d)\n", hov);
    return done(POLY_EUNSUPPORTED);
  }
  h->tf_smem = fwd_smem;
  h->tb_smem = bwd_smem;
  h->tb_lcap = lcap;
  if (cudaFuncSetAttribute((const void *)&k_strip_forward, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)h->tf_smem) != cudaSuccess ||
      cudaFuncSetAttribute((const void *)&k_tile_backward, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)h->tb_smem) != cudaSuccess) {
    cudaGetLastError();
    return done(POLY_EUNSUPPORTED);
  }
  h->tfwd = StripFwd{frec, fhdr, uoff, d_ustart, d_ctr, pz, n, m.NS, m.rows_img, m.cols_img, m.W, m.P};
  h->tbwd = TileBwd{brec, toff, bbase, list, loff, tcol, (int32_t)ntiles, npw, inter};
  {
    // part of the records kept in L2 across passes (evict-last); the rest streams evict-first
    double keep_f = kTiledKeepFwdMB, keep_b = kTiledKeepBwdMB;
    if (const char *e = getenv("POLY_L2_KEEP_MB")) {
      keep_f = keep_b = 0.0;
      sscanf(e, "%lf,%lf", &keep_f, &keep_b);
    }
    const double fmb = (double)frows * kFwdWarps * kRecBytes / 1e6, bmb = (double)brows * 2 * npw * kRecBytes / 1e6;
    h->tfwd.keep = fmb > 0 ? (int32_t)std::min(1024.0, std::max(0.0, keep_f / fmb * 1024.0)) : 0;
    h->tbwd.keep = bmb > 0 ? (int32_t)std::min(1024.0, std::max(0.0, keep_b / bmb * 1024.0)) : 0;
    h->keep_bytes = (int64_t)((h->tfwd.keep * fmb + h->tbwd.keep * bmb) / 1024.0 * 1e6);
  }
  h->tf_grid = (int)std::max<int64_t>(m.NS, (int64_t)h->sms / m.NS * m.NS);
  h->tb_grid = (int)ntiles;
  h->tf_groups = frows * kFwdWarps;
  h->tb_groups = brows * 2 * npw;
  // the fused step epilogue needs every warp's 32 columns to be one k_finalize block
  h->tile_epi = m.rows_img == 1 || m.cols_img % 32 == 0;
  // link blocks = loss partials (allocated for nrslices >= this grid); one
  // row per thread (two CTAs per SM, each thread looping over rows, measured
  // slower: 127.9 vs 117.9 us per C4 step)
  h->k4_grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)h->sms * 8);
  {
    // the fp32 iterate copies also hold the strips in the forward's layout
    // (one bulk copy per CTA instead of per-element staging); padding zero
    const int64_t SP = ((int64_t)m.rows_img * m.P + 3) & ~(int64_t)3, off = (d + 3) & ~(int64_t)3;
    const size_t n32 = (size_t)(off + (int64_t)m.NS * SP);
    float *b32[3] = {nullptr, nullptr, nullptr};
    for (int q = 0; q < 3; ++q) {
      if ((rc = dev_alloc(h, &b32[q], n32))) {
        for (int u = 0; u < q; ++u) dev_release(h, b32[u]);
        return done(rc);
      }
      cudaMemsetAsync(b32[q], 0, n32 * 4, st);
    }
    dev_release(h, h->xa32);
    dev_release(h, h->xh32);
    dev_release(h, h->xin32);
    h->xa32 = b32[0], h->xh32 = b32[1], h->xin32 = b32[2];
    h->xs = X32Strip{m.W, m.P, m.rows_img, m.cols_img, (int32_t)SP, off};
    h->tfwd.xs_off = off;
    h->tfwd.SP = (int32_t)SP;
  }
  h->tiled = true;
  h->tr_side = 0;  // the forward stages x itself: no transposed copy
  h->tr_slices = 0;
  return done(POLY_OK);
}

int build_sell(poly_handle *h) {
  const int rt = build_tiled(h);
  if (rt != POLY_EUNSUPPORTED) return rt;
  return h->p.dtype == POLY_F32 ? build_sell_t<float>(h) : build_sell_t<double>(h);
}

}  // namespace

namespace {

// ------------------------------------------------------------ K9-NVLS host side
// Driver entry points through the runtime (cudaGetDriverEntryPoint), so the
// library does not link libcuda and still loads on a CPU-only box.
struct DrvApi {
  bool ok = false;
  CUresult (*mcCreate)(CUmemGenericAllocationHandle *, const CUmulticastObjectProp *) = nullptr;
  CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                        unsigned long long) = nullptr;
  CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*mcGranularity)(size_t *, const CUmulticastObjectProp *, CUmulticastGranularity_flags) = nullptr;
  CUresult (*memCreate)(CUmemGenericAllocationHandle *, size_t, const CUmemAllocationProp *,
                        unsigned long long) = nullptr;
  CUresult (*memRelease)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*addrReserve)(CUdeviceptr *, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*addrFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*memUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc *, size_t) = nullptr;
  CUresult (*exportFd)(void *, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long) = nullptr;
  CUresult (*importFd)(CUmemGenericAllocationHandle *, void *, CUmemAllocationHandleType) = nullptr;
  CUresult (*devAttr)(int *, CUdevice_attribute, CUdevice) = nullptr;
};

DrvApi *drv_api() {
  static DrvApi api;
  static bool tried = false;
  if (tried) return api.ok ? &api : nullptr;
  tried = true;
  auto get = [](const char *name, void **fn) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !*fn) {
      cudaGetLastError();
      return false;
    }
    return true;
  };
  api.ok = get("cuMulticastCreate", (void **)&api.mcCreate) && get("cuMulticastAddDevice", (void **)&api.mcAddDevice) &&
           get("cuMulticastBindMem", (void **)&api.mcBindMem) && get("cuMulticastUnbind", (void **)&api.mcUnbind) &&
           get("cuMulticastGetGranularity", (void **)&api.mcGranularity) &&
           get("cuMemCreate", (void **)&api.memCreate) && get("cuMemRelease", (void **)&api.memRelease) &&
           get("cuMemAddressReserve", (void **)&api.addrReserve) && get("cuMemAddressFree", (void **)&api.addrFree) &&
           get("cuMemMap", (void **)&api.memMap) && get("cuMemUnmap", (void **)&api.memUnmap) &&
           get("cuMemSetAccess", (void **)&api.setAccess) &&
           get("cuMemExportToShareableHandle", (void **)&api.exportFd) &&
           get("cuMemImportFromShareableHandle", (void **)&api.importFd) &&
           get("cuDeviceGetAttribute", (void **)&api.devAttr);
  return api.ok ? &api : nullptr;
}

#define DRV(call)                                                                            \
  do {                                                                                       \
    CUresult r_ = (call);                                                                    \
    if (r_ != CUDA_SUCCESS) return fail(POLY_ECUDA, "%s failed: CUresult %d (%s:%d)", #call, \
                                        (int)r_, __FILE__, __LINE__);                        \
  } while (0)

// The 64-byte descriptor rank 0 hands to every rank (poly_nvls_handle ->
// caller's broadcast -> poly_nvls_open).
struct NvlsDesc {
  uint32_t magic;   // 'NVLS'
  int32_t world;
  uint64_t size;    // window bytes (multiple of the multicast granularity)
  char name[48];    // abstract unix socket on which rank 0 serves the multicast fd
};
static_assert(sizeof(NvlsDesc) == 64, "descriptor is 64 bytes");
constexpr uint32_t kNvlsMagic = 0x534c564eu;

sockaddr_un abstract_addr(const char *name, socklen_t *len) {
  sockaddr_un a{};
  a.sun_family = AF_UNIX;
  a.sun_path[0] = '\0';  // abstract namespace: nothing on the file system
  const size_t n = strnlen(name, sizeof(a.sun_path) - 2);
  memcpy(a.sun_path + 1, name, n);
  *len = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + n);
  return a;
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

extern "C" {
// File-descriptor exchange of poly_nvls_open (declared in poly.h): rank 0
// listens on the abstract unix socket `name` and sends fd_in to world-1
// connecting ranks with SCM_RIGHTS; the other ranks connect (retrying until
// timeout_s) and receive a duplicate in *fd_out.  Rank 0's *fd_out = fd_in.
int poly_share_fd(int32_t rank, int32_t world, const char *name, int fd_in, int *fd_out, double timeout_s) {
  if (!name || !fd_out || world < 1 || rank < 0 || rank >= world) return fail(POLY_EINVAL, "bad arguments");
  *fd_out = -1;
  socklen_t len = 0;
  const sockaddr_un addr = abstract_addr(name, &len);
  const double t_end = now_s() + timeout_s;
  if (rank == 0) {
    *fd_out = fd_in;
    if (world == 1) return POLY_OK;
    const int ls = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    if (ls < 0) return fail(POLY_ECUDA, "fd exchange: socket() failed");
    if (bind(ls, (const sockaddr *)&addr, len) != 0 || listen(ls, world) != 0) {
      close(ls);
      return fail(POLY_ECUDA, "fd exchange: cannot listen on @%s", name);
    }
    int served = 0;
    while (served < world - 1) {
      pollfd pf{ls, POLLIN, 0};
      const int left_ms = (int)std::max(0.0, (t_end - now_s()) * 1e3);
      if (left_ms == 0 || poll(&pf, 1, std::min(left_ms, 1000)) < 0) break;
      if (!(pf.revents & POLLIN)) continue;
      const int c = accept(ls, nullptr, nullptr);
      if (c < 0) continue;
      char byte = 'F';
      iovec io{&byte, 1};
      char ctrl[CMSG_SPACE(sizeof(int))] = {};
      msghdr m{};
      m.msg_iov = &io;
      m.msg_iovlen = 1;
      m.msg_control = ctrl;
      m.msg_controllen = sizeof(ctrl);
      cmsghdr *cm = CMSG_FIRSTHDR(&m);
      cm->cmsg_level = SOL_SOCKET;
      cm->cmsg_type = SCM_RIGHTS;
      cm->cmsg_len = CMSG_LEN(sizeof(int));
      memcpy(CMSG_DATA(cm), &fd_in, sizeof(int));
      if (sendmsg(c, &m, 0) == 1) ++served;
      close(c);
    }
    close(ls);
    if (served < world - 1) return fail(POLY_ENCCL, "fd exchange: %d of %d ranks connected within %.0f s", served,
                                        world - 1, timeout_s);
    return POLY_OK;
  }
  for (;;) {
    const int c = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    if (c < 0) return fail(POLY_ECUDA, "fd exchange: socket() failed");
    if (connect(c, (const sockaddr *)&addr, len) == 0) {
      char byte = 0;
      iovec io{&byte, 1};
      char ctrl[CMSG_SPACE(sizeof(int))] = {};
      msghdr m{};
      m.msg_iov = &io;
      m.msg_iovlen = 1;
      m.msg_control = ctrl;
      m.msg_controllen = sizeof(ctrl);
      const ssize_t r = recvmsg(c, &m, 0);
      cmsghdr *cm = CMSG_FIRSTHDR(&m);
      close(c);
      if (r == 1 && cm && cm->cmsg_type == SCM_RIGHTS) {
        memcpy(fd_out, CMSG_DATA(cm), sizeof(int));
        return POLY_OK;
      }
      return fail(POLY_ENCCL, "fd exchange: no descriptor received from rank 0");
    }
    close(c);
    if (now_s() > t_end) return fail(POLY_ENCCL, "fd exchange: rank 0 not reachable on @%s", name);
    std::this_thread::sleep_for(std::chrono::milliseconds(2));
  }
}
}  // extern "C"

namespace {

void nvls_release(poly_handle *h) {
  DrvApi *api = drv_api();
  auto &v = h->nv;
  if (api) {
    if (v.mc_mapped) api->memUnmap(v.mc_va, v.size);
    if (v.uc_mapped) api->memUnmap(v.uc_va, v.size);
    if (v.mc_va) api->addrFree(v.mc_va, v.size);
    if (v.uc_va) api->addrFree(v.uc_va, v.size);
    if (v.bound) api->mcUnbind(v.mc, h->dev, 0, v.size);
    if (v.have_mem) api->memRelease(v.mem);
    if (v.have_mc) api->memRelease(v.mc);
  }
  if (v.fd >= 0) close(v.fd);
  if (v.listen_fd >= 0) close(v.listen_fd);
  v = decltype(h->nv){};
}

// every rank's host: a barrier through the handle's communicator (one
// allreduce of one double, drained) — all devices are added to the multicast
// object before any binds, all bound before any kernel uses it
int comm_barrier(poly_handle *h) {
  if (!h->comm_path || h->p.world == 1) return POLY_OK;
  NcclApi *api = nccl_api();
  if (!h->nccl) return fail(POLY_ENCCL, "no communicator");
  const ncclResult_t r = api->allReduce(h->comm, h->comm, 1, ncclFloat64, ncclSum, h->nccl, h->work);
  if (r != ncclSuccess) return fail(POLY_ENCCL, "barrier: %s", api->errStr(r));
  return sync_work(h);
}

// K9-NVLS: the cross-rank sum of one F evaluation (csrc/nvls.cuh)
int enqueue_nvls_reduce(poly_handle *h) {
  ProfScope ps(h, 2);
  NvlsArgs a{};
  a.comm = h->comm;
  a.n = h->p.d + 1;
  a.world = (int32_t)h->p.world;
  a.rank = (int32_t)h->p.rank;
  a.uc = (char *)h->nv.uc_va;
  a.mc = (char *)h->nv.mc_va;
  a.epoch = h->nv.epoch;
  a.err = &h->state->comm_err;
  a.timeout_ns = (unsigned long long)(h->comm_timeout_s * 1e9);
  const int grid = (int)std::min<int64_t>(std::min(h->sms, kNvlsMaxBlocks), (a.n + 255) / 256);
  return launch(h, (const void *)&k_nvls_reduce, dim3(grid), dim3(256), 0, true, a);
}

}  // namespace

namespace {

constexpr int kPollEvery = 4;          // poll the device state every 4 replays (32 iterations)

// Enqueue a copy of the solver state to pinned host memory behind
// ev_poll[k & 1] and check the copy made at the previous poll (one poll
// behind, so the device always has work queued): a non-finite iterate
// is then seen within ~2 polls instead of after all T
// iterations, and with a communicator NCCL's async error state is checked.
int poll_state(poly_handle *h, int k) {
  if (k >= 1) TRY(wait_event(h, h->ev_poll[(k - 1) & 1]));
  TRY(check_comm(h));
  if (h->hstate->bad != 0 || h->hstate->comm_err != 0) return POLY_OK;
  CK(cudaMemcpyAsync(h->hstate, h->state, sizeof(SolveState), cudaMemcpyDeviceToHost, h->work));
  CK(cudaEventRecord(h->ev_poll[k & 1], h->work));
  return POLY_OK;
}

// Replay the U-iteration graph (and the 1-iteration graph for the tail) for
// T iterations, polling every kPollEvery replays; a non-finite iterate or a
// K9 wait timeout stops further launches.
int replay_solve(poly_handle *h, cudaGraphExec_t gU, cudaGraphExec_t g1, int T) {
  const int U = h->graph_U;
  int done = 0, replays = 0, polls = 0;
  while (done < T) {
    const int step = (T - done >= U) ? U : 1;
    CK(cudaGraphLaunch(step == U ? gU : g1, h->work));
    done += step;
    if (++replays % kPollEvery == 0 && done < T) {
      TRY(poll_state(h, polls++));
      if (h->hstate->bad != 0 || h->hstate->comm_err != 0) break;
    }
  }
  return POLY_OK;
}

void collect_profile(poly_handle *h) {
  double sum[3] = {0, 0, 0};
  int cnt[3] = {0, 0, 0};
  const bool dbg = getenv("POLY_PROF_DEBUG") != nullptr;
  for (auto &r : h->recs) {
    float ms = 0.f;
    const cudaError_t e = cudaEventElapsedTime(&ms, r.a, r.b);
    if (dbg) fprintf(stderr, "prof rec kind %d: %s %.4f ms\n", r.kind, cudaGetErrorString(e), ms);
    if (e != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    sum[r.kind] += ms;
    cnt[r.kind]++;
  }
  for (int k = 0; k < 3; ++k) h->ktimes[k] = cnt[k] ? sum[k] / cnt[k] : 0.0;
  h->ktimes[3] = cnt[0];
  h->ktimes[4] = cnt[0] + cnt[1];
  h->prof = false;
}

}  // namespace

extern "C" {


int poly_abi_version(void) { return POLY_ABI_VERSION; }
const char *poly_last_error(void) { return g_err; }

int poly_nccl_unique_id(void *out128) {
  if (!out128) return fail(POLY_EINVAL, "out is NULL");
  NcclApi *api = nccl_api();
  if (!api) return fail(POLY_ENCCL, "cannot load libnccl.so.2");
  ncclUniqueId id;
  ncclResult_t r = api->getUniqueId(&id);
  if (r != ncclSuccess) return fail(POLY_ENCCL, "ncclGetUniqueId: %s", api->errStr(r));
  memcpy(out128, &id, sizeof(id));
  return POLY_OK;
}

int poly_p2p_handle(poly_handle *h, void *out64) {
  if (!h || !out64) return fail(POLY_EINVAL, "NULL handle or out");
  if (!h->p2p_win) return fail(POLY_EINVAL, "handle was not created with POLY_FLAG_P2P");
  cudaIpcMemHandle_t m;
  CK(cudaIpcGetMemHandle(&m, h->p2p_win));
  static_assert(sizeof(m) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(out64, &m, 64);
  return POLY_OK;
}

int poly_p2p_open(poly_handle *h, const void *handles) {
  if (!h || !handles) return fail(POLY_EINVAL, "NULL handle or handles");
  if (!h->p2p_win) return fail(POLY_EINVAL, "handle was not created with POLY_FLAG_P2P");
  if (h->p2p) return fail(POLY_EINVAL, "poly_p2p_open called twice");
  const int P = (int)h->p.world;
  for (int r = 0; r < P; ++r) {
    if (r == h->p.rank) {
      h->p2p_peer[r] = h->p2p_win;
      continue;
    }
    cudaIpcMemHandle_t m;
    memcpy(&m, (const char *)handles + 64 * r, 64);
    void *ptr = nullptr;
    if (cudaIpcOpenMemHandle(&ptr, m, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      for (int q = 0; q < r; ++q)
        if (q != h->p.rank && h->p2p_peer[q]) cudaIpcCloseMemHandle(h->p2p_peer[q]);
      for (auto &q : h->p2p_peer) q = nullptr;
      return fail(POLY_ECUDA, "cudaIpcOpenMemHandle(rank %d) failed: no peer access to that GPU", r);
    }
    h->p2p_peer[r] = (char *)ptr;
  }
  // graphs captured so far hold the NCCL path
  for (auto &a : h->gexec)
    for (auto &g : a)
      if (g) cudaGraphExecDestroy(g), g = nullptr;
  for (auto &a : h->gexec_ex)
    for (auto &b : a)
      for (auto &g : b)
        if (g) cudaGraphExecDestroy(g), g = nullptr;
  h->p2p = true;
  return POLY_OK;
}

int poly_nvls_handle(poly_handle *h, void *out64) {
  if (!h || !out64) return fail(POLY_EINVAL, "NULL handle or out");
  if (!(h->p.flags & POLY_FLAG_NVLS)) return fail(POLY_EINVAL, "handle was not created with POLY_FLAG_NVLS");
  if (h->nv.have_mc) return fail(POLY_EINVAL, "poly_nvls_handle called twice");
  NvlsDesc dsc{};
  dsc.magic = kNvlsMagic;
  dsc.world = (int32_t)h->p.world;
  if (h->p.rank == 0) {
    DrvApi *api = drv_api();
    if (!api) return fail(POLY_EUNSUPPORTED, "NVLS: driver multicast entry points unavailable");
    int mcs = 0;
    if (api->devAttr(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, h->dev) != CUDA_SUCCESS || !mcs)
      return fail(POLY_EUNSUPPORTED, "NVLS: the device does not support multicast objects");
    CUmulticastObjectProp mp{};
    mp.numDevices = (unsigned)h->p.world;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = kNvlsHdr + (size_t)4 * (h->p.d + 1) * 8;
    size_t gran = 0;
    DRV(api->mcGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    mp.size = (mp.size + gran - 1) / gran * gran;
    DRV(api->mcCreate(&h->nv.mc, &mp));
    h->nv.have_mc = true;
    h->nv.size = mp.size;
    int fd = -1;
    DRV(api->exportFd(&fd, h->nv.mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
    h->nv.fd = fd;
    dsc.size = mp.size;
    static int counter = 0;
    snprintf(dsc.name, sizeof(dsc.name), "poly-nvls-%d-%d", (int)getpid(), ++counter);
  }
  memcpy(out64, &dsc, 64);
  return POLY_OK;
}

int poly_nvls_open(poly_handle *h, const void *desc64) {
  if (!h || !desc64) return fail(POLY_EINVAL, "NULL handle or descriptor");
  if (!(h->p.flags & POLY_FLAG_NVLS)) return fail(POLY_EINVAL, "handle was not created with POLY_FLAG_NVLS");
  if (h->nv.on) return fail(POLY_EINVAL, "poly_nvls_open called twice");
  NvlsDesc dsc;
  memcpy(&dsc, desc64, 64);
  if (dsc.magic != kNvlsMagic || dsc.world != h->p.world || dsc.size == 0)
    return fail(POLY_EINVAL, "NVLS: not a descriptor of this communicator (poly_nvls_handle on rank 0)");
  if (h->p.rank == 0 && !h->nv.have_mc) return fail(POLY_EINVAL, "NVLS: rank 0 must call poly_nvls_handle first");
  DrvApi *api = drv_api();
  if (!api) return fail(POLY_EUNSUPPORTED, "NVLS: driver multicast entry points unavailable");
  auto bail = [&](int rc) {
    nvls_release(h);
    return rc;
  };
  int rc = POLY_OK;
  // 1. every rank obtains the multicast object (rank 0 serves its fd)
  int fd = -1;
  if ((rc = poly_share_fd((int32_t)h->p.rank, (int32_t)h->p.world, dsc.name, h->nv.fd, &fd,
                          std::min(h->comm_timeout_s, 120.0))) != POLY_OK)
    return bail(rc);
  if (h->p.rank != 0) {
    h->nv.fd = fd;
    h->nv.size = dsc.size;
    CUresult r = api->importFd(&h->nv.mc, (void *)(intptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    if (r != CUDA_SUCCESS) return bail(fail(POLY_ECUDA, "NVLS: import of the multicast object failed (%d)", (int)r));
    h->nv.have_mc = true;
  }
  CUresult r = api->mcAddDevice(h->nv.mc, h->dev);
  if (r != CUDA_SUCCESS) return bail(fail(POLY_ECUDA, "NVLS: cuMulticastAddDevice failed (%d)", (int)r));
  if ((rc = comm_barrier(h)) != POLY_OK) return bail(rc);
  // 2. this rank's physical copy, bound to the object; unicast and multicast views
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = h->dev;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  const size_t sz = h->nv.size;
  if ((r = api->memCreate(&h->nv.mem, sz, &ap, 0)) != CUDA_SUCCESS)
    return bail(fail(POLY_ENOMEM, "NVLS: cuMemCreate(%zu) failed (%d)", sz, (int)r));
  h->nv.have_mem = true;
  if ((r = api->mcBindMem(h->nv.mc, 0, h->nv.mem, 0, sz, 0)) != CUDA_SUCCESS)
    return bail(fail(POLY_ECUDA, "NVLS: cuMulticastBindMem failed (%d)", (int)r));
  h->nv.bound = true;
  CUmemAccessDesc ad{};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = h->dev;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if ((r = api->addrReserve(&h->nv.uc_va, sz, sz, 0, 0)) != CUDA_SUCCESS ||
      (r = api->memMap(h->nv.uc_va, sz, 0, h->nv.mem, 0)) != CUDA_SUCCESS)
    return bail(fail(POLY_ECUDA, "NVLS: unicast mapping failed (%d)", (int)r));
  h->nv.uc_mapped = true;
  if ((r = api->setAccess(h->nv.uc_va, sz, &ad, 1)) != CUDA_SUCCESS ||
      (r = api->addrReserve(&h->nv.mc_va, sz, sz, 0, 0)) != CUDA_SUCCESS ||
      (r = api->memMap(h->nv.mc_va, sz, 0, h->nv.mc, 0)) != CUDA_SUCCESS)
    return bail(fail(POLY_ECUDA, "NVLS: multicast mapping failed (%d)", (int)r));
  h->nv.mc_mapped = true;
  if ((r = api->setAccess(h->nv.mc_va, sz, &ad, 1)) != CUDA_SUCCESS)
    return bail(fail(POLY_ECUDA, "NVLS: multicast access failed (%d)", (int)r));
  if (!h->nv.epoch && (rc = dev_alloc(h, &h->nv.epoch, (size_t)kNvlsMaxBlocks)) != POLY_OK) return bail(rc);
  if (cudaMemsetAsync((void *)h->nv.uc_va, 0, sz, h->work) != cudaSuccess ||
      cudaMemsetAsync(h->nv.epoch, 0, 8 * (size_t)kNvlsMaxBlocks, h->work) != cudaSuccess)
    return bail(fail(POLY_ECUDA, "NVLS: window reset failed"));
  if ((rc = sync_work(h)) != POLY_OK || (rc = comm_barrier(h)) != POLY_OK) return bail(rc);
  // graphs captured so far hold the NCCL path
  for (auto &a : h->gexec)
    for (auto &g : a)
      if (g) cudaGraphExecDestroy(g), g = nullptr;
  for (auto &a : h->gexec_ex)
    for (auto &b : a)
      for (auto &g : b)
        if (g) cudaGraphExecDestroy(g), g = nullptr;
  h->nv.on = true;
  return POLY_OK;
}

void poly_free(poly_handle *h) {
  if (!h) return;
  // drain first: a K9 launch may still be reading the peers' windows (the
  // caller must also barrier across ranks before freeing, poly.h)
  if (h->work) cudaStreamSynchronize(h->work);
  if (h->p2p)
    for (int r = 0; r < (int)h->p.world; ++r)
      if (r != h->p.rank && h->p2p_peer[r]) cudaIpcCloseMemHandle(h->p2p_peer[r]);
  nvls_release(h);
  for (auto &a : h->gexec)
    for (auto &g : a)
      if (g) cudaGraphExecDestroy(g);
  for (auto &a : h->gexec_ex)
    for (auto &b : a)
      for (auto &g : b)
        if (g) cudaGraphExecDestroy(g);
  if (h->nccl) {
    NcclApi *api = nccl_api();
    if (api) api->commDestroy(h->nccl);
  }
  for (void *p : h->owned) cudaFree(p);
  if (h->hstate) cudaFreeHost(h->hstate);
  for (cudaEvent_t e : h->evpool) cudaEventDestroy(e);
  if (h->ev_in) cudaEventDestroy(h->ev_in);
  if (h->ev_out) cudaEventDestroy(h->ev_out);
  for (cudaEvent_t e : {h->ev_poll[0], h->ev_poll[1], h->ev_sync})
    if (e) cudaEventDestroy(e);
  if (h->work) cudaStreamDestroy(h->work);
  delete h;
}

int poly_init(const poly_problem *pin, poly_handle **out) {
  if (!out) return fail(POLY_EINVAL, "out is NULL");
  *out = nullptr;
  TRY(validate(pin));
  poly_handle *h = new poly_handle();
  h->p = *pin;
  poly_problem &p = h->p;
  int rc = POLY_OK;
  auto bail = [&](int code) {
    poly_free(h);
    return code;
  };
  if (cudaGetDevice(&h->dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, h->dev) != cudaSuccess) {
    cudaGetLastError();
    delete h;
    return fail(POLY_ECUDA, "no CUDA device available");
  }
  h->elsize = p.dtype == POLY_F32 ? 4 : 8;
  h->Om = p.windows > 1 ? p.windows : 1;
  h->n_norm = (int64_t)h->Om * p.n_global;
  h->ysz = p.ytype == POLY_Y_F64 ? 8 : 4;
  h->user = (cudaStream_t)p.stream;
  h->pdl = !(p.flags & POLY_FLAG_NO_PDL);
  h->use_graph = !(p.flags & POLY_FLAG_NO_GRAPH);
  if (cudaStreamCreateWithFlags(&h->work, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_out, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_poll[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_poll[1], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_sync, cudaEventDisableTiming) != cudaSuccess)
    return bail(fail(POLY_ECUDA, "stream/event creation failed"));
  h->no_epi = getenv("POLY_NO_EPI") != nullptr;
  if (const char *t = getenv("POLY_COMM_TIMEOUT_S")) {
    const double v = atof(t);
    if (v > 0.0) h->comm_timeout_s = v;
  }
  if ((rc = sync_in(h)) != POLY_OK) return bail(rc);

  // host inputs -> library-owned device copies
  if (p.flags & POLY_FLAG_HOST_INPUTS) {
    const size_t n = (size_t)p.n_local;
    if (p.layout == POLY_DENSE) {
      if ((rc = copy_in(h, &p.A, n * p.lda * h->elsize)) != POLY_OK) return bail(rc);
    } else {
      const void *rp = p.row_ptr, *cl = p.col;
      if ((rc = copy_in(h, &rp, (n + 1) * 8)) != POLY_OK) return bail(rc);
      if ((rc = copy_in(h, &cl, (size_t)p.nnz * 4)) != POLY_OK) return bail(rc);
      if ((rc = copy_in(h, &p.val, (size_t)p.nnz * h->elsize)) != POLY_OK) return bail(rc);
      p.row_ptr = (const int64_t *)rp;
      p.col = (const int32_t *)cl;
    }
    if ((rc = copy_in(h, &p.y, n * h->ysz * (size_t)h->Om)) != POLY_OK) return bail(rc);
    const void *sr = p.s_row, *ir = p.I_row;
    if ((rc = copy_in(h, &sr, n * p.W * 4)) != POLY_OK) return bail(rc);
    if ((rc = copy_in(h, &ir, n * 4)) != POLY_OK) return bail(rc);
    p.s_row = (const float *)sr;
    p.I_row = (const float *)ir;
  }

  // spectrum [s | mu | 1/mu] and centre
  // Ω windows share a_i and μ_j, so Σ_ω [y_ωi - Ī_ω h_ω(z)] = y_i^Σ - Ī_Σ h̃(z) with
  // Ī_Σ = Σ_ω Ī_ω, s̃_j = Σ_ω Ī_ω s_ωj / Ī_Σ, y^Σ = Σ_ω y_ω: one link of W bins
  // per row; the loss is linear in y too.
  std::vector<double> s_eff(p.W, 0.0);
  if (h->Om == 1) {
    for (int j = 0; j < p.W; ++j) s_eff[j] = p.s[j];
  } else {
    double It = 0.0;
    for (int w = 0; w < h->Om; ++w) It += p.I_win[w];
    for (int j = 0; j < p.W; ++j) {
      double c = 0.0;
      for (int w = 0; w < h->Om; ++w) c += p.I_win[w] * p.s[(size_t)w * p.W + j];
      s_eff[j] = c / It;
    }
    p.I_bar = It;
  }
  std::vector<double> spec(3 * kMaxW, 0.0);
  for (int j = 0; j < p.W; ++j) {
    spec[j] = s_eff[j];
    spec[kMaxW + j] = p.mu[j];
    spec[2 * kMaxW + j] = 1.0 / p.mu[j];
  }
  // μ an arithmetic progression (e.g. linspace): the CSR link walks the bins
  // geometrically (tiled.cuh row_residual_serial); tolerance 8 ulp of max μ
  if (p.W >= 3 && !getenv("POLY_NO_GEO_MU")) {
    const double st = (p.mu[p.W - 1] - p.mu[0]) / (double)(p.W - 1);
    double mx = 0.0, dev = 0.0;
    for (int j = 0; j < p.W; ++j) mx = std::max(mx, std::fabs(p.mu[j]));
    for (int j = 0; j < p.W; ++j) dev = std::max(dev, std::fabs(p.mu[0] + j * st - p.mu[j]));
    bool pos = true;
    for (int j = 0; j < p.W; ++j) pos = pos && p.mu[j] > 0.0;
    if (st != 0.0 && pos && dev <= 8.0 * 2.220446049250313e-16 * mx) h->mu_step = st;
  }
  if ((rc = dev_alloc(h, &h->spec, 3 * kMaxW)) != POLY_OK) return bail(rc);
  if (cudaMemcpy(h->spec, spec.data(), spec.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess)
    return bail(fail(POLY_ECUDA, "spectrum upload failed"));
  if (p.center) {
    if ((rc = dev_alloc(h, &h->center, p.d)) != POLY_OK) return bail(rc);
    if (cudaMemcpy(h->center, p.center, p.d * 8, cudaMemcpyHostToDevice) != cudaSuccess)
      return bail(fail(POLY_ECUDA, "centre upload failed"));
  }
  p.s = p.mu = p.center = p.I_win = nullptr;  // host copies are not kept

  // tile configuration and workspaces
  if (p.layout == POLY_DENSE) {
    if ((rc = setup_dense(h)) != POLY_OK) return bail(rc);
    if ((rc = dev_alloc(h, &h->partials, (size_t)h->G * p.d)) != POLY_OK) return bail(rc);
    if ((rc = dev_alloc(h, &h->loss_partials, (size_t)h->G)) != POLY_OK) return bail(rc);
  } else {
    h->G = 1;
    h->nrslices = (int)std::max<int64_t>(1, (p.n_local + 31) / 32);
    h->k4_grid = h->nrslices;
    if ((rc = dev_alloc(h, &h->partials, (size_t)p.d)) != POLY_OK) return bail(rc);
    if (p.layout == POLY_PARALLEL_BEAM) {  // geometry table, per-view loss partials, view halves
      h->pb.N = p.pb_side;
      h->pb.V = p.pb_views;
      h->pb.B = p.pb_bins;
      h->pb.v0 = (int32_t)(p.row_offset / p.pb_bins);
      h->pb.nv = (int32_t)(p.n_local / p.pb_bins);
      if (h->pb.nv < 1) return bail(fail(POLY_EINVAL, "parallel beam: no views"));
      std::vector<double> trig((size_t)2 * p.pb_views);
      for (int k = 0; k < p.pb_views; ++k) {
        const double th = 3.14159265358979323846 * (double)k / (double)p.pb_views;
        double cs = std::cos(th), sn = std::sin(th);
        // axis-aligned views exactly (cos(π/2) is 6e-17 in fp64): edge rays then sit
        // exactly on pixel edges in both passes and take the same tie rule
        if (std::fabs(cs) < 1e-12) cs = 0.0, sn = sn > 0 ? 1.0 : -1.0;
        if (std::fabs(sn) < 1e-12) sn = 0.0, cs = cs > 0 ? 1.0 : -1.0;
        trig[2 * k] = cs;
        trig[2 * k + 1] = sn;
      }
      if ((rc = dev_alloc(h, &h->pb_trig, trig.size())) != POLY_OK) return bail(rc);
      if (cudaMemcpy(h->pb_trig, trig.data(), trig.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess)
        return bail(fail(POLY_ECUDA, "geometry upload failed"));
      h->pb.trig = h->pb_trig;
      if ((rc = dev_alloc(h, &h->pb_out2, (size_t)kPbParts * p.d)) != POLY_OK) return bail(rc);
      if ((rc = dev_alloc(h, &h->pb_zpart, (size_t)kPbRowSplit * p.n_local)) != POLY_OK) return bail(rc);
      if ((rc = dev_alloc(h, &h->pb_ticket, (size_t)h->pb.nv)) != POLY_OK) return bail(rc);
      if (cudaMemset(h->pb_ticket, 0, sizeof(int32_t) * (size_t)h->pb.nv) != cudaSuccess)
        return bail(fail(POLY_ECUDA, "parallel beam: ticket reset"));
      {
        const int tc = (p.pb_side + kPbTile - 1) / kPbTile;
        if ((rc = dev_alloc(h, &h->pb_tticket, (size_t)tc * tc)) != POLY_OK) return bail(rc);
        if (cudaMemset(h->pb_tticket, 0, sizeof(int32_t) * (size_t)tc * tc) != cudaSuccess)
          return bail(fail(POLY_ECUDA, "parallel beam: ticket reset"));
        h->pb.tticket = h->pb_tticket;
      }
      h->pb.zpart = h->pb_zpart;
      h->pb.ticket = h->pb_ticket;
      h->k4_grid = h->pb.nv;
      for (int f = 0; f < 2; ++f) {
        const void *fn = f ? (const void *)&k_pb_forward<true> : (const void *)&k_pb_forward<false>;
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kPbBufs * kPbRows * (p.pb_side + 2 * kPbPad) * 4) != cudaSuccess)
          return bail(fail(POLY_EUNSUPPORTED, "parallel beam: image too wide for the row stage"));
      }
    }
    if ((rc = dev_alloc(h, &h->loss_partials, (size_t)h->k4_grid)) != POLY_OK) return bail(rc);
    // r padded to whole float4s: K4tb copies aligned 4-row chunks of it
    if ((rc = dev_alloc(h, &h->rbuf, (size_t)((std::max<int64_t>(1, p.n_local) + 3) & ~(int64_t)3))) != POLY_OK)
      return bail(rc);
    {  // a square d may be an image: the fp32 copies get room for x transposed
      const int64_t s = (int64_t)llround(std::sqrt((double)p.d));
      if (s * s == p.d && s > 1) h->tr_side = (int)s;
    }
    const size_t n32 = (size_t)p.d * (h->tr_side ? 2 : 1);
    if ((rc = dev_alloc(h, &h->xa32, n32)) != POLY_OK) return bail(rc);
    if ((rc = dev_alloc(h, &h->xh32, n32)) != POLY_OK) return bail(rc);
    if ((rc = dev_alloc(h, &h->xin32, n32)) != POLY_OK) return bail(rc);
    if (cudaMemsetAsync(h->rbuf, 0, ((std::max<int64_t>(1, p.n_local) + 3) & ~(int64_t)3) * 4, h->work) != cudaSuccess)
      return bail(fail(POLY_ECUDA, "memset failed"));
  }
  h->fin_grid = (int)((p.d + 31) / 32);
  h->fin_split = (p.d > kSplitFinD || p.set == POLY_SET_TV_NONNEG || p.set == POLY_SET_TV) ? 1 : 0;
  if (p.set == POLY_SET_TV_NONNEG || p.set == POLY_SET_TV) {
    const int s = (int)llround(std::sqrt((double)p.d));
    h->tv_cl = std::min(kTvMaxCL, s);
    const int cap = ((s + h->tv_cl - 1) / h->tv_cl) * ((s + 31) & ~31);  // band rows x padded pitch
    h->tv_smem = ((size_t)5 * cap + tv_edge_doubles(s) + 8 + 4 + (kTvThreads / 32) * 4) * 8 + tv_xchg_bytes(s);
    if (s > 256 || h->tv_smem > kSmemLimit)
      return bail(fail(POLY_EUNSUPPORTED, "TV image side %d too large for one cluster", s));
    if (cudaFuncSetAttribute((const void *)&k_tv_project, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)h->tv_smem) != cudaSuccess ||
        cudaFuncSetAttribute((const void *)&k_tv_project, cudaFuncAttributeNonPortableClusterSizeAllowed,
                             1) != cudaSuccess)
      return bail(fail(POLY_ECUDA, "TV kernel attributes: %s", cudaGetErrorString(cudaGetLastError())));
    {  // λ values per round (clusters): the caller's tv_k, if that many can be resident
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(h->tv_cl);
      cfg.blockDim = dim3(kTvThreads);
      cfg.dynamicSmemBytes = h->tv_smem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = h->tv_cl;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int maxc = 0;
      if (cudaOccupancyMaxActiveClusters(&maxc, (const void *)&k_tv_project, &cfg) != cudaSuccess || maxc < 1) {
        cudaGetLastError();
        return bail(fail(POLY_EUNSUPPORTED, "TV: a %d-CTA cluster cannot be resident", h->tv_cl));
      }
      const int want = p.tv_k > 1 ? p.tv_k : 1;  // default: the paper's bisection (R22 measured slower)
      if (want > maxc || want > kTvMaxK)
        return bail(fail(POLY_EUNSUPPORTED, "TV: tv_k = %d clusters requested, %d can be resident", want,
                         std::min(maxc, kTvMaxK)));
      h->tv_k = want;
    }
    const size_t kd = (size_t)h->tv_k * p.d;
    if ((rc = dev_alloc(h, &h->tv_zk, kd)) || (rc = dev_alloc(h, &h->tv_p, kd)) || (rc = dev_alloc(h, &h->tv_q, kd)) ||
        (rc = dev_alloc(h, &h->tv_stats, 4)) || (rc = dev_alloc(h, &h->tv_vals, (size_t)2 * h->tv_k)) ||
        (rc = dev_alloc(h, &h->tv_gbar, 1)) || (rc = dev_alloc(h, &h->tv_xsel, (size_t)p.d)) ||
        (!p.tv_cold && (rc = dev_alloc(h, &h->tv_ustate, 2 * kd))))
      return bail(rc);
    if (cudaMemsetAsync(h->tv_stats, 0, 16, h->work) != cudaSuccess) return bail(fail(POLY_ECUDA, "memset"));
  }
  if ((rc = dev_alloc(h, &h->comm, (size_t)p.d + 1)) != POLY_OK) return bail(rc);
  if ((rc = dev_alloc(h, &h->xa, (size_t)p.d)) != POLY_OK) return bail(rc);
  if ((rc = dev_alloc(h, &h->xh, (size_t)p.d)) != POLY_OK) return bail(rc);
  if ((rc = dev_alloc(h, &h->xin, (size_t)p.d)) != POLY_OK) return bail(rc);
  if ((rc = dev_alloc(h, &h->gbuf, (size_t)p.d)) != POLY_OK) return bail(rc);
  if ((rc = dev_alloc(h, &h->vscratch, (size_t)p.d)) != POLY_OK) return bail(rc);
  if ((rc = dev_alloc(h, &h->block_norm, (size_t)h->fin_grid)) != POLY_OK) return bail(rc);
  if ((rc = dev_alloc(h, &h->state, 1)) != POLY_OK) return bail(rc);
  if (cudaMallocHost(&h->hstate, sizeof(SolveState)) != cudaSuccess)
    return bail(fail(POLY_ENOMEM, "cudaMallocHost failed"));
  memset(h->hstate, 0, sizeof(SolveState));
  if (cudaMemcpyAsync(h->state, h->hstate, sizeof(SolveState), cudaMemcpyHostToDevice, h->work) != cudaSuccess)
    return bail(fail(POLY_ECUDA, "state upload failed"));

  // input checks that need the device: counts >= 0, CSR structure
  if (p.n_local > 0) {
    int32_t *flag = nullptr;
    if ((rc = dev_alloc(h, &flag, 1)) != POLY_OK) return bail(rc);
    int32_t hv = 0;
    cudaMemsetAsync(flag, 0, 4, h->work);
    if (p.ytype == POLY_Y_I32) {
      k_min_i32<<<std::min<int64_t>(1024, (p.n_local * h->Om + 255) / 256), 256, 0, h->work>>>(
          (const int32_t *)p.y, p.n_local * h->Om, flag);
      cudaMemcpyAsync(&hv, flag, 4, cudaMemcpyDeviceToHost, h->work);
      if (cudaStreamSynchronize(h->work) != cudaSuccess)
        return bail(fail(POLY_ECUDA, "count check failed: %s", cudaGetErrorString(cudaGetLastError())));
      if (hv < 0) return bail(fail(POLY_EINVAL, "negative Poisson count in y (PAPER.md:876-878)"));
    }
    if (p.layout == POLY_CSR) {
      cudaMemsetAsync(flag, 0, 4, h->work);
      k_check_csr<<<1024, 256, 0, h->work>>>(p.row_ptr, p.col, p.n_local, p.nnz, (int)p.d, flag);
      cudaMemcpyAsync(&hv, flag, 4, cudaMemcpyDeviceToHost, h->work);
      if (cudaStreamSynchronize(h->work) != cudaSuccess)
        return bail(fail(POLY_ECUDA, "CSR check failed: %s", cudaGetErrorString(cudaGetLastError())));
      if (hv) return bail(fail(POLY_EINVAL, "invalid CSR structure (code %d)", hv));
    }
  }
  if (p.layout == POLY_CSR && (rc = build_sell(h)) != POLY_OK) return bail(rc);
  if (h->Om > 1 && p.n_local > 0) {  // y^Σ_i = Σ_ω y_ωi (ω ascending), library-owned
    const bool ints = p.ytype == POLY_Y_I32;
    void *ys = nullptr;
    if ((rc = dev_alloc(h, (unsigned char **)&ys, (size_t)p.n_local * (ints ? 4 : 8))) != POLY_OK)
      return bail(rc);
    int32_t *flag = nullptr;
    if ((rc = dev_alloc(h, &flag, 1)) != POLY_OK) return bail(rc);
    int32_t hv = 0;
    cudaMemsetAsync(flag, 0, 4, h->work);
    k_sum_windows<<<std::min<int64_t>(4096, (p.n_local + 255) / 256), 256, 0, h->work>>>(
        p.y, p.ytype, h->Om, p.n_local, ys, flag);
    cudaMemcpyAsync(&hv, flag, 4, cudaMemcpyDeviceToHost, h->work);
    if (cudaStreamSynchronize(h->work) != cudaSuccess)
      return bail(fail(POLY_ECUDA, "window sum failed: %s", cudaGetErrorString(cudaGetLastError())));
    if (hv) return bail(fail(POLY_EUNSUPPORTED, "sum of window counts exceeds int32"));
    p.y = ys;
    p.ytype = ints ? POLY_Y_I32 : POLY_Y_F64;
    h->ysz = ints ? 4 : 8;
  }

  h->comm_path = p.world > 1 || (p.flags & POLY_FLAG_COMM);
  if ((p.flags & POLY_FLAG_NVLS) && !h->comm_path)
    return bail(fail(POLY_EINVAL, "POLY_FLAG_NVLS needs world > 1 or POLY_FLAG_COMM"));
  if ((p.flags & POLY_FLAG_NVLS) && (p.flags & POLY_FLAG_P2P))
    return bail(fail(POLY_EINVAL, "POLY_FLAG_NVLS and POLY_FLAG_P2P are exclusive"));
  if (p.flags & POLY_FLAG_P2P) {
    if (!h->comm_path) return bail(fail(POLY_EINVAL, "POLY_FLAG_P2P needs world > 1 or POLY_FLAG_COMM"));
    if (p.world > kP2PMaxRanks) return bail(fail(POLY_EUNSUPPORTED, "POLY_FLAG_P2P: world > %d", kP2PMaxRanks));
    const size_t wb = kP2PFlagBytes + (size_t)2 * (p.d + 1) * 8;
    if ((rc = dev_alloc(h, &h->p2p_win, wb)) || (rc = dev_alloc(h, &h->p2p_epoch, (size_t)kP2PMaxBlocks)))
      return bail(rc);
    if (cudaMemsetAsync(h->p2p_win, 0, wb, h->work) != cudaSuccess ||
        cudaMemsetAsync(h->p2p_epoch, 0, 8 * (size_t)kP2PMaxBlocks, h->work) != cudaSuccess)
      return bail(fail(POLY_ECUDA, "p2p window reset"));
  }
  if (h->comm_path) {
    NcclApi *api = nccl_api();
    if (!api) return bail(fail(POLY_ENCCL, "world > 1 but libnccl.so.2 cannot be loaded"));
    ncclUniqueId id;
    memcpy(&id, p.nccl_id, sizeof(id));
    ncclResult_t r = api->commInitRank(&h->nccl, p.world, id, p.rank);
    if (r != ncclSuccess) {
      h->nccl = nullptr;
      return bail(fail(POLY_ENCCL, "ncclCommInitRank: %s", api->errStr(r)));
    }
  }
  p.nccl_id = nullptr;
  if (cudaStreamSynchronize(h->work) != cudaSuccess)
    return bail(fail(POLY_ECUDA, "init: %s", cudaGetErrorString(cudaGetLastError())));
  g_err[0] = 0;
  *out = h;
  return POLY_OK;
}

int poly_loss_grad(poly_handle *h, const double *x, double *g, double *loss) {
  if (!h || !x) return fail(POLY_EINVAL, "NULL handle or x");
  TRY(sync_in(h));
  TRY(check_comm(h));
  const double *xd = x;
  if (!is_device_ptr(x)) {
    CK(cudaMemcpyAsync(h->xin, x, h->p.d * 8, cudaMemcpyHostToDevice, h->work));
    xd = h->xin;
  }
  const bool g_dev = g && is_device_ptr(g);
  double *gd = g ? (g_dev ? g : h->gbuf) : nullptr;
  h->prof = false;
  TRY(enqueue_eval(h, xd, loss != nullptr, false, nullptr, nullptr, gd));
  if (g && !g_dev) CK(cudaMemcpyAsync(g, h->gbuf, h->p.d * 8, cudaMemcpyDeviceToHost, h->work));
  if (loss) {
    CK(cudaMemcpyAsync(&h->hstate->loss_cur, &h->state->loss_cur, 8, cudaMemcpyDeviceToHost, h->work));
    TRY(sync_work(h));
    *loss = h->hstate->loss_cur;
  } else if (g && !g_dev) {
    TRY(sync_work(h));
  }
  TRY(sync_out(h));
  CK(cudaGetLastError());
  return POLY_OK;
}

int poly_solve_ex(poly_handle *h, const poly_solve_opts *o, double *x, double *x_last,
                  poly_solve_info *info) {
  if (!h || !o || !x) return fail(POLY_EINVAL, "NULL handle, opts or x");
  if (o->T_max < 0) return fail(POLY_EINVAL, "T_max < 0");
  if (o->method != POLY_METHOD_EXTRAGRADIENT && o->method != POLY_METHOD_GD)
    return fail(POLY_EINVAL, "bad method");
  if (!(o->gamma > 0.0) || !std::isfinite(o->gamma)) return fail(POLY_EINVAL, "gamma must be > 0");
  if (!(o->tol >= 0.0)) return fail(POLY_EINVAL, "tol must be >= 0");
  if (info) memset(info, 0, sizeof(*info));
  const int d = (int)h->p.d;
  const bool avg = o->average != 0;
  const int method = o->method;
  TRY(sync_in(h));
  const bool x_dev = is_device_ptr(x);
  CK(cudaMemcpyAsync(h->xa, x, (size_t)d * 8, x_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                     h->work));
  if (avg) {
    const int cap = (o->T_max + 1) / 2 + 3;
    if (cap > h->avg_cap) {
      // graphs captured with the old ring baked in must be rebuilt
      for (auto &a : h->gexec_ex)
        for (auto &g : a[1])
          if (g) {
            cudaGraphExecDestroy(g);
            g = nullptr;
          }
      double *old = h->hist;
      TRY(dev_alloc(h, &h->hist, (size_t)cap * d));
      if (old) {  // no graph refers to it any more; the stream must drain first
        TRY(sync_work(h));
        dev_release(h, old);
      }
      if (!h->Ssum) {
        TRY(dev_alloc(h, &h->Ssum, (size_t)d));
        TRY(dev_alloc(h, &h->xbar, (size_t)d));
        TRY(dev_alloc(h, &h->avg_norm, (size_t)(d + 255) / 256));
      }
      h->avg_cap = cap;
    }
    CK(cudaMemsetAsync(h->hist, 0, (size_t)d * 8, h->work));  // slot 0: "x_0" = 0
    CK(cudaMemsetAsync(h->Ssum, 0, (size_t)d * 8, h->work));
    CK(cudaMemsetAsync(h->xbar, 0, (size_t)d * 8, h->work));
  }
  SolveState st{};
  st.gamma = o->gamma;
  st.tol = o->tol;
  *h->hstate = st;
  CK(cudaMemcpyAsync(h->state, h->hstate, sizeof(SolveState), cudaMemcpyHostToDevice, h->work));
  h->prof = (o->flags & POLY_SOLVE_PROFILE) != 0;
  h->recs.clear();
  h->evused = 0;
  {
    FinArgs f = fin_base(h, FIN_PROJECT);  // x_1 = P_X(x_in)
    f.anchor = h->xa;
    f.x_out = h->xa;
    f.x32_out = h->xa32;
    f.tr_side = h->tr_side;
    TRY(enqueue_fin(h, f));
  }
  if (avg) TRY(enqueue_avg(h));  // folds x_1: S = x_1, x̄_1 = x_1, k = 1
  const int T = o->T_max;
  const bool poll = avg && o->tol > 0.0;
  int done = 0;
  auto halted = [&]() { return h->hstate->bad != 0 || h->hstate->comm_err != 0 || (poll && h->hstate->stopped); };
  if (h->use_graph && !h->prof) {
    const int U = h->graph_U;
    cudaGraphExec_t *gU = &h->gexec_ex[method][avg ? 1 : 0][1];
    cudaGraphExec_t *g1 = &h->gexec_ex[method][avg ? 1 : 0][0];
    int rc = POLY_OK;
    if (T >= U && !*gU) rc = build_graph_ex(h, method, avg, U, gU);
    if (rc == POLY_OK && (T % U) && !*g1) rc = build_graph_ex(h, method, avg, 1, g1);
    if (rc != POLY_OK) return rc;
    // the stop rule is polled after every replay (one replay behind), the
    // non-finite / K9 flags every kPollEvery replays otherwise
    int replays = 0, polls = 0;
    while (done < T && !halted()) {
      const int step = (T - done >= U) ? U : 1;
      CK(cudaGraphLaunch(step == U ? *gU : *g1, h->work));
      done += step;
      if ((poll || ++replays % kPollEvery == 0) && done < T) TRY(poll_state(h, polls++));
    }
  } else {
    for (; done < T && !halted(); ++done) {
      TRY(enqueue_iteration_ex(h, method, avg));
      if (!h->prof && (done % 64) == 63) {
        CK(cudaMemcpyAsync(h->hstate, h->state, sizeof(SolveState), cudaMemcpyDeviceToHost, h->work));
        TRY(sync_work(h));
      }
    }
  }
  CK(cudaMemcpyAsync(h->hstate, h->state, sizeof(SolveState), cudaMemcpyDeviceToHost, h->work));
  TRY(sync_work(h));
  const SolveState fin = *h->hstate;
  const bool stopped = avg && fin.stopped;
  const double *last = stopped ? h->hist + (size_t)(fin.k_stop % h->avg_cap) * d : h->xa;
  const double *outv = avg ? h->xbar : h->xa;
  CK(cudaMemcpyAsync(x, outv, (size_t)d * 8, x_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                     h->work));
  if (x_last)
    CK(cudaMemcpyAsync(x_last, last, (size_t)d * 8,
                       is_device_ptr(x_last) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->work));
  TRY(sync_work(h));
  if (h->prof) collect_profile(h);
  TRY(sync_out(h));
  CK(cudaGetLastError());
  const int per = method == POLY_METHOD_EXTRAGRADIENT ? 2 : 1;
  if (fin.comm_err == 2) return fail(POLY_ECUDA, "K4p: grid barrier timed out (CTAs not co-resident)");
  if (fin.comm_err) {
    if (h->nccl) nccl_api()->commAbort(h->nccl);
    h->nccl = nullptr;
    return fail(POLY_ENCCL, "peer reduce: a peer did not publish within the wait bound; communicator aborted");
  }
  if (info) {
    info->stopped = stopped ? 1 : 0;
    info->iters = stopped ? fin.k_stop - 1 : done;
    info->move = avg ? fin.move : 0.0;
  }
  if (fin.bad != 0) {
    const int b = fin.bad > 0 ? (fin.bad + per - 1) / per : 0;
    if (info) info->bad_iter = b;
    return fail(POLY_ENONFINITE, "non-finite iterate at iteration %d", b);
  }
  return POLY_OK;
}

int poly_solve(poly_handle *h, double *x, int T, double gamma, uint32_t flags, double *trace,
               int *bad_iter) {
  if (!h || !x) return fail(POLY_EINVAL, "NULL handle or x");
  if (T < 0) return fail(POLY_EINVAL, "T < 0");
  if (!(gamma > 0.0) || !std::isfinite(gamma)) return fail(POLY_EINVAL, "gamma must be > 0");
  if (bad_iter) *bad_iter = 0;
  TRY(sync_in(h));
  TRY(check_comm(h));
  const bool x_dev = is_device_ptr(x);
  CK(cudaMemcpyAsync(h->xa, x, h->p.d * 8, x_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                     h->work));
  const bool want_trace = trace != nullptr;
  if (want_trace && h->trace_cap < 2 * T) {
    double *nt = nullptr;
    TRY(dev_alloc(h, &nt, (size_t)2 * T));
    // graphs hold the old trace pointer only through SolveState (read on the
    // device), so the old buffer can go once the stream has drained
    if (h->trace) {
      TRY(sync_work(h));
      dev_release(h, h->trace);
    }
    h->trace = nt;
    h->trace_cap = 2 * T;
  }
  SolveState st{};
  st.gamma = gamma;
  st.trace = want_trace ? h->trace : nullptr;
  st.trace_cap = want_trace ? 2 * T : 0;
  *h->hstate = st;
  CK(cudaMemcpyAsync(h->state, h->hstate, sizeof(SolveState), cudaMemcpyHostToDevice, h->work));

  {  // small dense problems: the whole solve in one cluster-resident kernel
    int C = 0;
    size_t smem = 0;
    if (!(flags & POLY_SOLVE_PROFILE) && T > 0 && small_solve_config(h, &C, &smem) == POLY_OK) {
      TRY(launch_small_solve(h, h->xa, T, want_trace, C, smem));
      CK(cudaMemcpyAsync(x, h->xa, h->p.d * 8, x_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                         h->work));
      if (want_trace)
        CK(cudaMemcpyAsync(trace, h->trace, (size_t)2 * T * 8, cudaMemcpyDeviceToHost, h->work));
      CK(cudaMemcpyAsync(h->hstate, h->state, sizeof(SolveState), cudaMemcpyDeviceToHost, h->work));
      TRY(sync_work(h));
      TRY(sync_out(h));
      CK(cudaGetLastError());
      if (h->hstate->bad != 0) {
        const int b = h->hstate->bad;
        if (bad_iter) *bad_iter = b > 0 ? (b + 1) / 2 : 0;
        return fail(POLY_ENONFINITE, "non-finite iterate at iteration %d", b > 0 ? (b + 1) / 2 : 0);
      }
      return POLY_OK;
    }
  }
  h->prof = (flags & POLY_SOLVE_PROFILE) != 0;
  h->recs.clear();
  h->evused = 0;
  // x_1 = P_X(x_in)
  {
    FinArgs f = fin_base(h, FIN_PROJECT);
    f.anchor = h->xa;
    f.x_out = h->xa;
    f.x32_out = h->xa32;
    f.tr_side = h->tr_side;
    TRY(enqueue_fin(h, f));
  }
  const bool loss = want_trace;
  int rc = POLY_OK;
  if (h->use_graph && !h->prof && T > 0) {
    int li = loss ? 1 : 0;
    // both graphs (U iterations and 1) are built and uploaded at the first
    // solve, whatever its T, so that a short warm-up call prepares a long one
    if (!h->gexec[li][1]) rc = build_graph(h, loss, h->graph_U, &h->gexec[li][1]);
    if (rc == POLY_OK && !h->gexec[li][0]) rc = build_graph(h, loss, 1, &h->gexec[li][0]);
    if (rc != POLY_OK && h->pdl) {  // retry capture without programmatic edges
      h->pdl = false;
      cudaGetLastError();
      rc = POLY_OK;
      if (!h->gexec[li][1]) rc = build_graph(h, loss, h->graph_U, &h->gexec[li][1]);
      if (rc == POLY_OK && !h->gexec[li][0]) rc = build_graph(h, loss, 1, &h->gexec[li][0]);
    }
    if (rc == POLY_OK) rc = replay_solve(h, h->gexec[li][1], h->gexec[li][0], T);
  } else {
    for (int t = 0; t < T && rc == POLY_OK; ++t) {
      rc = enqueue_iteration(h, loss);
      if (rc == POLY_OK && !h->prof && (t % kPollEvery) == kPollEvery - 1) rc = poll_state(h, t / kPollEvery);
      if (rc == POLY_OK && h->hstate->bad) break;
    }
  }
  if (rc != POLY_OK) {
    h->prof = false;
    sync_work(h);
    return rc;
  }
  CK(cudaMemcpyAsync(x, h->xa, h->p.d * 8, x_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                     h->work));
  if (want_trace) CK(cudaMemcpyAsync(trace, h->trace, (size_t)2 * T * 8, cudaMemcpyDeviceToHost, h->work));
  CK(cudaMemcpyAsync(h->hstate, h->state, sizeof(SolveState), cudaMemcpyDeviceToHost, h->work));
  TRY(sync_work(h));
  if (h->prof) collect_profile(h);
  TRY(sync_out(h));
  CK(cudaGetLastError());
  if (h->hstate->comm_err == 2) return fail(POLY_ECUDA, "K4p: grid barrier timed out (CTAs not co-resident)");
  if (h->hstate->comm_err) {
    if (h->nccl) nccl_api()->commAbort(h->nccl);
    h->nccl = nullptr;
    return fail(POLY_ENCCL, "peer reduce: a peer did not publish within the wait bound; communicator aborted");
  }
  TRY(check_tv_meet(h));
  if (h->hstate->bad != 0) {
    const int b = h->hstate->bad;
    if (bad_iter) *bad_iter = b > 0 ? (b + 1) / 2 : 0;
    return fail(POLY_ENONFINITE, "non-finite iterate at iteration %d", b > 0 ? (b + 1) / 2 : 0);
  }
  return POLY_OK;
}

}  // extern "C"

namespace {
int aux_rows(poly_handle *h, const double *x, double *out, int want_counts) {
  if (!h || !x || !out) return fail(POLY_EINVAL, "NULL argument");
  const poly_problem &p = h->p;
  if (p.layout == POLY_PARALLEL_BEAM) return fail(POLY_EUNSUPPORTED, "forward/expected counts: dense or CSR only");
  if (p.n_local == 0) return POLY_OK;
  TRY(sync_in(h));
  AuxArgs a{};
  a.layout = p.layout;
  a.dtype = p.dtype;
  a.A = p.A;
  a.lda = p.lda;
  a.row_ptr = p.row_ptr;
  a.col = p.col;
  a.val = p.val;
  a.n = p.n_local;
  a.d = (int32_t)p.d;
  a.W = p.W;
  a.relu = p.relu;
  a.s_row = p.s_row;
  a.I_row = p.I_row;
  a.I_bar = p.I_bar;
  a.x = x;
  a.spec = h->spec;
  a.out = out;
  a.want_counts = want_counts;
  const int grid = (int)std::min<int64_t>((int64_t)h->sms * 16, (p.n_local + 7) / 8);
  if (p.dtype == POLY_F32)
    k_aux_rows<float><<<grid, 256, 0, h->work>>>(a);
  else
    k_aux_rows<double><<<grid, 256, 0, h->work>>>(a);
  CK(cudaGetLastError());
  TRY(sync_out(h));
  return POLY_OK;
}
}  // namespace

extern "C" {

int poly_forward(poly_handle *h, const double *x, double *z) { return aux_rows(h, x, z, 0); }

int poly_expected_counts(poly_handle *h, const double *x, double *lam) {
  return aux_rows(h, x, lam, 1);
}

int poly_reparameterize(int32_t W, const double *s, const double *mu, double I_bar, int64_t n,
                        const double *b, int32_t clamp, float *s_row, float *I_row, void *stream) {
  if (W < 1 || W > kMaxW || !s || !mu || n < 0 || (n > 0 && (!b || !s_row || !I_row)))
    return fail(POLY_EINVAL, "poly_reparameterize: bad arguments");
  if (!(I_bar > 0.0)) return fail(POLY_EINVAL, "I_bar must be > 0");
  if (n == 0) return POLY_OK;
  ReparamArgs a{};
  a.W = W;
  a.clamp = clamp;
  a.n = n;
  a.I_bar = I_bar;
  for (int j = 0; j < W; ++j) {
    if (!(s[j] > 0.0) || !(mu[j] > 0.0)) return fail(POLY_EINVAL, "bad spectrum");
    a.s[j] = s[j];
    a.mu[j] = mu[j];
  }
  a.b = b;
  a.s_row = s_row;
  a.I_row = I_row;
  const int grid = (int)std::min<int64_t>(148 * 32, (n + 255) / 256);
  k_reparam<<<grid, 256, 0, (cudaStream_t)stream>>>(a);
  CK(cudaGetLastError());
  return POLY_OK;
}

int poly_project(poly_handle *h, const double *v, double *x, int64_t *stats) {
  if (!h || !v || !x) return fail(POLY_EINVAL, "NULL argument");
  TRY(sync_in(h));
  if (h->tv_stats) CK(cudaMemsetAsync(h->tv_stats, 0, 16, h->work));
  if (h->tv_cl) {
    TRY(enqueue_tv(h, v, x));
  } else {
    FinArgs f = fin_base(h, FIN_PROJECT);
    f.anchor = v;
    f.x_out = x;
    f.x32_out = nullptr;
    f.tr_side = 0;
    TRY(enqueue_fin(h, f));
  }
  int32_t hs[4] = {0, 0, 0, 0};
  if (h->tv_stats) CK(cudaMemcpyAsync(hs, h->tv_stats, 16, cudaMemcpyDeviceToHost, h->work));
  CK(cudaStreamSynchronize(h->work));
  if (stats)
    for (int k = 0; k < 3; ++k) stats[k] = hs[k];
  TRY(sync_out(h));
  CK(cudaGetLastError());
  if (hs[3]) return fail(POLY_ECUDA, "TV projection: the %d clusters did not meet (not co-resident)", h->tv_k);
  return POLY_OK;
}

int poly_stream_probe(poly_handle *h, int32_t reps, double *ms) {
  if (!h || !ms || reps < 1) return fail(POLY_EINVAL, "bad arguments");
  if (h->p.layout != POLY_DENSE) return fail(POLY_EUNSUPPORTED, "the probe streams dense A only");
  const poly_problem &p = h->p;
  const int64_t row_bytes = p.lda * h->elsize;
  const int rps = h->dv->RPS;
  const size_t smem = (size_t)h->k1_stages * rps * row_bytes + 2 * 8 * (size_t)h->k1_stages;
  CK(cudaFuncSetAttribute((const void *)&k_stream_probe, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)smem));
  TRY(sync_in(h));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  k_stream_probe<<<h->k1_grid, 64, smem, h->work>>>(p.A, row_bytes, p.n_local, rps, h->k1_stages);
  CK(cudaEventRecord(e0, h->work));
  for (int r = 0; r < reps; ++r)
    k_stream_probe<<<h->k1_grid, 64, smem, h->work>>>(p.A, row_bytes, p.n_local, rps, h->k1_stages);
  CK(cudaEventRecord(e1, h->work));
  CK(cudaEventSynchronize(e1));
  float t = 0.f;
  cudaEventElapsedTime(&t, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *ms = (double)t / reps;
  TRY(sync_out(h));
  CK(cudaGetLastError());
  return POLY_OK;
}

int poly_kernel_times(poly_handle *h, double *out, int32_t nout) {
  if (!h || !out || nout < 0 || nout > 5) return fail(POLY_EINVAL, "bad arguments");
  for (int i = 0; i < nout; ++i) out[i] = h->ktimes[i];
  return POLY_OK;
}

int poly_describe(poly_handle *h, int64_t *out, int32_t nout) {
  if (!h || !out || nout < 0 || nout > 14) return fail(POLY_EINVAL, "bad arguments");
  int64_t v[14] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  if (h->nccl) {
    int c = 0;
    if (nccl_api()->count(h->nccl, &c) == ncclSuccess) v[10] = c;
  }
  v[11] = h->nv.on ? 2 : (h->p2p ? 1 : 0);
  if (h->p.layout == POLY_DENSE) {
    v[0] = h->k1_grid;
    v[1] = h->k1_threads;
    v[2] = h->dv->RPS;
    v[3] = h->k1_stages;
    v[4] = (int64_t)h->k1_smem;
    v[6] = h->dv->V;     // K1 template <T, V, WPR, NW, RPS, LOSS, FULL>
    v[7] = h->dv->WPR;
    v[8] = h->dv->NW;
    v[9] = h->full;
  } else if (h->tiled) {
    v[0] = h->tf_grid;   // K4tf CTAs (one per SM), K4tb: one CTA per 32 x 8 tile
    v[1] = (kFwdWarps + 1) * 32;
    v[2] = h->tfwd.NS;   // column strips
    v[3] = h->tb_grid;
    v[4] = (int64_t)h->tf_smem;
  } else {
    v[0] = h->k4_grid;   // K4f blocks (32-row slices); K4b: one block per 32-column slice
    v[1] = 128;
    v[2] = h->nslices;
    v[3] = h->sell_steps;
    v[4] = 0;
  }
  // CSR layout: 0 wide SELL-32, 1 compact SELL16, 2 DSELL, 3 K4t (tiled.cuh); -1 dense / matrix-free
  v[12] = h->p.layout != POLY_CSR ? -1 : (h->tiled ? 3 : (h->dsell ? 2 : (h->sell16 ? 1 : 0)));
  v[5] = h->sms;
  v[13] = (h->p.layout == POLY_DENSE || h->tiled) ? h->keep_bytes : 0;
  for (int i = 0; i < nout; ++i) out[i] = v[i];
  return POLY_OK;
}

}  // extern "C"
