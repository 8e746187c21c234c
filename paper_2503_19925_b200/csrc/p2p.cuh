// K9 — the cross-GPU sum of step a6 as one
// kernel over NVLink peer memory instead of ncclAllReduce.
//
// Each rank owns a window (cudaIpc-exported, mapped by every peer):
//   flags[2][kP2PMaxBlocks] (uint64) | slot0[n] | slot1[n]   (n = d + 1 doubles)
// The grid (at most one block per SM) is the same on every rank, and block b
// owns the same chunk of the vector everywhere, so blocks never wait for each
// other — only for their namesakes on the other ranks.  Per F evaluation
// e = 1, 2, ... (block b's counter, advanced in lockstep on every rank), with
// parity q = e & 1, block b:
//   1. copies its chunk of the local unnormalised sums (comm) into its own
//      slot q, and after a block barrier publishes flags[q][b] = e with one
//      system-scope release store;
//   2. waits (system-scope acquire loads, bounded by timeout_ns) until every
//      rank's flags[q][b] == e,
//      then sums its chunk over ranks 0..P-1 in rank order straight from the
//      ranks' slots (NVLink loads) into comm — the same bits on every rank,
//      so the replicated iterates stay identical.
// Double buffering is enough: a block publishes e+2 into slot q only after its
// evaluation e+1 saw every namesake's e+1 flag, i.e. after each of them
// finished reading slot q of evaluation e.
#pragma once

#include "common.cuh"

namespace poly {

constexpr int kP2PMaxRanks = 8;
constexpr int kP2PMaxBlocks = 256;                     // >= SM count
constexpr int kP2PFlagBytes = 2 * kP2PMaxBlocks * 8;  // flags[2][kP2PMaxBlocks]

struct PeerArgs {
  double *comm;                    // [n] local sums in, rank-ordered total out
  int64_t n;                       // d + 1
  int32_t world, rank;
  char *win[kP2PMaxRanks];         // every rank's window (own one local, peers IPC-mapped)
  unsigned long long *epoch;       // [kP2PMaxBlocks] local evaluation counters, one per block
  int32_t *err;                    // set to 1 when a wait exceeds timeout_ns (SolveState.comm_err)
  unsigned long long timeout_ns;   // bound on every wait for a peer (globaltimer ns)
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed_sys(const double *p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(256) k_peer_reduce(const PeerArgs a) {
  const unsigned long long e = a.epoch[blockIdx.x] + 1;
  const int q = (int)(e & 1);
  auto slot = [&](int r) { return reinterpret_cast<double *>(a.win[r] + kP2PFlagBytes) + q * a.n; };
  auto flag = [&](int r) { return reinterpret_cast<unsigned long long *>(a.win[r]) + q * kP2PMaxBlocks + blockIdx.x; };
  const int64_t chunk = (a.n + gridDim.x - 1) / gridDim.x;
  const int64_t c0 = blockIdx.x * chunk, c1 = min(a.n, c0 + chunk);
  pdl_wait();  // comm is written by the reduce kernel before us
  // 1. publish this block's chunk
  double *own = slot(a.rank);
  for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) own[i] = a.comm[i];
  __syncthreads();
  if (threadIdx.x == 0) st_release_sys(flag(a.rank), e);
  // 2. wait (bounded) for the namesake blocks of every rank, then the
  // rank-ordered sum; a peer that never publishes ends the wait with err set
  // (the host aborts the communicator: no rank hangs)
  __shared__ int s_ok;
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  if (threadIdx.x < a.world) {
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_sys(flag(threadIdx.x)) != e) {
      if (globaltimer_ns() - t0 > a.timeout_ns) {
        s_ok = 0;
        atomicExch(a.err, 1);
        break;
      }
    }
  }
  __syncthreads();
  if (!s_ok) return;
  for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
    double v = 0.0;
    for (int r = 0; r < a.world; ++r) v += ld_relaxed_sys(slot(r) + i);
    a.comm[i] = v;
  }
  if (threadIdx.x == 0) a.epoch[blockIdx.x] = e;
}

}  // namespace poly
