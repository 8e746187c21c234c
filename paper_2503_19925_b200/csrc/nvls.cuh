// K9-NVLS — the cross-GPU sum of step a6
// as one kernel over an NVLink multicast object: the reduction itself runs
// in the NVSwitch (multimem.ld_reduce), the result is broadcast by the switch
// (multimem.st), and the ranks synchronise with multimem.red on flags that
// live in the same multicast window.  No NCCL launch, no protocol.
//
// Window (bound to a multicast object; every rank has a unicast view uc of
// its own physical copy and the common multicast view mc; same offsets):
//   flags[2][kNvlsMaxBlocks] (uint64, barrier 0 and 1) | pad to 4 KB |
//   data[2][n] | res[2][n]        (n = d + 1 doubles, slot q = parity of e)
// Per F evaluation e = 1, 2, ... (block b's counter, advanced in lockstep on
// every rank), block b owns chunk b of the vector and, within it, sub-chunk
// `rank` of `world`:
//   1. writes its chunk of the local unnormalised sums into data[q] (uc);
//   2. barrier 0: fence.acq_rel.sys, multimem.red.release.sys.add(flag0[b], 1)
//      — one add lands in every rank's copy — then waits (acquire, bounded
//      by timeout_ns) until its own copy of flag0[b] reaches world·e;
//   3. for its sub-chunk: v = multimem.ld_reduce.add.f64(data[q] mc) — the
//      switch sums the ranks' copies — and multimem.st(res[q] mc, v): each
//      element is reduced once and every rank receives the same bits;
//   4. barrier 1 (same pattern on flag1[b]), then copies res[q] (uc) back into
//      comm.
// Double buffering: a rank writes data/res slot q for e + 2 only after barrier
// 0 of e + 1, which every rank reaches only after finishing evaluation e.
#pragma once

#include "common.cuh"

namespace poly {

constexpr int kNvlsMaxBlocks = 256;
constexpr size_t kNvlsHdr = 4096;  // flags[2][kNvlsMaxBlocks] uint64, padded

struct NvlsArgs {
  double *comm;                   // [n] local sums in, total out
  int64_t n;                      // d + 1
  int32_t world, rank;
  char *uc;                       // this rank's unicast view of the window
  char *mc;                       // the multicast view
  unsigned long long *epoch;      // [kNvlsMaxBlocks] local evaluation counters
  int32_t *err;                   // set to 1 on a wait timeout (SolveState.comm_err)
  unsigned long long timeout_ns;
};

__device__ __forceinline__ unsigned long long nvls_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned long long nvls_ld_acquire(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// thread 0 of the block: arrive on barrier `which` of block b and wait for all
// ranks (flag value world·e); false on timeout
__device__ __forceinline__ bool nvls_barrier(const NvlsArgs &a, int which, unsigned long long target) {
  unsigned long long *mcf = reinterpret_cast<unsigned long long *>(a.mc) + which * kNvlsMaxBlocks + blockIdx.x;
  const unsigned long long *ucf =
      reinterpret_cast<const unsigned long long *>(a.uc) + which * kNvlsMaxBlocks + blockIdx.x;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  asm volatile("multimem.red.release.sys.global.add.u64 [%0], %1;" ::"l"(mcf), "l"(1ull) : "memory");
  const unsigned long long t0 = nvls_clock();
  while (nvls_ld_acquire(ucf) < target)
    if (nvls_clock() - t0 > a.timeout_ns) return false;
  return true;
}

__global__ void __launch_bounds__(256) k_nvls_reduce(const NvlsArgs a) {
  __shared__ int s_ok;
  const unsigned long long e = a.epoch[blockIdx.x] + 1;
  const int q = (int)(e & 1);
  const int64_t chunk = (a.n + gridDim.x - 1) / gridDim.x;
  const int64_t c0 = blockIdx.x * chunk, c1 = min(a.n, c0 + chunk);
  double *data_uc = reinterpret_cast<double *>(a.uc + kNvlsHdr) + q * a.n;
  double *data_mc = reinterpret_cast<double *>(a.mc + kNvlsHdr) + q * a.n;
  double *res_uc = reinterpret_cast<double *>(a.uc + kNvlsHdr) + (2 + q) * a.n;
  double *res_mc = reinterpret_cast<double *>(a.mc + kNvlsHdr) + (2 + q) * a.n;
  const unsigned long long target = (unsigned long long)a.world * e;
  pdl_wait();  // comm is written by the reduce kernel before us
  for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) data_uc[i] = a.comm[i];
  __syncthreads();
  if (threadIdx.x == 0) s_ok = nvls_barrier(a, 0, target);
  __syncthreads();
  if (!s_ok) {
    if (threadIdx.x == 0) atomicExch(a.err, 1);
    return;
  }
  const int64_t len = c1 - c0;
  const int64_t s0 = c0 + len * a.rank / a.world, s1 = c0 + len * (a.rank + 1) / a.world;
  for (int64_t i = s0 + threadIdx.x; i < s1; i += blockDim.x) {
    double v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f64 %0, [%1];" : "=d"(v) : "l"(data_mc + i) : "memory");
    asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(res_mc + i), "d"(v) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) s_ok = nvls_barrier(a, 1, target);
  __syncthreads();
  if (!s_ok) {
    if (threadIdx.x == 0) atomicExch(a.err, 1);
    return;
  }
  for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x)
    a.comm[i] = *reinterpret_cast<volatile double *>(res_uc + i);
  if (threadIdx.x == 0) a.epoch[blockIdx.x] = e;
}

}  // namespace poly
