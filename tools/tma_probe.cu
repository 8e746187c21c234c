// Bulk-copy (TMA) streaming ceiling on this GPU: each CTA streams contiguous
// chunks of S bytes through a ring of NST shared-memory stages (producer lane
// issues cp.async.bulk; consumer warps touch one word per stage and release
// it).  Usage: tma_probe [GB]; prints GB/s per (S, NST, CTAs/SM, interleave).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_probe(const uint8_t *src, int64_t chunks_per_cta, int S, int NST, int inter, int nwarps,
                        unsigned long long *sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t *full = (uint64_t *)(sm + (size_t)NST * S);
  uint64_t *empty = full + NST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(full + s)), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(empty + s)), "r"(nwarps));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == nwarps) {
    if (lane == 0) {
      for (int64_t k = 0; k < chunks_per_cta; ++k) {
        const int st = (int)(k % NST);
        if (k >= NST) {
          const uint32_t par = (uint32_t)((k / NST) - 1) & 1;
          asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(su(empty + st)), "r"(par) : "memory");
        }
        const int64_t c = inter ? k * gridDim.x + blockIdx.x : (int64_t)blockIdx.x * chunks_per_cta + k;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(full + st)), "r"(S) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(sm + (size_t)st * S)), "l"(src + c * S), "r"(S), "r"(su(full + st)) : "memory");
      }
    }
    return;
  }
  unsigned long long acc = 0;
  for (int64_t k = 0; k < chunks_per_cta; ++k) {
    const int st = (int)(k % NST);
    const uint32_t par = (uint32_t)(k / NST) & 1;
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(su(full + st)), "r"(par) : "memory");
    acc += *(const uint32_t *)(sm + (size_t)st * S + (warp * 32 + lane) * 4);
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(empty + st)) : "memory");
  }
  if (acc == 0x1234567) sink[0] = acc;
}

int main(int argc, char **argv) {
  const double gb = argc > 1 ? atof(argv[1]) : 2.0;
  const size_t bytes = (size_t)(gb * 1e9);
  uint8_t *buf;
  unsigned long long *sink;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 8);
  cudaMemset(buf, 1, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int Ss[] = {8192, 16384, 32768, 65536};
  printf("S_KB NST ctas_per_sm inter smem_KB GB/s\n");
  for (int S : Ss)
    for (int NST : {2, 3, 4, 6, 8, 12})
      for (int cps : {1, 2})
        for (int inter : {0, 1}) {
          const size_t smem = (size_t)NST * S + 2 * NST * 8;
          if (smem * cps > 226 * 1024) continue;
          const int grid = sms * cps;
          const int64_t cpc = (int64_t)(bytes / S / grid);
          if (cpc < 4) continue;
          for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            k_probe<<<grid, 9 * 32, smem>>>(buf, cpc, S, NST, inter, 8, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep == 1)
              printf("%d %d %d %d %zu %.0f\n", S / 1024, NST, cps, inter, smem / 1024,
                     (double)cpc * grid * S / (ms * 1e-3) / 1e9);
          }
        }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
