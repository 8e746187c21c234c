// Shared device helpers for the sm_100a product kernels: mbarrier / bulk-copy
// (TMA engine) / cp.async / PDL PTX wrappers and warp reductions.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace poly {

constexpr int kMaxW = 64;  // spectral bins supported by the kernels

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

#ifndef POLY_MBAR_SUSPEND_NS
#define POLY_MBAR_SUSPEND_NS 0  // > 0: try_wait suspend-time hint (a waiting warp sleeps instead of re-polling)
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
#if POLY_MBAR_SUSPEND_NS > 0
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity), "n"(POLY_MBAR_SUSPEND_NS)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#endif
}

// ------------------------------------------------------- bulk async copies
// 1D bulk copy global -> shared through the TMA engine, completing as
// transaction bytes on `bar`; L2 evict-first policy (A is streamed once).
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void bulk_g2s(void *smem_dst, const void *gmem_src, uint32_t bytes,
                                         uint64_t *bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Per-thread async copies (LDGSTS) whose completion arrives on an mbarrier.
__device__ __forceinline__ void cp_async4(void *smem_dst, const void *gmem_src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem_dst)),
               "l"(gmem_src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void *smem_dst, const void *gmem_src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem_dst)),
               "l"(gmem_src)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gmem_src)
               : "memory");
}
// arrive on `bar` once all prior cp.async of this thread completed (.noinc:
// the arrival is counted in the barrier's initial count).
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// --------------------------------------------- programmatic dependent launch
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Data written by the kernel that precedes this one in a programmatic-launch
// chain is read past L1 (ld.global.cg): this grid may have started while the
// writer was still running, so a const __restrict__ load (ld.global.nc) would
// break that path's "read-only for the kernel's lifetime" contract.
#ifndef POLY_HARDEN_LD
#define POLY_HARDEN_LD 1
#endif
template <typename T>
__device__ __forceinline__ T ld_prev(const T *p) {
#if POLY_HARDEN_LD
  return __ldcg(p);
#else
  return *p;
#endif
}
// (optional, off) fence.proxy.async after griddepcontrol.wait and before a bulk
// copy of data the previous grid wrote with ordinary stores: griddepcontrol.wait
// already makes the prerequisite grid's global writes visible to this grid, and
// the bulk copy reads global memory at L2; measured: +1.2 us per C4 pass, no
// effect on results
#ifndef POLY_PDL_PROXY_FENCE
#define POLY_PDL_PROXY_FENCE 0
#endif
__device__ __forceinline__ void pdl_proxy_fence() {
#if POLY_PDL_PROXY_FENCE
  asm volatile("fence.proxy.async;" ::: "memory");
#endif
}

// ------------------------------------------------------------ named barrier
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// exp(x) for x <= 0 in fp64: Cody-Waite reduction x = k ln2 + r, |r| <= ln2/2,
// Taylor polynomial of degree DEG, scale by 2^k.  Branch-free: x is clamped at
// -708 (exp(-708) ~ 3e-308, below any count the link can resolve).  Truncation
// r^(DEG+1)/(DEG+1)! relative: DEG 13 -> 5e-18 (fp64 path), DEG 9 -> 7e-12
// (fp32 path, whose budget is 1e-4).  Compact replacement for libm exp.
__host__ __device__ constexpr double inv_factorial(int n) {
  double f = 1.0;
  for (int i = 2; i <= n; ++i) f *= (double)i;
  return 1.0 / f;
}

// DEG = 0: the fraction 2^f, |f| <= 1/2, by the SFU (ex2.approx.ftz.f32) on a
// fp64 Cody-Waite reduction: relative error ~3e-7 (the fp32-A link's option
// POLY_K1_MUFU_EXP; x >= -87 keeps 2^f·2^k inside the fp32 SFU's range).
__device__ __forceinline__ double exp_nonpos_sfu(double x) {
  x = fmax(x, -87.0);
  const double k = rint(x * 1.4426950408889634);
  double r = fma(-k, 6.93147180369123816490e-01, x);
  r = fma(-k, 1.90821492927058770002e-10, r);
  float e2;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e2) : "f"((float)(r * 1.4426950408889634)));
  return (double)e2 * __longlong_as_double((long long)(1023 + (int)k) << 52);
}

#ifndef POLY_EXP_CONST
#define POLY_EXP_CONST 0   // 1: the polynomial's constants as constant-bank operands of the DFMAs (measured slower)
#endif
// 1/i! (i = 0..15), then log2 e and the two parts of ln 2: as 64-bit immediates each constant costs two
// UMOVs per use (24 of the 48 instructions of one evaluation); from the constant bank they are operands
__device__ __constant__ double kExpTab[19] = {
    inv_factorial(0),  inv_factorial(1),  inv_factorial(2),  inv_factorial(3),  inv_factorial(4),  inv_factorial(5),
    inv_factorial(6),  inv_factorial(7),  inv_factorial(8),  inv_factorial(9),  inv_factorial(10), inv_factorial(11),
    inv_factorial(12), inv_factorial(13), inv_factorial(14), inv_factorial(15), 1.4426950408889634,
    6.93147180369123816490e-01, 1.90821492927058770002e-10};

template <int DEG = 13>
__device__ __forceinline__ double exp_nonpos(double x) {
  if (DEG == 0) return exp_nonpos_sfu(x);
  static_assert(DEG <= 15, "table");
  x = fmax(x, -708.0);
#if POLY_EXP_CONST
  const double k = rint(x * kExpTab[16]);
  double r = fma(-k, kExpTab[17], x);
  r = fma(-k, kExpTab[18], r);
  double p = kExpTab[DEG];
#pragma unroll
  for (int i = DEG - 1; i >= 0; --i) p = fma(p, r, kExpTab[i]);
#else
  const double k = rint(x * 1.4426950408889634);
  double r = fma(-k, 6.93147180369123816490e-01, x);
  r = fma(-k, 1.90821492927058770002e-10, r);
  // Horner on the Taylor coefficients 1/i!, i = DEG .. 0
  double p = inv_factorial(DEG);
#pragma unroll
  for (int i = DEG - 1; i >= 0; --i) p = fma(p, r, inv_factorial(i));
#endif
  return p * __longlong_as_double((long long)(1023 + (int)k) << 52);
}

// --------------------------------------------------------- warp reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace poly
