/*
 * polysynth.h — CUDA twin of the seeded input generators in gen/rng.py.
 *
 * Not part of the method: these calls only draw random numbers (Philox4x32-10
 * counters, polar-method normals, inversion/PTRS Poisson) so that the large
 * workloads (BASELINE.json configs[1,2,4]: up to 131 GB of A) can be built
 * in HBM.  Every draw is a pure function of (seed, stream id, counter) and is
 * bit-identical to gen/rng.py (tests/test_gpu_synth.py checks sampled rows).
 * The means λ passed to polysynth_poisson come from poly_expected_counts.
 *
 * All pointers are device pointers; work is enqueued on `stream`
 * (cudaStream_t, NULL = default).  Return 0 on success, nonzero on error
 * with a message from polysynth_last_error().
 */
#ifndef POLYSYNTH_H_
#define POLYSYNTH_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* A[r, c] = N(0,1) draw keyed (row0 + r, col0 + c), r < n, c < d; dtype 0:
 * float (fp64 draw rounded to nearest), 1: double.  Row pitch lda >= d
 * elements; padding columns d..lda-1 are set to 0. */
int polysynth_gaussian_matrix(void *A, int32_t dtype, int64_t n, int64_t d, int64_t lda,
                              int64_t row0, int64_t col0, uint32_t seed, uint32_t stream_id,
                              void *stream);

/* y[r] = Poisson(lam[r]) draw keyed row0 + r (int32; lam must be < 2^31). */
int polysynth_poisson(const double *lam, int32_t *y, int64_t n, int64_t row0, uint32_t seed,
                      uint32_t stream_id, void *stream);

/* y[r] = float(k[r] + sigma * N(0,1)), normal keyed (row0 + r, 0). */
int polysynth_add_noise(const int32_t *k, float *y, int64_t n, int64_t row0, double sigma,
                        uint32_t seed, uint32_t stream_id, void *stream);

const char *polysynth_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* POLYSYNTH_H_ */
