/*
 * lsgd_b200_testing.h — conformance hooks of liblsgd_b200.so (not part of the reference-facing surface).
 * Used by tests/ to check the tensor-core GEMM against a float64 host product.
 */
#ifndef LSGD_B200_TESTING_H_
#define LSGD_B200_TESTING_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* D = A * B^T on device 0 through the tcgen05 split-TF32 path (gemm_tc.cu). A is M x K stored K-major
 * ([M][K], a_mn = 0) or MN-major ([K][M], a_mn = 1); B likewise N x K. epi: 0 forward (+bias[n], ReLU if relu),
 * 1 weight gradient (/div), 2 input gradient (zero where mask[m*N+n] <= 0). out [M*N]. Shapes must be multiples
 * of 128 (M), 256 (N) and 32 (K). */
int lsgd_b200_test_gemm(int32_t a_mn, int32_t b_mn, int32_t epi, int32_t M, int32_t N, int32_t K, const float* A,
                        const float* B, const float* bias, const float* mask, float div, int32_t relu, float* out);

/* Device time (CUDA events, average over reps launches) of the tensor-core GEMM of that shape and majors. */
int lsgd_b200_test_gemm_timed(int32_t a_mn, int32_t b_mn, int32_t epi, int32_t M, int32_t N, int32_t K, int32_t reps,
                              double* avg_ms);

/* One forward + backward of the tensor-core path on host buffers (w [P], x [batch*layers[0]] fp32, y [batch]),
 * returning the activations of every layer (concatenated), the top delta, the gradient [P] and the mean loss. */
int lsgd_b200_test_tc_step(int32_t n_layers, const int32_t* layers, int32_t batch, const float* w, const float* x,
                           const int32_t* y, float* act, float* delta, float* grad, float* loss);

/* Every launch timed since lsgd_b200_rank_timing(r, 1), one "family<TAB>start_ms<TAB>end_ms" line each (device
 * clock via CUDA events, relative to the timing call), into buf (NUL-terminated, truncated to cap). */
typedef struct lsgd_b200_rank lsgd_b200_rank;
int lsgd_b200_test_rank_timeline(lsgd_b200_rank* r, char* buf, int64_t cap);

/* One production exchange kernel in isolation (no flags, no other work), from device 0 against buffers on devices
 * 1..n_dev-1 over NVLink, so a profiler can replay it: kind 0 = K6 reduce_push (k local sub-slices summed, +0.0, /N,
 * pushed to 1 local + n_dev-1 remote owners), 1 = member->owner scatter with SM stores (n_dev-1 pairs), 2 = K7+K8
 * global_update of the owner's slot (k sub-slices + 1 group sum, momentum update, average pushed to n_dev-1
 * members), 3 = K8 update (local), 4 = copy-engine peer copies (n_dev-1), 5 = kind 2 with the NVLS multicast
 * fan-out (one multimem.st per vector into the n_dev devices' buffers). len = slot elements (fp32). Returns the
 * average device time over reps launches and the algorithmic NVLink / local HBM bytes of one launch. */
int lsgd_b200_test_exchange_kernel(int32_t kind, int32_t n_dev, int32_t k, int64_t len, int32_t reps, double* avg_ms,
                                   double* bytes_nvlink, double* bytes_local);

/* The cross-GPU flag protocol check (wait_flags_kernel) on device 0: one flag holding `value`, waited for `target`
 * with `max_lead`. *code = 0 passed, 2 protocol violation (value > target + max_lead), 1 timed out (50 ms). */
int lsgd_b200_test_wait_flag(uint64_t value, uint64_t target, uint64_t max_lead, int32_t* code);

#ifdef __cplusplus
}
#endif
#endif /* LSGD_B200_TESTING_H_ */
