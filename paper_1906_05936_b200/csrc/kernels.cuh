// Kernel launchers of the LSGD step (K1 gather, K2-K5 MLP, K6 ordered reduce, K7 ordered
// global sum, K8 broadcast-pull + fused SGD/momentum update + finite check) and the cross-GPU flag primitives.
// All launchers are asynchronous on `st` and count their launches in `launches` (the bench's gpu_launches).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.hpp"

namespace lsgd_b200 {


// GEMM epilogues of the SIMT path.
enum GemmEpi : int { kEpiForward = 0, kEpiWeightGrad = 1, kEpiInputGrad = 2 };

struct LaunchCounter {
  int64_t n = 0;
};

// --- K1: gather the shard's rows (device-resident dataset, or pinned host dataset through UVA) -------------
template <typename T>
void launch_gather(const T* rows, const int32_t* labels, const int32_t* idx, int b, int d, T* x_out, int32_t* y_out,
                   cudaStream_t st, LaunchCounter& lc);

// --- K2/K4/K5 SIMT GEMM with sequential-k accumulation:
//     C[m,n] = init(n) + sum_{k=0..K-1} A(m,k) * B(k,n)   (k strictly ascending, one rounding per op when EXACT)
// init = bias[n] (forward) or 0; epilogue: ReLU (forward hidden), / divisor (weight grad), mask (input grad).
template <typename T>
void launch_gemm_simt(int epi, bool exact, int M, int N, int K, const T* A, int64_t lda_m, int64_t lda_k, const T* B,
                      int64_t ldb_k, int64_t ldb_n, T* C, int64_t ldc, const T* bias, int relu, T divisor,
                      const T* mask, cudaStream_t st, LaunchCounter& lc);

// --- K3: softmax cross-entropy head, one sequential pass per sample (mlp.cpp:79-102) -----------------------
template <typename T>
void launch_softmax_xent(const T* logits, const int32_t* labels, int b, int c, T* delta, T* sample_loss,
                         cudaStream_t st, LaunchCounter& lc);
// mean loss in batch order (mlp.cpp:262-271) -> *out
template <typename T>
void launch_mean_loss(const T* sample_loss, int b, T* out, cudaStream_t st, LaunchCounter& lc);
// bias gradient: db[j] = (sum_s delta[s,j]) / b, s ascending
template <typename T>
void launch_bias_grad(const T* delta, int b, int n_out, T* db, cudaStream_t st, LaunchCounter& lc);

// --- K6/K7: ordered sum over peer slices: dst[e] = ((src0[e] + src1[e]) + ... [+ 0.0]) [/ divisor] --------
template <typename T>
struct SrcList {
  const T* p[kMaxPeers];
};
template <typename T>
void launch_ordered_sum(SrcList<T> src, int n_src, int64_t len, T* dst, bool add_zero, T divisor,
                        cudaStream_t st, LaunchCounter& lc);

// --- K8: pull the averaged gradient slices and apply the postponed update (optimizer.cpp:24-42) ------------
// delta[e] = ((slices[e / S][e % S] [+ 0.0]) [/ post_div]): post_div is the CSGD per-worker /N, add_zero + /N the
// single-worker group's communicator arithmetic when the reduce is skipped. Optionally writes the TF32 hi/lo split
// of the updated weights for the tensor-core GEMMs.
template <typename T>
struct UpdateArgs {
  SrcList<T> slices;
  int64_t slice_len;
  int64_t n_params;
  T* w;
  T* v;
  int mode;
  T lr, momentum, weight_decay, post_div;
  int add_zero;
  int scalar_only;    // set by the launcher when a bucket's w/v base is not 16-byte aligned
  T* loss_out;        // receives delta[n_params] (the loss slot), may be null
  unsigned* bad;      // OR-ed 1 when a non-finite parameter is produced
  float* w_hi;        // fp32 only, may be null
  float* w_lo;
  int64_t skip_lo = 0, skip_hi = 0;  // bucket-local elements [skip_lo, skip_hi) are updated elsewhere (own slot)
};
template <typename T>
void launch_update(const UpdateArgs<T>& a, bool exact, cudaStream_t st, LaunchCounter& lc);

// --- broadcast as a push: copy an averaged slice into n destinations (the group members' full-gradient
// buffers, k-1 of them over NVLink) so the update kernel reads local HBM only.
template <typename T>
struct DstList {
  T* p[kMaxPeers];
};
template <typename T>
void launch_push(const T* src, int64_t len, DstList<T> dst, int n_dst, cudaStream_t st, LaunchCounter& lc);

// --- K7 + broadcast + K8 for the owner's own slot, fused: per element of slot j the owner recomputes its group's
// ordered sum (+0.0, /N) from the local member sub-slices, adds the other groups' sums (local gstage) in ascending
// group order, stores the average into the other members' gfull (NVLink) and applies the SGD / momentum update to its
// own parameters of that slot (same arithmetic as update_kernel; the loss slot goes to the loss history). The own
// slot's average never touches HBM.
template <typename T>
struct GlobalUpdateArgs {
  SrcList<T> src;       // k member sub-slices of the slot (local), ascending member order
  int k = 1;
  SrcList<T> gsum;      // [G]: other groups' slot sums (local gstage); own entry unused
  int G = 1, g = 0;
  bool gsum_raw = false; // k = 1: gstage holds the other owners' raw payload (DMA copy), apply (+0.0, /N) here
  bool direct = false;   // src holds all N = k*G sub-slices (group-major); every group's sum is formed here
  T* mc = nullptr;       // NVLS: multicast view of the members' gfull at the slot; one multimem.st per vector
  bool add_zero = false;
  T divisor = T(0);
  int64_t len = 0;      // slot length S
  DstList<T> push;      // the other members' gfull for this slot
  int n_push = 0;
  T* out_local = nullptr;  // also store the average here (the copy engines forward it when pushing by DMA)
  int64_t first = 0;    // bucket-local index of slot element 0
  int64_t n_params = 0; // bucket parameters (index n_params = the loss slot, beyond = padding)
  T* w = nullptr;       // bucket parameter 0
  T* v = nullptr;
  int mode = 0;
  T lr = T(0), momentum = T(0), weight_decay = T(0);
  T* loss_out = nullptr;
  unsigned* bad = nullptr;
  float* w_hi = nullptr;  // fp32 only, may be null: TF32 hi/lo split of the updated weights (bucket parameter 0),
  float* w_lo = nullptr;  // for the GEMMs that read pre-split weights (LSGD_TC_WSPLIT=0)
};
template <typename T>
void launch_global_update(const GlobalUpdateArgs<T>& a, bool exact, cudaStream_t st, LaunchCounter& lc);

// --- push exchange (K6/K7 without remote reads): ordered sum of local sources written to n destinations (local or
// peer), and member -> owner scatter copies (pair p: src_p[0, len) -> dst_p). Grids capped at LSGD_B200_COMM_CTAS.
template <typename T>
void launch_reduce_push(SrcList<T> src, int n_src, int64_t len, DstList<T> dst, int n_dst, bool add_zero, T divisor,
                        cudaStream_t st, LaunchCounter& lc);
template <typename T>
void launch_copy_pairs(SrcList<T> src, DstList<T> dst, int n_pairs, int64_t len, cudaStream_t st, LaunchCounter& lc);

// --- cross-GPU flags: monotone step counters in peer memory -------------------------------------------------
struct SignalList {
  unsigned long long* f[kMaxPeers];
};
// System-scope release store of `value` into n (possibly remote) flags after all prior work of the stream.
void launch_signal_many(SignalList flags, int n, unsigned long long value, cudaStream_t st, LaunchCounter& lc);
struct FlagList {
  const volatile unsigned long long* f[kMaxPeers];
};
// Spin (one CTA) until every flag >= target; on timeout writes 1 to *timed_out (host-mapped) and returns.
// max_lead: a flag above target + max_lead is a protocol violation (code 2 in timed_out); ~0 disables the check.
void launch_wait_flags(FlagList flags, int n, unsigned long long target, unsigned long long timeout_ns,
                       volatile int* timed_out, cudaStream_t st, LaunchCounter& lc,
                       unsigned long long max_lead = ~0ull);
// Version tracking (executors.hpp:102 version_at_compute, measured): `*ver = value` after the prior work of the
// stream, and `*dst = min ver[b0..b1)` (the oldest update any of a layer's buckets has received when its forward
// reads it). One thread each.
void launch_store_u64(unsigned long long* ver, unsigned long long value, cudaStream_t st, LaunchCounter& lc);
void launch_min_u64(const unsigned long long* ver, int b0, int b1, long long* dst, cudaStream_t st, LaunchCounter& lc);
// System-scope release store of `value` after all prior work of the stream.
void launch_signal_flag(unsigned long long* flag, unsigned long long value, cudaStream_t st, LaunchCounter& lc);
// Device-side sleep for the injected io / link delays (executors.hpp:213-216).
void launch_sleep(double seconds, cudaStream_t st, LaunchCounter& lc);

// Convert a host-uploaded float64 buffer into T on device.
template <typename T>
void launch_from_f64(const double* src, int64_t n, T* dst, cudaStream_t st, LaunchCounter& lc);
template <typename T>
void launch_to_f64(const T* src, int64_t n, double* dst, cudaStream_t st, LaunchCounter& lc);

}  // namespace lsgd_b200
