// Tensor-core path of the fp32 step: the dense-layer GEMMs as tcgen05.mma kind::tf32
// with the split-TF32 ("3xTF32") decomposition  a*b ~= a_hi*b_lo + a_lo*b_hi + a_hi*b_hi, where
// a_hi = rna_tf32(a), a_lo = rna_tf32(a - a_hi); the dropped a_lo*b_lo term is ~2^-22 relative, so products are
// fp32-grade (the parity contract needs fp32 accuracy: SURVEY §7 "hard parts" 1, 6). The tensor pipe's fp32
// accumulation does not round to nearest, so K runs in 512-wide chunks whose TMEM partial sums are folded with
// round-to-nearest adds (gemm_tc.cu): 3.6e-6 norm-wise vs float64 at any K instead of growing linearly with K.
// Operands are staged by TMA from hi/lo copies their producers write (the forward/backward epilogues for
// activations and deltas); the weights are split in shared memory by the forward / dX kernels themselves (WS).
// Accumulators live in TMEM.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "host.hpp"
#include "kernels.cuh"

namespace lsgd_b200 {

struct TcLayer;

struct TcWorkspace {
  bool ready = false;
  int batch = 0;
  std::vector<void*> bufs;     // owned device allocations
  float* w_hi = nullptr;       // [P], same layout as w (only weight blocks are written)
  float* w_lo = nullptr;
  float* x_hi = nullptr;       // [B, d]
  float* x_lo = nullptr;
  std::vector<float*> act, act_hi, act_lo;  // [B, out_k] per layer
  // deltas [B, out_k] per layer: dX and dW interleave in either backward order (rank.cu bwd_reverse), so every
  // layer keeps its own delta
  std::vector<float*> dlt, dlt_hi, dlt_lo;
  float* partial = nullptr;    // split-K workspace
  size_t partial_elems = 0;
  std::vector<TcLayer*> layers;
  bool weights_split_in_smem = false;  // the updates need not write w_hi / w_lo
};

// Every layer width a multiple of 256 and the local batch a multiple of 128 (tile 128 x 256, BK = 16).
bool tc_shapes_supported(const std::vector<int32_t>& layers, int batch);
// w_master (the fp32 weights, fixed address): when given (and LSGD_TC_WSPLIT != 0) the forward and input-gradient
// GEMMs read it raw and split it in shared memory, so w_hi / w_lo need not be kept current.
void tc_alloc(TcWorkspace& ws, const Layout& L, int batch, int n_features, const float* w_master = nullptr);
void tc_free(TcWorkspace& ws);
// w -> (w_hi, w_lo) for the whole parameter vector (initial parameters; afterwards the fused update writes it).
void tc_split_weights(TcWorkspace& ws, const Layout& L, const float* w, cudaStream_t st, LaunchCounter& lc);
// Gather of the batch rows (dataset in HBM) straight into (x_hi, x_lo) + labels; d % 4 == 0.
void tc_gather_split(TcWorkspace& ws, const Layout& L, const float* rows, const int32_t* labels, const int32_t* idx,
                     int32_t* y, cudaStream_t st, LaunchCounter& lc);
// Gathered batch x -> (x_hi, x_lo), the operand of the first forward GEMM.
void tc_split_input(TcWorkspace& ws, const Layout& L, const float* x, cudaStream_t st, LaunchCounter& lc);
// Forward layer k: act_k = ReLU?(in . W_k^T + b_k) and its split.
void tc_forward_layer(TcWorkspace& ws, const Layout& L, int k, const float* w, cudaStream_t st, LaunchCounter& lc);
// Softmax-CE head: delta of the top layer (+ split), per-sample losses, mean loss -> *loss_out.
void tc_head(TcWorkspace& ws, const Layout& L, const int32_t* y, float* sample_loss, float* loss_out, cudaStream_t st,
             LaunchCounter& lc);
// Backward layer k: dW_k -> gW ([out x in], /B), db_k -> gb, and (k > 0) the masked delta of layer k-1.
void tc_backward_layer(TcWorkspace& ws, const Layout& L, int k, float* gW, float* gb, cudaStream_t st,
                       LaunchCounter& lc);
// Gradient-bucket scatter (the first hop of the push exchange fused into the producers): bucket-local element e is
// written to dst[e / S] + e % S — sub-slice j straight into its owner's stage (over NVLink), the own one locally.
struct BucketScatter {
  int n = 0;        // owners (k); 0 = plain local write
  int64_t S = 0;    // sub-slice length (elements, multiple of 64)
  int64_t e0 = 0;   // bucket-local index of the first element this producer writes
  float* dst[kMaxPeers] = {};
};
// SGD / momentum update fused into the gradient producers (one worker, one group: the gradient is final as soon as
// it is produced): the epilogue applies the K8 arithmetic of update_kernel (pre_delta, sgd_one with FMAs, finite
// check, TF32 split of the new weights) to the bucket's parameters instead of storing the gradient. Pointers are
// the bucket's first parameter; loss_in -> loss_out copies the (folded) loss slot.
struct FusedUpdate {
  float* w = nullptr;
  float* v = nullptr;
  float* hi = nullptr;
  float* lo = nullptr;
  float lr = 0.f, momentum = 0.f, weight_decay = 0.f, post_div = 0.f;
  int mode = 0, add_zero = 0;
  unsigned* bad = nullptr;
  const float* loss_in = nullptr;
  float* loss_out = nullptr;
};
// The same in pieces: rows [row0, row0+rows) of dW_k -> gW (row stride in_k), then db_k, then dX_k.
void tc_backward_dw(TcWorkspace& ws, const Layout& L, int k, int row0, int rows, float* gW, cudaStream_t st,
                    LaunchCounter& lc, const BucketScatter* scat = nullptr, const FusedUpdate* upd = nullptr);
void tc_backward_bias(TcWorkspace& ws, const Layout& L, int k, float* gb, cudaStream_t st, LaunchCounter& lc,
                      const BucketScatter* scat = nullptr, const FusedUpdate* upd = nullptr);
void tc_backward_dx(TcWorkspace& ws, const Layout& L, int k, cudaStream_t st, LaunchCounter& lc);

// Standalone GEMM for conformance tests: D = A * B^T with A [M x K], B [N x K] given in their storage major
// (K-major: [rows][K]; MN-major: [K][rows]), epilogue 0 forward (bias, relu), 1 weight-grad (/div), 2 input-grad
// (mask). Host buffers.
void tc_test_gemm(int a_mn, int b_mn, int epi, int M, int N, int K, int reps, const float* A, const float* B,
                  const float* bias, const float* mask, float div, int relu, float* out, double* avg_ms = nullptr);

}  // namespace lsgd_b200

namespace lsgd_b200 {
void tc_debug_step(const std::vector<int32_t>& layers, int batch, const float* w_host, const float* x_host,
                   const int32_t* y_host, float* act_out, float* delta_out, float* grad_out, float* loss_out);
}
