// Transport and optimizer seams of the C-ABI on one device (conformance surface for the reference's
// collective and update tests: test_transport.cpp:135-269, test_optimizer.cpp:64-120). The ranks of the
// collective are emulated as rows on device 0 and summed by the same ordered-sum kernel the step uses (K6/K7).
#include <cuda_runtime.h>

#include <cstring>
#include <string>
#include <vector>

#include "../../include/lsgd_b200.h"
#include "common.hpp"
#include "kernels.cuh"

using namespace lsgd_b200;

namespace {

template <typename F>
int seam_guard(F&& f) {
  try {
    f();
    return LSGD_B200_OK;
  } catch (const ConfigError& e) {
    last_error_slot() = e.what();
    return LSGD_B200_ERR_CONFIG;
  } catch (const TransportError& e) {
    last_error_slot() = e.what();
    return LSGD_B200_ERR_TRANSPORT;
  } catch (const std::exception& e) {
    last_error_slot() = e.what();
    return LSGD_B200_ERR_RUNTIME;
  }
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(size_t n) { LSGD_CUDA(cudaMalloc(&p, sizeof(T) * (n ? n : 1))); }
  ~DevBuf() { cudaFree(p); }
};

template <typename T>
void upload(T* dst, const double* src, int64_t n) {
  std::vector<T> t(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) t[static_cast<size_t>(i)] = static_cast<T>(src[i]);
  LSGD_CUDA(cudaMemcpy(dst, t.data(), sizeof(T) * n, cudaMemcpyHostToDevice));
}
template <typename T>
void download(double* dst, const T* src, int64_t n) {
  std::vector<T> t(static_cast<size_t>(n));
  LSGD_CUDA(cudaMemcpy(t.data(), src, sizeof(T) * n, cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < n; ++i) dst[i] = static_cast<double>(t[static_cast<size_t>(i)]);
}

template <typename T>
void collective_impl(int op, int world, int root, int64_t n, const double* contrib, double* out) {
  check<Error>(world >= 1 && world <= kMaxPeers, "collective: world must be in [1, ", kMaxPeers, "]");
  check<TransportError>(root >= 0 && root < world, "CommGroup: root ", root, " is not a member");
  LSGD_CUDA(cudaSetDevice(0));
  const int64_t ld = (n + 63) / 64 * 64;
  DevBuf<T> rows(static_cast<size_t>(world * ld)), res(static_cast<size_t>(ld));
  LSGD_CUDA(cudaMemset(rows.p, 0, sizeof(T) * world * ld));
  for (int r = 0; r < world; ++r) upload(rows.p + r * ld, contrib + r * n, n);
  LaunchCounter lc;
  if (op == 1) {
    LSGD_CUDA(cudaMemcpy(res.p, rows.p + root * ld, sizeof(T) * ld, cudaMemcpyDeviceToDevice));
  } else {
    SrcList<T> src{};
    for (int r = 0; r < world; ++r) src.p[r] = rows.p + r * ld;  // ascending member id (transport.cpp:92)
    launch_ordered_sum<T>(src, world, ld, res.p, false, T(0), 0, lc);
  }
  LSGD_CUDA(cudaDeviceSynchronize());
  std::vector<double> one(static_cast<size_t>(n));
  download(one.data(), res.p, n);
  for (int r = 0; r < world; ++r) {
    if (op == 0 && r != root) continue;  // non-roots of reduce_to_root receive nothing (transport.hpp:54-56)
    std::memcpy(out + r * n, one.data(), sizeof(double) * n);
  }
}

template <typename T>
void update_impl(int64_t n, double* w, const double* delta, double* v, int mode, double mom, double wd, double lr) {
  check<Error>(lr > 0.0, "sgd_update: lr must be > 0");
  LSGD_CUDA(cudaSetDevice(0));
  const int64_t S = (n + 1 + 63) / 64 * 64;
  DevBuf<T> dw(static_cast<size_t>(n)), dv(static_cast<size_t>(n)), dd(static_cast<size_t>(S));
  LSGD_CUDA(cudaMemset(dd.p, 0, sizeof(T) * S));
  upload(dw.p, w, n);
  upload(dd.p, delta, n);
  if (mode == LSGD_B200_MOMENTUM) {
    if (v) upload(dv.p, v, n);
    else LSGD_CUDA(cudaMemset(dv.p, 0, sizeof(T) * n));
  }
  unsigned* bad = nullptr;
  LSGD_CUDA(cudaMalloc(&bad, sizeof(unsigned)));
  LSGD_CUDA(cudaMemset(bad, 0, sizeof(unsigned)));
  UpdateArgs<T> a{};
  a.slices.p[0] = dd.p;
  a.slice_len = S;
  a.n_params = n;
  a.w = dw.p;
  a.v = mode == LSGD_B200_MOMENTUM ? dv.p : nullptr;
  a.mode = mode;
  a.lr = static_cast<T>(lr);
  a.momentum = static_cast<T>(mom);
  a.weight_decay = static_cast<T>(wd);
  a.bad = bad;
  LaunchCounter lc;
  launch_update<T>(a, sizeof(T) == 8, 0, lc);
  LSGD_CUDA(cudaDeviceSynchronize());
  unsigned hb = 0;
  LSGD_CUDA(cudaMemcpy(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost));
  cudaFree(bad);
  download(w, dw.p, n);
  if (mode == LSGD_B200_MOMENTUM && v) download(v, dv.p, n);
  check<Error>(hb == 0, "non-finite value in parameters after update");
}
}  // namespace

extern "C" {

int lsgd_b200_collective(int32_t op, int32_t dtype, int32_t world, int32_t root, int64_t n, const double* contrib,
                         double* out) {
  int rc = seam_guard([&] {
    check<Error>(op >= 0 && op <= 2, "collective: op must be 0 (reduce), 1 (broadcast) or 2 (allreduce)");
    if (dtype == LSGD_B200_FP64) collective_impl<double>(op, world, root, n, contrib, out);
    else collective_impl<float>(op, world, root, n, contrib, out);
  });
  return rc;
}

int lsgd_b200_sgd_update(int32_t dtype, int64_t n, double* w, const double* delta, double* velocity, int32_t mode,
                         double momentum, double weight_decay, double lr) {
  return seam_guard([&] {
    if (dtype == LSGD_B200_FP64) update_impl<double>(n, w, delta, velocity, mode, momentum, weight_decay, lr);
    else update_impl<float>(n, w, delta, velocity, mode, momentum, weight_decay, lr);
  });
}

}  // extern "C"

#include "../../include/lsgd_b200_testing.h"
#include "gemm_tc.cuh"

extern "C" int lsgd_b200_test_gemm(int32_t a_mn, int32_t b_mn, int32_t epi, int32_t M, int32_t N, int32_t K,
                                   const float* A, const float* B, const float* bias, const float* mask, float div,
                                   int32_t relu, float* out) {
  return seam_guard([&] { tc_test_gemm(a_mn, b_mn, epi, M, N, K, 1, A, B, bias, mask, div, relu, out); });
}

extern "C" int lsgd_b200_test_gemm_timed(int32_t a_mn, int32_t b_mn, int32_t epi, int32_t M, int32_t N, int32_t K,
                                         int32_t reps, double* avg_ms) {
  return seam_guard([&] {
    std::vector<float> A(static_cast<size_t>(M) * K, 0.5f), B(static_cast<size_t>(N) * K, 0.25f),
        bias(static_cast<size_t>(N), 0.f), mask(static_cast<size_t>(M) * N, 1.f), out(static_cast<size_t>(M) * N);
    tc_test_gemm(a_mn, b_mn, epi, M, N, K, reps, A.data(), B.data(), bias.data(), mask.data(), 512.f, 0, out.data(),
                 avg_ms);
  });
}

extern "C" int lsgd_b200_test_tc_step(int32_t n_layers, const int32_t* layers, int32_t batch, const float* w,
                                      const float* x, const int32_t* y, float* act, float* delta, float* grad,
                                      float* loss) {
  return seam_guard([&] {
    tc_debug_step(std::vector<int32_t>(layers, layers + n_layers), batch, w, x, y, act, delta, grad, loss);
  });
}
