// Exchange-kernel probe (testing surface, lsgd_b200_testing.h): runs ONE production exchange kernel of the LSGD step
// (K6 reduce_push, member->owner scatter, K7+K8 global_update, K8 update, or a copy-engine peer copy for
// comparison) from device 0 against buffers on devices 1..n_dev-1 over NVLink, with no flags and no other work, so
// a profiler can replay it in isolation (ncu serialises kernels, which would deadlock the live cross-GPU flag
// protocol) and read its NVLink (nvltx/nvlrx) and DRAM counters. Same kernels, same launch grids as the step.
#include <cuda_runtime.h>

#include <vector>

#include "../../include/lsgd_b200.h"
#include "../../include/lsgd_b200_testing.h"
#include "common.hpp"
#include "kernels.cuh"
#include "nvls.hpp"

using namespace lsgd_b200;

namespace {

struct Bufs {
  std::vector<std::pair<int, void*>> all;
  float* alloc(int dev, int64_t n) {
    LSGD_CUDA(cudaSetDevice(dev));
    void* p = nullptr;
    LSGD_CUDA(cudaMalloc(&p, sizeof(float) * n));
    LSGD_CUDA(cudaMemset(p, 0, sizeof(float) * n));
    all.emplace_back(dev, p);
    return static_cast<float*>(p);
  }
  ~Bufs() {
    for (auto& d : all) {
      cudaSetDevice(d.first);
      cudaFree(d.second);
    }
  }
};

__global__ void fill_kernel(float* p, int64_t n, float base) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = base + 1e-3f * static_cast<float>(i % 977);
}

}  // namespace

extern "C" int lsgd_b200_test_exchange_kernel(int32_t kind, int32_t n_dev, int32_t k, int64_t len, int32_t reps,
                                              double* avg_ms, double* bytes_nvlink, double* bytes_local) {
  try {
    int ndev = 0;
    LSGD_CUDA(cudaGetDeviceCount(&ndev));
    check<ConfigError>(n_dev >= 2 && n_dev <= ndev && n_dev <= kMaxPeers, "exchange probe needs 2..", ndev,
                       " devices");
    check<ConfigError>(k >= 1 && k <= kMaxPeers && len > 0 && reps >= 1, "exchange probe: bad k / len / reps");
    for (int d = 1; d < n_dev; ++d) {
      LSGD_CUDA(cudaSetDevice(0));
      cudaError_t e = cudaDeviceEnablePeerAccess(d, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else LSGD_CUDA(e);
    }
    Bufs b;
    const int R = n_dev - 1;  // remote destinations
    std::vector<float*> src, remote;
    for (int m = 0; m < std::max(k, 2); ++m) src.push_back(b.alloc(0, len));
    for (int d = 1; d < n_dev; ++d) remote.push_back(b.alloc(d, len));
    float* local = b.alloc(0, len);
    float* w = b.alloc(0, len);
    float* v = b.alloc(0, len);
    unsigned* bad = nullptr;
    LSGD_CUDA(cudaSetDevice(0));
    LSGD_CUDA(cudaMalloc(&bad, sizeof(unsigned)));
    for (size_t m = 0; m < src.size(); ++m) fill_kernel<<<592, 256>>>(src[m], len, 0.1f * static_cast<float>(m + 1));
    fill_kernel<<<592, 256>>>(w, len, 0.5f);
    std::vector<NvlsBuffer> mcb;
    uint64_t mc = 0;
    float* mc_ptr = nullptr;
    if (kind == 5) {  // one multicast object over n_dev devices, each binding len floats
      const size_t size = nvls_size(sizeof(float) * static_cast<size_t>(len), n_dev);
      mc = nvls_create(size, n_dev, nullptr);
      for (int d = 0; d < n_dev; ++d) nvls_add_device(mc, d);
      mcb.resize(static_cast<size_t>(n_dev));
      for (int d = 0; d < n_dev; ++d) {
        nvls_bind_map(mcb[static_cast<size_t>(d)], mc, size, d);
        mcb[static_cast<size_t>(d)].own_mc = false;
      }
      mc_ptr = reinterpret_cast<float*>(mcb[0].mc_va);
      LSGD_CUDA(cudaSetDevice(0));
    }
    cudaStream_t st;
    LSGD_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    LaunchCounter lc;
    double nv = 0, loc = 0;
    auto launch = [&] {
      switch (kind) {
        case 0: {  // K6: ordered sum of k local member sub-slices (+0.0, /N) pushed to 1 local + R remote owners
          SrcList<float> s{};
          for (int m = 0; m < k; ++m) s.p[m] = src[static_cast<size_t>(m)];
          DstList<float> d{};
          d.p[0] = local;
          for (int r = 0; r < R; ++r) d.p[1 + r] = remote[static_cast<size_t>(r)];
          launch_reduce_push<float>(s, k, len, d, 1 + R, true, 4.0f, st, lc);
          nv = 4.0 * len * R;
          loc = 4.0 * len * (k + 1);
          break;
        }
        case 1: {  // member -> owner scatter with SM stores: R pairs, local sub-slice -> remote stage
          SrcList<float> s{};
          DstList<float> d{};
          for (int r = 0; r < R; ++r) {
            s.p[r] = src[static_cast<size_t>(r % src.size())];
            d.p[r] = remote[static_cast<size_t>(r)];
          }
          launch_copy_pairs<float>(s, d, R, len, st, lc);
          nv = 4.0 * len * R;
          loc = 4.0 * len * R;
          break;
        }
        case 2: {  // K7 + broadcast + K8 of the owner's slot: k member sums, G = 2 group sums, update w / v, push the
                   // average to R members
          GlobalUpdateArgs<float> a;
          for (int m = 0; m < k; ++m) a.src.p[m] = src[static_cast<size_t>(m)];
          a.k = k;
          a.gsum.p[0] = nullptr;
          a.gsum.p[1] = src[1];
          a.G = 2;
          a.g = 0;
          a.add_zero = true;
          a.divisor = 4.0f;
          a.len = len;
          for (int r = 0; r < R; ++r) a.push.p[r] = remote[static_cast<size_t>(r)];
          a.n_push = R;
          a.first = 0;
          a.n_params = len;
          a.w = w;
          a.v = v;
          a.mode = 1;
          a.lr = 1e-3f;
          a.momentum = 0.9f;
          a.weight_decay = 1e-4f;
          a.bad = bad;
          launch_global_update<float>(a, false, st, lc);
          nv = 4.0 * len * R;
          loc = 4.0 * len * (k + 1 + 4);  // k sub-slices + 1 group sum read; w, v read + written
          break;
        }
        case 3: {  // K8 on the other slots: average (local gfull) -> momentum update of w / v
          UpdateArgs<float> a{};
          a.slices.p[0] = src[0];
          a.slice_len = len;
          a.n_params = len;
          a.w = w;
          a.v = v;
          a.mode = 1;
          a.lr = 1e-3f;
          a.momentum = 0.9f;
          a.weight_decay = 1e-4f;
          a.bad = bad;
          launch_update<float>(a, false, st, lc);
          nv = 0;
          loc = 20.0 * len;
          break;
        }
        case 5: {  // kind 2 with the NVLS fan-out: one multimem.st per vector into the n_dev members' buffers
          GlobalUpdateArgs<float> a;
          for (int m = 0; m < k; ++m) a.src.p[m] = src[static_cast<size_t>(m)];
          a.k = k;
          a.gsum.p[1] = src[1];
          a.G = 2;
          a.g = 0;
          a.add_zero = true;
          a.divisor = 4.0f;
          a.len = len;
          a.mc = mc_ptr;
          a.n_params = len;
          a.w = w;
          a.v = v;
          a.mode = 1;
          a.lr = 1e-3f;
          a.momentum = 0.9f;
          a.weight_decay = 1e-4f;
          a.bad = bad;
          launch_global_update<float>(a, false, st, lc);
          nv = 4.0 * len;  // one copy leaves this GPU; the switch replicates it to the n_dev members
          loc = 4.0 * len * (k + 1 + 4);
          break;
        }
        case 4: {  // copy-engine peer copies (the LSGD_B200_DMA path): R concurrent copies local -> remote
          for (int r = 0; r < R; ++r)
            LSGD_CUDA(cudaMemcpyAsync(remote[static_cast<size_t>(r)], src[static_cast<size_t>(r % src.size())],
                                      sizeof(float) * len, cudaMemcpyDeviceToDevice, st));
          nv = 4.0 * len * R;
          loc = 4.0 * len * R;
          break;
        }
        default:
          throw ConfigError(cat("exchange probe: unknown kind ", kind));
      }
    };
    launch();  // warm-up (and the single launch a profiler replays)
    LSGD_CUDA(cudaStreamSynchronize(st));
    cudaEvent_t e0, e1;
    LSGD_CUDA(cudaEventCreate(&e0));
    LSGD_CUDA(cudaEventCreate(&e1));
    LSGD_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < reps; ++i) launch();
    LSGD_CUDA(cudaEventRecord(e1, st));
    LSGD_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    LSGD_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (avg_ms) *avg_ms = ms / reps;
    if (bytes_nvlink) *bytes_nvlink = nv;
    if (bytes_local) *bytes_local = loc;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(st);
    cudaFree(bad);
    for (auto& b : mcb) nvls_free(b);
    if (mc) nvls_release(mc);
    LSGD_CUDA(cudaSetDevice(0));
    return LSGD_B200_OK;
  } catch (const ConfigError& e) {
    last_error_slot() = e.what();
    return LSGD_B200_ERR_CONFIG;
  } catch (const std::exception& e) {
    last_error_slot() = e.what();
    return LSGD_B200_ERR_RUNTIME;
  }
}

// The flag-protocol check of wait_flags_kernel on one device: a flag holding `value`, waited for `target` with
// `max_lead`; *code = 0 (passed), 2 (protocol violation reported), 1 (timed out after 50 ms).
extern "C" int lsgd_b200_test_wait_flag(uint64_t value, uint64_t target, uint64_t max_lead, int32_t* code) {
  try {
    LSGD_CUDA(cudaSetDevice(0));
    unsigned long long* f = nullptr;
    LSGD_CUDA(cudaMalloc(&f, sizeof(unsigned long long)));
    LSGD_CUDA(cudaMemcpy(f, &value, sizeof(value), cudaMemcpyHostToDevice));
    int* h = nullptr;
    LSGD_CUDA(cudaHostAlloc(&h, sizeof(int), cudaHostAllocMapped));
    *h = 0;
    int* d = nullptr;
    LSGD_CUDA(cudaHostGetDevicePointer(&d, h, 0));
    FlagList fl{};
    fl.f[0] = f;
    LaunchCounter lc;
    launch_wait_flags(fl, 1, target, 50000000ull, d, 0, lc, max_lead);
    LSGD_CUDA(cudaDeviceSynchronize());
    *code = *h;
    cudaFreeHost(h);
    cudaFree(f);
    return LSGD_B200_OK;
  } catch (const std::exception& e) {
    last_error_slot() = e.what();
    return LSGD_B200_ERR_RUNTIME;
  }
}
