// extern "C" boundary of include/lsgd_b200.h. Exceptions never cross it: each entry point maps
// Error / ConfigError / TransportError (common.hpp; the reference's common.hpp:16-29) onto 1 / 2 / 3 and keeps the
// message for lsgd_b200_last_error().
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <unistd.h>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/lsgd_b200.h"
#include "engine.hpp"
#include "nvls.hpp"
#include "host.hpp"

using namespace lsgd_b200;

namespace {


template <typename F>
int guarded(F&& f) {
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

constexpr int64_t kIpcBytes = sizeof(cudaIpcMemHandle_t);  // 64
constexpr int64_t kUidBytes = sizeof(ncclUniqueId);         // 128
constexpr int64_t kNvlsOff = kIpcBytes + 2 * kUidBytes;   // group leader: pid, multicast fd, object size
constexpr int64_t kBlobBytes = kNvlsOff + 16;

}  // namespace

struct lsgd_b200_rank;
namespace {
char* leader_block_of(lsgd_b200_rank* r, int leader);
}

struct lsgd_b200_rank {
  std::unique_ptr<RunSpec> spec;
  std::unique_ptr<Rank> rank;
  int id = 0;
  ncclUniqueId slice_uid{}, flat_uid{};
  std::map<int, char*> peer_bases;  // IPC-mapped peer blocks (connect)
  uint64_t nvls_mc = 0;  // group leader: the multicast object created at export (attached at connect)
  size_t nvls_size = 0;
};

namespace {
char* leader_block_of(lsgd_b200_rank* r, int leader) {
  auto it = r->peer_bases.find(leader);
  check<Error>(it != r->peer_bases.end(), "NVLS: leader ", leader, "'s block is not mapped");
  return it->second;
}
}  // namespace

extern "C" {

const char* lsgd_b200_last_error(void) { return last_error_slot().c_str(); }
const char* lsgd_b200_version(void) { return "lsgd_b200 0.1 (sm_100a)"; }

int lsgd_b200_config_init(lsgd_b200_config* c) {
  return guarded([&] {
    check<ConfigError>(c != nullptr, "config_init: null config");
    std::memset(c, 0, sizeof(*c));
    // reference defaults: executors.hpp:203-242, optimizer.hpp:16-33
    c->algorithm = LSGD_B200_SEQUENTIAL;
    c->n_workers = 1;
    c->n_groups = 1;
    c->n_samples = 5000;
    c->n_features = 32;
    c->n_classes = 10;
    c->spread = 10.0;
    c->mode = LSGD_B200_MOMENTUM;
    c->base_lr = 0.1;
    c->momentum = 0.9;
    c->weight_decay = 1e-4;
    c->warmup_epochs = 5.0;
    c->decay_every_epochs = 30;
    c->decay_factor = 0.1;
    c->local_batch = 64;
    c->epochs = 1;
    c->iterations = 0;
    c->seed = 42;
    c->init_scale = 0.05;
    c->collective_timeout_s = 30.0;
    c->shared_minibatch = 1;
    c->dtype = LSGD_B200_FP32;
    c->global_algo = LSGD_B200_GLOBAL_ORDERED;  // push exchange in the reference order (NCCL: opt-in)
    c->gemm = LSGD_B200_GEMM_AUTO;
    c->data_source = LSGD_B200_DATA_DEVICE;
    c->model = LSGD_B200_MODEL_MLP;
  });
}

int lsgd_b200_config_validate(const lsgd_b200_config* c) {
  return guarded([&] { RunSpec(*c).validate(); });
}

int lsgd_b200_device_count(int32_t* out) {
  return guarded([&] {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    *out = n;
  });
}

int lsgd_b200_splitmix(uint64_t seed, int64_t n, uint64_t* out) {
  return guarded([&] {
    SplitMix64 r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.u64();
  });
}

int lsgd_b200_generate_synthetic(uint64_t seed, int64_t n, int32_t d, int32_t c, double spread, double* x,
                                 int32_t* y) {
  return guarded([&] { generate_blobs_parallel(seed, n, d, c, spread, x, y); });
}

int lsgd_b200_init_params(int32_t n_layers, const int32_t* layers, uint64_t seed, double scale, double* w) {
  return guarded([&] {
    check<ConfigError>(n_layers >= 2, "model.layer_sizes must list at least input and output dims");
    Layout L(std::vector<int32_t>(layers, layers + n_layers));
    init_weights(L, seed, scale, w);
  });
}

int64_t lsgd_b200_n_params(int32_t n_layers, const int32_t* layers) {
  if (n_layers < 2 || !layers) return -1;
  return Layout(std::vector<int32_t>(layers, layers + n_layers)).n_params;
}

int lsgd_b200_minibatch_indices(const lsgd_b200_config* c, int64_t t0, int64_t n_steps, int32_t* out) {
  return guarded([&] {
    RunSpec spec(*c);
    check<ConfigError>(spec.global_batch() <= spec.c.n_samples, "global batch exceeds dataset size");
    ShardStream s(spec);
    std::vector<int32_t> row(static_cast<size_t>(spec.global_batch()));
    for (int64_t t = 0; t < t0 + n_steps; ++t) {
      s.next(row.data());
      if (t >= t0) std::memcpy(out + (t - t0) * spec.global_batch(), row.data(), row.size() * sizeof(int32_t));
    }
  });
}

int lsgd_b200_learning_rate(const lsgd_b200_config* c, int64_t t, double* out) {
  return guarded([&] {
    RunSpec spec(*c);
    check<Error>(t >= 0, "learning_rate: epoch_float must be >= 0");
    *out = spec.lr(t);
  });
}

int lsgd_b200_topology(const lsgd_b200_config* c, int32_t* role, int32_t* group, int32_t* device_of_worker) {
  return guarded([&] {
    RunSpec spec(*c);
    const int N = c->n_workers;
    const int G = spec.G();
    check<ConfigError>(N >= 1 && G >= 1 && N % G == 0, "n_groups (", G, ") must divide n_workers (", N, ")");
    const int per = N / G;
    const int world = c->algorithm == LSGD_B200_LSGD ? N + G : N;
    for (int r = 0; r < world; ++r) {
      // executors.cpp:405-413: communicators are ranks N..N+G-1
      if (role) role[r] = r >= N ? 1 : 0;
      if (group) group[r] = r >= N ? r - N : r / per;
    }
    int visible = 0;
    if (cudaGetDeviceCount(&visible) != cudaSuccess) {
      cudaGetLastError();
      visible = 0;
    }
    int ndev = c->n_devices > 0 ? c->n_devices : (visible > 0 ? visible : N);
    ndev = ndev < N ? ndev : N;
    if (device_of_worker)
      for (int i = 0; i < N; ++i) device_of_worker[i] = static_cast<int32_t>(static_cast<int64_t>(i) * ndev / N);
  });
}

int lsgd_b200_run_train(const lsgd_b200_config* c, lsgd_b200_result* out) {
  return guarded([&] {
    RunSpec spec(*c);
    spec.validate();
    TrainOutputs o;
    run_world(spec, c->record_history != 0 || out->history != nullptr, out->worker_finals != nullptr ||
                                                                           out->version_at_compute != nullptr,
              o);
    const int64_t T = spec.iterations();
    if (out->final_params) std::memcpy(out->final_params, o.final_params.data(), o.final_params.size() * 8);
    if (out->loss) std::memcpy(out->loss, o.loss.data(), static_cast<size_t>(T) * 8);
    if (out->lr) std::memcpy(out->lr, o.lr.data(), static_cast<size_t>(T) * 8);
    if (out->history && !o.history.empty()) std::memcpy(out->history, o.history.data(), o.history.size() * 8);
    if (out->worker_finals && !o.worker_finals.empty())
      std::memcpy(out->worker_finals, o.worker_finals.data(), o.worker_finals.size() * 8);
    if (out->version_at_compute && !o.version_at_compute.empty())
      std::memcpy(out->version_at_compute, o.version_at_compute.data(), o.version_at_compute.size() * 8);
    if (out->phase_spans && !o.phase_spans.empty())
      std::memcpy(out->phase_spans, o.phase_spans.data(), o.phase_spans.size() * 8);
    out->total_wall_s = o.total_wall_s;
    out->throughput_sps = o.total_wall_s > 0 && T > 0
                              ? static_cast<double>(T) * static_cast<double>(spec.global_batch()) / o.total_wall_s
                              : 0.0;
    out->gpu_launches = o.launches;
  });
}

// ------------------------------------------------------------------------------------------ rank API
int lsgd_b200_rank_create(const lsgd_b200_config* c, int32_t rank, int32_t device, lsgd_b200_rank** out) {
  return guarded([&] {
    auto h = std::make_unique<lsgd_b200_rank>();
    h->spec = std::make_unique<RunSpec>(*c);
    h->spec->validate();
    check<ConfigError>(rank >= 0 && rank < c->n_workers, "rank ", rank, " out of range");
    h->id = rank;
    h->rank = make_rank(*h->spec, device, {rank}, 0);
    const RunSpec& s = *h->spec;
    if (s.c.model == LSGD_B200_MODEL_MLP) {
      std::vector<double> x(static_cast<size_t>(s.c.n_samples) * s.c.n_features);
      std::vector<int32_t> y(static_cast<size_t>(s.c.n_samples));
      generate_blobs_parallel(s.c.seed, s.c.n_samples, s.c.n_features, s.c.n_classes, s.c.spread, x.data(), y.data());
      h->rank->upload_dataset(x.data(), y.data(), s.c.n_samples);
      Layout L(s.layers);
      std::vector<double> w0(static_cast<size_t>(L.n_params));
      init_weights(L, s.c.seed + 1, s.c.init_scale, w0.data());
      h->rank->set_params(w0.data());
    } else {
      std::vector<double> w0(static_cast<size_t>(s.c.synthetic_params), 0.0);
      SplitMix64 r(s.c.seed + 1);
      for (auto& v : w0) v = r.sym(s.c.init_scale);
      h->rank->set_params(w0.data());
    }
    h->rank->synchronize();
    *out = h.release();
  });
}

int lsgd_b200_rank_upload_dataset(lsgd_b200_rank* r, const double* x, const int32_t* y, int64_t n_samples,
                                  int32_t n_features) {
  return guarded([&] {
    const RunSpec& s = *r->spec;
    check<ConfigError>(s.c.model == LSGD_B200_MODEL_MLP, "upload_dataset: the synthetic-gradient model has no data");
    check<ConfigError>(n_features == s.c.n_features, "upload_dataset: dataset has ", n_features,
                       " features, model.layer_sizes[0] is ", s.c.n_features);
    // the sampler draws from data.n_samples (executors.cpp:73, sampler.cpp:15-43): the config must say the size
    check<ConfigError>(n_samples == s.c.n_samples, "upload_dataset: dataset has ", n_samples,
                       " samples, the config's data.n_samples is ", s.c.n_samples);
    for (int64_t i = 0; i < n_samples; ++i)
      check<ConfigError>(y[i] >= 0 && y[i] < s.c.n_classes, "upload_dataset: label ", y[i], " of sample ", i,
                         " is outside [0, ", s.c.n_classes, ")");
    r->rank->upload_dataset(x, y, n_samples);
  });
}

int lsgd_b200_rank_blob_size(int64_t* out) {
  *out = kBlobBytes;
  return LSGD_B200_OK;
}

int lsgd_b200_rank_export(lsgd_b200_rank* r, void* blob) {
  return guarded([&] {
    char* b = static_cast<char*>(blob);
    std::memset(b, 0, kBlobBytes);
    LSGD_CUDA(cudaSetDevice(r->rank->device()));
    cudaIpcMemHandle_t h;
    LSGD_CUDA(cudaIpcGetMemHandle(&h, r->rank->peer_block(r->id)));
    std::memcpy(b, &h, kIpcBytes);
    const RunSpec& s = *r->spec;
    const int k = s.k();
    if (s.c.algorithm == LSGD_B200_LSGD && s.G() > 1 && s.c.global_algo == LSGD_B200_GLOBAL_NCCL && r->id < k) {
      LSGD_NCCL(ncclGetUniqueId(&r->slice_uid));  // group 0 slot j publishes the id of slice comm j
      std::memcpy(b + kIpcBytes, &r->slice_uid, kUidBytes);
    }
    if (s.c.algorithm == LSGD_B200_CSGD && s.c.csgd_nccl && r->id == 0) {
      LSGD_NCCL(ncclGetUniqueId(&r->flat_uid));
      std::memcpy(b + kIpcBytes + kUidBytes, &r->flat_uid, kUidBytes);
    }
    if (r->rank->nvls_wanted() && r->id % k == 0 && !r->nvls_mc) {  // group leader: the NVLS multicast object
      r->nvls_size = nvls_size(r->rank->nvls_bytes(), k);
      int fd = -1;
      r->nvls_mc = nvls_create(r->nvls_size, k, &fd);
      const int32_t pid = static_cast<int32_t>(getpid());
      const int32_t fd32 = fd;
      const uint64_t sz = r->nvls_size;
      std::memcpy(b + kNvlsOff, &pid, 4);
      std::memcpy(b + kNvlsOff + 4, &fd32, 4);
      std::memcpy(b + kNvlsOff + 8, &sz, 8);
    }
  });
}

int lsgd_b200_rank_connect(lsgd_b200_rank* r, const void* all_blobs) {
  return guarded([&] {
    const char* all = static_cast<const char*>(all_blobs);
    const RunSpec& s = *r->spec;
    const int N = s.N(), G = s.G(), k = s.k();
    LSGD_CUDA(cudaSetDevice(r->rank->device()));
    for (int w = 0; w < N; ++w) {
      if (w == r->id) continue;
      cudaIpcMemHandle_t h;
      std::memcpy(&h, all + w * kBlobBytes, kIpcBytes);
      void* p = nullptr;
      LSGD_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      r->rank->set_peer_base(w, static_cast<char*>(p));
      r->peer_bases[w] = static_cast<char*>(p);
      note_ipc_mapping(r->rank.get(), static_cast<char*>(p));
    }
    ncclComm_t slice = nullptr, flat = nullptr;
    if (s.c.algorithm == LSGD_B200_LSGD && G > 1 && s.c.global_algo == LSGD_B200_GLOBAL_NCCL) {
      const int j = r->id % k, g = r->id / k;
      ncclUniqueId uid;
      std::memcpy(&uid, all + j * kBlobBytes + kIpcBytes, kUidBytes);
      slice = static_cast<ncclComm_t>(nccl_init_rank(G, &uid, g, init_timeout(s.c.collective_timeout_s)));
    }
    if (s.c.algorithm == LSGD_B200_CSGD && s.c.csgd_nccl && N > 1) {
      ncclUniqueId uid;
      std::memcpy(&uid, all + kIpcBytes + kUidBytes, kUidBytes);
      flat = static_cast<ncclComm_t>(nccl_init_rank(N, &uid, r->id, init_timeout(s.c.collective_timeout_s)));
    }
    r->rank->set_nccl(slice, flat);
    if (r->rank->nvls_wanted()) {  // join the group's multicast object (leader's blob: pid, fd, size)
      const int leader = (r->id / k) * k;
      const char* lb = all + leader * kBlobBytes + kNvlsOff;
      int32_t pid = 0, fd = -1;
      uint64_t sz = 0;
      std::memcpy(&pid, lb, 4);
      std::memcpy(&fd, lb + 4, 4);
      std::memcpy(&sz, lb + 8, 8);
      check<Error>(sz > 0, "NVLS: the group leader published no multicast object");
      const uint64_t mc = leader == r->id ? r->nvls_mc : nvls_import(pid, fd);
      char* lblock = leader == r->id ? r->rank->peer_block(r->id) : leader_block_of(r, leader);
      r->rank->nvls_join(mc, static_cast<size_t>(sz), lblock, r->id % k, k, init_timeout(s.c.collective_timeout_s));
    }
    enable_phase_recording(r->rank.get());
  });
}

int lsgd_b200_rank_step(lsgd_b200_rank* r, int64_t n_steps, const int32_t* host_indices) {
  return guarded([&] { r->rank->issue_steps(n_steps, host_indices, host_indices != nullptr); });
}
int lsgd_b200_rank_step_rows(lsgd_b200_rank* r, int64_t n_steps, const void* x, const int32_t* y) {
  return guarded([&] { r->rank->issue_steps_rows(n_steps, x, y); });
}
int lsgd_b200_rank_drain(lsgd_b200_rank* r) {
  return guarded([&] { r->rank->drain(); });
}
int lsgd_b200_rank_synchronize(lsgd_b200_rank* r) {
  return guarded([&] { r->rank->synchronize(); });
}
int lsgd_b200_rank_last_loss(lsgd_b200_rank* r, double* loss) {
  return guarded([&] { *loss = r->rank->last_loss(); });
}
int lsgd_b200_rank_get_params(lsgd_b200_rank* r, double* w, int64_t n) {
  return guarded([&] {
    (void)n;
    r->rank->get_params(r->id, w);
  });
}
int lsgd_b200_rank_set_params(lsgd_b200_rank* r, const double* w, int64_t n) {
  return guarded([&] {
    (void)n;
    r->rank->set_params(w);
  });
}
int lsgd_b200_rank_history(lsgd_b200_rank* r, double* loss, double* lr, int64_t n) {
  return guarded([&] { r->rank->history(loss, lr, n); });
}
int lsgd_b200_rank_launches(lsgd_b200_rank* r, int64_t* out) {
  return guarded([&] { *out = r->rank->launches(); });
}
int lsgd_b200_rank_stream(lsgd_b200_rank* r, void** stream) {
  return guarded([&] { *stream = r->rank->main_stream(); });
}
int lsgd_b200_rank_join(lsgd_b200_rank* r) {
  return guarded([&] { r->rank->join(); });
}
int lsgd_b200_rank_kernel_time(lsgd_b200_rank* r, const char* family, double* avg_ms, int64_t* count) {
  return guarded([&] { r->rank->kernel_time(family, avg_ms, count); });
}
int lsgd_b200_rank_loss_async(lsgd_b200_rank* r, void* host_pinned, int32_t* elem_bytes) {
  return guarded([&] {
    const int n = r->rank->loss_async(host_pinned);
    if (elem_bytes) *elem_bytes = n;
  });
}
int lsgd_b200_test_rank_timeline(lsgd_b200_rank* r, char* buf, int64_t cap) {
  return guarded([&] {
    const std::string t = r->rank->timeline();
    check<Error>(cap > 0, "timeline buffer is empty");
    const size_t n = std::min(t.size(), static_cast<size_t>(cap - 1));
    std::memcpy(buf, t.data(), n);
    buf[n] = '\0';
  });
}
int lsgd_b200_rank_timing(lsgd_b200_rank* r, int32_t enable) {
  return guarded([&] { r->rank->set_timing(enable != 0); });
}
int lsgd_b200_rank_destroy(lsgd_b200_rank* r) {
  return guarded([&] { delete r; });
}

// ------------------------------------------------------------------------------------------ kernel seam
int lsgd_b200_batch_gradient(int32_t n_layers, const int32_t* layers, int32_t dtype, int32_t gemm, const double* w,
                             int64_t n_rows, const double* x, const int32_t* y, const int32_t* idx, int64_t b,
                             double* grad, double* mean_loss) {
  return guarded([&] {
    check<Error>(b >= 1, "batch dimension check: empty batch");
    check<Error>(n_layers >= 2, "model.layer_sizes must list at least input and output dims");
    for (int64_t i = 0; i < b; ++i) {
      check<Error>(idx[i] >= 0 && idx[i] < n_rows, "batch index ", idx[i], " out of range");
      int32_t lab = y[idx[i]];
      check<Error>(lab >= 0 && lab < layers[n_layers - 1], "batch dimension check: label ", lab, " out of range [0, ",
                   layers[n_layers - 1], ")");
    }
    lsgd_b200_config c;
    lsgd_b200_config_init(&c);
    c.algorithm = LSGD_B200_LSGD;
    c.n_layers = n_layers;
    c.layer_sizes = layers;
    c.n_samples = n_rows;
    c.n_features = layers[0];
    c.n_classes = layers[n_layers - 1];
    c.local_batch = static_cast<int32_t>(b);
    c.dtype = dtype;
    c.gemm = gemm;
    c.mode = LSGD_B200_PLAIN;
    c.iterations = 1;
    RunSpec spec(c);
    check<ConfigError>(b <= n_rows, "batch larger than the dataset");
    auto rank = make_rank(spec, 0, {0}, 0);
    rank->upload_dataset(x, y, n_rows);
    rank->set_params(w);
    rank->compute_gradient(idx, grad, mean_loss);
  });
}

}  // extern "C"
