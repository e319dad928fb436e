// In-process world (run_train seam, executors.cpp:481-521) and the row-parallel blob generator.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <thread>

#include "engine.hpp"
#include "nvls.hpp"

namespace lsgd_b200 {

// ================================================================================================ blobs
void generate_blobs_parallel(uint64_t seed, int64_t n, int d, int c, double spread, double* x, int32_t* y) {
  // Every row consumes exactly 2*ceil(d/2) draws; SplitMix64's state after m draws is seed + m*gamma, so rows
  // can be produced independently and stay bit-identical to the sequential generator (dataset.cpp:32-70).
  const int64_t per_row = 2 * ((d + 1) / 2);
  std::vector<int32_t> ylab(static_cast<size_t>(c));
  if (n * static_cast<int64_t>(d) < (1 << 22)) {
    generate_blobs(seed, n, d, c, spread, x, y);
    return;
  }
  // centres first (sequential, small), by generating a c-row prefix with the reference routine's stream
  std::vector<double> centre(static_cast<size_t>(c) * d);
  {
    check<ConfigError>(c >= 2 && n >= c && d >= 1 && spread > 0.0, "generate_synthetic: invalid arguments");
    SplitMix64 r(seed);
    for (int cls = 0; cls < c; ++cls) {
      double* mu = &centre[static_cast<size_t>(cls) * d];
      for (int i = 0; i < d; i += 2) {
        double a, b;
        r.normal_pair(a, b);
        mu[i] = a;
        if (i + 1 < d) mu[i + 1] = b;
      }
      double ss = 0.0;
      for (int j = 0; j < d; ++j) ss += mu[j] * mu[j];
      double len = std::sqrt(ss);
      if (len == 0.0) len = 1.0;
      for (int j = 0; j < d; ++j) mu[j] = spread * mu[j] / len;
    }
  }
  const uint64_t gamma = 0x9E3779B97F4A7C15ULL;
  const uint64_t rows_base = seed + static_cast<uint64_t>(c) * static_cast<uint64_t>(per_row) * gamma;
  unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (unsigned q = 0; q < nt; ++q) {
    th.emplace_back([&, q] {
      int64_t lo = n * q / nt, hi = n * (q + 1) / nt;
      SplitMix64 r(rows_base + static_cast<uint64_t>(lo) * static_cast<uint64_t>(per_row) * gamma);
      for (int64_t i = lo; i < hi; ++i) {
        int32_t cls = static_cast<int32_t>(i % c);
        y[i] = cls;
        double* row = x + i * d;
        for (int j = 0; j < d; j += 2) {
          double a, b;
          r.normal_pair(a, b);
          row[j] = a;
          if (j + 1 < d) row[j + 1] = b;
        }
        const double* mu = &centre[static_cast<size_t>(cls) * d];
        for (int j = 0; j < d; ++j) row[j] += mu[j];
      }
    });
  }
  for (auto& t : th) t.join();
}

// ================================================================================================ world
void run_world(const RunSpec& spec, bool want_history, bool want_workers, TrainOutputs& out) {
  spec.validate();
  int visible = 0;
  LSGD_CUDA(cudaGetDeviceCount(&visible));
  check<Error>(visible > 0, "no CUDA device visible: the b200 backend has no CPU fallback");
  const int N = spec.N(), G = spec.G(), k = spec.k();
  int ndev = spec.c.n_devices > 0 ? std::min(spec.c.n_devices, visible) : visible;
  ndev = std::max(1, std::min(ndev, N));
  const int64_t T = spec.iterations();
  const int64_t P = Geometry(spec, 4).P;

  // contiguous worker blocks per device (worker i -> GPU i when ndev == N)
  std::vector<std::vector<int>> blocks(static_cast<size_t>(ndev));
  for (int i = 0; i < N; ++i) blocks[static_cast<size_t>(static_cast<int64_t>(i) * ndev / N)].push_back(i);
  RunSpec rspec = spec;  // outlives the ranks (cleared below)
  rspec.track_versions = want_workers;
  std::vector<std::unique_ptr<Rank>> ranks;
  for (int r = 0; r < ndev; ++r)
    ranks.push_back(make_rank(rspec, r, blocks[static_cast<size_t>(r)], r == 0 && want_history ? T + 1 : 0));

  for (int a = 0; a < ndev; ++a) {
    LSGD_CUDA(cudaSetDevice(a));
    for (int b = 0; b < ndev; ++b) {
      if (a == b) continue;
      int can = 0;
      LSGD_CUDA(cudaDeviceCanAccessPeer(&can, a, b));
      check<TransportError>(can == 1, "GPU ", a, " cannot access GPU ", b, " peer memory (no NVLink/NVSwitch path)");
      cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else LSGD_CUDA(e);
    }
  }
  for (auto& r : ranks)
    for (auto& q : ranks)
      for (int w : q->workers()) r->set_peer_base(w, q->peer_block(w));

  // NCCL only when every rank hosts a single worker (one NCCL rank per device).
  const bool one_each = ndev == N;
  if (one_each && spec.c.algorithm == LSGD_B200_LSGD && G > 1 && spec.c.global_algo == LSGD_B200_GLOBAL_NCCL) {
    for (int j = 0; j < k; ++j) {
      std::vector<int> devs;
      for (int g = 0; g < G; ++g) devs.push_back(g * k + j);
      std::vector<void*> cs = nccl_init_all(devs, init_timeout(spec.c.collective_timeout_s));
      for (int g = 0; g < G; ++g) ranks[static_cast<size_t>(g * k + j)]->set_nccl(cs[static_cast<size_t>(g)], nullptr);
    }
  }
  if (one_each && spec.c.algorithm == LSGD_B200_CSGD && spec.c.csgd_nccl && N > 1) {
    std::vector<int> devs;
    for (int i = 0; i < N; ++i) devs.push_back(i);
    std::vector<void*> cs = nccl_init_all(devs, init_timeout(spec.c.collective_timeout_s));
    for (int i = 0; i < N; ++i) ranks[static_cast<size_t>(i)]->set_nccl(nullptr, cs[static_cast<size_t>(i)]);
  }

  // NVLS multicast fan-out (LSGD_B200_NVLS): one object per group, every member's device added before any binds;
  // the handles stay with this function until the ranks are gone
  std::vector<uint64_t> mcs;
  if (one_each && ranks[0]->nvls_wanted()) {
    for (int g = 0; g < G; ++g) {
      const size_t size = nvls_size(ranks[static_cast<size_t>(g * k)]->nvls_bytes(), k);
      const uint64_t mc = nvls_create(size, k, nullptr);
      mcs.push_back(mc);
      for (int m = 0; m < k; ++m) nvls_add_device(mc, ranks[static_cast<size_t>(g * k + m)]->device());
      for (int m = 0; m < k; ++m) ranks[static_cast<size_t>(g * k + m)]->nvls_attach(mc, size, false);
    }
  }

  // inputs: host-generated with the reference-identical streams, data = seed, init = seed + 1
  if (spec.c.model == LSGD_B200_MODEL_MLP) {
    const int64_t n = spec.c.n_samples;
    const int d = spec.c.n_features;
    std::vector<double> x(static_cast<size_t>(n) * d);
    std::vector<int32_t> y(static_cast<size_t>(n));
    generate_blobs_parallel(spec.c.seed, n, d, spec.c.n_classes, spec.c.spread, x.data(), y.data());
    for (size_t r = 0; r < ranks.size(); ++r) {
      if (r > 0 && spec.c.data_source == LSGD_B200_DATA_HOST) ranks[r]->share_dataset_from(ranks[0].get());
      else ranks[r]->upload_dataset(x.data(), y.data(), n);
    }
  }
  std::vector<double> w0(static_cast<size_t>(P), 0.0);
  if (spec.c.model == LSGD_B200_MODEL_MLP) {
    init_weights(Layout(spec.layers), spec.c.seed + 1, spec.c.init_scale, w0.data());
  } else {
    SplitMix64 r(spec.c.seed + 1);  // synthetic-gradient model: w0 uniform in [-init_scale, init_scale]
    for (auto& v : w0) v = r.sym(spec.c.init_scale);
  }
  for (auto& r : ranks) r->set_params(w0.data());
  for (auto& r : ranks) {
    r->synchronize();
    enable_phase_recording(r.get());
  }

  // one host thread per GPU (executors.cpp:497-515); the first error aborts every rank's flag waits
  std::vector<std::exception_ptr> errors(ranks.size());
  std::atomic<bool> failed{false};
  auto t_start = std::chrono::steady_clock::now();
  std::vector<std::thread> threads;
  for (size_t r = 0; r < ranks.size(); ++r) {
    threads.emplace_back([&, r] {
      try {
        LSGD_CUDA(cudaSetDevice(ranks[r]->device()));
        for (int64_t t = 0; t < T && !failed.load(); ++t) ranks[r]->issue_steps(1, nullptr, false);
        ranks[r]->drain();
      } catch (const std::exception& e) {
        std::string msg = cat("rank ", ranks[r]->workers().front(), " in phase ", current_phase(), ": ", e.what());
        if (dynamic_cast<const TransportError*>(&e)) errors[r] = std::make_exception_ptr(TransportError(msg));
        else if (dynamic_cast<const ConfigError*>(&e)) errors[r] = std::make_exception_ptr(ConfigError(msg));
        else errors[r] = std::make_exception_ptr(Error(msg));
        failed = true;
        for (auto& q : ranks) q->abort();
      }
    });
  }
  for (auto& t : threads) t.join();
  for (auto& e : errors)
    if (e) std::rethrow_exception(e);
  out.total_wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();

  out.final_params.assign(static_cast<size_t>(P), 0.0);
  ranks[0]->get_params(0, out.final_params.data());
  out.loss.assign(static_cast<size_t>(T), 0.0);
  out.lr.assign(static_cast<size_t>(T), 0.0);
  ranks[0]->history(out.loss.data(), out.lr.data(), T);
  if (want_history) {
    out.history.assign(static_cast<size_t>((T + 1) * P), 0.0);
    ranks[0]->param_history(out.history.data(), T + 1);
  }
  if (want_workers) {
    out.worker_finals.assign(static_cast<size_t>(N * P), 0.0);
    out.version_at_compute.assign(static_cast<size_t>(N * T), 0);
    for (auto& r : ranks)
      for (int w : r->workers()) {
        r->get_params(w, out.worker_finals.data() + static_cast<int64_t>(w) * P);
        // measured on the device: the update rounds every layer had received when the forward of t read it
        // (executors.cpp:244 records opt.iteration at the gradient pass)
        r->versions(w, out.version_at_compute.data() + static_cast<int64_t>(w) * T, T);
      }
  }
  if (spec.c.record_phases) {
    out.phase_spans.assign(static_cast<size_t>(N * T * 12), 0.0);
    for (auto& r : ranks)
      for (int w : r->workers()) r->phase_spans(w, out.phase_spans.data() + static_cast<int64_t>(w) * T * 12, T);
  }
  out.launches = 0;
  for (auto& r : ranks) out.launches += r->launches();
  ranks.clear();  // destroys comms too (each rank owns its handles)
  for (uint64_t mc : mcs) nvls_release(mc);
}

}  // namespace lsgd_b200
