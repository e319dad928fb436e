// Test infrastructure, NOT product code.
//
// C-ABI harness around the UNMODIFIED reference library (/root/reference/proj/src/*.cpp), compiled by
// oracle/Makefile into oracle/_ref/liblsgd_ref.so. It exists for two purposes only:
//   1. generate golden vectors (tests/golden/make_golden.py) that pin oracle/lsgd_oracle.c and the
//      CUDA path to the reference's own numbers;
//   2. the CPU baseline leg of bench.py (`--impl reference`), which times the reference's own
//      run_train (proj/src/executors.cpp:481-521) on the host cores.
// Nothing under paper_1906_05936_b200/ links or loads this file.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "lsgd/common.hpp"
#include "lsgd/dataset.hpp"
#include "lsgd/executors.hpp"
#include "lsgd/mlp.hpp"
#include "lsgd/optimizer.hpp"
#include "lsgd/rng.hpp"
#include "lsgd/sampler.hpp"
#include "lsgd/transport.hpp"
#include "lsgd/inprocess.hpp"

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const lsgd::ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // namespace

extern "C" {

// Flat mirror of lsgd::TrainConfig (executors.hpp:218-242).
struct lsgd_ref_config {
  int algorithm;  // 0 sequential, 1 csgd, 2 lsgd (executors.hpp:180)
  int n_workers;
  int n_groups;
  int n_layers;
  const int* layer_sizes;
  int64_t n_samples;
  int n_features;
  int n_classes;
  double spread;
  int mode;  // 0 plain, 1 momentum (optimizer.hpp:14)
  double base_lr, momentum, weight_decay, warmup_epochs;
  int decay_every_epochs;
  double decay_factor;
  int local_batch;
  int epochs;
  int64_t iterations;
  uint64_t seed;
  double init_scale;
  double io_delay_s, global_link_delay_s;
  int shared_minibatch;
};

// Caller-owned output buffers; any pointer may be null.
struct lsgd_ref_result {
  double* final_params;      // [P]            worker 0
  double* loss;              // [T]
  double* lr;                // [T]
  double* history;           // [(T+1) * P]    w_0..w_T (forces record_history)
  double* worker_finals;     // [N * P]        every worker's final parameters
  int64_t* version_at_compute;  // [N * T]     per worker
  double* phase_spans;       // [world * T * 6 * 2] (begin,end) per rank/iteration/phase
  double total_wall_s;
  double throughput_sps;
};

const char* lsgd_ref_last_error(void) { return g_err.c_str(); }

static lsgd::TrainConfig to_train_config(const lsgd_ref_config* c) {
  lsgd::TrainConfig t;
  t.algorithm = static_cast<lsgd::Algorithm>(c->algorithm);
  t.topology.n_workers = c->n_workers;
  t.topology.n_groups = c->n_groups;
  t.model.layer_sizes.assign(c->layer_sizes, c->layer_sizes + c->n_layers);
  t.data.n_samples = c->n_samples;
  t.data.n_features = c->n_features;
  t.data.n_classes = c->n_classes;
  t.data.spread = c->spread;
  t.optim.mode = c->mode == 0 ? lsgd::UpdateMode::plain : lsgd::UpdateMode::momentum;
  t.optim.base_lr = c->base_lr;
  t.optim.momentum = c->momentum;
  t.optim.weight_decay = c->weight_decay;
  t.optim.warmup_epochs = c->warmup_epochs;
  t.optim.decay_every_epochs = c->decay_every_epochs;
  t.optim.decay_factor = c->decay_factor;
  t.local_batch = c->local_batch;
  t.epochs = c->epochs;
  t.iterations = c->iterations;
  t.seed = c->seed;
  t.init_scale = c->init_scale;
  t.delays.io_delay_s = c->io_delay_s;
  t.delays.global_link_delay_s = c->global_link_delay_s;
  t.shared_minibatch = c->shared_minibatch != 0;
  return t;
}

int lsgd_ref_run_train(const lsgd_ref_config* c, lsgd_ref_result* r) {
  return guarded([&] {
    lsgd::TrainConfig t = to_train_config(c);
    t.record_history = r->history != nullptr;
    lsgd::TrainResult res = lsgd::run_train(t);
    size_t P = res.final_params.size();
    if (r->final_params) std::memcpy(r->final_params, res.final_params.data(), P * sizeof(double));
    if (r->loss) std::memcpy(r->loss, res.loss_history.data(), res.loss_history.size() * sizeof(double));
    if (r->lr) {
      for (size_t i = 0; i < res.rows.size(); ++i) r->lr[i] = res.rows[i].lr;
    }
    if (r->history) {
      for (size_t i = 0; i < res.param_history.size(); ++i)
        std::memcpy(r->history + i * P, res.param_history[i].data(), P * sizeof(double));
    }
    int n_workers = t.topology.n_workers;
    for (const lsgd::RankResult& rr : res.ranks) {
      if (rr.role != lsgd::Role::worker) continue;
      if (r->worker_finals)
        std::memcpy(r->worker_finals + static_cast<size_t>(rr.rank) * P, rr.final_params.data(),
                    P * sizeof(double));
      if (r->version_at_compute) {
        for (size_t i = 0; i < rr.iterations.size(); ++i)
          r->version_at_compute[static_cast<size_t>(rr.rank) * rr.iterations.size() + i] =
              rr.iterations[i].version_at_compute;
      }
    }
    (void)n_workers;
    if (r->phase_spans) {
      size_t w = 0;
      for (const lsgd::RankResult& rr : res.ranks) {
        for (size_t i = 0; i < rr.iterations.size(); ++i) {
          for (int p = 0; p < lsgd::kNumPhases; ++p) {
            const lsgd::PhaseSpan& s = rr.iterations[i].phase[static_cast<size_t>(p)];
            size_t at = ((w * rr.iterations.size() + i) * lsgd::kNumPhases + static_cast<size_t>(p)) * 2;
            r->phase_spans[at] = s.begin;
            r->phase_spans[at + 1] = s.end;
          }
        }
        ++w;
      }
    }
    r->total_wall_s = res.total_wall_s;
    r->throughput_sps = res.throughput_sps;
  });
}

// rng.hpp:14-19 — raw SplitMix64 stream.
void lsgd_ref_splitmix(uint64_t seed, int64_t n, uint64_t* out) {
  lsgd::Rng rng(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = rng.next_u64();
}

// dataset.cpp:32-70.
int lsgd_ref_generate_synthetic(uint64_t seed, int64_t n, int d, int c, double spread, double* x,
                                int32_t* y) {
  return guarded([&] {
    lsgd::Dataset data = lsgd::generate_synthetic(seed, n, d, c, spread);
    std::memcpy(x, data.features.data(), data.features.size() * sizeof(double));
    std::memcpy(y, data.labels.data(), data.labels.size() * sizeof(int32_t));
  });
}

// sampler.cpp:15-43 + partition 45-57: `n_draws` global batches of `size`, concatenated.
int lsgd_ref_sampler(int64_t n, uint64_t seed, int64_t size, int64_t n_draws, int with_replacement,
                     int32_t* out, int64_t* epochs_started) {
  return guarded([&] {
    lsgd::MinibatchSampler s(n, lsgd::Rng(seed), with_replacement != 0);
    for (int64_t k = 0; k < n_draws; ++k) {
      lsgd::Minibatch m = s.draw(size);
      std::memcpy(out + k * size, m.indices.data(), static_cast<size_t>(size) * sizeof(int32_t));
    }
    if (epochs_started) *epochs_started = s.epochs_started();
  });
}

int lsgd_ref_partition(const int32_t* idx, int64_t size, int n_workers, int32_t* out) {
  return guarded([&] {
    lsgd::Minibatch m;
    m.indices.assign(idx, idx + size);
    std::vector<lsgd::Shard> shards = lsgd::partition_minibatch(m, n_workers);
    int64_t at = 0;
    for (const lsgd::Shard& s : shards) {
      std::memcpy(out + at, s.indices.data(), s.indices.size() * sizeof(int32_t));
      at += static_cast<int64_t>(s.indices.size());
    }
  });
}

// mlp.cpp:174-186.
int lsgd_ref_init_params(int n_layers, const int* layers, uint64_t seed, double scale, double* w) {
  return guarded([&] {
    lsgd::MlpModel m;
    m.layer_sizes.assign(layers, layers + n_layers);
    lsgd::ParamVector v = lsgd::init_params(m, lsgd::Rng(seed), scale);
    std::memcpy(w, v.data(), v.size() * sizeof(double));
  });
}

// mlp.cpp:238-273 (serial=1 selects batch_gradient_serial :217-236).
int lsgd_ref_batch_gradient(int n_layers, const int* layers, const double* w, int64_t n_rows,
                            const double* x, const int32_t* y, const int32_t* idx, int64_t b, int serial,
                            double* grad, double* mean_loss) {
  return guarded([&] {
    lsgd::MlpModel m;
    m.layer_sizes.assign(layers, layers + n_layers);
    lsgd::Dataset d;
    d.n_samples = n_rows;
    d.n_features = layers[0];
    d.n_classes = layers[n_layers - 1];
    d.features.assign(x, x + n_rows * layers[0]);
    d.labels.assign(y, y + n_rows);
    lsgd::ParamVector wv(w, w + m.n_params());
    std::span<const int32_t> view(idx, static_cast<size_t>(b));
    lsgd::BatchGrad bg = serial ? lsgd::batch_gradient_serial(m, wv, lsgd::BatchView{&d, view})
                                : lsgd::batch_gradient(m, wv, lsgd::BatchView{&d, view});
    std::memcpy(grad, bg.grad.data(), bg.grad.size() * sizeof(double));
    *mean_loss = bg.mean_loss;
  });
}

// optimizer.cpp:8-22.
int lsgd_ref_learning_rate(double base_lr, double warmup_epochs, int decay_every, double decay_factor,
                           int n_workers, int local_batch, double epoch, double* out) {
  return guarded([&] {
    lsgd::HyperParams hp;
    hp.base_lr = base_lr;
    hp.warmup_epochs = warmup_epochs;
    hp.decay_every_epochs = decay_every;
    hp.decay_factor = decay_factor;
    *out = lsgd::learning_rate(hp, n_workers, local_batch, epoch);
  });
}

// optimizer.cpp:24-42; `velocity` may be null in plain mode.
int lsgd_ref_sgd_update(int64_t n, double* w, const double* delta, double* velocity, int mode,
                        double momentum, double weight_decay, double lr) {
  return guarded([&] {
    lsgd::HyperParams hp;
    hp.mode = mode == 0 ? lsgd::UpdateMode::plain : lsgd::UpdateMode::momentum;
    hp.momentum = momentum;
    hp.weight_decay = weight_decay;
    lsgd::ParamVector wv(w, w + n);
    lsgd::OptimizerState st;
    if (velocity) st.velocity.assign(velocity, velocity + n);
    lsgd::sgd_update(wv, std::span<const double>(delta, static_cast<size_t>(n)), st, hp, lr);
    std::memcpy(w, wv.data(), static_cast<size_t>(n) * sizeof(double));
    if (velocity && !st.velocity.empty())
      std::memcpy(velocity, st.velocity.data(), static_cast<size_t>(n) * sizeof(double));
  });
}

// Reference collectives (transport.cpp:17-96) over the in-process fabric, one thread per rank.
// contributions: [world * n]; op 0 reduce_to_root, 1 broadcast (root's row), 2 allreduce.
// out: [world * n] (rows of ranks that receive nothing are left untouched).
int lsgd_ref_collective(int op, int world, int root, int64_t n, const double* contributions, double* out) {
  return guarded([&] {
    lsgd::InProcessRouter router(world, 30.0);
    std::vector<int> ids;
    for (int i = 0; i < world; ++i) ids.push_back(i);
    lsgd::CommGroup g = lsgd::CommGroup::of(ids, root);
    std::vector<std::exception_ptr> errs(static_cast<size_t>(world));
    std::vector<std::thread> th;
    for (int r = 0; r < world; ++r) {
      th.emplace_back([&, r] {
        try {
          lsgd::InProcessEndpoint ep = router.endpoint(r);
          std::span<const double> mine(contributions + static_cast<int64_t>(r) * n, static_cast<size_t>(n));
          lsgd::ParamVector res;
          if (op == 0) res = lsgd::reduce_to_root(ep, g, mine);
          else if (op == 1) res = lsgd::broadcast(ep, g, r == root ? mine : std::span<const double>{});
          else res = lsgd::allreduce(ep, g, mine);
          if (!res.empty()) std::memcpy(out + static_cast<int64_t>(r) * n, res.data(), res.size() * sizeof(double));
        } catch (...) {
          errs[static_cast<size_t>(r)] = std::current_exception();
        }
      });
    }
    for (auto& t : th) t.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  });
}

}  // extern "C"
