#include "host.hpp"

#include <cmath>
#include <numeric>

namespace lsgd_b200 {

std::string& last_error_slot() {
  thread_local std::string msg;
  return msg;
}

const char*& current_phase() {
  thread_local const char* phase = "setup";
  return phase;
}

void SplitMix64::normal_pair(double& a, double& b) {
  const double tau = 6.283185307179586476925286766559;
  double u = 1.0 - unit();  // (0, 1]: keeps log finite
  double v = unit();
  double rad = std::sqrt(-2.0 * std::log(u));
  a = rad * std::cos(tau * v);
  b = rad * std::sin(tau * v);
}

Layout::Layout(std::vector<int32_t> s) : sizes(std::move(s)) {
  int64_t off = 0;
  for (int k = 0; k < depth(); ++k) {
    w_off.push_back(off);
    off += static_cast<int64_t>(in(k)) * out(k);
    b_off.push_back(off);
    off += out(k);
  }
  n_params = off;
}

int Layout::widest() const {
  int m = 0;
  for (int k = 0; k < depth(); ++k) m = out(k) > m ? out(k) : m;
  return m;
}

namespace {
// d standard normals from consecutive Box-Muller pairs; an odd tail burns its pair (dataset.cpp:18-28).
void normals(SplitMix64& r, double* dst, int d) {
  for (int i = 0; i < d; i += 2) {
    double a, b;
    r.normal_pair(a, b);
    dst[i] = a;
    if (i + 1 < d) dst[i + 1] = b;
  }
}
}  // namespace

void generate_blobs(uint64_t seed, int64_t n, int d, int c, double spread, double* x, int32_t* y) {
  check<ConfigError>(c >= 2, "generate_synthetic: n_classes must be >= 2, got ", c);
  check<ConfigError>(n >= c, "generate_synthetic: n_samples (", n, ") must be >= n_classes (", c, ")");
  check<ConfigError>(d >= 1, "generate_synthetic: n_features must be >= 1");
  check<ConfigError>(spread > 0.0, "generate_synthetic: spread must be > 0");
  SplitMix64 r(seed);
  std::vector<double> centre(static_cast<size_t>(c) * d);
  for (int cls = 0; cls < c; ++cls) {
    double* mu = &centre[static_cast<size_t>(cls) * d];
    normals(r, mu, d);
    double ss = 0.0;
    for (int j = 0; j < d; ++j) ss += mu[j] * mu[j];
    double len = std::sqrt(ss);
    if (len == 0.0) len = 1.0;
    for (int j = 0; j < d; ++j) mu[j] = spread * mu[j] / len;
  }
  for (int64_t i = 0; i < n; ++i) {
    int32_t cls = static_cast<int32_t>(i % c);
    y[i] = cls;
    double* row = x + i * d;
    normals(r, row, d);
    const double* mu = &centre[static_cast<size_t>(cls) * d];
    for (int j = 0; j < d; ++j) row[j] += mu[j];
  }
}

void init_weights(const Layout& L, uint64_t seed, double scale, double* w) {
  check<Error>(scale >= 0.0, "init_params: scale must be >= 0");
  SplitMix64 r(seed);
  for (int64_t i = 0; i < L.n_params; ++i) w[i] = 0.0;
  for (int k = 0; k < L.depth(); ++k) {
    double* wk = w + L.w_off[static_cast<size_t>(k)];
    int64_t cnt = static_cast<int64_t>(L.in(k)) * L.out(k);
    for (int64_t i = 0; i < cnt; ++i) wk[i] = r.sym(scale);
  }
}

EpochSampler::EpochSampler(int64_t n, uint64_t seed, bool with_replacement)
    : n_(n), rng_(seed), repl_(with_replacement) {
  check<Error>(n_ >= 1, "MinibatchSampler: dataset size must be >= 1, got ", n_);
  if (!repl_) shuffle();
}

void EpochSampler::shuffle() {
  perm_.resize(static_cast<size_t>(n_));
  std::iota(perm_.begin(), perm_.end(), 0);
  for (int64_t i = n_ - 1; i > 0; --i) {
    auto j = static_cast<int64_t>(rng_.below(static_cast<uint64_t>(i + 1)));
    std::swap(perm_[static_cast<size_t>(i)], perm_[static_cast<size_t>(j)]);
  }
  cursor_ = 0;
  ++epochs_;
}

void EpochSampler::draw(int64_t size, int32_t* out) {
  check<Error>(size >= 1, "draw_minibatch: size must be >= 1");
  check<Error>(size <= n_, "draw_minibatch: size ", size, " exceeds dataset size ", n_);
  if (repl_) {
    for (int64_t i = 0; i < size; ++i) out[i] = static_cast<int32_t>(rng_.below(static_cast<uint64_t>(n_)));
    return;
  }
  if (cursor_ + size > n_) shuffle();
  for (int64_t i = 0; i < size; ++i) out[i] = perm_[static_cast<size_t>(cursor_ + i)];
  cursor_ += size;
}

RunSpec::RunSpec(const lsgd_b200_config& cfg) : c(cfg) {
  check<ConfigError>(cfg.layer_sizes != nullptr && cfg.n_layers >= 0, "model.layer_sizes must be given");
  layers.assign(cfg.layer_sizes, cfg.layer_sizes + cfg.n_layers);
  c.layer_sizes = layers.data();
}

int64_t RunSpec::iterations() const {
  if (c.iterations > 0) return c.iterations;
  return static_cast<int64_t>(c.epochs) * (c.n_samples / global_batch());
}

double RunSpec::epoch_float(int64_t t) const {
  return static_cast<double>(t) * static_cast<double>(global_batch()) / static_cast<double>(c.n_samples);
}

double RunSpec::lr(int64_t t) const {
  double e = epoch_float(t);
  double gb = static_cast<double>(c.n_workers) * static_cast<double>(c.local_batch);
  double target = c.base_lr * gb / 256.0;
  if (c.warmup_epochs > 0.0 && e < c.warmup_epochs) return c.base_lr + (target - c.base_lr) * (e / c.warmup_epochs);
  double rate = target;
  auto decays = static_cast<int64_t>(std::floor(e / static_cast<double>(c.decay_every_epochs)));
  while (decays-- > 0) rate *= c.decay_factor;
  return rate;
}

void RunSpec::validate() const {
  using CE = ConfigError;
  check<CE>(c.algorithm >= 0 && c.algorithm <= 2, "algorithm: expected sequential|csgd|lsgd");
  check<CE>(c.n_workers >= 1, "n_workers must be >= 1");
  check<CE>(c.n_groups >= 1, "n_groups must be >= 1");
  if (c.algorithm == LSGD_B200_SEQUENTIAL) check<CE>(c.n_workers == 1, "sequential runs require n_workers = 1");
  if (c.algorithm == LSGD_B200_LSGD)
    check<CE>(c.n_workers % c.n_groups == 0, "n_groups (", c.n_groups, ") must divide n_workers (", c.n_workers, ")");
  check<CE>(layers.size() >= 2, "model.layer_sizes must list at least input and output dims");
  for (int32_t s : layers) check<CE>(s >= 1, "model.layer_sizes entries must be positive");
  check<CE>(layers.back() >= 2, "model.layer_sizes: class count must be >= 2");
  check<CE>(c.base_lr > 0.0, "optim.base_lr must be > 0");
  check<CE>(c.momentum >= 0.0 && c.momentum < 1.0, "optim.momentum must be in [0, 1)");
  check<CE>(c.weight_decay >= 0.0, "optim.weight_decay must be >= 0");
  check<CE>(c.warmup_epochs >= 0.0, "optim.warmup_epochs must be >= 0");
  check<CE>(c.decay_every_epochs >= 1, "optim.decay_every_epochs must be >= 1");
  check<CE>(c.decay_factor > 0.0 && c.decay_factor <= 1.0, "optim.decay_factor must be in (0, 1]");
  check<CE>(c.mode == LSGD_B200_PLAIN || c.mode == LSGD_B200_MOMENTUM, "optim.mode: expected plain|momentum");
  check<CE>(c.local_batch >= 1, "local_batch must be >= 1");
  check<CE>(c.epochs >= 0, "epochs must be >= 0");
  check<CE>(c.iterations >= 0, "iterations must be >= 0");
  check<CE>(c.init_scale >= 0.0, "init_scale must be >= 0");
  check<CE>(c.io_delay_s >= 0.0 && c.global_link_delay_s >= 0.0, "delays must be >= 0");
  check<CE>(c.collective_timeout_s > 0.0, "transport.timeout_s must be > 0");
  check<CE>(c.n_samples >= 1, "data.n_samples must be >= 1");
  check<CE>(c.n_features == layers.front(), "data.n_features (", c.n_features, ") must match model input dim (",
            layers.front(), ")");
  check<CE>(c.n_classes == layers.back(), "data.n_classes (", c.n_classes, ") must match model class count (",
            layers.back(), ")");
  check<CE>(global_batch() <= c.n_samples, "global batch ", global_batch(), " exceeds dataset size ", c.n_samples);
  check<CE>(c.dtype == LSGD_B200_FP32 || c.dtype == LSGD_B200_FP64, "b200.dtype: expected fp32|fp64");
  check<CE>(c.global_algo == LSGD_B200_GLOBAL_NCCL || c.global_algo == LSGD_B200_GLOBAL_ORDERED,
            "b200.global_allreduce: expected nccl|ordered");
  check<CE>(c.gemm >= 0 && c.gemm <= 2, "b200.gemm: expected auto|simt|tcgen05");
  check<CE>(c.data_source == LSGD_B200_DATA_DEVICE || c.data_source == LSGD_B200_DATA_HOST,
            "b200.data: expected device|host");
  check<CE>(c.model == LSGD_B200_MODEL_MLP || c.model == LSGD_B200_MODEL_SYNTHETIC_GRADIENT,
            "b200.model: expected mlp|synthetic_gradient");
  check<CE>(c.n_devices >= 0, "b200.n_devices must be >= 0");
}

ShardStream::ShardStream(const RunSpec& spec) : spec_(spec) {
  const auto& c = spec.c;
  if (c.shared_minibatch) {
    samplers_.emplace_back(c.n_samples, c.seed + 2);
  } else {
    for (int i = 0; i < c.n_workers; ++i) samplers_.emplace_back(c.n_samples, c.seed + 3 + static_cast<uint64_t>(i));
  }
}

void ShardStream::next(int32_t* out) {
  const auto& c = spec_.c;
  if (c.shared_minibatch) {
    samplers_[0].draw(spec_.global_batch(), out);  // contiguous shards are views of this row
    return;
  }
  for (int i = 0; i < c.n_workers; ++i) samplers_[static_cast<size_t>(i)].draw(c.local_batch, out + i * c.local_batch);
}

}  // namespace lsgd_b200
