// Host-side, bit-exact pieces of the LSGD step that never touch the GPU: the SplitMix64 stream, the synthetic
// blob generator, the epoch-wise Fisher-Yates sampler, shard partition, parameter layout/init, the learning-rate
// schedule and the worker/communicator topology. Each mirrors a reference routine bit for bit (cited per item);
// they run on the host because the reference generates every input there.
#pragma once

#include <cstdint>
#include <vector>

#include "common.hpp"
#include "../../include/lsgd_b200.h"

namespace lsgd_b200 {

// SplitMix64 (rng.hpp:14-51).
struct SplitMix64 {
  uint64_t s;
  explicit SplitMix64(uint64_t seed) : s(seed) {}
  uint64_t u64() {
    s += 0x9E3779B97F4A7C15ULL;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double unit() { return static_cast<double>(u64() >> 11) * 0x1.0p-53; }    // [0,1), 53 bits
  double sym(double scale) { return scale * (2.0 * unit() - 1.0); }           // [-scale, scale]
  uint64_t below(uint64_t bound) { return u64() % bound; }                    // modulo draw
  void normal_pair(double& a, double& b);                                    // Box-Muller, 2 draws
};

// Model geometry: layer_sizes = {input, hidden..., classes}; layer k = W_k [out x in] row-major then b_k.
struct Layout {
  std::vector<int32_t> sizes;
  std::vector<int64_t> w_off, b_off;
  int64_t n_params = 0;
  explicit Layout(std::vector<int32_t> s);
  int depth() const { return static_cast<int>(sizes.size()) - 1; }
  int in(int k) const { return sizes[static_cast<size_t>(k)]; }
  int out(int k) const { return sizes[static_cast<size_t>(k) + 1]; }
  int widest() const;
};

// Reference-identical Gaussian blobs (dataset.cpp:18-70); x row-major [n x d].
void generate_blobs(uint64_t seed, int64_t n, int d, int c, double spread, double* x, int32_t* y);
// Weights uniform in [-scale, scale] in layout order; biases zero, no draws consumed (mlp.cpp:174-186).
void init_weights(const Layout& L, uint64_t seed, double scale, double* w);

// Epoch-wise Fisher-Yates without replacement, drop-last refresh; or i.i.d. with replacement (sampler.cpp:9-43).
class EpochSampler {
 public:
  EpochSampler(int64_t n, uint64_t seed, bool with_replacement = false);
  void draw(int64_t size, int32_t* out);
  int64_t epochs() const { return epochs_; }

 private:
  void shuffle();
  int64_t n_;
  SplitMix64 rng_;
  bool repl_;
  std::vector<int32_t> perm_;
  int64_t cursor_ = 0, epochs_ = 0;
};

// Owned copy of lsgd_b200_config with the derived quantities the engine needs.
struct RunSpec {
  lsgd_b200_config c{};
  std::vector<int32_t> layers;
  bool track_versions = false;  // run_train asked for version_at_compute (measured on the device)
  explicit RunSpec(const lsgd_b200_config& cfg);
  int N() const { return c.n_workers; }
  int G() const { return c.algorithm == LSGD_B200_LSGD ? c.n_groups : 1; }
  int k() const { return N() / G(); }                      // workers per group
  int64_t global_batch() const { return static_cast<int64_t>(c.local_batch) * c.n_workers; }
  int64_t iterations() const;                              // executors.cpp:435-439
  double epoch_float(int64_t t) const;                     // executors.cpp:441-444
  double lr(int64_t t) const;                              // optimizer.cpp:8-22
  void validate() const;                                   // executors.cpp:389-399, 446-466, 484-489
};

// The shared minibatch stream, as every rank of the reference redraws it (ShardSource, executors.cpp:67-85).
class ShardStream {
 public:
  explicit ShardStream(const RunSpec& spec);
  // Global batch of iteration `next` -> out[global_batch]; worker i owns [i*B_loc, (i+1)*B_loc).
  void next(int32_t* out);

 private:
  const RunSpec& spec_;
  std::vector<EpochSampler> samplers_;
};

}  // namespace lsgd_b200
