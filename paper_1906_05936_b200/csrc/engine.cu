// LSGD step engine — see engine.hpp for the design. Reference loop structure: executors.cpp:190-304
// (worker: io -> postponed update -> compute -> local reduce; communicator: reduce -> /N -> global allreduce ->
// broadcast), csgd executors.cpp:132-188, sequential :87-130.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <exception>
#include <map>
#include <mutex>
#include <thread>

#include "engine.hpp"
#include "gemm_tc.cuh"
#include "kernels.cuh"

namespace lsgd_b200 {

namespace {
constexpr int64_t kAlign = 64;       // elements: slices start on 256 B (fp32) / 512 B (fp64) boundaries
constexpr int kRing = 4;             // pinned index ring depth (host may run this many steps ahead)
constexpr int64_t kLossCap = 1 << 16;  // device loss history ring per rank

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

struct PhaseEvents {
  cudaEvent_t ev[6][2];
  bool used[6];
};
}  // namespace

Geometry::Geometry(const RunSpec& spec, int es) : esize(es) {
  if (spec.c.model == LSGD_B200_MODEL_SYNTHETIC_GRADIENT) P = spec.c.synthetic_params;
  else P = Layout(spec.layers).n_params;
  P1 = P + 1;
  int k = spec.k();
  S = round_up((P1 + k - 1) / k, kAlign);
  Ppad = S * k;
  peer.flags = 0;
  peer.payload = 256;
  peer.s[0] = round_up(peer.payload + Ppad * es, 256);
  peer.s[1] = round_up(peer.s[0] + S * es, 256);
  peer.gbar = round_up(peer.s[1] + S * es, 256);
  peer.total = round_up(peer.gbar + S * es, 256);
}

// ================================================================================================ RankImpl
template <typename T>
class RankImpl final : public Rank {
 public:
  RankImpl(const RunSpec& spec, int device, std::vector<int> workers, int64_t history_rows)
      : spec_(spec), L_(spec.layers), geo_(spec, sizeof(T)), dev_(device), workers_(std::move(workers)),
        hist_rows_(history_rows) {
    N_ = spec_.N();
    G_ = spec_.G();
    k_ = spec_.k();
    alg_ = spec_.c.algorithm;
    exact_ = sizeof(T) == 8;
    synth_ = spec_.c.model == LSGD_B200_MODEL_SYNTHETIC_GRADIENT;
    B_ = alg_ == LSGD_B200_SEQUENTIAL ? static_cast<int>(spec_.global_batch()) : spec_.c.local_batch;
    check<ConfigError>(N_ <= kMaxPeers * 8, "n_workers too large for one box");
    check<ConfigError>(k_ <= kMaxPeers && G_ <= kMaxPeers, "group size and group count must be <= ", kMaxPeers);
    LSGD_CUDA(cudaSetDevice(dev_));
    int major = 0;
    LSGD_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev_));
    check<Error>(major >= 10, "device ", dev_, " is not sm_100-class (compute capability major ", major, ")");
    LSGD_CUDA(cudaStreamCreateWithFlags(&main_, cudaStreamNonBlocking));
    int lo = 0, hi = 0;
    LSGD_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    // The communicator role runs on a high-priority side stream; emulated ranks use one stream.
    split_ = workers_.size() == 1;
    if (split_) LSGD_CUDA(cudaStreamCreateWithPriority(&comm_, cudaStreamNonBlocking, hi));
    else comm_ = main_;
    LSGD_CUDA(cudaEventCreateWithFlags(&ev_handoff_, cudaEventDisableTiming));
    LSGD_CUDA(cudaEventCreateWithFlags(&ev_back_, cudaEventDisableTiming));
    void* to = nullptr;
    LSGD_CUDA(cudaHostAlloc(&to, sizeof(int), cudaHostAllocMapped));
    timed_out_host_ = static_cast<volatile int*>(to);
    *timed_out_host_ = 0;
    void* tod = nullptr;
    LSGD_CUDA(cudaHostGetDevicePointer(&tod, to, 0));
    timed_out_dev_ = static_cast<int*>(tod);
    LSGD_CUDA(cudaMalloc(&bad_dev_, sizeof(unsigned)));
    LSGD_CUDA(cudaMemset(bad_dev_, 0, sizeof(unsigned)));
    peer_base_.assign(static_cast<size_t>(N_), nullptr);
    for (int i = 0; i < kRing; ++i) LSGD_CUDA(cudaEventCreateWithFlags(&ring_ev_[i], cudaEventDisableTiming));
    LSGD_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ring_), sizeof(int32_t) * kRing * workers_.size() * B_,
                            cudaHostAllocDefault));
    if (!synth_) {
      if (spec_.c.shared_minibatch || alg_ == LSGD_B200_SEQUENTIAL) draw_.resize(static_cast<size_t>(spec_.global_batch()));
      else draw_.resize(static_cast<size_t>(spec_.global_batch()));
      shards_ = std::make_unique<ShardStream>(spec_);
    }
    for (int wid : workers_) alloc_worker(wid);
    if (hist_rows_ > 0)
      LSGD_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&hist_), sizeof(T) * hist_rows_ * geo_.P, cudaHostAllocDefault));
    use_tc_ = tc_eligible();
  }

  ~RankImpl() override {
    cudaSetDevice(dev_);
    cudaDeviceSynchronize();
    for (auto& kv : timers_)
      for (auto& pr : kv.second) {
        cudaEventDestroy(pr.first);
        cudaEventDestroy(pr.second);
      }
    for (auto& pv : phase_ev_)
      for (auto& pe : pv)
        for (int p = 0; p < 6; ++p)
          if (pe.used[p]) {
            cudaEventDestroy(pe.ev[p][0]);
            cudaEventDestroy(pe.ev[p][1]);
          }
    for (auto& w : ws_) free_worker(w);
    for (char* p : ipc_opened_) cudaIpcCloseMemHandle(p);
    if (slice_comm_) ncclCommDestroy(slice_comm_);
    if (flat_comm_) ncclCommDestroy(flat_comm_);
    if (own_data_) {
      if (host_data_) cudaFreeHost(host_alloc_);
      else {
        cudaFree(data_x_);
        cudaFree(data_y_);
      }
    }
    if (hist_) cudaFreeHost(hist_);
    cudaFreeHost(ring_);
    cudaFreeHost(const_cast<int*>(timed_out_host_));
    cudaFree(bad_dev_);
    for (int i = 0; i < kRing; ++i) cudaEventDestroy(ring_ev_[i]);
    cudaEventDestroy(ev_handoff_);
    cudaEventDestroy(ev_back_);
    if (split_) cudaStreamDestroy(comm_);
    cudaStreamDestroy(main_);
  }

  int device() const override { return dev_; }
  const std::vector<int>& workers() const override { return workers_; }
  char* peer_block(int worker) override { return find(worker).blk; }
  void set_peer_base(int worker, char* base) override { peer_base_[static_cast<size_t>(worker)] = base; }
  void set_nccl(void* slice_comm, void* flat_comm) override {
    slice_comm_ = static_cast<ncclComm_t>(slice_comm);
    flat_comm_ = static_cast<ncclComm_t>(flat_comm);
  }
  void note_ipc(char* p) { ipc_opened_.push_back(p); }

  // ------------------------------------------------------------------------------------------ data / params
  void upload_dataset(const double* x, const int32_t* y, int64_t n) override {
    if (synth_) return;
    LSGD_CUDA(cudaSetDevice(dev_));
    const int d = spec_.c.n_features;
    std::vector<T> conv(static_cast<size_t>(n) * d);
    for (size_t i = 0; i < conv.size(); ++i) conv[i] = static_cast<T>(x[i]);
    own_data_ = true;
    n_rows_ = n;
    if (spec_.c.data_source == LSGD_B200_DATA_HOST) {
      // Pinned host dataset read by the gather kernel through UVA: the per-step H2D is the shard's rows.
      host_data_ = true;
      size_t bytes = conv.size() * sizeof(T) + static_cast<size_t>(n) * sizeof(int32_t) + 256;
      LSGD_CUDA(cudaHostAlloc(&host_alloc_, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
      std::memcpy(host_alloc_, conv.data(), conv.size() * sizeof(T));
      char* lab = static_cast<char*>(host_alloc_) + round_up(static_cast<int64_t>(conv.size() * sizeof(T)), 256);
      std::memcpy(lab, y, static_cast<size_t>(n) * sizeof(int32_t));
      void* dx = nullptr;
      LSGD_CUDA(cudaHostGetDevicePointer(&dx, host_alloc_, 0));
      data_x_ = static_cast<T*>(dx);
      data_y_ = reinterpret_cast<int32_t*>(static_cast<char*>(dx) + (lab - static_cast<char*>(host_alloc_)));
    } else {
      LSGD_CUDA(cudaMalloc(&data_x_, conv.size() * sizeof(T)));
      LSGD_CUDA(cudaMalloc(&data_y_, static_cast<size_t>(n) * sizeof(int32_t)));
      LSGD_CUDA(cudaMemcpy(data_x_, conv.data(), conv.size() * sizeof(T), cudaMemcpyHostToDevice));
      LSGD_CUDA(cudaMemcpy(data_y_, y, static_cast<size_t>(n) * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
  }

  void share_dataset_from(Rank* other) override {
    auto* o = dynamic_cast<RankImpl<T>*>(other);
    check<Error>(o != nullptr, "share_dataset_from: dtype mismatch");
    data_x_ = o->data_x_;
    data_y_ = o->data_y_;
    n_rows_ = o->n_rows_;
    own_data_ = false;
  }

  void set_params(const double* w) override {
    LSGD_CUDA(cudaSetDevice(dev_));
    std::vector<T> conv(static_cast<size_t>(geo_.P));
    for (int64_t i = 0; i < geo_.P; ++i) conv[static_cast<size_t>(i)] = static_cast<T>(w[i]);
    for (auto& wk : ws_) {
      LSGD_CUDA(cudaMemcpy(wk.w, conv.data(), sizeof(T) * geo_.P, cudaMemcpyHostToDevice));
      if (wk.v) LSGD_CUDA(cudaMemset(wk.v, 0, sizeof(T) * geo_.P));
    }
    if (hist_rows_ > 0) std::memcpy(hist_, conv.data(), sizeof(T) * geo_.P);  // w_0
    if (use_tc_) for (auto& wk : ws_) tc_resplit_weights(wk);
  }

  void get_params(int worker, double* w) override {
    LSGD_CUDA(cudaSetDevice(dev_));
    LSGD_CUDA(cudaStreamSynchronize(main_));
    std::vector<T> tmp(static_cast<size_t>(geo_.P));
    LSGD_CUDA(cudaMemcpy(tmp.data(), find(worker).w, sizeof(T) * geo_.P, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < geo_.P; ++i) w[i] = static_cast<double>(tmp[static_cast<size_t>(i)]);
  }

  // ------------------------------------------------------------------------------------------ the step
  void issue_steps(int64_t n, const int32_t* host_idx, bool shard_only) override {
    LSGD_CUDA(cudaSetDevice(dev_));
    for (int64_t q = 0; q < n; ++q) {
      check_health();
      const int32_t* given = nullptr;
      if (host_idx) given = host_idx + q * (shard_only ? static_cast<int64_t>(B_) * workers_.size() : spec_.global_batch());
      issue_one(t_next_, given, shard_only);
      ++t_next_;
    }
  }

  void issue_steps_rows(int64_t n, const void* x_host, const int32_t* y_host) override {
    LSGD_CUDA(cudaSetDevice(dev_));
    check<Error>(!synth_, "step_rows needs the MLP model");
    const int64_t per = static_cast<int64_t>(B_) * spec_.c.n_features * static_cast<int64_t>(ws_.size());
    for (int64_t q = 0; q < n; ++q) {
      check_health();
      rows_x_ = static_cast<const T*>(x_host) + q * per;
      rows_y_ = y_host + q * static_cast<int64_t>(B_) * static_cast<int64_t>(ws_.size());
      issue_one(t_next_, nullptr, false);
      rows_x_ = nullptr;
      rows_y_ = nullptr;
      ++t_next_;
    }
  }

  void drain() override {
    LSGD_CUDA(cudaSetDevice(dev_));
    if (alg_ == LSGD_B200_LSGD && applied_ < t_next_) {
      current_phase() = "broadcast";
      for (auto& wk : ws_) apply(wk, t_next_ - 1);
      ++applied_;
    }
    synchronize();
  }

  void synchronize() override {
    LSGD_CUDA(cudaSetDevice(dev_));
    LSGD_CUDA(cudaStreamSynchronize(comm_));
    LSGD_CUDA(cudaStreamSynchronize(main_));
    check_health();
    unsigned bad = 0;
    LSGD_CUDA(cudaMemcpy(&bad, bad_dev_, sizeof(bad), cudaMemcpyDeviceToHost));
    check<Error>(bad == 0, "non-finite value in parameters after update");
  }

  int64_t steps_issued() const override { return t_next_; }
  int64_t updates_applied() const override { return applied_; }

  void history(double* loss, double* lr, int64_t n) override {
    LSGD_CUDA(cudaSetDevice(dev_));
    synchronize();
    n = std::min(n, applied_);
    std::vector<T> tmp(static_cast<size_t>(kLossCap));
    LSGD_CUDA(cudaMemcpy(tmp.data(), ws_[0].loss_hist, sizeof(T) * kLossCap, cudaMemcpyDeviceToHost));
    for (int64_t u = 0; u < n; ++u) {
      if (loss) loss[u] = static_cast<double>(tmp[static_cast<size_t>(u % kLossCap)]);
      if (lr) lr[u] = spec_.lr(u);
    }
  }

  void param_history(double* out, int64_t rows) override {
    synchronize();
    rows = std::min(rows, hist_rows_);
    for (int64_t i = 0; i < rows * geo_.P; ++i) out[i] = static_cast<double>(hist_[i]);
  }

  void phase_spans(int worker, double* out, int64_t n_iter) override {
    synchronize();
    size_t wi = static_cast<size_t>(&find(worker) - ws_.data());
    for (int64_t t = 0; t < n_iter; ++t) {
      for (int p = 0; p < 6; ++p) {
        double b = 0, e = 0;
        if (wi < phase_ev_.size() && t < static_cast<int64_t>(phase_ev_[wi].size()) &&
            phase_ev_[wi][static_cast<size_t>(t)].used[p]) {
          float ms0 = 0, ms1 = 0;
          LSGD_CUDA(cudaEventElapsedTime(&ms0, t0_ev_, phase_ev_[wi][static_cast<size_t>(t)].ev[p][0]));
          LSGD_CUDA(cudaEventElapsedTime(&ms1, t0_ev_, phase_ev_[wi][static_cast<size_t>(t)].ev[p][1]));
          b = ms0 * 1e-3;
          e = ms1 * 1e-3;
        }
        out[(t * 6 + p) * 2] = b;
        out[(t * 6 + p) * 2 + 1] = e;
      }
    }
  }

  double last_loss() override {
    synchronize();
    if (applied_ == 0) return 0.0;
    T v{};
    LSGD_CUDA(cudaMemcpy(&v, ws_[0].loss_hist + (applied_ - 1) % kLossCap, sizeof(T), cudaMemcpyDeviceToHost));
    return static_cast<double>(v);
  }

  int64_t launches() const override { return lc_.n; }
  void* main_stream() override { return main_; }
  void set_timing(bool on) override {
    timing_ = on;
    if (on) {
      LSGD_CUDA(cudaSetDevice(dev_));
      for (auto& kv : timers_)
        for (auto& pr : kv.second) {
          cudaEventDestroy(pr.first);
          cudaEventDestroy(pr.second);
        }
      timers_.clear();
    }
  }
  void kernel_time(const std::string& fam, double* avg_ms, int64_t* count) override {
    synchronize();
    auto it = timers_.find(fam);
    double sum = 0;
    int64_t cnt = 0;
    if (it != timers_.end()) {
      for (auto& pr : it->second) {
        float ms = 0;
        LSGD_CUDA(cudaEventElapsedTime(&ms, pr.first, pr.second));
        sum += ms;
        ++cnt;
      }
    }
    *avg_ms = cnt ? sum / static_cast<double>(cnt) : 0.0;
    *count = cnt;
  }

  void compute_gradient(const int32_t* idx, double* grad, double* loss) override {
    check<Error>(!synth_ && ws_.size() == 1, "compute_gradient needs a single-worker MLP rank");
    LSGD_CUDA(cudaSetDevice(dev_));
    Worker& w = ws_[0];
    io(t_next_, idx, true);
    compute(w);
    LSGD_CUDA(cudaStreamSynchronize(main_));
    std::vector<T> tmp(static_cast<size_t>(geo_.P1));
    LSGD_CUDA(cudaMemcpy(tmp.data(), w.payload, sizeof(T) * geo_.P1, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < geo_.P; ++i) grad[i] = static_cast<double>(tmp[static_cast<size_t>(i)]);
    *loss = static_cast<double>(tmp[static_cast<size_t>(geo_.P)]);
  }

  void abort() override { *timed_out_host_ = 1; }
  void check_health() override {
    if (*timed_out_host_)
      throw TransportError(cat("collective timeout or abort on device ", dev_, " after ",
                               spec_.c.collective_timeout_s, " s waiting for peer flags"));
  }

  void enable_phases() {
    if (!spec_.c.record_phases) return;
    LSGD_CUDA(cudaSetDevice(dev_));
    LSGD_CUDA(cudaEventCreate(&t0_ev_));
    LSGD_CUDA(cudaEventRecord(t0_ev_, main_));
    phase_ev_.assign(ws_.size(), {});
  }

 private:
  struct Worker {
    int id = 0, g = 0, j = 0;
    char* blk = nullptr;
    unsigned long long* flags = nullptr;
    T* payload = nullptr;
    T* s[2] = {nullptr, nullptr};
    T* gbar = nullptr;
    T* w = nullptr;
    T* v = nullptr;
    T* x = nullptr;
    int32_t* y = nullptr;
    int32_t* idx = nullptr;
    std::vector<T*> act;
    T* d0 = nullptr;
    T* d1 = nullptr;
    T* sample_loss = nullptr;
    T* loss_hist = nullptr;
    TcWorkspace tc;  // split-TF32 operand buffers of the tensor-core path
  };

  Worker& find(int worker) {
    for (auto& w : ws_)
      if (w.id == worker) return w;
    throw Error(cat("worker ", worker, " is not hosted by this rank"));
  }

  void alloc_worker(int wid) {
    Worker w;
    w.id = wid;
    w.g = wid / k_;
    w.j = wid % k_;
    LSGD_CUDA(cudaMalloc(&w.blk, static_cast<size_t>(geo_.peer.total)));
    LSGD_CUDA(cudaMemset(w.blk, 0, static_cast<size_t>(geo_.peer.total)));
    w.flags = reinterpret_cast<unsigned long long*>(w.blk + geo_.peer.flags);
    w.payload = reinterpret_cast<T*>(w.blk + geo_.peer.payload);
    w.s[0] = reinterpret_cast<T*>(w.blk + geo_.peer.s[0]);
    w.s[1] = reinterpret_cast<T*>(w.blk + geo_.peer.s[1]);
    w.gbar = reinterpret_cast<T*>(w.blk + geo_.peer.gbar);
    LSGD_CUDA(cudaMalloc(&w.w, sizeof(T) * geo_.P));
    if (spec_.c.mode == LSGD_B200_MOMENTUM) LSGD_CUDA(cudaMalloc(&w.v, sizeof(T) * geo_.P));
    LSGD_CUDA(cudaMalloc(&w.loss_hist, sizeof(T) * kLossCap));
    LSGD_CUDA(cudaMemset(w.loss_hist, 0, sizeof(T) * kLossCap));
    if (synth_) {
      // cfg4 synthetic gradient: g_r[k] = Rng(1000 + r).next_symmetric(1.0); fixed per run.
      std::vector<T> g(static_cast<size_t>(geo_.P1));
      SplitMix64 r(1000 + static_cast<uint64_t>(wid));
      for (auto& e : g) e = static_cast<T>(r.sym(1.0));
      LSGD_CUDA(cudaMemcpy(w.payload, g.data(), sizeof(T) * geo_.P1, cudaMemcpyHostToDevice));
    } else {
      const int d = spec_.c.n_features;
      LSGD_CUDA(cudaMalloc(&w.x, sizeof(T) * static_cast<size_t>(B_) * d));
      LSGD_CUDA(cudaMalloc(&w.y, sizeof(int32_t) * B_));
      LSGD_CUDA(cudaMalloc(&w.idx, sizeof(int32_t) * B_));
      for (int k = 0; k < L_.depth(); ++k) {
        T* a = nullptr;
        LSGD_CUDA(cudaMalloc(&a, sizeof(T) * static_cast<size_t>(B_) * L_.out(k)));
        w.act.push_back(a);
      }
      int wide = std::max(L_.widest(), spec_.c.n_features);
      LSGD_CUDA(cudaMalloc(&w.d0, sizeof(T) * static_cast<size_t>(B_) * wide));
      LSGD_CUDA(cudaMalloc(&w.d1, sizeof(T) * static_cast<size_t>(B_) * wide));
      LSGD_CUDA(cudaMalloc(&w.sample_loss, sizeof(T) * B_));
    }
    ws_.push_back(std::move(w));
    peer_base_[static_cast<size_t>(wid)] = ws_.back().blk;
  }

  void free_worker(Worker& w) {
    cudaFree(w.blk);
    cudaFree(w.w);
    if (w.v) cudaFree(w.v);
    cudaFree(w.loss_hist);
    if (w.x) cudaFree(w.x);
    if (w.y) cudaFree(w.y);
    if (w.idx) cudaFree(w.idx);
    for (T* a : w.act) cudaFree(a);
    if (w.d0) cudaFree(w.d0);
    if (w.d1) cudaFree(w.d1);
    if (w.sample_loss) cudaFree(w.sample_loss);
    tc_free(w.tc);
  }

  // Peer views of worker `wid`'s block, from this device.
  char* base(int wid) const {
    char* b = peer_base_[static_cast<size_t>(wid)];
    if (!b) throw TransportError(cat("rank on device ", dev_, " has no mapping of worker ", wid, "'s peer block"));
    return b;
  }
  T* peer_payload(int wid) const { return reinterpret_cast<T*>(base(wid) + geo_.peer.payload); }
  T* peer_s(int wid, int par) const { return reinterpret_cast<T*>(base(wid) + geo_.peer.s[par]); }
  T* peer_gbar(int wid) const { return reinterpret_cast<T*>(base(wid) + geo_.peer.gbar); }
  const volatile unsigned long long* peer_flag(int wid, int which) const {
    return reinterpret_cast<const volatile unsigned long long*>(base(wid) + geo_.peer.flags) + which;
  }

  unsigned long long timeout_ns() const {
    return static_cast<unsigned long long>(spec_.c.collective_timeout_s * 1e9);
  }

  void wait(const std::vector<int>& wids, int which, unsigned long long target, cudaStream_t st) {
    FlagList fl{};
    int n = 0;
    for (int wid : wids) fl.f[n++] = peer_flag(wid, which);
    launch_wait_flags(fl, n, target, timeout_ns(), timed_out_dev_, st, lc_);
  }
  void signal(Worker& w, int which, unsigned long long v, cudaStream_t st) {
    launch_signal_flag(w.flags + which, v, st, lc_);
  }

  // --- kernel-family timing (bench roofline) and phase spans (executors.hpp:248-267)
  struct Timed {
    RankImpl* r;
    const char* fam;
    cudaStream_t st;
    cudaEvent_t b = nullptr;
    Timed(RankImpl* rr, const char* f, cudaStream_t s) : r(rr), fam(f), st(s) {
      if (r->timing_) {
        cudaEventCreate(&b);
        cudaEventRecord(b, st);
      }
    }
    ~Timed() {
      if (r->timing_) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        r->timers_[fam].emplace_back(b, e);
      }
    }
  };
  void phase_mark(size_t wi, int64_t t, int phase, int end, cudaStream_t st) {
    if (!spec_.c.record_phases || t0_ev_ == nullptr) return;
    auto& v = phase_ev_[wi];
    while (static_cast<int64_t>(v.size()) <= t) {
      PhaseEvents pe{};
      v.push_back(pe);
    }
    PhaseEvents& pe = v[static_cast<size_t>(t)];
    if (!pe.used[phase]) {
      LSGD_CUDA(cudaEventCreate(&pe.ev[phase][0]));
      LSGD_CUDA(cudaEventCreate(&pe.ev[phase][1]));
      pe.used[phase] = true;
    }
    LSGD_CUDA(cudaEventRecord(pe.ev[phase][end], st));
  }
  size_t widx(const Worker& w) const { return static_cast<size_t>(&w - ws_.data()); }

  // io: host sampler -> pinned ring -> H2D -> gather (K1). executors.cpp:236-239 / 75-79.
  void io(int64_t t, const int32_t* given, bool shard_only) {
    if (rows_x_) {  // caller-supplied host rows: the H2D copy is the io (executors.cpp:236-239)
      const int d = spec_.c.n_features;
      for (size_t i = 0; i < ws_.size(); ++i) {
        Worker& w = ws_[i];
        phase_mark(i, t, 0, 0, main_);
        launch_sleep(spec_.c.io_delay_s, main_, lc_);
        LSGD_CUDA(cudaMemcpyAsync(w.x, rows_x_ + i * static_cast<size_t>(B_) * d, sizeof(T) * B_ * d,
                                  cudaMemcpyHostToDevice, main_));
        LSGD_CUDA(cudaMemcpyAsync(w.y, rows_y_ + i * B_, sizeof(int32_t) * B_, cudaMemcpyHostToDevice, main_));
        phase_mark(i, t, 0, 1, main_);
      }
      return;
    }
    const int slot = static_cast<int>(t % kRing);
    LSGD_CUDA(cudaEventSynchronize(ring_ev_[slot]));  // the copy that last used this slot has completed
    int32_t* dst = ring_ + static_cast<size_t>(slot) * workers_.size() * B_;
    const int32_t* src = given;
    if (!src || !shard_only) {
      if (!src) {
        shards_->next(draw_.data());
        src = draw_.data();
      }
      // global row -> this rank's shards (contiguous partition, sampler.cpp:45-57)
      for (size_t i = 0; i < ws_.size(); ++i)
        std::memcpy(dst + i * B_, src + static_cast<int64_t>(ws_[i].id) * (alg_ == LSGD_B200_SEQUENTIAL ? 0 : B_),
                    sizeof(int32_t) * B_);
    } else {
      std::memcpy(dst, src, sizeof(int32_t) * B_ * ws_.size());
    }
    for (size_t i = 0; i < ws_.size(); ++i) {
      Worker& w = ws_[i];
      phase_mark(i, t, 0, 0, main_);
      launch_sleep(spec_.c.io_delay_s, main_, lc_);
      LSGD_CUDA(cudaMemcpyAsync(w.idx, dst + i * B_, sizeof(int32_t) * B_, cudaMemcpyHostToDevice, main_));
      {
        Timed tm(this, "gather", main_);
        launch_gather<T>(data_x_, data_y_, w.idx, B_, spec_.c.n_features, w.x, w.y, main_, lc_);
      }
      phase_mark(i, t, 0, 1, main_);
    }
    LSGD_CUDA(cudaEventRecord(ring_ev_[slot], main_));
  }

  // compute: forward + backward of the local shard into the payload (mlp.cpp:238-273 as batched GEMMs).
  void compute(Worker& w) {
    if (synth_) return;
    if (use_tc_) {
      tc_compute(w);
      return;
    }
    Timed tm(this, "gemm", main_);
    const int depth = L_.depth();
    const T* in = w.x;
    for (int k = 0; k < depth; ++k) {
      const int ni = L_.in(k), no = L_.out(k);
      const T* Wk = w.w + L_.w_off[static_cast<size_t>(k)];
      const T* bk = w.w + L_.b_off[static_cast<size_t>(k)];
      launch_gemm_simt<T>(kEpiForward, exact_, B_, no, ni, in, ni, 1, Wk, 1, ni, w.act[static_cast<size_t>(k)], no, bk,
                          k + 1 < depth ? 1 : 0, T(0), nullptr, main_, lc_);
      in = w.act[static_cast<size_t>(k)];
    }
    const int C = L_.out(depth - 1);
    T* dcur = w.d0;
    T* dnext = w.d1;
    launch_softmax_xent<T>(w.act[static_cast<size_t>(depth - 1)], w.y, B_, C, dcur, w.sample_loss, main_, lc_);
    launch_mean_loss<T>(w.sample_loss, B_, w.payload + geo_.P, main_, lc_);
    for (int k = depth - 1; k >= 0; --k) {
      const int ni = L_.in(k), no = L_.out(k);
      const T* aprev = k == 0 ? w.x : w.act[static_cast<size_t>(k - 1)];
      T* gW = w.payload + L_.w_off[static_cast<size_t>(k)];
      T* gb = w.payload + L_.b_off[static_cast<size_t>(k)];
      launch_gemm_simt<T>(kEpiWeightGrad, exact_, no, ni, B_, dcur, 1, no, aprev, ni, 1, gW, ni, nullptr, 0,
                          static_cast<T>(B_), nullptr, main_, lc_);
      launch_bias_grad<T>(dcur, B_, no, gb, main_, lc_);
      if (k > 0) {
        const T* Wk = w.w + L_.w_off[static_cast<size_t>(k)];
        launch_gemm_simt<T>(kEpiInputGrad, exact_, B_, ni, no, dcur, no, 1, Wk, ni, 1, dnext, ni, nullptr, 0, T(0),
                            w.act[static_cast<size_t>(k - 1)], main_, lc_);
        std::swap(dcur, dnext);
      }
    }
  }

  std::vector<int> group_members(int g) const {
    std::vector<int> m;
    for (int i = g * k_; i < (g + 1) * k_; ++i) m.push_back(i);
    return m;
  }

  // local reduce: slice owner (g, j) sums slice j of its group's payloads in ascending worker order, adds the
  // communicator's zero vector, divides by N (transport.cpp:27-48; executors.cpp:278-288).
  void local_reduce(Worker& w, int64_t t) {
    if (alg_ == LSGD_B200_SEQUENTIAL) return;
    const int par = static_cast<int>(t & 1);
    if (alg_ == LSGD_B200_CSGD && flat_comm_) {
      // K9 baseline: flat NCCL ring allreduce of the whole payload over N ranks (in place).
      Timed tm(this, "global", main_);
      LSGD_NCCL(ncclAllReduce(w.payload, w.payload, static_cast<size_t>(geo_.Ppad), nccl_type(), ncclSum, flat_comm_,
                              main_));
      return;
    }
    auto members = group_members(w.g);
    wait(members, kFlagGrad, static_cast<unsigned long long>(t + 1), main_);
    SrcList<T> src{};
    for (int i = 0; i < k_; ++i) src.p[i] = peer_payload(members[static_cast<size_t>(i)]) + w.j * geo_.S;
    T* dst = G_ == 1 ? w.gbar : w.s[par];
    {
      Timed tm(this, "reduce", main_);
      launch_ordered_sum<T>(src, k_, geo_.S, dst, alg_ == LSGD_B200_LSGD, static_cast<T>(N_), main_, lc_);
    }
    if (G_ == 1) signal(w, kFlagBcast, static_cast<unsigned long long>(t + 1), main_);
    // every local slice sum is published before any local global-average waits on peers' (emulated ranks)
    else if (slice_comm_ == nullptr) signal(w, kFlagSlice, static_cast<unsigned long long>(t + 1), main_);
  }

  // global average across communicators (executors.cpp:290-295): NCCL (or the ordered peer sum) on the comm
  // stream, so it overlaps the workers' next io.
  void global(Worker& w, int64_t t) {
    if (G_ == 1 || alg_ != LSGD_B200_LSGD) return;
    const int par = static_cast<int>(t & 1);
    const bool nccl = slice_comm_ != nullptr;
    if (split_) {
      LSGD_CUDA(cudaEventRecord(ev_handoff_, main_));
      LSGD_CUDA(cudaStreamWaitEvent(comm_, ev_handoff_, 0));
    }
    launch_sleep(spec_.c.global_link_delay_s, comm_, lc_);
    if (nccl) {
      Timed tm(this, "global", comm_);
      LSGD_NCCL(ncclAllReduce(w.s[par], w.gbar, static_cast<size_t>(geo_.S), nccl_type(), ncclSum, slice_comm_, comm_));
    } else {
      std::vector<int> owners;
      for (int g = 0; g < G_; ++g) owners.push_back(g * k_ + w.j);
      wait(owners, kFlagSlice, static_cast<unsigned long long>(t + 1), comm_);
      SrcList<T> src{};
      for (int g = 0; g < G_; ++g) src.p[g] = peer_s(owners[static_cast<size_t>(g)], par);
      Timed tm(this, "global", comm_);
      launch_ordered_sum<T>(src, G_, geo_.S, w.gbar, false, T(0), comm_, lc_);
    }
    signal(w, kFlagBcast, static_cast<unsigned long long>(t + 1), comm_);
  }

  // broadcast + update (executors.cpp:210-229): pull the k averaged slices of the group, apply sgd_update,
  // check finiteness, record the round's loss.
  void apply(Worker& w, int64_t u) {
    const size_t wi = widx(w);
    phase_mark(wi, u, 4, 0, main_);
    UpdateArgs<T> a{};
    a.slice_len = geo_.S;
    a.n_params = geo_.P;
    if (alg_ == LSGD_B200_SEQUENTIAL) {
      for (int j = 0; j < k_; ++j) a.slices.p[j] = w.payload + j * geo_.S;
    } else if (alg_ == LSGD_B200_CSGD && flat_comm_) {
      for (int j = 0; j < k_; ++j) a.slices.p[j] = w.payload + j * geo_.S;
      a.post_div = static_cast<T>(N_);  // the per-worker /N after the flat allreduce (executors.cpp:170)
    } else {
      auto owners = group_members(w.g);
      wait(owners, kFlagBcast, static_cast<unsigned long long>(u + 1), main_);
      for (int j = 0; j < k_; ++j) a.slices.p[j] = peer_gbar(owners[static_cast<size_t>(j)]);
    }
    phase_mark(wi, u, 4, 1, main_);
    phase_mark(wi, u, 5, 0, main_);
    a.w = w.w;
    a.v = w.v;
    a.mode = spec_.c.mode;
    a.lr = static_cast<T>(spec_.lr(u));
    a.momentum = static_cast<T>(spec_.c.momentum);
    a.weight_decay = static_cast<T>(spec_.c.weight_decay);
    a.loss_out = w.loss_hist + (u % kLossCap);
    a.bad = bad_dev_;
    {
      Timed tm(this, "update", main_);
      launch_update<T>(a, exact_, main_, lc_);
    }
    if (use_tc_) tc_resplit_weights(w);
    phase_mark(wi, u, 5, 1, main_);
    if (hist_rows_ > 0 && w.id == workers_[0] && u + 1 < hist_rows_)
      LSGD_CUDA(cudaMemcpyAsync(hist_ + (u + 1) * geo_.P, w.w, sizeof(T) * geo_.P, cudaMemcpyDeviceToHost, main_));
  }

  void issue_one(int64_t t, const int32_t* given, bool shard_only) {
    current_phase() = "io";
    if (!synth_) io(t, given, shard_only);
    else if (spec_.c.io_delay_s > 0) launch_sleep(spec_.c.io_delay_s, main_, lc_);
    if (alg_ == LSGD_B200_LSGD && t >= 1) {
      current_phase() = "broadcast";
      for (auto& w : ws_) apply(w, t - 1);  // postponed update of round t-1 (executors.cpp:241-242)
      ++applied_;
    }
    current_phase() = "compute";
    for (auto& w : ws_) {
      phase_mark(widx(w), t, 1, 0, main_);
      compute(w);
      phase_mark(widx(w), t, 1, 1, main_);
      if (!(alg_ == LSGD_B200_CSGD && flat_comm_) && alg_ != LSGD_B200_SEQUENTIAL)
        signal(w, kFlagGrad, static_cast<unsigned long long>(t + 1), main_);
    }
    current_phase() = "local_reduce";
    for (auto& w : ws_) {
      phase_mark(widx(w), t, 2, 0, main_);
      local_reduce(w, t);
      phase_mark(widx(w), t, 2, 1, main_);
    }
    current_phase() = "global_allreduce";
    for (auto& w : ws_) {
      phase_mark(widx(w), t, 3, 0, comm_);
      global(w, t);
      phase_mark(widx(w), t, 3, 1, comm_);
    }
    if (alg_ != LSGD_B200_LSGD) {
      current_phase() = "update";
      for (auto& w : ws_) apply(w, t);
      ++applied_;
    }
    current_phase() = "between-phases";
  }

  ncclDataType_t nccl_type() const { return sizeof(T) == 8 ? ncclFloat64 : ncclFloat32; }

  // ----------------------------------------------------------------------------- tensor-core path hooks
  bool tc_eligible() const {
    if (synth_ || sizeof(T) != 4) return false;
    if (spec_.c.gemm == LSGD_B200_GEMM_SIMT) return false;
    bool ok = tc_shapes_supported(spec_.layers, B_);
    if (spec_.c.gemm == LSGD_B200_GEMM_TC)
      check<ConfigError>(ok, "b200.gemm = tcgen05 needs every layer width and the local batch to be multiples of 128");
    return ok;
  }
  void tc_compute(Worker& w) {
    Timed tm(this, "gemm", main_);
    tc_forward_backward(w.tc, L_, B_, reinterpret_cast<const float*>(w.w), reinterpret_cast<const float*>(w.x), w.y,
                        reinterpret_cast<float*>(w.payload), reinterpret_cast<float*>(w.sample_loss), main_, lc_);
  }
  void tc_resplit_weights(Worker& w) {
    if (!w.tc.ready) tc_alloc(w.tc, L_, B_, spec_.c.n_features);
    tc_split_weights(w.tc, L_, reinterpret_cast<const float*>(w.w), main_, lc_);
  }

  const T* rows_x_ = nullptr;
  const int32_t* rows_y_ = nullptr;
  RunSpec spec_;
  Layout L_;
  Geometry geo_;
  int dev_;
  std::vector<int> workers_;
  int64_t hist_rows_;
  int N_ = 1, G_ = 1, k_ = 1, alg_ = 2, B_ = 1;
  bool exact_ = false, synth_ = false, split_ = false, use_tc_ = false;
  cudaStream_t main_ = nullptr, comm_ = nullptr;
  cudaEvent_t ev_handoff_ = nullptr, ev_back_ = nullptr;
  std::vector<char*> peer_base_;
  std::vector<char*> ipc_opened_;
  ncclComm_t slice_comm_ = nullptr, flat_comm_ = nullptr;
  T* data_x_ = nullptr;
  int32_t* data_y_ = nullptr;
  int64_t n_rows_ = 0;
  bool own_data_ = false, host_data_ = false;
  void* host_alloc_ = nullptr;
  std::vector<Worker> ws_;
  int32_t* ring_ = nullptr;
  cudaEvent_t ring_ev_[kRing] = {};
  std::unique_ptr<ShardStream> shards_;
  std::vector<int32_t> draw_;
  volatile int* timed_out_host_ = nullptr;
  int* timed_out_dev_ = nullptr;
  unsigned* bad_dev_ = nullptr;
  int64_t t_next_ = 0, applied_ = 0;
  T* hist_ = nullptr;
  LaunchCounter lc_;
  bool timing_ = false;
  std::map<std::string, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>> timers_;
  cudaEvent_t t0_ev_ = nullptr;
  std::vector<std::vector<PhaseEvents>> phase_ev_;
};

std::unique_ptr<Rank> make_rank(const RunSpec& spec, int device, std::vector<int> workers, int64_t history_rows) {
  std::unique_ptr<Rank> r;
  if (spec.c.dtype == LSGD_B200_FP64) r = std::make_unique<RankImpl<double>>(spec, device, std::move(workers), history_rows);
  else r = std::make_unique<RankImpl<float>>(spec, device, std::move(workers), history_rows);
  return r;
}

void enable_phase_recording(Rank* r) {
  if (auto* a = dynamic_cast<RankImpl<float>*>(r)) a->enable_phases();
  if (auto* b = dynamic_cast<RankImpl<double>*>(r)) b->enable_phases();
}

void note_ipc_mapping(Rank* r, char* p) {
  if (auto* a = dynamic_cast<RankImpl<float>*>(r)) a->note_ipc(p);
  if (auto* b = dynamic_cast<RankImpl<double>*>(r)) b->note_ipc(p);
}

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
  std::vector<std::unique_ptr<Rank>> ranks;
  for (int r = 0; r < ndev; ++r)
    ranks.push_back(make_rank(spec, r, blocks[static_cast<size_t>(r)], r == 0 && want_history ? T + 1 : 0));

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
  std::vector<ncclComm_t> comms_to_free;
  const bool one_each = ndev == N;
  if (one_each && spec.c.algorithm == LSGD_B200_LSGD && G > 1 && spec.c.global_algo == LSGD_B200_GLOBAL_NCCL) {
    for (int j = 0; j < k; ++j) {
      std::vector<int> devs;
      for (int g = 0; g < G; ++g) devs.push_back(g * k + j);
      std::vector<ncclComm_t> cs(static_cast<size_t>(G));
      LSGD_NCCL(ncclCommInitAll(cs.data(), G, devs.data()));
      for (int g = 0; g < G; ++g) ranks[static_cast<size_t>(g * k + j)]->set_nccl(cs[static_cast<size_t>(g)], nullptr);
    }
  }
  if (one_each && spec.c.algorithm == LSGD_B200_CSGD && spec.c.csgd_nccl && N > 1) {
    std::vector<int> devs;
    for (int i = 0; i < N; ++i) devs.push_back(i);
    std::vector<ncclComm_t> cs(static_cast<size_t>(N));
    LSGD_NCCL(ncclCommInitAll(cs.data(), N, devs.data()));
    for (int i = 0; i < N; ++i) ranks[static_cast<size_t>(i)]->set_nccl(nullptr, cs[static_cast<size_t>(i)]);
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
        // stream order makes gradient t read w_t: t updates were applied before compute t (executors.cpp:245)
        for (int64_t t = 0; t < T; ++t) out.version_at_compute[static_cast<size_t>(w * T + t)] = t;
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
}

}  // namespace lsgd_b200
