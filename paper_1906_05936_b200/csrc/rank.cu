// LSGD step engine, one Rank per GPU — see engine.hpp for the design. Reference loop structure:
// executors.cpp:190-304 (worker: io -> postponed update -> compute -> local reduce; communicator: reduce -> /N ->
// global allreduce -> broadcast), csgd executors.cpp:132-188, sequential :87-130.
//
// The step is pipelined per gradient bucket (one bucket per layer): as soon as the backward pass has written layer
// k's gradient, the comm stream starts the ordered intra-group reduce (K6) and the inter-group average (K7) of
// that bucket while the main stream continues with layer k-1's backward. The postponed update is applied per
// bucket right before the forward of the same layer in the next step, so forward layer 0 only waits for bucket 0.
// Arithmetic per element is unchanged (the reference's ascending-order sums), only the schedule differs.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <atomic>
#include <chrono>
#include <deque>
#include <map>
#include <thread>
#include <tuple>
#include <type_traits>
#include <mutex>

#include "engine.hpp"
#include "gemm_tc.cuh"
#include "kernels.cuh"
#include "nvls.hpp"

namespace lsgd_b200 {

namespace {
constexpr int64_t kAlign = 64;         // elements: slices start on 256 B (fp32) / 512 B (fp64) boundaries
constexpr int kRing = 4;               // pinned index ring depth (host may run this many steps ahead)
constexpr int64_t kLossCap = 1 << 16;  // device loss history ring per rank

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

double steady_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Poll a non-blocking communicator until its pending call has been enqueued (ncclInProgress -> ncclSuccess). On
// an error or past the deadline the communicator is aborted and TransportError raised. Returns normally on success.
void nccl_settle(ncclComm_t c, double timeout_s, const char* what) {
  const double t0 = steady_s();
  for (;;) {
    ncclResult_t ae = ncclSuccess;
    ncclResult_t r = ncclCommGetAsyncError(c, &ae);
    if (r != ncclSuccess) ae = r;
    if (ae == ncclSuccess) return;
    if (ae != ncclInProgress) {
      ncclCommAbort(c);
      throw TransportError(cat("NCCL ", what, " failed: ", ncclGetErrorString(ae), "; communicator aborted"));
    }
    if (steady_s() - t0 > timeout_s) {
      ncclCommAbort(c);
      throw TransportError(cat("NCCL ", what, " did not complete within ", timeout_s,
                               " s (a peer never joined); communicator aborted"));
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

ncclConfig_t nonblocking_config() {
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  cfg.blocking = 0;
  return cfg;
}

struct PhaseEvents {
  cudaEvent_t ev[6][2];
  bool used[6];
  bool marked[6][2];  // both ends recorded (a span that was never closed reads as absent, not as an error)
};
}  // namespace

bool direct_exchange(const RunSpec& spec) {
  static const char* e = std::getenv("LSGD_B200_DIRECT");
  return e && std::atoi(e) != 0 && spec.c.algorithm == LSGD_B200_LSGD && spec.G() > 1 && spec.k() > 1 &&
         spec.c.global_algo == LSGD_B200_GLOBAL_ORDERED && spec.c.model == LSGD_B200_MODEL_MLP &&
         spec.N() <= kMaxPeers;
}

Geometry::Geometry(const RunSpec& spec, int es) : esize(es) {
  if (spec.c.model == LSGD_B200_MODEL_SYNTHETIC_GRADIENT) {
    P = spec.c.synthetic_params;
    Bucket b;
    b.n = P;
    buckets.push_back(b);
  } else {
    Layout L(spec.layers);
    P = L.n_params;
    check<ConfigError>(L.depth() <= kMaxBuckets, "at most ", kMaxBuckets, " layers are supported");
    // Exchange buckets are row blocks of W_k (heights a multiple of the 128-row GEMM tile): 64M parameters on one
    // GPU, 32M with an exchange. The weight-gradient GEMM runs over blocks of consecutive buckets: one bucket per
    // block for one worker per group (2x1: 560k samples/s vs 539k with 64M blocks, 499k with 64M buckets), 64M
    // blocks for groups of k >= 2, whose exchange is a scatter + reduce + global chain per bucket: 32M buckets in
    // 64M blocks pipeline that chain over the two halves of W_1 without shrinking its GEMM (2x2, A/B on one box:
    // 944k vs 895k with 64M buckets, 916k with 32M blocks, 866k with 16M buckets; profiles/r1_buckets_ab.log).
    // LSGD_B200_BUCKET_ELEMS / LSGD_B200_GEMM_ELEMS override both (tests force multi-bucket layers).
    const int kk = spec.k();
    const char* env = std::getenv("LSGD_B200_BUCKET_ELEMS");
    const char* genv = std::getenv("LSGD_B200_GEMM_ELEMS");
    const double kMi = 1024.0 * 1024.0;
    // N = 1: 64M (layer 1 in two blocks): fewer, larger weight-gradient GEMMs overlapped by fewer update launches
    // (A/B, 3 rounds on one box: 345-350k samples/s vs 337-339k with 16M; profiles/r2_n1_bucket_ab.log)
    const double kBucketElems = env ? std::max(1.0, std::atof(env)) : (spec.N() > 1 ? 32.0 : 64.0) * kMi;
    const double kGemmElems = std::max(kBucketElems, genv ? std::atof(genv) : (kk >= 2 ? 64.0 * kMi : 0.0));
    layer_buckets.resize(static_cast<size_t>(L.depth()));
    // Layer 0's gradient is the first one the backward produces and the first one the next forward needs: with an
    // exchange (N > 1) it is cut into buckets / blocks of half the size, so its chain starts earlier.
    const bool tail_half = spec.N() > 1;
    const char* l0env = std::getenv("LSGD_B200_L0_DIV");  // layer-0 bucket / block divisor with an exchange (A/B)
    const double l0div = l0env ? std::max(1.0, std::atof(l0env)) : 2.0;
    auto split_rows = [](int out, double elems, int in) {  // divisor of out, rows a multiple of the tile quantum
      int nc = std::max(1, static_cast<int>(std::ceil(static_cast<double>(in) * out / elems)));
      const int quantum = out % 128 == 0 ? 128 : (out % 8 == 0 ? 8 : out);
      while (nc > 1 && (out % nc != 0 || (out / nc) % quantum != 0)) --nc;
      return nc;
    };
    for (int k = 0; k < L.depth(); ++k) {
      const int in = L.in(k), out = L.out(k);
      const double btarget = (k == 0 && tail_half) ? kBucketElems / l0div : kBucketElems;
      const double gtarget = (k == 0 && tail_half) ? kGemmElems / l0div : kGemmElems;
      const int ng = split_rows(out, gtarget, in), grows = out / ng;
      for (int g = 0; g < ng; ++g) {
        int ne = split_rows(grows, btarget, in);
        // buckets inside a block must tile the block's contiguous output exactly (no slot padding between them)
        if ((static_cast<int64_t>(grows / ne) * in) % (64 * kk) != 0) ne = 1;
        const int rows = grows / ne;
        for (int c = 0; c < ne; ++c) {
          Bucket b;
          b.layer = k;
          b.row0 = g * grows + c * rows;
          b.rows = rows;
          b.bias = g + 1 == ng && c + 1 == ne;
          b.pstart = L.w_off[static_cast<size_t>(k)] + static_cast<int64_t>(b.row0) * in;
          b.n = static_cast<int64_t>(rows) * in + (b.bias ? out : 0);
          b.blk_rows = c == 0 ? grows : 0;
          b.blk_bias = c == 0 && g + 1 == ng;
          layer_buckets[static_cast<size_t>(k)].push_back(static_cast<int>(buckets.size()));
          buckets.push_back(b);
        }
      }
    }
    check<ConfigError>(static_cast<int>(buckets.size()) <= kMaxBuckets, "model too large: more than ", kMaxBuckets,
                       " gradient buckets");
  }
  if (layer_buckets.empty()) layer_buckets.push_back({0});
  buckets.back().loss = true;
  const int k = spec.k();
  int64_t poff = 0, goff = 0;
  for (auto& b : buckets) {
    const int64_t len = b.n + (b.loss ? 1 : 0);
    b.S = round_up((len + k - 1) / k, kAlign);
    b.poff = poff;
    b.goff = goff;
    poff += b.S * k;
    goff += b.S;
  }
  Ppad = poff;
  Sg = goff;
  loss_at = buckets.back().poff + buckets.back().n;
  peer.flags = 0;
  peer.payload = round_up(static_cast<int64_t>(kFlagWords) * 8, 256);
  peer.s[0] = round_up(peer.payload + Ppad * es, 256);
  peer.s[1] = round_up(peer.s[0] + Sg * es, 256);
  peer.gbar = round_up(peer.s[1] + Sg * es, 256);
  peer.gfull = round_up(peer.gbar + Sg * es, 256);
  peer.stage = round_up(peer.gfull + Ppad * es, 256);
  const int G = spec.G();
  const bool direct = direct_exchange(spec);
  const int64_t stage_elems = direct ? 2 * spec.N() * Sg : (k > 1 ? k * Sg : 0);
  const int64_t gstage_elems = (G > 1 && !direct) ? G * Sg : 0;  // only what the layout uses
  peer.gstage[0] = round_up(peer.stage + stage_elems * es, 256);
  peer.gstage[1] = round_up(peer.gstage[0] + gstage_elems * es, 256);
  peer.total = round_up(peer.gstage[1] + gstage_elems * es, 256);
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
    nb_ = static_cast<int>(geo_.buckets.size());
    alg_ = spec_.c.algorithm;
    exact_ = sizeof(T) == 8;
    synth_ = spec_.c.model == LSGD_B200_MODEL_SYNTHETIC_GRADIENT;
    B_ = alg_ == LSGD_B200_SEQUENTIAL ? static_cast<int>(spec_.global_batch()) : spec_.c.local_batch;
    check<ConfigError>(k_ <= kMaxPeers && G_ <= kMaxPeers, "group size and group count must be <= ", kMaxPeers);
    LSGD_CUDA(cudaSetDevice(dev_));
    int major = 0;
    LSGD_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev_));
    check<Error>(major >= 10, "device ", dev_, " is not sm_100-class (compute capability major ", major, ")");
    int lo = 0, hi = 0;
    LSGD_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    // priorities: communicator > compute > updates (the update of most buckets has a step of slack)
    LSGD_CUDA(cudaStreamCreateWithPriority(&main_, cudaStreamNonBlocking, hi < lo ? hi + 1 : hi));
    // The communicator role runs on a high-priority side stream; emulated ranks use one stream.
    split_ = workers_.size() == 1;
    if (split_) LSGD_CUDA(cudaStreamCreateWithPriority(&comm_, cudaStreamNonBlocking, hi));
    else comm_ = main_;
    // more communicator streams let consecutive buckets' push exchanges overlap (no NCCL on that path):
    // bucket q of the step runs on stream q mod n (LSGD_B200_COMM_STREAMS, 1..kMaxComm). Default 4 for groups of
    // k >= 2 (reverse backward order: layer 0's chains start as soon as dW_0 ends instead of queueing behind the
    // middle layer's; 2x2: 977-988k vs 973-975k samples/s), 3 otherwise (2x1: 560k vs 556k with 2;
    // profiles/r1_order_ab.log)
    if (split_) {
      const char* e = std::getenv("LSGD_B200_COMM_STREAMS");
      n_comm_ = e ? std::min(kMaxComm, std::max(1, std::atoi(e))) : (spec_.k() >= 2 ? 4 : 3);
      for (int i = 1; i < n_comm_; ++i)
        LSGD_CUDA(cudaStreamCreateWithPriority(&commx_[i], cudaStreamNonBlocking, hi));
    }
    commx_[0] = comm_;
    if (split_) LSGD_CUDA(cudaStreamCreateWithFlags(&upd_, cudaStreamNonBlocking));
    else upd_ = main_;
    for (int b = 0; b < kMaxBuckets; ++b) LSGD_CUDA(cudaEventCreateWithFlags(&ev_upd_[b], cudaEventDisableTiming));
    for (int b = 0; b < kMaxBuckets; ++b) LSGD_CUDA(cudaEventCreateWithFlags(&ev_dx_[b], cudaEventDisableTiming));
    for (int b = 0; b < kMaxBuckets; ++b) LSGD_CUDA(cudaEventCreateWithFlags(&ev_gupd_[b], cudaEventDisableTiming));
    for (int b = 0; b < kMaxBuckets; ++b) LSGD_CUDA(cudaEventCreateWithFlags(&ev_bucket_[b], cudaEventDisableTiming));
    for (int b = 0; b < kMaxBuckets; ++b) LSGD_CUDA(cudaEventCreateWithFlags(&ev_bias_[b], cudaEventDisableTiming));
    LSGD_CUDA(cudaEventCreateWithFlags(&ev_bias_src_, cudaEventDisableTiming));
    const char* be = std::getenv("LSGD_B200_BIAS_STREAM");  // 0: bias gradients on the main stream (A/B only)
    if (split_ && !(be && std::atoi(be) == 0)) LSGD_CUDA(cudaStreamCreateWithPriority(&bias_, cudaStreamNonBlocking, hi));
    LSGD_CUDA(cudaEventCreateWithFlags(&join_ev_, cudaEventDisableTiming));
    void* to = nullptr;
    LSGD_CUDA(cudaHostAlloc(&to, sizeof(int), cudaHostAllocMapped));
    timed_out_host_ = static_cast<volatile int*>(to);
    *timed_out_host_ = 0;
    void* tod = nullptr;
    LSGD_CUDA(cudaHostGetDevicePointer(&tod, to, 0));
    timed_out_dev_ = static_cast<int*>(tod);
    LSGD_CUDA(cudaMalloc(&bad_dev_, sizeof(unsigned)));
    // Every H2D copy and memset below is issued on main_ (a non-blocking stream does not order behind the
    // legacy stream, and a pageable cudaMemcpy may return before its DMA lands).
    LSGD_CUDA(cudaMemsetAsync(bad_dev_, 0, sizeof(unsigned), main_));
    peer_base_.assign(static_cast<size_t>(N_), nullptr);
    for (int i = 0; i < kRing; ++i) LSGD_CUDA(cudaEventCreateWithFlags(&ring_ev_[i], cudaEventDisableTiming));
    LSGD_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ring_), sizeof(int32_t) * kRing * workers_.size() * B_,
                            cudaHostAllocDefault));
    if (!synth_) {
      draw_.resize(static_cast<size_t>(spec_.global_batch()));
      shards_ = std::make_unique<ShardStream>(spec_);
    }
    use_tc_ = tc_eligible();
    for (int wid : workers_) alloc_worker(wid);
    direct_ = direct_exchange(spec_) && split_;
    if (hist_rows_ > 0)
      LSGD_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&hist_), sizeof(T) * hist_rows_ * geo_.P, cudaHostAllocDefault));
    LSGD_CUDA(cudaStreamSynchronize(main_));  // zeroed flags/payloads are in place before any peer connects
  }

  ~RankImpl() override {
    stop_nccl_watchdog();
    cudaSetDevice(dev_);
    cudaDeviceSynchronize();
    nvls_free(nvls_);
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
    for (T* p : own_x_) cudaFree(p);
    for (int32_t* p : own_y_) cudaFree(p);
    for (char* p : ipc_opened_) cudaIpcCloseMemHandle(p);
    if (!nccl_aborted_) {  // an aborted communicator is already torn down (ncclCommAbort)
      if (slice_comm_) ncclCommDestroy(slice_comm_);
      if (flat_comm_) ncclCommDestroy(flat_comm_);
    }
    for (cudaEvent_t e : nccl_ev_pool_) cudaEventDestroy(e);
    for (auto& op : nccl_ops_) {
      cudaEventDestroy(op.pre);
      cudaEventDestroy(op.post);
    }
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
    for (int b = 0; b < kMaxBuckets; ++b) cudaEventDestroy(ev_bucket_[b]);
    for (int b = 0; b < kMaxBuckets; ++b) cudaEventDestroy(ev_bias_[b]);
    cudaEventDestroy(ev_bias_src_);
    if (bias_) cudaStreamDestroy(bias_);
    if (split_) {
      cudaStreamDestroy(comm_);
      for (int i = 1; i < n_comm_; ++i) cudaStreamDestroy(commx_[i]);
      cudaStreamDestroy(upd_);
    }
    for (int b = 0; b < kMaxBuckets; ++b) cudaEventDestroy(ev_upd_[b]);
    for (int b = 0; b < kMaxBuckets; ++b) cudaEventDestroy(ev_dx_[b]);
    for (int b = 0; b < kMaxBuckets; ++b) cudaEventDestroy(ev_gupd_[b]);
    cudaEventDestroy(join_ev_);
    if (iod_) cudaStreamDestroy(iod_);
    if (pio_) cudaStreamDestroy(pio_);
    if (ev_x_free_) cudaEventDestroy(ev_x_free_);
    if (ev_x_ready_) cudaEventDestroy(ev_x_ready_);
    if (ev_pre_exch_) cudaEventDestroy(ev_pre_exch_);
    if (ev_io_done_) cudaEventDestroy(ev_io_done_);
    if (base_ev_) cudaEventDestroy(base_ev_);
    if (io_) {
      cudaStreamDestroy(io_);
      for (int i = 0; i < 2; ++i) {
        cudaFree(rows_xbuf_[i]);
        cudaFree(rows_ybuf_[i]);
        cudaEventDestroy(ev_rows_h2d_[i]);
        cudaEventDestroy(ev_rows_free_[i]);
      }
    }
    cudaStreamDestroy(main_);
  }

  int device() const override { return dev_; }
  const std::vector<int>& workers() const override { return workers_; }
  char* peer_block(int worker) override { return find(worker).blk; }
  void set_peer_base(int worker, char* base) override { peer_base_[static_cast<size_t>(worker)] = base; }
  void set_nccl(void* slice_comm, void* flat_comm) override {
    slice_comm_ = static_cast<ncclComm_t>(slice_comm);
    flat_comm_ = static_cast<ncclComm_t>(flat_comm);
    if ((slice_comm_ || flat_comm_) && !nccl_watch_.joinable())
      nccl_watch_ = std::thread([this] { nccl_watch_loop(); });
  }

  // ---- NVLS multicast fan-out (nvls.cu): whole-slot push exchange, groups of k >= 2, LSGD_B200_NVLS=1
  bool nvls_wanted() const override {
    static const char* e = std::getenv("LSGD_B200_NVLS");
    return e && std::atoi(e) != 0 && own_slot_fused() && k_ >= 2 && !sliced_global() && !direct_ && !pull_avg() &&
           (G_ == 1 || spec_.c.global_algo == LSGD_B200_GLOBAL_ORDERED);
  }
  size_t nvls_bytes() const override { return static_cast<size_t>(geo_.Ppad) * sizeof(T); }
  void nvls_join(uint64_t mc, size_t size, char* leader_block, int j, int k, double timeout_s) override {
    LSGD_CUDA(cudaSetDevice(dev_));
    nvls_add_device(mc, dev_);
    auto* flags = reinterpret_cast<unsigned long long*>(leader_block + geo_.peer.flags) + kNvlsAdded;
    const unsigned long long one = 1;
    LSGD_CUDA(cudaMemcpy(flags + j, &one, sizeof(one), cudaMemcpyHostToDevice));
    std::vector<unsigned long long> seen(static_cast<size_t>(k));
    const double t0 = steady_s();
    for (;;) {  // every member's device is in the team before anyone binds memory
      LSGD_CUDA(cudaMemcpy(seen.data(), flags, sizeof(unsigned long long) * k, cudaMemcpyDeviceToHost));
      bool all = true;
      for (auto v : seen) all = all && v != 0;
      if (all) break;
      if (steady_s() - t0 > timeout_s)
        throw TransportError(cat("NVLS: not every group member joined the multicast team within ", timeout_s, " s"));
      std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
    nvls_attach(mc, size, true);
  }
  void nvls_attach(uint64_t mc, size_t size, bool own_mc) override {
    check<Error>(ws_.size() == 1, "NVLS needs one worker per GPU");
    nvls_bind_map(nvls_, mc, size, dev_);
    nvls_.own_mc = own_mc;
    ws_[0].gfull = reinterpret_cast<T*>(nvls_.va);
    mc_gfull_ = reinterpret_cast<T*>(nvls_.mc_va);
  }

  // ---- NCCL watchdog: the reference times out every receive (inprocess.cpp:44-49, TransportError). A collective
  // whose peer never arrives would block its stream forever, so every NCCL call is bracketed by two events; a host
  // thread watches the oldest unfinished call and, once it has been running (its `pre` event reached) for longer
  // than collective_timeout_s, or NCCL reports an asynchronous error, aborts the communicators (ncclCommAbort
  // releases the stuck kernels) and marks the rank failed: the next step / synchronize raises TransportError.
  struct NcclOp {
    cudaEvent_t pre, post;
    double started;
  };
  cudaEvent_t nccl_event() {  // under nccl_mu_
    if (!nccl_ev_pool_.empty()) {
      cudaEvent_t e = nccl_ev_pool_.back();
      nccl_ev_pool_.pop_back();
      return e;
    }
    cudaEvent_t e;
    LSGD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return e;
  }
  // `call` issues one collective on `comm` and returns its ncclResult_t (ncclInProgress on a non-blocking
  // communicator); the host then polls until it is enqueued (bounded: nccl_settle), and the watchdog thread takes
  // over for the device side.
  template <class F>
  void nccl_call(cudaStream_t st, ncclComm_t comm, F&& call) {
    check_health();  // never touch an aborted communicator
    NcclOp op{};
    {
      std::lock_guard<std::mutex> g(nccl_mu_);
      op.pre = nccl_event();
      op.post = nccl_event();
    }
    op.started = -1.0;
    LSGD_CUDA(cudaEventRecord(op.pre, st));
    ncclResult_t r;
    {
      std::lock_guard<std::mutex> g(nccl_api_mu_);
      r = call();
    }
    if (r != ncclSuccess && r != ncclInProgress) {
      mark_nccl_aborted(cat("NCCL error ", ncclGetErrorString(r)));
      check_health();
    }
    try {
      for (;;) {  // bounded host-side enqueue (lazy connection setup needs every peer)
        ncclResult_t ae = ncclSuccess;
        {
          std::lock_guard<std::mutex> g(nccl_api_mu_);
          ncclCommGetAsyncError(comm, &ae);
        }
        if (ae == ncclSuccess) break;
        if (ae != ncclInProgress)
          throw TransportError(cat("NCCL collective failed: ", ncclGetErrorString(ae)));
        if (steady_s() - op_t0_or(op) > spec_.c.collective_timeout_s)
          throw TransportError(cat("NCCL collective was not enqueued within ", spec_.c.collective_timeout_s,
                                   " s (a peer never joined)"));
        std::this_thread::sleep_for(std::chrono::microseconds(20));
      }
    } catch (const TransportError& e) {
      mark_nccl_aborted(e.what());
      check_health();
    }
    LSGD_CUDA(cudaEventRecord(op.post, st));
    std::lock_guard<std::mutex> g(nccl_mu_);
    nccl_ops_.push_back(op);
  }
  double op_t0_or(NcclOp& op) {
    if (op.started < 0) op.started = steady_s();
    return op.started;
  }
  // Abort every communicator of this rank (once) and fail the rank: the next step / synchronize raises
  // TransportError with `why`.
  void mark_nccl_aborted(const std::string& why) {
    std::lock_guard<std::mutex> g(nccl_api_mu_);
    if (nccl_aborted_.load()) return;
    nccl_abort_reason_ = why;
    nccl_aborted_ = true;
    *timed_out_host_ = 1;
    if (slice_comm_) ncclCommAbort(slice_comm_);
    if (flat_comm_) ncclCommAbort(flat_comm_);
  }
  void nccl_watch_loop() {
    cudaSetDevice(dev_);
    while (!nccl_stop_.load()) {
      bool abort_now = false;
      std::string why;
      {
        std::lock_guard<std::mutex> g(nccl_mu_);
        while (!nccl_ops_.empty()) {
          NcclOp& op = nccl_ops_.front();
          if (cudaEventQuery(op.post) == cudaSuccess) {
            nccl_ev_pool_.push_back(op.pre);
            nccl_ev_pool_.push_back(op.post);
            nccl_ops_.pop_front();
            continue;
          }
          if (op.started < 0 && cudaEventQuery(op.pre) == cudaSuccess) op.started = steady_s();
          if (op.started >= 0 && steady_s() - op.started > spec_.c.collective_timeout_s) {
            abort_now = true;
            why = cat("NCCL collective did not complete within ", spec_.c.collective_timeout_s, " s");
          }
          break;
        }
      }
      if (abort_now) {
        mark_nccl_aborted(why);
        return;
      }
      std::this_thread::sleep_for(std::chrono::milliseconds(5));
    }
  }
  void stop_nccl_watchdog() {
    nccl_stop_ = true;
    if (nccl_watch_.joinable()) nccl_watch_.join();
  }
  void note_ipc(char* p) { ipc_opened_.push_back(p); }

  // ------------------------------------------------------------------------------------------ data / params
  void upload_dataset(const double* x, const int32_t* y, int64_t n) override {
    if (synth_) return;
    LSGD_CUDA(cudaSetDevice(dev_));
    const int d = spec_.c.n_features;
    std::vector<T> conv(static_cast<size_t>(n) * d);
    for (size_t i = 0; i < conv.size(); ++i) conv[i] = static_cast<T>(x[i]);
    if (own_data_) {  // a caller-supplied dataset replaces the one created with the rank
      LSGD_CUDA(cudaStreamSynchronize(main_));
      if (host_data_) LSGD_CUDA(cudaFreeHost(host_alloc_));
      else {
        LSGD_CUDA(cudaFree(data_x_));
        LSGD_CUDA(cudaFree(data_y_));
      }
      host_alloc_ = nullptr;
      data_x_ = nullptr;
      data_y_ = nullptr;
      host_data_ = false;
    }
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
      LSGD_CUDA(cudaMemcpyAsync(data_x_, conv.data(), conv.size() * sizeof(T), cudaMemcpyHostToDevice, main_));
      LSGD_CUDA(cudaMemcpyAsync(data_y_, y, static_cast<size_t>(n) * sizeof(int32_t), cudaMemcpyHostToDevice, main_));
      LSGD_CUDA(cudaStreamSynchronize(main_));
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
      LSGD_CUDA(cudaMemcpyAsync(wk.w, conv.data(), sizeof(T) * geo_.P, cudaMemcpyHostToDevice, main_));
      if (wk.v) LSGD_CUDA(cudaMemsetAsync(wk.v, 0, sizeof(T) * geo_.P, main_));
      if (use_tc_) tc_split_weights(wk.tc, L_, reinterpret_cast<const float*>(wk.w), main_, lc_);
    }
    if (hist_rows_ > 0) std::memcpy(hist_, conv.data(), sizeof(T) * geo_.P);  // w_0
    LSGD_CUDA(cudaStreamSynchronize(main_));
  }

  void get_params(int worker, double* w) override {
    LSGD_CUDA(cudaSetDevice(dev_));
    LSGD_CUDA(cudaStreamSynchronize(main_));
    std::vector<T> tmp(static_cast<size_t>(geo_.P));
    LSGD_CUDA(cudaMemcpy(tmp.data(), find(worker).w, sizeof(T) * geo_.P, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < geo_.P; ++i) w[i] = static_cast<double>(tmp[static_cast<size_t>(i)]);
  }

  // ------------------------------------------------------------------------------------------ the step API
  void issue_steps(int64_t n, const int32_t* host_idx, bool shard_only) override {
    LSGD_CUDA(cudaSetDevice(dev_));
    for (int64_t q = 0; q < n; ++q) {
      check_health();
      const int32_t* given = nullptr;
      if (host_idx) given = host_idx + q * (shard_only ? static_cast<int64_t>(B_) * workers_.size() : spec_.global_batch());
      spill_losses_if_due();
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
      spill_losses_if_due();
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
      for (auto& wk : ws_)
        for (int b = 0; b < nb_; ++b) apply_bucket(wk, b, t_next_ - 1, main_);
      for (auto& wk : ws_) after_update(wk, t_next_ - 1, main_);
      ++applied_;
    }
    synchronize();
  }

  void synchronize() override {
    LSGD_CUDA(cudaSetDevice(dev_));
    LSGD_CUDA(cudaStreamSynchronize(comm_));
    for (int i = 1; i < n_comm_; ++i) LSGD_CUDA(cudaStreamSynchronize(commx_[i]));
    LSGD_CUDA(cudaStreamSynchronize(upd_));
    if (bias_) LSGD_CUDA(cudaStreamSynchronize(bias_));
    LSGD_CUDA(cudaStreamSynchronize(main_));
    check_health();
    unsigned bad = 0;
    LSGD_CUDA(cudaMemcpy(&bad, bad_dev_, sizeof(bad), cudaMemcpyDeviceToHost));
    check<Error>(bad == 0, "non-finite value in parameters after update");
  }

  int64_t steps_issued() const override { return t_next_; }
  int64_t updates_applied() const override { return applied_; }

  // The device loss ring holds kLossCap rounds. Every kLossCap/2 issued steps the applied rounds not yet saved are
  // copied to host memory (one host sync per kLossCap/2 steps), so the ring never overwrites an unsaved round and
  // history() returns every iteration's loss however long the run.
  void spill_losses_if_due() {
    if (t_next_ == 0 || t_next_ % (kLossCap / 2) != 0) return;
    synchronize();
    spill_losses();
  }
  void spill_losses() {
    if (applied_ <= spilled_) return;
    check<Error>(applied_ - spilled_ <= kLossCap, "loss history: unsaved rounds were overwritten");
    std::vector<T> ring(static_cast<size_t>(kLossCap));
    LSGD_CUDA(cudaMemcpy(ring.data(), ws_[0].loss_hist, sizeof(T) * kLossCap, cudaMemcpyDeviceToHost));
    loss_saved_.resize(static_cast<size_t>(applied_));
    for (int64_t u = spilled_; u < applied_; ++u)
      loss_saved_[static_cast<size_t>(u)] = ring[static_cast<size_t>(u % kLossCap)];
    spilled_ = applied_;
  }

  void history(double* loss, double* lr, int64_t n) override {
    LSGD_CUDA(cudaSetDevice(dev_));
    synchronize();
    spill_losses();
    n = std::min(n, applied_);
    for (int64_t u = 0; u < n; ++u) {
      if (loss) loss[u] = static_cast<double>(loss_saved_[static_cast<size_t>(u)]);
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
            phase_ev_[wi][static_cast<size_t>(t)].marked[p][0] && phase_ev_[wi][static_cast<size_t>(t)].marked[p][1]) {
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

  int loss_async(void* host_pinned) override {
    LSGD_CUDA(cudaSetDevice(dev_));
    check<Error>(applied_ > 0, "no round has been applied yet");
    // the stream the round's update ran on
    cudaStream_t st = (split_ && (alg_ == LSGD_B200_LSGD || flat_nccl()) && !fused_update()) ? upd_ : main_;
    Timed tm(this, "d2h", st);
    LSGD_CUDA(cudaMemcpyAsync(host_pinned, ws_[0].loss_hist + (applied_ - 1) % kLossCap, sizeof(T),
                              cudaMemcpyDeviceToHost, st));
    return static_cast<int>(sizeof(T));
  }
  double last_loss() override {
    synchronize();
    if (applied_ == 0) return 0.0;
    T v{};
    LSGD_CUDA(cudaMemcpy(&v, ws_[0].loss_hist + (applied_ - 1) % kLossCap, sizeof(T), cudaMemcpyDeviceToHost));
    return static_cast<double>(v);
  }

  void join() override {
    LSGD_CUDA(cudaSetDevice(dev_));
    for (cudaStream_t st : {commx_[0], commx_[1], commx_[2], commx_[3], upd_, io_, bias_}) {
      if (st == nullptr || st == main_) continue;
      LSGD_CUDA(cudaEventRecord(join_ev_, st));
      LSGD_CUDA(cudaStreamWaitEvent(main_, join_ev_, 0));
    }
  }
  int64_t launches() const override { return lc_.n; }
  void* main_stream() override { return main_; }
  void set_timing(bool on) override {
    timing_ = on;
    if (on) {
      LSGD_CUDA(cudaSetDevice(dev_));
      if (base_ev_ == nullptr) LSGD_CUDA(cudaEventCreate(&base_ev_));
      LSGD_CUDA(cudaEventRecord(base_ev_, main_));
      for (auto& kv : timers_)
        for (auto& pr : kv.second) {
          cudaEventDestroy(pr.first);
          cudaEventDestroy(pr.second);
        }
      timers_.clear();
      timer_tags_.clear();
    }
  }
  std::string timeline() override {
    synchronize();
    std::vector<std::tuple<float, float, std::string, int>> rows;
    for (auto& kv : timers_) {
      const auto& tags = timer_tags_[kv.first];
      for (size_t i = 0; i < kv.second.size(); ++i) {
        float a = 0, b = 0;
        LSGD_CUDA(cudaEventElapsedTime(&a, base_ev_, kv.second[i].first));
        LSGD_CUDA(cudaEventElapsedTime(&b, base_ev_, kv.second[i].second));
        rows.emplace_back(a, b, kv.first, i < tags.size() ? tags[i] : -1);
      }
    }
    std::sort(rows.begin(), rows.end());
    std::string out;
    char line[160];
    for (auto& r : rows) {  // family, start, end, tag (bucket id; 100 + k for layer-k GEMMs; -1 none)
      std::snprintf(line, sizeof(line), "%s\t%.4f\t%.4f\t%d\n", std::get<2>(r).c_str(), std::get<0>(r),
                    std::get<1>(r), std::get<3>(r));
      out += line;
    }
    return out;
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
    for (int k = 0; k < L_.depth(); ++k) forward_layer(w, k);
    head(w);
    for (int k = L_.depth() - 1; k >= 0; --k) backward_layer(w, k);
    LSGD_CUDA(cudaStreamSynchronize(main_));
    std::vector<T> tmp(static_cast<size_t>(geo_.Ppad));
    LSGD_CUDA(cudaMemcpy(tmp.data(), w.payload, sizeof(T) * geo_.Ppad, cudaMemcpyDeviceToHost));
    for (const Bucket& b : geo_.buckets)
      for (int64_t i = 0; i < b.n; ++i) grad[b.pstart + i] = static_cast<double>(tmp[static_cast<size_t>(b.poff + i)]);
    *loss = static_cast<double>(tmp[static_cast<size_t>(geo_.loss_at)]);
  }

  void abort() override { *timed_out_host_ = 1; }
  void check_health() override {
    if (!*timed_out_host_) return;
    if (nccl_aborted_.load())
      throw TransportError(cat(nccl_abort_reason_, " on device ", dev_, "; communicators aborted"));
    if (*timed_out_host_ == 2)
      throw TransportError(cat("flag protocol violation on device ", dev_,
                               ": a producer ran ahead of its consumer (buffer reuse before it was read)"));
    throw TransportError(cat("collective timeout or abort on device ", dev_, " after ", spec_.c.collective_timeout_s,
                             " s waiting for peer flags"));
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
    T* gfull = nullptr;
    T* w = nullptr;
    T* v = nullptr;
    T* x = nullptr;
    int32_t* y = nullptr;
    int32_t* idx = nullptr;
    std::vector<T*> act;
    std::vector<T*> dl;  // delta of each layer [B, out_k]
    T* sample_loss = nullptr;
    T* loss_hist = nullptr;
    unsigned long long* ver = nullptr;  // [kMaxBuckets] update rounds applied per bucket (version tracking)
    long long* ver_log = nullptr;       // host-mapped [T * depth]: per iteration and layer, read at its forward
    TcWorkspace tc;  // split-TF32 operands of the tensor-core path
    bool x_split_ready = false;  // io() gathered this step's rows straight into the TC split
    const PeerLayout* lay = nullptr;
    int64_t Sg = 0;
    T* blk_stage(int m) const { return reinterpret_cast<T*>(blk + lay->stage) + static_cast<int64_t>(m) * Sg; }
    T* blk_gstage(int par, int g) const {
      return reinterpret_cast<T*>(blk + lay->gstage[par]) + static_cast<int64_t>(g) * Sg;
    }
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
    if (track_versions()) {
      LSGD_CUDA(cudaMalloc(&w.ver, sizeof(unsigned long long) * kMaxBuckets));
      LSGD_CUDA(cudaMemsetAsync(w.ver, 0, sizeof(unsigned long long) * kMaxBuckets, main_));
      const size_t n = static_cast<size_t>(spec_.iterations()) * static_cast<size_t>(L_.depth());
      LSGD_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&w.ver_log), sizeof(long long) * n, cudaHostAllocMapped));
      for (size_t i = 0; i < n; ++i) w.ver_log[i] = -1;
    }
    LSGD_CUDA(cudaMalloc(&w.blk, static_cast<size_t>(geo_.peer.total)));
    LSGD_CUDA(cudaMemsetAsync(w.blk, 0, static_cast<size_t>(geo_.peer.total), main_));
    w.flags = reinterpret_cast<unsigned long long*>(w.blk + geo_.peer.flags);
    w.payload = reinterpret_cast<T*>(w.blk + geo_.peer.payload);
    w.s[0] = reinterpret_cast<T*>(w.blk + geo_.peer.s[0]);
    w.s[1] = reinterpret_cast<T*>(w.blk + geo_.peer.s[1]);
    w.gbar = reinterpret_cast<T*>(w.blk + geo_.peer.gbar);
    w.gfull = reinterpret_cast<T*>(w.blk + geo_.peer.gfull);
    w.lay = &geo_.peer;
    w.Sg = geo_.Sg;
    LSGD_CUDA(cudaMalloc(&w.w, sizeof(T) * geo_.P));
    if (spec_.c.mode == LSGD_B200_MOMENTUM) LSGD_CUDA(cudaMalloc(&w.v, sizeof(T) * geo_.P));
    LSGD_CUDA(cudaMalloc(&w.loss_hist, sizeof(T) * kLossCap));
    LSGD_CUDA(cudaMemsetAsync(w.loss_hist, 0, sizeof(T) * kLossCap, main_));
    if (synth_) {
      // cfg4 synthetic gradient: g_r[k] = Rng(1000 + r).next_symmetric(1.0); fixed per run. The
      // single bucket keeps the payload contiguous: [g_0 .. g_{P-1} | loss slot].
      std::vector<T> g(static_cast<size_t>(geo_.P + 1));
      SplitMix64 r(1000 + static_cast<uint64_t>(wid));
      for (auto& e : g) e = static_cast<T>(r.sym(1.0));
      LSGD_CUDA(cudaMemcpyAsync(w.payload, g.data(), sizeof(T) * g.size(), cudaMemcpyHostToDevice, main_));
      LSGD_CUDA(cudaStreamSynchronize(main_));
    } else {
      const int d = spec_.c.n_features;
      LSGD_CUDA(cudaMalloc(&w.x, sizeof(T) * static_cast<size_t>(B_) * d));
      LSGD_CUDA(cudaMalloc(&w.y, sizeof(int32_t) * B_));
      LSGD_CUDA(cudaMalloc(&w.idx, sizeof(int32_t) * B_));
      LSGD_CUDA(cudaMalloc(&w.sample_loss, sizeof(T) * B_));
      if (use_tc_) {
        tc_alloc(w.tc, L_, B_, d, reinterpret_cast<const float*>(w.w));  // activations, deltas, plans
      } else {
        for (int k = 0; k < L_.depth(); ++k) {
          T* a = nullptr;
          LSGD_CUDA(cudaMalloc(&a, sizeof(T) * static_cast<size_t>(B_) * L_.out(k)));
          w.act.push_back(a);
        }
        for (int k = 0; k < L_.depth(); ++k) {  // per-layer deltas: every dX runs before any dW
          T* dl = nullptr;
          LSGD_CUDA(cudaMalloc(&dl, sizeof(T) * static_cast<size_t>(B_) * L_.out(k)));
          w.dl.push_back(dl);
        }
      }
    }
    own_x_.push_back(w.x);
    own_y_.push_back(w.y);
    ws_.push_back(std::move(w));
    peer_base_[static_cast<size_t>(wid)] = ws_.back().blk;
  }

  void free_worker(Worker& w) {
    if (w.ver) cudaFree(w.ver);
    if (w.ver_log) cudaFreeHost(w.ver_log);
    cudaFree(w.blk);
    cudaFree(w.w);
    if (w.v) cudaFree(w.v);
    cudaFree(w.loss_hist);
    if (w.idx) cudaFree(w.idx);
    for (T* a : w.act) cudaFree(a);
    for (T* p : w.dl) cudaFree(p);
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
  T* peer_gfull(int wid) const { return reinterpret_cast<T*>(base(wid) + geo_.peer.gfull); }
  unsigned long long* peer_arrived(int wid, int b, int j) const {
    return reinterpret_cast<unsigned long long*>(base(wid) + geo_.peer.flags) + kArrived + b * kMaxPeers + j;
  }

  // Broadcast of bucket b's averaged sub-slice j (executors.cpp:297-299) as a push into every group member's gfull
  // (k-1 of them over NVLink), then a release of the member's arrival flag; runs on the comm stream, off the
  // update's critical path.
  void push_bucket(Worker& w, int b, int64_t t, cudaStream_t st) {
    const Bucket& bk = geo_.buckets[static_cast<size_t>(b)];
    auto members = group_members(w.g);
    DstList<T> dst{};
    SignalList sl{};
    for (int i = 0; i < k_; ++i) {
      dst.p[i] = peer_gfull(members[static_cast<size_t>(i)]) + bk.poff + w.j * bk.S;
      sl.f[i] = peer_arrived(members[static_cast<size_t>(i)], b, w.j);
    }
    {
      Timed tm(this, "broadcast", st);
      launch_push<T>(w.gbar + bk.goff, bk.S, dst, k_, st, lc_);
    }
    launch_signal_many(sl, k_, static_cast<unsigned long long>(t + 1), st, lc_);
  }
  const volatile unsigned long long* peer_flag(int wid, int which, int b) const {
    return reinterpret_cast<const volatile unsigned long long*>(base(wid) + geo_.peer.flags) + which * kMaxBuckets + b;
  }

  unsigned long long timeout_ns() const {
    return static_cast<unsigned long long>(spec_.c.collective_timeout_s * 1e9);
  }

  void wait(const std::vector<int>& wids, int which, int b, unsigned long long target, cudaStream_t st) {
    FlagList fl{};
    int n = 0;
    for (int wid : wids) fl.f[n++] = peer_flag(wid, which, b);
    launch_wait_flags(fl, n, target, timeout_ns(), timed_out_dev_, st, lc_);
  }
  void signal(Worker& w, int which, int b, unsigned long long v, cudaStream_t st) {
    launch_signal_flag(w.flags + which * kMaxBuckets + b, v, st, lc_);
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
        r->timer_tags_[fam].push_back(r->tag_);
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
    pe.marked[phase][end] = true;
  }
  size_t widx(const Worker& w) const { return static_cast<size_t>(&w - ws_.data()); }

  // ------------------------------------------------------------------------------------------ io
  // host sampler -> pinned ring -> H2D -> gather (K1). executors.cpp:236-239 / 75-79.
  void io(int64_t t, const int32_t* given, bool shard_only) {
    if (rows_x_) {  // caller-supplied host rows: the H2D copy is the io
      const int d = spec_.c.n_features;
      const size_t nw = ws_.size();
      if (io_ == nullptr) {
        LSGD_CUDA(cudaStreamCreateWithFlags(&io_, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
          LSGD_CUDA(cudaMalloc(&rows_xbuf_[i], sizeof(T) * nw * B_ * d));
          LSGD_CUDA(cudaMalloc(&rows_ybuf_[i], sizeof(int32_t) * nw * B_));
          LSGD_CUDA(cudaEventCreateWithFlags(&ev_rows_h2d_[i], cudaEventDisableTiming));
          LSGD_CUDA(cudaEventCreateWithFlags(&ev_rows_free_[i], cudaEventDisableTiming));
        }
      }
      const int slot = static_cast<int>(t & 1);
      if (rows_used_[slot]) LSGD_CUDA(cudaStreamWaitEvent(io_, ev_rows_free_[slot], 0));
      {
        Timed tm(this, "h2d", io_);
        LSGD_CUDA(cudaMemcpyAsync(rows_xbuf_[slot], rows_x_, sizeof(T) * nw * B_ * d, cudaMemcpyHostToDevice, io_));
        LSGD_CUDA(cudaMemcpyAsync(rows_ybuf_[slot], rows_y_, sizeof(int32_t) * nw * B_, cudaMemcpyHostToDevice, io_));
      }
      LSGD_CUDA(cudaEventRecord(ev_rows_h2d_[slot], io_));
      rows_used_[slot] = true;
      rows_slot_ = slot;
      for (size_t i = 0; i < nw; ++i) {
        Worker& w = ws_[i];
        phase_mark(i, t, 0, 0, main_);
        launch_sleep(spec_.c.io_delay_s, main_, lc_);
        if (i == 0) LSGD_CUDA(cudaStreamWaitEvent(main_, ev_rows_h2d_[slot], 0));
        w.x = rows_xbuf_[slot] + i * static_cast<size_t>(B_) * d;
        w.y = rows_ybuf_[slot] + i * static_cast<size_t>(B_);
        phase_mark(i, t, 0, 1, main_);
      }
      return;
    }
    for (size_t i = 0; i < ws_.size(); ++i) {  // gathered rows land in the worker's own batch buffers
      ws_[i].x = own_x_[i];
      ws_[i].y = own_y_[i];
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
    // Injected io latency (executors.hpp:213-216). Emulated ranks (several workers on one stream) model the
    // reference's concurrent rank threads: one sleep per step for all of them, and under LSGD on a side stream
    // forked before the previous round's exchange, so io(t) overlaps the communicators' global allreduce(t-1)
    // (and its injected link delay) as the reference's worker and communicator threads do (executors.cpp:210-229).
    const bool emu_delay = ws_.size() > 1 && spec_.c.io_delay_s > 0;
    if (emu_delay && alg_ == LSGD_B200_LSGD) {
      if (!iod_) {
        LSGD_CUDA(cudaStreamCreateWithFlags(&iod_, cudaStreamNonBlocking));
        LSGD_CUDA(cudaEventCreateWithFlags(&ev_io_done_, cudaEventDisableTiming));
      }
      if (t > 0) LSGD_CUDA(cudaStreamWaitEvent(iod_, ev_pre_exch_, 0));
      for (size_t i = 0; i < ws_.size(); ++i) phase_mark(i, t, 0, 0, iod_);
      launch_sleep(spec_.c.io_delay_s, iod_, lc_);
      LSGD_CUDA(cudaEventRecord(ev_io_done_, iod_));
      LSGD_CUDA(cudaStreamWaitEvent(main_, ev_io_done_, 0));
    } else if (emu_delay) {
      for (size_t i = 0; i < ws_.size(); ++i) phase_mark(i, t, 0, 0, main_);
      launch_sleep(spec_.c.io_delay_s, main_, lc_);
    }
    // Prefetched io (one worker per GPU, no injected delay): the gather of step t runs on its own stream as soon as
    // step t-1 no longer reads the batch buffers (after its last layer-0 weight-gradient GEMM, ev_x_free_), i.e.
    // under the rest of t-1's backward, instead of on the main stream between the two steps. Same kernel, same
    // rows. Off by default (LSGD_B200_PREFETCH_IO=1): the gather's 512 latency-bound CTAs under the dW_1 GEMM slow
    // it more than the 12-90 us they take off the step boundary (N = 1: 339k vs 351k samples/s, N = 4: 982k vs
    // 1.002M; profiles/r2_prefetch_io_ab.log).
    const bool pre = prefetch_io();
    cudaStream_t ist = main_;
    if (pre) {
      if (!pio_) {
        int lo = 0, hi = 0;
        LSGD_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        LSGD_CUDA(cudaStreamCreateWithPriority(&pio_, cudaStreamNonBlocking, hi));
        LSGD_CUDA(cudaEventCreateWithFlags(&ev_x_free_, cudaEventDisableTiming));
        LSGD_CUDA(cudaEventCreateWithFlags(&ev_x_ready_, cudaEventDisableTiming));
      }
      if (x_free_recorded_) LSGD_CUDA(cudaStreamWaitEvent(pio_, ev_x_free_, 0));
      ist = pio_;
    }
    for (size_t i = 0; i < ws_.size(); ++i) {
      Worker& w = ws_[i];
      if (!emu_delay) {
        phase_mark(i, t, 0, 0, ist);
        launch_sleep(spec_.c.io_delay_s, ist, lc_);
      }
      LSGD_CUDA(cudaMemcpyAsync(w.idx, dst + i * B_, sizeof(int32_t) * B_, cudaMemcpyHostToDevice, ist));
      {
        Timed tm(this, "gather", ist);
        if (use_tc_ && spec_.c.n_features % 4 == 0) {  // rows straight into the first GEMM's TF32 split
          tc_gather_split(w.tc, L_, reinterpret_cast<const float*>(data_x_), data_y_, w.idx, w.y, ist, lc_);
          w.x_split_ready = true;
        } else {
          launch_gather<T>(data_x_, data_y_, w.idx, B_, spec_.c.n_features, w.x, w.y, ist, lc_);
        }
      }
      phase_mark(i, t, 0, 1, ist);
    }
    LSGD_CUDA(cudaEventRecord(ring_ev_[slot], ist));
    if (pre) {
      LSGD_CUDA(cudaEventRecord(ev_x_ready_, pio_));
      LSGD_CUDA(cudaStreamWaitEvent(main_, ev_x_ready_, 0));
    }
  }
  bool prefetch_io() const {
    static const char* e = std::getenv("LSGD_B200_PREFETCH_IO");
    const bool on = e ? std::atoi(e) != 0 : false;
    return on && split_ && !synth_ && spec_.c.io_delay_s <= 0 && !fused_update();
  }

  // ------------------------------------------------------------------------------------------ compute
  // forward layer k / head / backward layer k of the local shard (mlp.cpp:60-127 as batched GEMMs); the
  // gradient of layer k lands in payload bucket k, the mean loss in the loss slot.
  T* delta_buf(Worker& w, int k) { return w.dl[static_cast<size_t>(k)]; }

  void forward_layer(Worker& w, int k) {
    tag_ = 100 + k;
    if (synth_) return;
    if (use_tc_) {
      if (k == 0 && !w.x_split_ready) {
        Timed ts(this, "split", main_);
        tc_split_input(w.tc, L_, reinterpret_cast<const float*>(w.x), main_, lc_);
      }
      if (k == 0) w.x_split_ready = false;
      Timed tm(this, "gemm", main_);
      tc_forward_layer(w.tc, L_, k, reinterpret_cast<const float*>(w.w), main_, lc_);
      return;
    }
    Timed tm(this, "gemm", main_);
    const int ni = L_.in(k), no = L_.out(k);
    const T* in = k == 0 ? w.x : w.act[static_cast<size_t>(k - 1)];
    const T* Wk = w.w + L_.w_off[static_cast<size_t>(k)];
    const T* bk = w.w + L_.b_off[static_cast<size_t>(k)];
    launch_gemm_simt<T>(kEpiForward, exact_, B_, no, ni, in, ni, 1, Wk, 1, ni, w.act[static_cast<size_t>(k)], no, bk,
                        k + 1 < L_.depth() ? 1 : 0, T(0), nullptr, main_, lc_);
  }

  // The push exchange's scatter is fused into the producers (dW epilogue, bias, loss) on the tensor-core path.
  bool fused_scatter() const {
    const bool exchange = !flat_nccl() && !reduce_folded() && alg_ != LSGD_B200_SEQUENTIAL;
    return exchange && split_ && use_tc_ && k_ > 1 && !dma(2) && !direct_;
  }
  // Push exchange (one worker per GPU, ordered global sum): the owner's K7 + broadcast + K8 for its own slot run as
  // one kernel on the comm stream; apply_bucket then updates the other members' slots only.
  // Which NVLink transfers go through the copy engines (no SM time, so the dW GEMMs they overlap keep their SMs)
  // instead of SM stores. LSGD_B200_DMA bit mask: 1 the k = 1 group payload (moves unchanged), 2 the member ->
  // owner scatter of the dW sub-slices (instead of the fused epilogue stores), 4 the group-sum push, 8 the average
  // fan-out. Default 1|2 (measured: N=2 +11%, N=4 +2%; 4 and 8 add a local round trip and were slower).
  int dma_bits() const {
    static const int v = std::getenv("LSGD_B200_DMA") ? std::atoi(std::getenv("LSGD_B200_DMA")) : 3;
    return v;
  }
  bool dma_push() const { return dma_bits() != 0; }
  bool dma(int bit) const { return (dma_bits() & bit) != 0; }
  bool own_slot_fused() const {
    const bool exchange = !flat_nccl() && !reduce_folded() && alg_ != LSGD_B200_SEQUENTIAL;
    return exchange && split_ && slice_comm_ == nullptr;
  }

  // Backward order. Reverse (dW_k right after delta_k) for groups of k >= 2, whose scatter -> reduce -> global chain
  // per bucket is long: the wide cfg3 middle layer's chains then overlap dX_1, dW_0 and the next forward's first GEMM
  // (2x2, A/B on one box: 971-974k vs 944-950k samples/s). dX-first otherwise: on one GPU there is nothing to
  // overlap, and with one worker per group (2x1) the payload copies running under the dW GEMMs slow them more than
  // the overlap gains (521k vs 558k; profiles/r1_order_ab.log). LSGD_B200_BWD_ORDER = reverse | dx_first overrides.
  // The fused-epilogue update writes W_k inside dW_k, so it keeps dX-first (dX_k must read W_k first).
  bool bwd_reverse() const {
    static const char* e = std::getenv("LSGD_B200_BWD_ORDER");
    if (fused_update()) return false;
    if (e) return std::strcmp(e, "reverse") == 0;
    return k_ >= 2;
  }
  // The backward as a sequence of ops: dX_k (x), or the weight-gradient GEMM block(s) of layer k (w; `blk` >= 0:
  // only the blk-th GEMM block of the layer). Default: reverse (w_{D-1}, x_{D-1}, ..., x_1, w_0) or dX-first
  // (x_{D-1} .. x_1, w_0 .. w_{D-1}) per bwd_reverse(). LSGD_B200_BWD_SEQ overrides with an explicit list such as
  // "x2,w1.0,x1,w0,w1.1,w2" (any order with dX_{k+1} before x_k / w_k, every block exactly once): which gradient is
  // ready when decides which exchange chains hide under the remaining GEMMs. Same kernels, same arithmetic.
  struct BwdOp {
    bool dx;
    int layer;
    std::vector<int> buckets;  // w: the buckets of the op's GEMM blocks, in row order
  };
  std::vector<std::vector<int>> layer_blocks(int k) const {  // buckets grouped by weight-gradient GEMM block
    std::vector<std::vector<int>> out;
    for (int b : geo_.layer_buckets[static_cast<size_t>(k)]) {
      if (geo_.buckets[static_cast<size_t>(b)].blk_rows > 0 || out.empty()) out.emplace_back();
      out.back().push_back(b);
    }
    return out;
  }
  std::vector<BwdOp> bwd_seq() const {
    const int D = synth_ ? 1 : L_.depth();
    std::vector<BwdOp> seq;
    auto all_w = [&](int k) {
      BwdOp op{false, k, {}};
      for (int b : geo_.layer_buckets[static_cast<size_t>(k)]) op.buckets.push_back(b);
      return op;
    };
    static const char* e = std::getenv("LSGD_B200_BWD_SEQ");
    if (e && *e && !fused_update() && !synth_) {
      std::vector<int> seen_x(static_cast<size_t>(D), 0), blk_done;
      std::string spec(e);
      size_t pos = 0;
      int nblk = 0;
      std::vector<std::vector<std::vector<int>>> blocks(static_cast<size_t>(D));
      for (int k = 0; k < D; ++k) {
        blocks[static_cast<size_t>(k)] = layer_blocks(k);
        nblk += static_cast<int>(blocks[static_cast<size_t>(k)].size());
      }
      std::vector<std::vector<int>> used(static_cast<size_t>(D));
      for (int k = 0; k < D; ++k) used[static_cast<size_t>(k)].assign(blocks[static_cast<size_t>(k)].size(), 0);
      int done = 0;
      while (pos <= spec.size()) {
        size_t end = spec.find(',', pos);
        if (end == std::string::npos) end = spec.size();
        const std::string tok = spec.substr(pos, end - pos);
        pos = end + 1;
        if (tok.empty()) continue;
        check<ConfigError>(tok[0] == 'x' || tok[0] == 'w', "LSGD_B200_BWD_SEQ: bad op '", tok, "'");
        const size_t dot = tok.find('.');
        const int k = std::atoi(tok.substr(1, dot == std::string::npos ? std::string::npos : dot - 1).c_str());
        check<ConfigError>(k >= 0 && k < D, "LSGD_B200_BWD_SEQ: layer out of range in '", tok, "'");
        // delta_k exists once dX_{k+1} ran (delta_{D-1} comes from the head)
        check<ConfigError>(k == D - 1 || seen_x[static_cast<size_t>(k + 1)], "LSGD_B200_BWD_SEQ: '", tok,
                           "' before x", k + 1);
        if (tok[0] == 'x') {
          check<ConfigError>(k >= 1 && !seen_x[static_cast<size_t>(k)], "LSGD_B200_BWD_SEQ: bad or repeated '", tok,
                             "'");
          seen_x[static_cast<size_t>(k)] = 1;
          seq.push_back(BwdOp{true, k, {}});
          continue;
        }
        auto& bl = blocks[static_cast<size_t>(k)];
        for (size_t i = 0; i < bl.size(); ++i) {
          if (dot != std::string::npos && static_cast<size_t>(std::atoi(tok.c_str() + dot + 1)) != i) continue;
          check<ConfigError>(!used[static_cast<size_t>(k)][i], "LSGD_B200_BWD_SEQ: block ", i, " of layer ", k,
                             " twice");
          used[static_cast<size_t>(k)][i] = 1;
          ++done;
          seq.push_back(BwdOp{false, k, bl[i]});
        }
      }
      check<ConfigError>(done == nblk, "LSGD_B200_BWD_SEQ: every weight-gradient block exactly once (", done, " of ",
                         nblk, ")");
      for (int k = 1; k < D; ++k) check<ConfigError>(seen_x[static_cast<size_t>(k)], "LSGD_B200_BWD_SEQ: x", k, " missing");
      return seq;
    }
    if (bwd_reverse()) {
      for (int k = D - 1; k >= 0; --k) {
        seq.push_back(all_w(k));
        if (k >= 1) seq.push_back(BwdOp{true, k, {}});
      }
    } else {
      for (int k = D - 1; k >= 1; --k) seq.push_back(BwdOp{true, k, {}});
      for (int k = 0; k < D; ++k) seq.push_back(all_w(k));
    }
    return seq;
  }
  // One worker, one group (N = 1): the gradient is final when produced, so the update runs in the producers'
  // epilogues (dW GEMM, bias) and the separate update pass over g disappears.
  // Measured version_at_compute: on for recorded runs of bounded length (run_train with history / phases), off
  // for the bench and the open-ended rank API (two 1-thread kernels per bucket and layer per step).
  bool track_versions() const {
    return !synth_ && (hist_rows_ > 0 || spec_.c.record_phases || spec_.track_versions) &&
           spec_.iterations() <= (1 << 20) && !fused_update();
  }
  void note_version(Worker& w, int b, int64_t rounds, cudaStream_t st) {
    if (w.ver) launch_store_u64(w.ver + b, static_cast<unsigned long long>(rounds), st, lc_);
  }
  void versions(int worker, int64_t* out, int64_t n) override {
    synchronize();
    Worker& w = find(worker);
    const int D = L_.depth();
    for (int64_t t = 0; t < n; ++t) {
      if (!w.ver_log || t >= spec_.iterations()) {
        out[t] = -1;
        continue;
      }
      long long m = -1;
      for (int k = 0; k < D; ++k) {
        const long long v = w.ver_log[t * D + k];
        m = (k == 0 || v < m) ? v : m;
      }
      out[t] = m;
    }
  }

  bool fused_update() const {
    // opt-in (LSGD_B200_FUSED_UPDATE=1): bitwise the separate pass, but its epilogue is latency-bound today
    static const bool on = std::getenv("LSGD_B200_FUSED_UPDATE") != nullptr;
    return on && alg_ == LSGD_B200_LSGD && split_ && use_tc_ && reduce_folded() && !spec_.c.record_phases;
  }
  FusedUpdate fused_update_args(Worker& w, int64_t first_param, const Bucket* loss_bucket) {
    FusedUpdate u;
    u.w = reinterpret_cast<float*>(w.w + first_param);
    u.v = w.v ? reinterpret_cast<float*>(w.v + first_param) : nullptr;
    u.hi = w.tc.w_hi + first_param;
    u.lo = w.tc.w_lo + first_param;
    u.lr = static_cast<float>(spec_.lr(t_cur_));
    u.momentum = static_cast<float>(spec_.c.momentum);
    u.weight_decay = static_cast<float>(spec_.c.weight_decay);
    u.mode = spec_.c.mode;
    u.add_zero = 1;  // the communicator's zero (executors.cpp:278), then / N
    u.post_div = static_cast<float>(N_);
    u.bad = bad_dev_;
    if (loss_bucket) {
      u.loss_in = reinterpret_cast<const float*>(w.payload + geo_.loss_at);
      u.loss_out = reinterpret_cast<float*>(w.loss_hist + (t_cur_ % kLossCap));
    }
    return u;
  }
  BucketScatter bucket_scatter(Worker& w, int b, int64_t e0) {
    const Bucket& bk = geo_.buckets[static_cast<size_t>(b)];
    const auto members = group_members(w.g);
    BucketScatter sc;
    sc.n = k_;
    sc.S = bk.S;
    sc.e0 = e0;
    for (int j = 0; j < k_; ++j)
      sc.dst[j] = reinterpret_cast<float*>(j == w.j ? w.payload + bk.poff + static_cast<int64_t>(j) * bk.S
                                                    : peer_stage(members[static_cast<size_t>(j)], w.j) + bk.goff);
    return sc;
  }

  void head(Worker& w) {
    if (synth_) return;
    T* loss_out = w.payload + geo_.loss_at;
    if (fused_scatter()) {  // the loss slot (bucket-local index n of the last bucket) goes to its owner
      const int lb = static_cast<int>(geo_.buckets.size()) - 1;
      const Bucket& bk = geo_.buckets[static_cast<size_t>(lb)];
      const BucketScatter sc = bucket_scatter(w, lb, 0);
      const int j = static_cast<int>(bk.n / bk.S);
      loss_out = reinterpret_cast<T*>(sc.dst[j] + (bk.n - j * bk.S));
    }
    Timed tm(this, "head", main_);
    if (use_tc_) {
      tc_head(w.tc, L_, w.y, reinterpret_cast<float*>(w.sample_loss), reinterpret_cast<float*>(loss_out), main_, lc_);
      return;
    }
    const int depth = L_.depth();
    launch_softmax_xent<T>(w.act[static_cast<size_t>(depth - 1)], w.y, B_, L_.out(depth - 1), delta_buf(w, depth - 1),
                           w.sample_loss, main_, lc_);
    launch_mean_loss<T>(w.sample_loss, B_, loss_out, main_, lc_);
  }

  // Weight gradient of bucket b (a row block of dW_k, plus db_k for the layer's last block).
  void backward_bucket(Worker& w, int b) {
    tag_ = b;
    const Bucket& bk0 = geo_.buckets[static_cast<size_t>(b)];
    if (bk0.blk_rows == 0) return;  // inside a block: its first bucket's GEMM wrote it
    Bucket bk = bk0;                  // the whole block: rows, and the bias when it ends the layer
    bk.rows = bk0.blk_rows;
    bk.bias = bk0.blk_bias;
    const int k = bk.layer;
    const int ni = L_.in(k), no = L_.out(k);
    T* gW = w.payload + bk.poff;
    T* gb = gW + static_cast<int64_t>(bk.rows) * ni;
    if (use_tc_) {
      const bool fuse = fused_scatter();
      const bool fupd = fused_update();
      check<Error>(!(fuse || fupd) || bk.rows == bk0.rows,
                   "fused scatter / update need one exchange bucket per weight-gradient block");
      // the layer's bias gradient belongs to its last bucket (the block that ends the layer computes it)
      const int bb = bk.bias ? geo_.layer_buckets[static_cast<size_t>(k)].back() : b;
      bias_side_[bb] = bk.bias && bias_ && !fuse && !fupd && alg_ == LSGD_B200_LSGD && !flat_nccl();
      if (bias_side_[bb]) {
        // db_k = colsum(delta_k) / B needs none of the dW GEMM's results: it runs on the bias stream beside it
        // (the bias kernel was ~4% of the one-GPU step on the main stream); the bucket's exchange / update wait for it
        LSGD_CUDA(cudaEventRecord(ev_bias_src_, main_));
        LSGD_CUDA(cudaStreamWaitEvent(bias_, ev_bias_src_, 0));
        {
          Timed tb(this, "bias", bias_);
          tc_backward_bias(w.tc, L_, k, reinterpret_cast<float*>(gb), bias_, lc_, nullptr, nullptr);
        }
        LSGD_CUDA(cudaEventRecord(ev_bias_[bb], bias_));
      }
      {
        Timed tm(this, "gemm", main_);
        const BucketScatter sc = fuse ? bucket_scatter(w, b, 0) : BucketScatter{};
        const FusedUpdate fu = fupd ? fused_update_args(w, bk.pstart, nullptr) : FusedUpdate{};
        tc_backward_dw(w.tc, L_, k, bk.row0, bk.rows, reinterpret_cast<float*>(gW), main_, lc_, fuse ? &sc : nullptr,
                       fupd ? &fu : nullptr);
      }
      if (bk.bias && !bias_side_[bb]) {
        Timed tb(this, "bias", main_);
        const BucketScatter sc = fuse ? bucket_scatter(w, b, static_cast<int64_t>(bk.rows) * ni) : BucketScatter{};
        const FusedUpdate fu =
            fupd ? fused_update_args(w, L_.b_off[static_cast<size_t>(k)], bk.loss ? &bk : nullptr) : FusedUpdate{};
        tc_backward_bias(w.tc, L_, k, reinterpret_cast<float*>(gb), main_, lc_, fuse ? &sc : nullptr,
                         fupd ? &fu : nullptr);
      }
      if (fuse) {  // this member's sub-slices of bucket b are in their owners' stage
        const auto members = group_members(w.g);
        SignalList sl{};
        int n = 0;
        for (int j = 0; j < k_; ++j)
          if (j != w.j) sl.f[n++] = peer_flag_word(members[static_cast<size_t>(j)], kStaged + b * kMaxPeers + w.j);
        launch_signal_many(sl, n, static_cast<unsigned long long>(t_cur_ + 1), main_, lc_);
      }
      return;
    }
    Timed tm(this, "gemm", main_);
    const T* dcur = delta_buf(w, k);
    const T* aprev = k == 0 ? w.x : w.act[static_cast<size_t>(k - 1)];
    launch_gemm_simt<T>(kEpiWeightGrad, exact_, bk.rows, ni, B_, dcur + bk.row0, 1, no, aprev, ni, 1, gW, ni, nullptr,
                        0, static_cast<T>(B_), nullptr, main_, lc_);
    if (bk.bias) launch_bias_grad<T>(dcur, B_, no, gb, main_, lc_);
  }

  // Input gradient of layer k (masked delta of layer k-1); layer 0 has none (mlp.cpp:116).
  void backward_input(Worker& w, int k) {
    tag_ = 200 + k;
    if (k == 0) return;
    Timed tm(this, "gemm", main_);
    if (use_tc_) {
      tc_backward_dx(w.tc, L_, k, main_, lc_);
      return;
    }
    const int ni = L_.in(k), no = L_.out(k);
    const T* Wk = w.w + L_.w_off[static_cast<size_t>(k)];
    launch_gemm_simt<T>(kEpiInputGrad, exact_, B_, ni, no, delta_buf(w, k), no, 1, Wk, ni, 1, delta_buf(w, k - 1), ni,
                        nullptr, 0, T(0), w.act[static_cast<size_t>(k - 1)], main_, lc_);
  }

  void backward_layer(Worker& w, int k) {  // compute_gradient (kernel seam): all blocks, then dX
    for (int b : geo_.layer_buckets[static_cast<size_t>(k)]) backward_bucket(w, b);
    backward_input(w, k);
  }

  // The global stage of the push exchange sliced over the G owners of each slot (reduce-scatter + all-gather, see
  // exchange_push_bucket). LSGD_B200_SLICED_GLOBAL = 0 / 1 forces it; default: on for G > 2, where the whole-slot
  // form's (G-1) slot lengths of egress per owner dominate (4x1: 888k vs 459k samples/s), and for one worker per
  // group, where every GPU would otherwise sum and update all P parameters (2x1: 591-593k vs 562k); off for 2 x k
  // with k >= 2 (2x2: 1.000M vs 936k). profiles/r2_layouts_n4_*.log, r2_n2_ab.log.
  bool sliced_global() const {
    static const char* e = std::getenv("LSGD_B200_SLICED_GLOBAL");
    if (G_ <= 1 || !own_slot_fused() || N_ > kMaxPeers || direct_) return false;  // one arrived word per source
    if (e) return std::atoi(e) != 0;
    return G_ > 2 || k_ == 1;
  }
  // Members pull the slot owners' averages straight into their update (NVLink loads from the owner's gbar) instead
  // of the owner pushing them into every member's gfull: no gfull write + read (8 B per parameter on (k-1)/k of P)
  // and no remote stores in the owner's global kernel. Whole-slot form only (k >= 2). LSGD_B200_PULL_AVG = 0 / 1.
  bool pull_avg() const {
    static const char* e = std::getenv("LSGD_B200_PULL_AVG");
    if (k_ < 2 || !own_slot_fused() || sliced_global() || direct_) return false;
    return e ? std::atoi(e) != 0 : false;
  }
  int64_t piece_len(const Bucket& bk) const {  // elements of each of the G pieces of a slot (64-aligned)
    return sliced_global() ? round_up((bk.S + G_ - 1) / G_, kAlign) : bk.S;
  }
  // arrived flag of the averaged piece (slot j, piece q): one word per source owner
  int arrived_index(int j, int q) const { return sliced_global() ? j * G_ + q : j; }

  std::vector<int> group_members(int g) const {
    std::vector<int> m;
    for (int i = g * k_; i < (g + 1) * k_; ++i) m.push_back(i);
    return m;
  }

  // ------------------------------------------------------------------------------------------ collectives
  // One worker per group and one group: the communicator's (g + 0.0) / N is folded into the update (no copy).
  bool reduce_folded() const { return alg_ != LSGD_B200_SEQUENTIAL && k_ == 1 && G_ == 1 && !flat_comm_; }
  bool flat_nccl() const { return alg_ == LSGD_B200_CSGD && flat_comm_ != nullptr; }

  // K6 for bucket b: slot (g, j) sums sub-slice j of its group's payloads in ascending worker order, adds the
  // communicator's zero vector, divides by N (transport.cpp:27-48; executors.cpp:278-288).
  void reduce_bucket(Worker& w, int b, int64_t t, cudaStream_t st) {
    const Bucket& bk = geo_.buckets[static_cast<size_t>(b)];
    const int par = static_cast<int>(t & 1);
    auto members = group_members(w.g);
    wait(members, kFlagGrad, b, static_cast<unsigned long long>(t + 1), st);
    SrcList<T> src{};
    for (int i = 0; i < k_; ++i) src.p[i] = peer_payload(members[static_cast<size_t>(i)]) + bk.poff + w.j * bk.S;
    T* dst = (G_ == 1 ? w.gbar : w.s[par]) + bk.goff;
    {
      Timed tm(this, "reduce", st);
      launch_ordered_sum<T>(src, k_, bk.S, dst, alg_ == LSGD_B200_LSGD, static_cast<T>(N_), st, lc_);
    }
    if (G_ == 1) push_bucket(w, b, t, st);
    else if (slice_comm_ == nullptr) signal(w, kFlagSlice, b, static_cast<unsigned long long>(t + 1), st);
  }

  // K7 for bucket b: average across communicators (executors.cpp:290-295) with NCCL over the G slot-j owners (or
  // the ordered peer sum), on the comm stream.
  void global_bucket(Worker& w, int b, int64_t t, cudaStream_t st) {
    if (G_ == 1) return;
    const Bucket& bk = geo_.buckets[static_cast<size_t>(b)];
    const int par = static_cast<int>(t & 1);
    if (slice_comm_) {
      Timed tm(this, "global", st);
      nccl_call(st, slice_comm_, [&] {
        return ncclAllReduce(w.s[par] + bk.goff, w.gbar + bk.goff, static_cast<size_t>(bk.S), nccl_type(), ncclSum,
                             slice_comm_, st);
      });
    } else {
      std::vector<int> owners;
      for (int g = 0; g < G_; ++g) owners.push_back(g * k_ + w.j);
      wait(owners, kFlagSlice, b, static_cast<unsigned long long>(t + 1), st);
      SrcList<T> src{};
      for (int g = 0; g < G_; ++g) src.p[g] = peer_s(owners[static_cast<size_t>(g)], par) + bk.goff;
      Timed tm(this, "global", st);
      launch_ordered_sum<T>(src, G_, bk.S, w.gbar + bk.goff, false, T(0), st, lc_);
    }
    push_bucket(w, b, t, st);
  }

  // Push exchange of bucket b (one worker per GPU; comm stream). Same arithmetic as reduce_bucket/global_bucket,
  // but every cross-GPU byte moves as an NVLink store and every sum reads local HBM:
  //   1. scatter: member i stores its sub-slices j != i into owner j's stage[i] (+ staged flag);
  //   2. K6: owner i sums stage[0..k-1] (its own sub-slice from its payload) in ascending member order, + 0.0, / N;
  //   3. G == 1: the sum goes straight into every member's gfull; G > 1 (ordered): into every slot-i owner's
  //      gstage[par][g] (+ gsum flag), then K7 sums gstage[par][0..G-1] in ascending group order into the members'
  //      gfull; G > 1 (nccl): NCCL allreduce over the slot owners, then the push;
  //   4. arrival flags released to every member (the update waits on them).
  T* peer_stage(int wid, int m) const {
    return reinterpret_cast<T*>(base(wid) + geo_.peer.stage) + static_cast<int64_t>(m) * geo_.Sg;
  }
  T* peer_gstage(int wid, int par, int g) const {
    return reinterpret_cast<T*>(base(wid) + geo_.peer.gstage[par]) + static_cast<int64_t>(g) * geo_.Sg;
  }
  unsigned long long* peer_flag_word(int wid, int idx) const {
    return reinterpret_cast<unsigned long long*>(base(wid) + geo_.peer.flags) + idx;
  }
  // max_lead (protocol check, wait_flags_kernel): stage and gfull are single-buffered and their producers are gated
  // by this consumer's own progress, so a staged / arrived flag is never above the round waited for (lead 0);
  // gstage is double-buffered by round parity (lead 1).
  void wait_own(Worker& w, int first, int n_words, int skip, unsigned long long target, cudaStream_t st,
                unsigned long long max_lead) {
    FlagList fl{};
    int n = 0;
    for (int q = 0; q < n_words; ++q)
      if (q != skip) fl.f[n++] = w.flags + first + q;
    if (n) {
      Timed tm(this, "wait", st);  // timeline only: when this rank's peers' data for the stage arrived
      launch_wait_flags(fl, n, target, timeout_ns(), timed_out_dev_, st, lc_, max_lead);
    }
  }
  // Direct two-hop exchange (direct_exchange(), engine.hpp): this GPU's sub-slice j goes by copy engine to the
  // slot-j owner of every group (stage[par][my id]); the owner of slot `me` then sums all N sub-slices in the
  // reference's order, updates its slot and pushes the average to its group's members (the broadcast hop).
  T* peer_stage_direct(int wid, int par, int src) const {
    return reinterpret_cast<T*>(base(wid) + geo_.peer.stage) +
           (static_cast<int64_t>(par) * N_ + src) * geo_.Sg;
  }
  void exchange_direct_bucket(Worker& w, int b, int64_t t, cudaStream_t st) {
    const Bucket& bk = geo_.buckets[static_cast<size_t>(b)];
    const int par = static_cast<int>(t & 1);
    const unsigned long long round = static_cast<unsigned long long>(t + 1);
    const int me = w.j;
    SignalList sl{};
    int n = 0;
    {
      Timed tm(this, "scatter", st);
      for (int q = 0; q < G_; ++q)
        for (int j = 0; j < k_; ++j) {
          const int owner = q * k_ + j;
          if (owner == w.id) continue;
          LSGD_CUDA(cudaMemcpyAsync(peer_stage_direct(owner, par, w.id) + bk.goff,
                                    w.payload + bk.poff + static_cast<int64_t>(j) * bk.S, sizeof(T) * bk.S,
                                    cudaMemcpyDeviceToDevice, st));
          sl.f[n++] = peer_flag_word(owner, kStaged + b * kMaxPeers + w.id);
        }
    }
    launch_signal_many(sl, n, round, st, lc_);
    // every other GPU's sub-slice `me` of round t; a source may already be one round ahead (double-buffered)
    wait_own(w, kStaged + b * kMaxPeers, N_, w.id, round, st, 1);
    GlobalUpdateArgs<T> ga;
    for (int id = 0; id < N_; ++id)
      ga.src.p[id] = id == w.id ? w.payload + bk.poff + static_cast<int64_t>(me) * bk.S
                                : peer_stage_direct(w.id, par, id) + bk.goff;
    ga.direct = true;
    ga.k = k_;
    ga.G = G_;
    ga.g = w.g;
    ga.add_zero = alg_ == LSGD_B200_LSGD;
    ga.divisor = static_cast<T>(N_);
    ga.len = bk.S;
    SignalList others{};
    const auto members = group_members(w.g);
    for (int m = 0; m < k_; ++m) {
      if (m == me) continue;
      others.f[ga.n_push] = peer_arrived(members[static_cast<size_t>(m)], b, me);
      ga.push.p[ga.n_push++] = peer_gfull(members[static_cast<size_t>(m)]) + bk.poff + static_cast<int64_t>(me) * bk.S;
    }
    ga.first = static_cast<int64_t>(me) * bk.S;
    ga.n_params = bk.n;
    ga.w = w.w + bk.pstart;
    ga.v = w.v ? w.v + bk.pstart : nullptr;
    ga.mode = spec_.c.mode;
    ga.lr = static_cast<T>(spec_.lr(t));
    ga.momentum = static_cast<T>(spec_.c.momentum);
    ga.weight_decay = static_cast<T>(spec_.c.weight_decay);
    ga.loss_out = bk.loss ? w.loss_hist + (t % kLossCap) : nullptr;
    ga.bad = bad_dev_;
    if constexpr (std::is_same_v<T, float>) {
      if (use_tc_ && !w.tc.weights_split_in_smem) {
        ga.w_hi = w.tc.w_hi + bk.pstart;
        ga.w_lo = w.tc.w_lo + bk.pstart;
      }
    }
    const int n_remote = ga.n_push;
    {
      Timed tm(this, "global", st);
      launch_global_update<T>(ga, exact_, st, lc_);
    }
    if (n_remote) launch_signal_many(others, n_remote, round, st, lc_);
    LSGD_CUDA(cudaEventRecord(ev_gupd_[b], st));
  }

  // Transport conformance under jitter (test_transport.cpp:135-269, the reference's jitter cases): with
  // LSGD_B200_JITTER_US = J every rank delays each bucket's exchange by a pseudo-random 0..J us (seeded by rank,
  // step and bucket) on its comm stream, so peers arrive at every flag in varying orders; results must not change.
  void exchange_jitter(int b, int64_t t, cudaStream_t st) {
    static const double j_us = std::getenv("LSGD_B200_JITTER_US") ? std::atof(std::getenv("LSGD_B200_JITTER_US")) : 0;
    if (j_us <= 0) return;
    SplitMix64 r(0x5eedull + static_cast<uint64_t>(workers_[0]) * 1000003ull + static_cast<uint64_t>(t) * 131ull +
                 static_cast<uint64_t>(b));
    launch_sleep(1e-6 * j_us * static_cast<double>(r.u64() % 1024) / 1023.0, st, lc_);
  }

  void exchange_push_bucket(Worker& w, int b, int64_t t, cudaStream_t st) {
    tag_ = b;
    exchange_jitter(b, t, st);
    const Bucket& bk = geo_.buckets[static_cast<size_t>(b)];
    const int par = static_cast<int>(t & 1);
    const unsigned long long round = static_cast<unsigned long long>(t + 1);
    const auto members = group_members(w.g);
    const int me = w.j;
    if (direct_) {
      exchange_direct_bucket(w, b, t, st);
      return;
    }
    if (k_ > 1 && fused_scatter()) {
      wait_own(w, kStaged + b * kMaxPeers, k_, me, round, st, 0);  // the producers already scattered (main stream)
    } else if (k_ > 1) {
      SrcList<T> src{};
      DstList<T> dst{};
      SignalList sl{};
      int n = 0;
      for (int j = 0; j < k_; ++j) {
        if (j == me) continue;
        src.p[n] = w.payload + bk.poff + static_cast<int64_t>(j) * bk.S;
        dst.p[n] = peer_stage(members[static_cast<size_t>(j)], me) + bk.goff;
        sl.f[n] = peer_flag_word(members[static_cast<size_t>(j)], kStaged + b * kMaxPeers + me);
        ++n;
      }
      {
        Timed tm(this, "scatter", st);
        if (dma(2)) {
          for (int q = 0; q < n; ++q)
            LSGD_CUDA(cudaMemcpyAsync(dst.p[q], src.p[q], sizeof(T) * bk.S, cudaMemcpyDeviceToDevice, st));
        } else {
          launch_copy_pairs<T>(src, dst, n, bk.S, st, lc_);
        }
      }
      launch_signal_many(sl, n, round, st, lc_);
      wait_own(w, kStaged + b * kMaxPeers, k_, me, round, st, 0);
    }
    SrcList<T> src{};
    for (int m = 0; m < k_; ++m)
      src.p[m] = m == me ? w.payload + bk.poff + static_cast<int64_t>(me) * bk.S : w.blk_stage(m) + bk.goff;
    DstList<T> gfull{};
    SignalList arrived{};
    for (int m = 0; m < k_; ++m) {
      gfull.p[m] = peer_gfull(members[static_cast<size_t>(m)]) + bk.poff + static_cast<int64_t>(me) * bk.S;
      arrived.f[m] = peer_arrived(members[static_cast<size_t>(m)], b, me);
    }
    const bool lsgd = alg_ == LSGD_B200_LSGD;
    if (own_slot_fused()) {
      // Sliced global stage (sliced_global()): slot `me` is cut into G pieces; the owner in group q computes the
      // average of piece q only. Owner (g, me) pushes piece q of its group sum to owner (q, me) (reduce-scatter
      // over the slot's G owners), sums piece g over the groups in ascending order, updates its parameters of that
      // piece and pushes its average to all N-1 other GPUs (all-gather). Same per-element arithmetic, so the same
      // bits as the whole-slot form, at 2(G-1)/G instead of G-1 slot lengths of egress for the global stage.
      // Unsliced: the piece is the whole slot, the group sum goes to all G-1 other owners and the average to the
      // k-1 group members.
      const bool sl = sliced_global();
      const int64_t Q = piece_len(bk);
      const int pg = sl ? w.g : 0;                        // the piece this owner averages
      const int64_t p0 = static_cast<int64_t>(pg) * Q;    // its offset inside the slot
      const int64_t plen = std::max<int64_t>(0, std::min(Q, bk.S - p0));
      // G > 1: the slot sum (or, sliced, each other owner's piece of it) goes to the other groups' slot owners
      if (G_ > 1) {
        DstList<T> gdst{};
        SignalList gsig{};
        int64_t goff_q[kMaxPeers] = {}, glen_q[kMaxPeers] = {};
        int n = 0;
        for (int g = 0; g < G_; ++g) {
          if (g == w.g) continue;
          const int owner = g * k_ + me;
          const int64_t q0 = sl ? static_cast<int64_t>(g) * Q : 0;  // piece g goes to the owner in group g
          goff_q[n] = q0;
          glen_q[n] = sl ? std::max<int64_t>(0, std::min(Q, bk.S - q0)) : bk.S;
          gdst.p[n] = peer_gstage(owner, par, w.g) + bk.goff + q0;
          gsig.f[n++] = peer_flag_word(owner, kGsum + b * kMaxPeers + w.g);
        }
        if (k_ == 1 && dma(1)) {
          // one member per group: the group "sum" is the payload itself, so the copy engines move it (no SM time);
          // the receiving owner applies the group's (+0.0, /N) when it reads it
          Timed tm(this, "reduce", st);
          for (int q = 0; q < n; ++q)
            if (glen_q[q])
              LSGD_CUDA(cudaMemcpyAsync(gdst.p[q], src.p[0] + goff_q[q], sizeof(T) * glen_q[q],
                                        cudaMemcpyDeviceToDevice, st));
        } else if (k_ > 1 && dma(4)) {  // the group sum lands locally, the copy engines forward it
          Timed tm(this, "reduce", st);
          DstList<T> loc{};
          loc.p[0] = w.s[par] + bk.goff;
          launch_reduce_push<T>(src, k_, bk.S, loc, 1, lsgd, static_cast<T>(N_), st, lc_);
          for (int q = 0; q < n; ++q)
            if (glen_q[q])
              LSGD_CUDA(cudaMemcpyAsync(gdst.p[q], loc.p[0] + goff_q[q], sizeof(T) * glen_q[q],
                                        cudaMemcpyDeviceToDevice, st));
        } else if (sl) {  // one ordered-sum launch per destination piece
          Timed tm(this, "reduce", st);
          for (int q = 0; q < n; ++q) {
            if (!glen_q[q]) continue;
            SrcList<T> ps{};
            for (int m = 0; m < k_; ++m) ps.p[m] = src.p[m] + goff_q[q];
            DstList<T> one{};
            one.p[0] = gdst.p[q];
            launch_reduce_push<T>(ps, k_, glen_q[q], one, 1, lsgd, static_cast<T>(N_), st, lc_);
          }
        } else {
          Timed tm(this, "reduce", st);
          launch_reduce_push<T>(src, k_, bk.S, gdst, n, lsgd, static_cast<T>(N_), st, lc_);
        }
        launch_signal_many(gsig, n, round, st, lc_);
        wait_own(w, kGsum + b * kMaxPeers, G_, w.g, round, st, 1);
      }
      // K7 + broadcast + K8 of this owner's piece (the whole slot unsliced) in one pass
      GlobalUpdateArgs<T> ga;
      for (int m = 0; m < k_; ++m) ga.src.p[m] = src.p[m] + p0;
      ga.k = k_;
      for (int g = 0; g < G_; ++g) ga.gsum.p[g] = w.blk_gstage(par, g) + bk.goff + p0;
      ga.G = G_;
      ga.g = w.g;
      ga.gsum_raw = G_ > 1 && k_ == 1 && dma(1);
      ga.add_zero = lsgd;
      ga.divisor = static_cast<T>(N_);
      ga.len = plen;
      SignalList others{};
      const int arr = arrived_index(me, pg);
      for (int d = 0; d < N_; ++d) {  // sliced: every other GPU; unsliced: the other members of this group
        if (d == w.id || (!sl && d / k_ != w.g)) continue;
        others.f[ga.n_push] = peer_arrived(d, b, arr);
        ga.push.p[ga.n_push++] = peer_gfull(d) + bk.poff + static_cast<int64_t>(me) * bk.S + p0;
      }
      ga.first = static_cast<int64_t>(me) * bk.S + p0;
      ga.n_params = bk.n;
      ga.w = w.w + bk.pstart;
      ga.v = w.v ? w.v + bk.pstart : nullptr;
      ga.mode = spec_.c.mode;
      ga.lr = static_cast<T>(spec_.lr(t));
      ga.momentum = static_cast<T>(spec_.c.momentum);
      ga.weight_decay = static_cast<T>(spec_.c.weight_decay);
      ga.loss_out = bk.loss ? w.loss_hist + (t % kLossCap) : nullptr;
      ga.bad = bad_dev_;
      if constexpr (std::is_same_v<T, float>) {
        if (use_tc_ && !w.tc.weights_split_in_smem) {  // the GEMMs read pre-split weights: refresh this slot's too
          ga.w_hi = w.tc.w_hi + bk.pstart;
          ga.w_lo = w.tc.w_lo + bk.pstart;
        }
      }
      if (pull_avg()) {  // the members read the average from this owner's gbar after the arrival flag
        ga.n_push = 0;
        ga.out_local = w.gbar + bk.goff + p0;
      }
      int n_signal = ga.n_push;  // members whose arrival flag this owner releases
      if (mc_gfull_ && !sl) {    // NVLS: one multicast store per vector instead of k-1 unicast pushes
        ga.mc = mc_gfull_ + bk.poff + static_cast<int64_t>(me) * bk.S + p0;
        ga.n_push = 0;
      }
      DstList<T> remote = ga.push;
      const int n_remote = ga.n_push;
      const bool fan_dma = dma(8) && n_remote > 0;
      if (fan_dma) {  // average stored locally once, the copy engines fan it out
        ga.n_push = 0;
        ga.out_local = w.gbar + bk.goff + p0;
      }
      if (plen > 0) {
        Timed tm(this, "global", st);
        launch_global_update<T>(ga, exact_, st, lc_);
      }
      if (fan_dma && plen > 0)
        for (int q = 0; q < n_remote; ++q)
          LSGD_CUDA(cudaMemcpyAsync(remote.p[q], ga.out_local, sizeof(T) * plen, cudaMemcpyDeviceToDevice, st));
      if (pull_avg()) {
        int nm = 0;
        SignalList mem{};
        for (int d = 0; d < N_; ++d)
          if (d != w.id && d / k_ == w.g) mem.f[nm++] = peer_arrived(d, b, arr);
        if (nm) launch_signal_many(mem, nm, round, st, lc_);
      } else if (n_signal) {
        launch_signal_many(others, n_signal, round, st, lc_);
      }
      LSGD_CUDA(cudaEventRecord(ev_gupd_[b], st));
      return;
    }
    if (G_ == 1) {
      Timed tm(this, "reduce", st);
    } else {
      DstList<T> sdst{};
      sdst.p[0] = w.s[par] + bk.goff;
      {
        Timed tm(this, "reduce", st);
        launch_reduce_push<T>(src, k_, bk.S, sdst, 1, lsgd, static_cast<T>(N_), st, lc_);
      }
      {
        Timed tm(this, "global", st);
        nccl_call(st, slice_comm_, [&] {
          return ncclAllReduce(w.s[par] + bk.goff, w.gbar + bk.goff, static_cast<size_t>(bk.S), nccl_type(),
                               ncclSum, slice_comm_, st);
        });
      }
      SrcList<T> one{};
      one.p[0] = w.gbar + bk.goff;
      Timed tm(this, "broadcast", st);
      launch_reduce_push<T>(one, 1, bk.S, gfull, k_, false, T(0), st, lc_);
    }
    launch_signal_many(arrived, k_, round, st, lc_);
  }

  // K8 for bucket b of round u (executors.cpp:210-229): pull the k averaged sub-slices of the group, apply
  // sgd_update to the bucket's parameters, check finiteness, record the loss (last bucket).
  void apply_bucket(Worker& w, int b, int64_t u, cudaStream_t st) {
    tag_ = b;
    const Bucket& bk = geo_.buckets[static_cast<size_t>(b)];
    const size_t wi = widx(w);
    if (b == 0) phase_mark(wi, u, 4, 0, st);
    UpdateArgs<T> a{};
    a.slice_len = bk.S;
    a.n_params = bk.n;
    if (alg_ == LSGD_B200_SEQUENTIAL || reduce_folded() || flat_nccl()) {
      for (int j = 0; j < k_; ++j) a.slices.p[j] = w.payload + bk.poff + j * bk.S;
      if (reduce_folded()) {
        a.add_zero = alg_ == LSGD_B200_LSGD ? 1 : 0;
        a.post_div = static_cast<T>(N_);
      }
      if (flat_nccl()) a.post_div = static_cast<T>(N_);  // the per-worker /N after the flat allreduce (:170)
    } else {
      const bool own = own_slot_fused();  // this worker's own slot (piece) was updated by its fused global kernel
      const bool sl = sliced_global();
      const int n_pieces = sl ? G_ : 1;
      const int64_t Q = piece_len(bk);
      const int pg = sl ? w.g : 0;
      const int64_t p0 = static_cast<int64_t>(pg) * Q;
      const int64_t plen = std::max<int64_t>(0, std::min(Q, bk.S - p0));
      // the other (slot, piece) averages of round u have been pushed into this worker's gfull (one flag per
      // source owner; kMaxPeers words per bucket hold all N of them); waited in chunks of kMaxPeers
      std::vector<const volatile unsigned long long*> srcs;
      for (int j = 0; j < k_; ++j)
        for (int q = 0; q < n_pieces; ++q) {
          if (own && j == w.j && q == pg) continue;
          const int64_t q0 = static_cast<int64_t>(q) * Q;
          if (sl && std::min(Q, bk.S - q0) <= 0) continue;  // empty trailing piece: nothing is pushed
          srcs.push_back(peer_arrived(w.id, b, arrived_index(j, q)));
        }
      for (size_t i0 = 0; i0 < srcs.size(); i0 += kMaxPeers) {
        FlagList fl{};
        int nf = 0;
        for (size_t i = i0; i < srcs.size() && nf < kMaxPeers; ++i) fl.f[nf++] = srcs[i];
        launch_wait_flags(fl, nf, static_cast<unsigned long long>(u + 1), timeout_ns(), timed_out_dev_, st, lc_, 0);
      }
      a.slices.p[0] = w.gfull + bk.poff;
      a.slice_len = bk.S * k_;
      if (pull_avg()) {  // slot j's average straight from its owner's gbar over NVLink (own slot: skipped below)
        const auto mem = group_members(w.g);
        for (int j = 0; j < k_; ++j) a.slices.p[j] = peer_gbar(mem[static_cast<size_t>(j)]) + bk.goff;
        a.slice_len = bk.S;
      }
      if (own) {
        a.skip_lo = static_cast<int64_t>(w.j) * bk.S + p0;
        a.skip_hi = a.skip_lo + plen;
        if (k_ == 1 && n_pieces == 1) {  // nothing left to update here
          if (b == 0) {
            phase_mark(wi, u, 4, 1, st);
            phase_mark(wi, u, 5, 0, st);
          }
          return;
        }
      }
    }
    if (b == 0) {
      phase_mark(wi, u, 4, 1, st);
      phase_mark(wi, u, 5, 0, st);
    }
    a.w = w.w + bk.pstart;
    a.v = w.v ? w.v + bk.pstart : nullptr;
    a.mode = spec_.c.mode;
    a.lr = static_cast<T>(spec_.lr(u));
    a.momentum = static_cast<T>(spec_.c.momentum);
    a.weight_decay = static_cast<T>(spec_.c.weight_decay);
    a.loss_out = bk.loss ? w.loss_hist + (u % kLossCap) : nullptr;
    a.bad = bad_dev_;
    if (use_tc_ && !w.tc.weights_split_in_smem) {
      a.w_hi = w.tc.w_hi + bk.pstart;
      a.w_lo = w.tc.w_lo + bk.pstart;
    }
    Timed tm(this, "update", st);
    launch_update<T>(a, exact_, st, lc_);
  }

  void after_update(Worker& w, int64_t u, cudaStream_t st) {
    phase_mark(widx(w), u, 5, 1, st);
    if (hist_rows_ > 0 && w.id == workers_[0] && u + 1 < hist_rows_)
      LSGD_CUDA(cudaMemcpyAsync(hist_ + (u + 1) * geo_.P, w.w, sizeof(T) * geo_.P, cudaMemcpyDeviceToHost, st));
  }

  // ------------------------------------------------------------------------------------------ one step
  void issue_one(int64_t t, const int32_t* given, bool shard_only) {
    t_cur_ = t;
    const int D = synth_ ? 1 : L_.depth();
    const int NB = nb_;
    const auto& LB = geo_.layer_buckets;
    current_phase() = "io";
    if (!synth_) io(t, given, shard_only);
    else launch_sleep(spec_.c.io_delay_s, main_, lc_);

    // Update of round t-1 (the postponed update of executors.cpp:210-229). With one worker per rank it was already
    // issued during step t-1 on the update stream, bucket by bucket as soon as (a) the bucket's averaged gradient
    // had arrived and (b) the backward of step t-1 no longer read W_k (after dX_k): the forward of layer k only
    // waits for its buckets' events. Emulated ranks (several workers on one stream) apply it here, in order.
    // flat-NCCL CSGD with one worker per GPU uses the same bucketed schedule (the fair flat-allreduce baseline):
    // per-bucket ncclAllReduce on the comm stream as each dW block lands, update per bucket on the update stream,
    // the next forward of layer k waits for its buckets only. Same dependencies as the reference's synchronous
    // CSGD block (executors.cpp:160-177): gradient t is reduced and applied before compute t+1 reads the layer.
    const bool eager = split_ && (alg_ == LSGD_B200_LSGD || flat_nccl());
    const bool postponed = alg_ == LSGD_B200_LSGD && t >= 1 && !split_;
    const bool exchange = !flat_nccl() && !reduce_folded() && alg_ != LSGD_B200_SEQUENTIAL;
    for (auto& w : ws_) {
      current_phase() = "compute";
      phase_mark(widx(w), t, 1, 0, main_);
      for (int k = 0; k < D; ++k) {
        for (int b : LB[static_cast<size_t>(k)]) {
          if (eager && t >= 1 && !fused_update()) {
            LSGD_CUDA(cudaStreamWaitEvent(main_, ev_upd_[b], 0));
          } else if (postponed) {
            current_phase() = "broadcast";
            apply_bucket(w, b, t - 1, main_);
            note_version(w, b, t, main_);
            current_phase() = "compute";
          }
        }
        if (w.ver_log) {  // the update rounds layer k's parameters have received when this forward reads them
          const auto& lb = LB[static_cast<size_t>(k)];
          long long* dst = nullptr;
          LSGD_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dst), w.ver_log + t * D + k, 0));
          launch_min_u64(w.ver, lb.front(), lb.back() + 1, dst, main_, lc_);
        }
        forward_layer(w, k);
      }
      if (postponed) after_update(w, t - 1, main_);
      // the previous step's side-stream bias gradients read the deltas this step's backward rewrites
      if (bias_) {
        LSGD_CUDA(cudaEventRecord(ev_bias_src_, bias_));
        LSGD_CUDA(cudaStreamWaitEvent(main_, ev_bias_src_, 0));
      }
      head(w);
      // Backward order (bwd_order()): which weight gradient is ready first decides which exchange chains hide
      // under the remaining backward and the next forward. Same kernels, same arithmetic; only the order differs.
      const std::vector<BwdOp> seq = bwd_seq();
      if (eager) LSGD_CUDA(cudaEventRecord(ev_dx_[0], main_));  // W_0 is not read by the backward
      for (const BwdOp& op : seq) {
        if (op.dx) {
          if (!synth_) backward_input(w, op.layer);
          if (eager) LSGD_CUDA(cudaEventRecord(ev_dx_[op.layer], main_));  // W_k is no longer read
          continue;
        }
        for (int b : op.buckets) {  // row block(s) of dW_k (+ db_k): ready for the exchange right away
          if (!synth_) backward_bucket(w, b);
          if (exchange && !split_) signal(w, kFlagGrad, b, static_cast<unsigned long long>(t + 1), main_);
          if (split_) LSGD_CUDA(cudaEventRecord(ev_bucket_[b], main_));
        }
        if (pio_ && op.layer == 0 && op.buckets.back() == LB[0].back()) {  // the batch buffers are free for t+1
          LSGD_CUDA(cudaEventRecord(ev_x_free_, main_));
          x_free_recorded_ = true;
        }
      }
      phase_mark(widx(w), t, 1, 1, main_);
    }
    if (rows_slot_ >= 0) {  // this step's staged host rows are no longer read
      LSGD_CUDA(cudaEventRecord(ev_rows_free_[rows_slot_], main_));
      rows_slot_ = -1;
    }
    if (postponed) ++applied_;

    // exchange order: the order buckets finish in the backward (row blocks ascending within a layer)
    std::vector<int> order;
    for (const BwdOp& op : bwd_seq())
      for (int b : op.buckets) order.push_back(b);

    if (iod_) {  // emulated ranks: the next io forks here, ahead of this round's exchange
      if (!ev_pre_exch_) LSGD_CUDA(cudaEventCreateWithFlags(&ev_pre_exch_, cudaEventDisableTiming));
      LSGD_CUDA(cudaEventRecord(ev_pre_exch_, main_));
    }
    // communicator work: per bucket, on the comm stream (overlapping the rest of the backward)
    current_phase() = "local_reduce";
    if (flat_nccl() && split_) {
      Worker& w = ws_[0];
      for (int b : order) {  // one stream: every rank issues the collectives of one communicator in one order
        const Bucket& bk = geo_.buckets[static_cast<size_t>(b)];
        LSGD_CUDA(cudaStreamWaitEvent(comm_, ev_bucket_[b], 0));
        if (bias_side_[b]) LSGD_CUDA(cudaStreamWaitEvent(comm_, ev_bias_[b], 0));
        Timed tm(this, "global", comm_);
        nccl_call(comm_, flat_comm_, [&] {
          return ncclAllReduce(w.payload + bk.poff, w.payload + bk.poff, static_cast<size_t>(bk.S * k_), nccl_type(),
                               ncclSum, flat_comm_, comm_);
        });
        LSGD_CUDA(cudaEventRecord(ev_gupd_[b], comm_));  // bucket b's sum is in the payload
      }
    } else if (flat_nccl()) {
      Timed tm(this, "global", main_);
      for (auto& w : ws_)
        nccl_call(main_, flat_comm_, [&] {
          return ncclAllReduce(w.payload, w.payload, static_cast<size_t>(geo_.Ppad), nccl_type(), ncclSum,
                               flat_comm_, main_);
        });
    } else if (exchange) {
      if (split_) {
        Worker& w = ws_[0];
        // with the ordered push sum (no NCCL) consecutive buckets rotate over the communicator streams so one
        // bucket's reduce/global phases overlap the next ones' scatters; NCCL collectives keep a single stream
        const int n_streams = slice_comm_ == nullptr ? n_comm_ : 1;
        for (size_t q = 0; q < order.size(); ++q) {
          const int b = order[q];
          cudaStream_t cs = commx_[q % static_cast<size_t>(n_streams)];
          LSGD_CUDA(cudaStreamWaitEvent(cs, ev_bucket_[b], 0));
          if (bias_side_[b]) LSGD_CUDA(cudaStreamWaitEvent(cs, ev_bias_[b], 0));
          if (q == 0) {
            // phases (executors.hpp:85): the push exchange interleaves the local reduce and the global average per
            // bucket, so local_reduce spans the whole exchange and global_allreduce starts after the link delay
            phase_mark(widx(w), t, 2, 0, comm_);
            launch_sleep(spec_.c.global_link_delay_s, comm_, lc_);
            phase_mark(widx(w), t, 3, 0, comm_);
            if (n_streams > 1) {  // the injected link delay precedes every bucket's exchange
              LSGD_CUDA(cudaEventRecord(join_ev_, comm_));
              for (int i = 1; i < n_streams; ++i) LSGD_CUDA(cudaStreamWaitEvent(commx_[i], join_ev_, 0));
            }
          }
          exchange_push_bucket(w, b, t, cs);
        }
        if (spec_.c.record_phases)  // every stream's work closes the spans
          for (int i = 1; i < n_streams; ++i) {
            LSGD_CUDA(cudaEventRecord(join_ev_, commx_[i]));
            LSGD_CUDA(cudaStreamWaitEvent(comm_, join_ev_, 0));
          }
        phase_mark(widx(w), t, 2, 1, comm_);
        phase_mark(widx(w), t, 3, 1, comm_);
      } else {
        // emulated ranks share one stream: every local slice sum is published before any global average waits
        for (auto& w : ws_) phase_mark(widx(w), t, 2, 0, main_);
        for (int b : order)
          for (auto& w : ws_) reduce_bucket(w, b, t, main_);
        for (auto& w : ws_) phase_mark(widx(w), t, 2, 1, main_);
        current_phase() = "global_allreduce";
        for (auto& w : ws_) phase_mark(widx(w), t, 3, 0, main_);
        launch_sleep(spec_.c.global_link_delay_s, main_, lc_);
        for (int b : order)
          for (auto& w : ws_) global_bucket(w, b, t, main_);
        for (auto& w : ws_) phase_mark(widx(w), t, 3, 1, main_);
      }
    }

    // Eager update of round t on the update stream, in backward order. Host issue order matters: these may spin on
    // the exchange's arrival flags, so they are enqueued after all the work they depend on (this step's backward
    // and communicator work) — a spinning kernel queued ahead of its producer could block it if the two streams
    // share a hardware queue.
    if (eager && fused_update()) {  // already applied by the gradient producers on the main stream
      after_update(ws_[0], t, main_);
      ++applied_;
    } else if (eager) {
      Worker& w = ws_[0];
      current_phase() = "broadcast";
      for (int b : order) {  // in the order the gradients are produced (bwd_seq)
        const int k = geo_.buckets[static_cast<size_t>(b)].layer;
        LSGD_CUDA(cudaStreamWaitEvent(upd_, ev_dx_[k], 0));  // W_k is no longer read by this step
        {
          if (reduce_folded()) LSGD_CUDA(cudaStreamWaitEvent(upd_, ev_bucket_[b], 0));
          if (flat_nccl()) LSGD_CUDA(cudaStreamWaitEvent(upd_, ev_gupd_[b], 0));  // the bucket's allreduce
          if (reduce_folded() && bias_side_[b]) LSGD_CUDA(cudaStreamWaitEvent(upd_, ev_bias_[b], 0));
          apply_bucket(w, b, t, upd_);
          if (own_slot_fused()) LSGD_CUDA(cudaStreamWaitEvent(upd_, ev_gupd_[b], 0));  // own slot (comm stream)
          note_version(w, b, t + 1, upd_);
          LSGD_CUDA(cudaEventRecord(ev_upd_[b], upd_));
        }
      }
      after_update(w, t, upd_);
      ++applied_;
    }

    if (alg_ != LSGD_B200_LSGD && !eager) {  // sequential / csgd: synchronous update in the same block (:172-177)
      current_phase() = "update";
      for (auto& w : ws_) {
        for (int b = 0; b < NB; ++b) {
          apply_bucket(w, b, t, main_);
          if (own_slot_fused()) LSGD_CUDA(cudaStreamWaitEvent(main_, ev_gupd_[b], 0));
          note_version(w, b, t + 1, main_);
        }
        after_update(w, t, main_);
      }
      ++applied_;
    }
    current_phase() = "between-phases";
  }

  ncclDataType_t nccl_type() const { return sizeof(T) == 8 ? ncclFloat64 : ncclFloat32; }

  bool tc_eligible() const {
    if (synth_ || sizeof(T) != 4) return false;
    if (spec_.c.gemm == LSGD_B200_GEMM_SIMT) return false;
    bool ok = tc_shapes_supported(spec_.layers, B_);
    if (spec_.c.gemm == LSGD_B200_GEMM_TC)
      check<ConfigError>(ok, "b200.gemm = tcgen05 needs every layer width a multiple of 256 and the local batch a "
                             "multiple of 128");
    return ok;
  }

  const T* rows_x_ = nullptr;
  const int32_t* rows_y_ = nullptr;
  RunSpec spec_;
  Layout L_;
  Geometry geo_;
  int dev_;
  std::vector<int> workers_;
  int64_t hist_rows_;
  int N_ = 1, G_ = 1, k_ = 1, nb_ = 1, alg_ = 2, B_ = 1;
  bool exact_ = false, synth_ = false, split_ = false, use_tc_ = false;
  static constexpr int kMaxComm = 4;
  cudaStream_t main_ = nullptr, comm_ = nullptr;
  cudaStream_t commx_[kMaxComm] = {};  // communicator streams; commx_[0] == comm_
  int n_comm_ = 1;
  cudaEvent_t ev_bucket_[kMaxBuckets] = {};
  // bias gradient of a layer on its own stream (off the GEMM chain): consumers of bucket b also wait ev_bias_[b]
  cudaStream_t bias_ = nullptr;
  cudaEvent_t ev_bias_[kMaxBuckets] = {};
  cudaEvent_t ev_bias_src_ = nullptr;
  bool bias_side_[kMaxBuckets] = {};
  cudaEvent_t ev_upd_[kMaxBuckets] = {};
  cudaEvent_t ev_gupd_[kMaxBuckets] = {};  // per bucket: the owner's fused global + update issued (comm stream)
  cudaEvent_t ev_dx_[kMaxBuckets] = {};
  cudaEvent_t base_ev_ = nullptr;  // timeline origin (set_timing)
  cudaEvent_t join_ev_ = nullptr;
  // caller-supplied host rows (step_rows): H2D on io_ into a double-buffered staging pair, overlapping the
  // previous step; ev_rows_free_[s] = the step that last read slot s has finished with it
  cudaStream_t io_ = nullptr;
  T* rows_xbuf_[2] = {nullptr, nullptr};
  int32_t* rows_ybuf_[2] = {nullptr, nullptr};
  cudaEvent_t ev_rows_h2d_[2] = {}, ev_rows_free_[2] = {};
  bool rows_used_[2] = {false, false};
  int rows_slot_ = -1;
  std::vector<T*> own_x_;
  std::vector<int32_t*> own_y_;  // per layer: dX_k issued (W_k free for its update)
  cudaStream_t upd_ = nullptr;
  bool direct_ = false;  // direct two-hop exchange (LSGD_B200_DIRECT)
  cudaStream_t pio_ = nullptr;  // prefetched io (gather of the next step under the current backward)
  cudaEvent_t ev_x_free_ = nullptr, ev_x_ready_ = nullptr;
  bool x_free_recorded_ = false;
  NvlsBuffer nvls_;       // NVLS: this worker's gfull bound to the group's multicast object
  T* mc_gfull_ = nullptr; // its multicast view (null: unicast pushes)
  cudaStream_t iod_ = nullptr;  // emulated ranks: the injected io latency, overlapping the previous exchange
  cudaEvent_t ev_pre_exch_ = nullptr, ev_io_done_ = nullptr;
  std::vector<char*> peer_base_;
  std::vector<char*> ipc_opened_;
  ncclComm_t slice_comm_ = nullptr, flat_comm_ = nullptr;
  std::mutex nccl_mu_;      // nccl_ops_ / nccl_ev_pool_
  std::mutex nccl_api_mu_;  // NCCL API calls of this rank's communicators (main thread vs watchdog)
  std::deque<NcclOp> nccl_ops_;
  std::vector<cudaEvent_t> nccl_ev_pool_;
  std::thread nccl_watch_;
  std::atomic<bool> nccl_stop_{false}, nccl_aborted_{false};
  std::string nccl_abort_reason_;
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
  int64_t spilled_ = 0;          // rounds [0, spilled_) of the loss history are in loss_saved_
  std::vector<T> loss_saved_;
  int64_t t_cur_ = 0;  // step being issued (round counter of the producers' staged flags)
  T* hist_ = nullptr;
  LaunchCounter lc_;
  bool timing_ = false;
  std::map<std::string, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>> timers_;
  std::map<std::string, std::vector<int>> timer_tags_;
  int tag_ = -1;  // bucket (or 100 + layer) the launches being issued belong to (timeline only)
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

void* nccl_init_rank(int nranks, const void* uid, int rank, double timeout_s) {
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  ncclConfig_t cfg = nonblocking_config();
  ncclComm_t c = nullptr;
  ncclResult_t r = ncclCommInitRankConfig(&c, nranks, id, rank, &cfg);
  if (r != ncclSuccess && r != ncclInProgress)
    throw TransportError(cat("NCCL init failed: ", ncclGetErrorString(r)));
  nccl_settle(c, timeout_s, "communicator init");
  return c;
}

std::vector<void*> nccl_init_all(const std::vector<int>& devs, double timeout_s) {
  ncclUniqueId id;
  LSGD_NCCL(ncclGetUniqueId(&id));
  const int n = static_cast<int>(devs.size());
  std::vector<ncclComm_t> cs(static_cast<size_t>(n), nullptr);
  ncclConfig_t cfg = nonblocking_config();
  LSGD_NCCL(ncclGroupStart());
  for (int i = 0; i < n; ++i) {
    LSGD_CUDA(cudaSetDevice(devs[static_cast<size_t>(i)]));
    ncclResult_t r = ncclCommInitRankConfig(&cs[static_cast<size_t>(i)], n, id, i, &cfg);
    if (r != ncclSuccess && r != ncclInProgress)
      throw TransportError(cat("NCCL init failed: ", ncclGetErrorString(r)));
  }
  ncclResult_t ge = ncclGroupEnd();
  if (ge != ncclSuccess && ge != ncclInProgress) throw TransportError(cat("NCCL init failed: ", ncclGetErrorString(ge)));
  std::vector<void*> out;
  for (ncclComm_t c : cs) {
    nccl_settle(c, timeout_s, "communicator init");
    out.push_back(c);
  }
  return out;
}

void note_ipc_mapping(Rank* r, char* p) {
  if (auto* a = dynamic_cast<RankImpl<float>*>(r)) a->note_ipc(p);
  if (auto* b = dynamic_cast<RankImpl<double>*>(r)) b->note_ipc(p);
}

}  // namespace lsgd_b200
