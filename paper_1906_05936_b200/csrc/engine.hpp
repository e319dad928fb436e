// The LSGD step engine (executors.cpp:190-304 re-designed for one box of B200s).
//
// A Rank = one host thread + one GPU + three streams (main: io/forward/backward, comm: the communicator's
// reduce/average/broadcast, upd: the postponed updates). It hosts one or more workers (one per GPU in production;
// several when fewer GPUs than workers are visible, which emulates the ranks on one device with identical
// arithmetic on a single stream). Every worker owns a peer-visible block
//     [flags | payload | s[0] | s[1] | gbar | gfull]
// which other GPUs read and write over NVLink (CUDA IPC when ranks are processes, direct peer pointers when
// threads). The gradient is split into per-layer buckets (Bucket); the communicator of group g is not a separate
// rank: each bucket's reduction is sliced across the group's k GPUs — slot j sums sub-slice j of all members'
// payloads in ascending worker order (the exact order of transport.cpp:27-48), so the result is bitwise the rooted
// reduce while each GPU moves only (k-1)/k of the vector over NVLink per direction. Slot owners then average
// across groups (NCCL on the comm stream, or the ordered peer variant) and push their averaged sub-slice into every
// member's gfull, so the update reads local HBM only.
// Cross-GPU ordering uses monotone step counters (ld.acquire / st.release at system scope) in the peer block.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "host.hpp"

namespace lsgd_b200 {

// Byte layout of a worker's peer-visible block; identical on every rank.
struct PeerLayout {
  int64_t flags = 0;     // u64 [which * kMaxBuckets + bucket]: which 0 = grad ready, 1 = slice sum, 2 = averaged
  int64_t payload = 0;   // Ppad elements
  int64_t s[2] = {0, 0};  // Sg elements each (double-buffered by step parity)
  int64_t gbar = 0;      // Sg elements
  int64_t gfull = 0;     // Ppad elements: the whole averaged gradient, pushed here by the group's slot owners
  // push exchange (one worker per GPU): stage[m] (Sg each) = member m's sub-slices of this worker's slot, pushed
  // by m after its weight-gradient GEMMs; gstage[par][g] (Sg each) = group g's slot sum, pushed by g's owner
  int64_t stage = 0;
  int64_t gstage[2] = {0, 0};
  int64_t total = 0;
};
enum : int { kFlagGrad = 0, kFlagSlice = 1, kFlagBcast = 2 };
constexpr int kMaxBuckets = 32;
// flags[kArrived + b * kMaxPeers + j]: round counter of the averaged sub-slice j of bucket b pushed by slot j
constexpr int kArrived = 3 * kMaxBuckets;
// flags[kStaged + b * kMaxPeers + m]: member m's sub-slice of bucket b is in this owner's stage[m]
constexpr int kStaged = kArrived + kMaxBuckets * kMaxPeers;
// flags[kGsum + b * kMaxPeers + g]: group g's slot sum of bucket b is in this owner's gstage[par][g]
constexpr int kGsum = kStaged + kMaxBuckets * kMaxPeers;
// flags[kNvlsAdded + j] (in the group leader's block): member j added its device to the group's multicast object
constexpr int kNvlsAdded = kGsum + kMaxBuckets * kMaxPeers;
constexpr int kFlagWords = kNvlsAdded + kMaxPeers;

// Gradient buckets: one per layer (that layer's [W_k | b_k] block, contiguous in the reference's parameter
// layout, mlp.hpp:14-18), the loss slot riding the last layer's bucket. Each bucket is split into k sub-slices of
// S elements; sub-slice j lives in the payload at poff + j*S and in slot j's s/gbar regions at goff.
// A large layer is split into row blocks of W_k (contiguous in the layout), so the exchange of the first blocks
// overlaps the weight-gradient GEMMs of the later ones; the layer's bias rides its last block.
struct Bucket {
  int64_t pstart = 0;  // first parameter index
  int64_t n = 0;       // parameters (the loss slot, when carried, is bucket-local index n)
  bool loss = false;
  int layer = 0;       // MLP layer k
  int row0 = 0;        // first output row of W_k in this bucket
  int rows = 0;        // output rows of W_k in this bucket
  bool bias = false;   // carries b_k (the layer's last block)
  int64_t S = 0;       // sub-slice length, multiple of 64 elements
  int64_t poff = 0;    // payload offset (elements, 64-aligned)
  int64_t goff = 0;    // offset inside each slot's s/gbar region (64-aligned)
  // The weight-gradient GEMM runs per block of consecutive buckets (one launch, contiguous payload): the block's
  // first bucket carries its row count (0 on the others) and whether it ends with the layer's bias.
  int blk_rows = 0;
  bool blk_bias = false;
};

// Direct two-hop exchange for groups of k >= 2 and G >= 2 (LSGD_B200_DIRECT=1): every member's sub-slice j goes by
// copy engine straight to the slot-j owner of EVERY group; owners sum all N sub-slices in the reference's order
// (groups ascending, members ascending within a group, + 0.0, / N per group) — no owner reduce kernel, no group-sum
// hop. Stage holds one sub-slice per source GPU, double-buffered by round parity.
bool direct_exchange(const RunSpec& spec);

struct Geometry {
  int64_t P = 0, Ppad = 0, Sg = 0;  // params, padded payload, per-slot slice elements (sum of bucket S)
  int esize = 4;
  std::vector<Bucket> buckets;
  std::vector<std::vector<int>> layer_buckets;  // bucket indices of each layer, in row order
  int64_t loss_at = 0;             // payload index of the loss slot
  PeerLayout peer;
  Geometry(const RunSpec& spec, int elem_size);
};

// Type-erased rank interface (the engine is instantiated for float and double).
class Rank {
 public:
  virtual ~Rank() = default;
  virtual int device() const = 0;
  virtual const std::vector<int>& workers() const = 0;
  virtual char* peer_block(int worker) = 0;                 // own blocks only
  virtual void set_peer_base(int worker, char* base) = 0;   // as addressable from this rank's device
  virtual void set_nccl(void* slice_comm, void* flat_comm) = 0;
  // NVLS multicast average fan-out (nvls.cu, LSGD_B200_NVLS): wanted by this layout/config; gfull bytes per
  // worker; bind this rank's gfull to the group's multicast object (after every member added its device)
  virtual bool nvls_wanted() const = 0;
  virtual size_t nvls_bytes() const = 0;
  virtual void nvls_attach(uint64_t mc, size_t size, bool own_mc) = 0;
  // processes: add this device to the group's object, wait until all k members have (flags in the leader's peer
  // block, mapped at leader_block), then attach
  virtual void nvls_join(uint64_t mc, size_t size, char* leader_block, int j, int k, double timeout_s) = 0;
  virtual void upload_dataset(const double* x, const int32_t* y, int64_t n) = 0;
  virtual void share_dataset_from(Rank* other) = 0;         // same-device or host-mapped dataset reuse
  virtual void set_params(const double* w) = 0;             // every local worker
  virtual void get_params(int worker, double* w) = 0;
  virtual void issue_steps(int64_t n, const int32_t* host_global_or_shard_indices, bool shard_only) = 0;
  virtual void issue_steps_rows(int64_t n, const void* x_host, const int32_t* y_host) = 0;
  virtual void drain() = 0;
  // version_at_compute (executors.hpp:102), measured on the device: for each iteration t < n, the number of update
  // rounds every layer had received when the forward pass of t read it (min over layers). -1 where not tracked.
  virtual void versions(int worker, int64_t* out, int64_t n) = 0;
  virtual void synchronize() = 0;
  virtual int64_t steps_issued() const = 0;
  virtual int64_t updates_applied() const = 0;
  virtual void history(double* loss, double* lr, int64_t n) = 0;
  virtual void param_history(double* out, int64_t rows) = 0;   // worker0 w_0..w_{rows-1}
  virtual void phase_spans(int worker, double* out, int64_t T) = 0;
  virtual double last_loss() = 0;
  // Enqueue the D2H copy of the latest applied round's loss into pinned host memory; returns its size in bytes.
  virtual int loss_async(void* host_pinned) = 0;
  virtual int64_t launches() const = 0;
  virtual void* main_stream() = 0;
  virtual void join() = 0;  // main_stream waits for everything issued so far on the rank's other streams
  virtual void set_timing(bool on) = 0;
  virtual void kernel_time(const std::string& family, double* avg_ms, int64_t* count) = 0;
  // Every timed launch since set_timing(true) as "family<TAB>start_ms<TAB>end_ms" lines (relative to that call).
  virtual std::string timeline() = 0;
  // Kernel seam (batch_gradient, mlp.hpp:54): gather `idx`, forward/backward, return grad [P] and mean loss.
  virtual void compute_gradient(const int32_t* idx, double* grad, double* loss) = 0;
  virtual void abort() = 0;
  virtual void check_health() = 0;
};

// Build a rank hosting `workers` on `device`. history_rows > 0 keeps w_0..w_{rows-1} of worker 0 on the host.
std::unique_ptr<Rank> make_rank(const RunSpec& spec, int device, std::vector<int> workers, int64_t history_rows);

// In-process world (executor seam): one Rank per device, one host thread per Rank.
struct TrainOutputs {
  std::vector<double> final_params, loss, lr, history, worker_finals, phase_spans;
  std::vector<int64_t> version_at_compute;
  double total_wall_s = 0.0;
  int64_t launches = 0;
};
void run_world(const RunSpec& spec, bool want_history, bool want_workers, TrainOutputs& out);
void enable_phase_recording(Rank* r);
// Non-blocking NCCL communicators (ncclConfig_t.blocking = 0): every NCCL call returns at once and the host polls
// ncclCommGetAsyncError with a deadline, so a peer that never joins an init or a collective surfaces as
// TransportError (ncclCommAbort) instead of blocking the host thread (inprocess.cpp:44-49).
// uid: the ncclUniqueId bytes. nccl_init_all: one communicator per device of `devs` from one thread (grouped).
void* nccl_init_rank(int nranks, const void* uid, int rank, double timeout_s);
// communicator setup (bootstrap, topology, channel connections) takes seconds: at least a minute, never less than
// the collective timeout
inline double init_timeout(double collective_timeout_s) { return collective_timeout_s > 60.0 ? collective_timeout_s : 60.0; }
std::vector<void*> nccl_init_all(const std::vector<int>& devs, double timeout_s);
void note_ipc_mapping(Rank* r, char* p);

// Parallel, bit-exact blob generator (SplitMix64 is a counter: draw k of Rng(s) = mix(s + (k+1)*gamma)).
void generate_blobs_parallel(uint64_t seed, int64_t n, int d, int c, double spread, double* x, int32_t* y);

}  // namespace lsgd_b200
