/*
 * lsgd_b200.h — C-ABI of the B200-native Layered-SGD synchronous update step.
 *
 * The reference (arXiv 1906.05936 re-implementation, /root/reference/proj) exposes no FFI; its hot path sits
 * behind three C++ seams. Each entry point below names the reference interface it replaces.
 *   executor seam : run_train  (include/lsgd/executors.hpp:138, src/executors.cpp:481-521)
 *                   run_rank   (include/lsgd/executors.hpp:143-144, src/executors.cpp:474-479)
 *   transport seam: reduce_to_root / broadcast / allreduce (include/lsgd/transport.hpp:56-63)
 *   kernel seam   : batch_gradient (include/lsgd/mlp.hpp:54), sgd_update (include/lsgd/optimizer.hpp:51-52)
 * Host-side pieces that must be bit-exact (SplitMix64, Fisher-Yates sampler, partition, topology, LR schedule,
 * synthetic blobs, init) are exported too, so a caller can verify them without a GPU.
 *
 * Conventions (mirroring the reference's error model, include/lsgd/common.hpp:16-29, tools/lsgd_main.cpp:282-288):
 *   every function returns int: 0 ok, 1 runtime/CUDA/NCCL error (lsgd::Error), 2 configuration error
 *   (lsgd::ConfigError), 3 transport error incl. collective timeout (lsgd::TransportError).
 *   lsgd_b200_last_error() returns the calling thread's last message ("rank R in phase P: ...").
 * Ownership: all buffers are caller-owned host memory; nothing returned aliases library storage except the
 *   opaque handles. Threading: a handle is owned by one host thread and is not re-entrant; run_train spawns one
 *   host thread per GPU internally (the reference spawns one per rank, executors.cpp:497-515).
 * There is no CPU fallback: every compute entry point fails with code 1 when no sm_100 device is present.
 */
#ifndef LSGD_B200_H_
#define LSGD_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSGD_B200_OK 0
#define LSGD_B200_ERR_RUNTIME 1
#define LSGD_B200_ERR_CONFIG 2
#define LSGD_B200_ERR_TRANSPORT 3

/* Algorithm (executors.hpp:180), update mode (optimizer.hpp:14). */
enum { LSGD_B200_SEQUENTIAL = 0, LSGD_B200_CSGD = 1, LSGD_B200_LSGD = 2 };
enum { LSGD_B200_PLAIN = 0, LSGD_B200_MOMENTUM = 1 };
/* Backend knobs (config key "b200", the new transport.backend = "b200" of config.cpp:176-178). */
enum { LSGD_B200_FP32 = 0, LSGD_B200_FP64 = 1 };                  /* dtype */
enum { LSGD_B200_GLOBAL_NCCL = 0, LSGD_B200_GLOBAL_ORDERED = 1 };  /* inter-communicator allreduce */
enum { LSGD_B200_GEMM_AUTO = 0, LSGD_B200_GEMM_SIMT = 1, LSGD_B200_GEMM_TC = 2 };
enum { LSGD_B200_DATA_DEVICE = 0, LSGD_B200_DATA_HOST = 1 };      /* dataset in HBM, or pinned host (UVA) */
enum { LSGD_B200_MODEL_MLP = 0, LSGD_B200_MODEL_SYNTHETIC_GRADIENT = 1 };

/* Flat mirror of lsgd::TrainConfig (executors.hpp:218-242) + lsgd::DataSpec/HyperParams/DelaySpec, plus the
 * B200 backend block. lsgd_b200_config_init() fills the reference defaults. */
typedef struct lsgd_b200_config {
  int32_t algorithm;
  int32_t n_workers;          /* N; GPU i hosts worker i when enough GPUs are visible */
  int32_t n_groups;           /* G, must divide N (executors.cpp:395-398) */
  int32_t n_layers;           /* entries in layer_sizes: input, hidden..., classes (mlp.hpp:20) */
  const int32_t* layer_sizes;
  int64_t n_samples;          /* synthetic blobs (dataset.hpp:40) */
  int32_t n_features;
  int32_t n_classes;
  double spread;
  int32_t mode;
  double base_lr, momentum, weight_decay, warmup_epochs;
  int32_t decay_every_epochs;
  double decay_factor;
  int32_t local_batch;
  int32_t epochs;
  int64_t iterations;         /* 0: epochs * floor(n_samples / global_batch) (executors.cpp:435-439) */
  uint64_t seed;              /* data = seed, init = seed+1, sampler = seed+2 (executors.hpp:244-246) */
  double init_scale;
  double io_delay_s;          /* injected per-iteration io latency (device-side sleep on the io stream) */
  double global_link_delay_s; /* injected latency ahead of the global allreduce (comm stream) */
  double collective_timeout_s;
  int32_t record_history;     /* keep w_0..w_T of worker 0 (and per-worker finals) */
  int32_t shared_minibatch;
  /* ---- B200 backend ---- */
  int32_t dtype;              /* LSGD_B200_FP32 | LSGD_B200_FP64 (parity mode) */
  int32_t n_devices;          /* GPUs to use (0: min(visible, N)); fewer GPUs than workers = ranks emulated */
  int32_t global_algo;        /* LSGD_B200_GLOBAL_* */
  int32_t gemm;               /* LSGD_B200_GEMM_* */
  int32_t data_source;        /* LSGD_B200_DATA_* */
  int32_t model;              /* LSGD_B200_MODEL_* */
  int32_t record_phases;      /* CUDA-event phase spans per iteration (executors.hpp:248-267) */
  int32_t csgd_nccl;          /* csgd only: 1 = flat ncclAllReduce baseline, 0 = ordered (reference order) */
  int64_t synthetic_params;   /* model = synthetic_gradient: P (gradient g_r[k] = Rng(1000+r).next_symmetric(1)) */
} lsgd_b200_config;

/* Caller-owned outputs of run_train; any pointer may be NULL. T = resolved iterations, P = n_params. */
typedef struct lsgd_b200_result {
  double* final_params;        /* [P]          worker 0 (executors.hpp:289) */
  double* loss;                /* [T]          minibatch mean loss per iteration (the payload's loss slot) */
  double* lr;                  /* [T] */
  double* history;             /* [(T+1)*P]    w_0..w_T, requires record_history */
  double* worker_finals;       /* [N*P]        every replica's final parameters */
  int64_t* version_at_compute; /* [N*T]        updates applied before each gradient pass (executors.hpp:266) */
  double* phase_spans;         /* [N*T*6*2]    (begin,end) seconds per worker/iteration/phase, record_phases */
  double total_wall_s;
  double throughput_sps;       /* T * global_batch / total_wall_s (executors.cpp:363-366) */
  int64_t gpu_launches;        /* kernels of this library launched during the run */
} lsgd_b200_result;

/* ---------------------------------------------------------------- misc */
const char* lsgd_b200_last_error(void);
const char* lsgd_b200_version(void);
int lsgd_b200_config_init(lsgd_b200_config* cfg);
/* TrainConfig::validate (executors.cpp:446-466) + run_train's dataset checks (executors.cpp:484-489). */
int lsgd_b200_config_validate(const lsgd_b200_config* cfg);
int lsgd_b200_device_count(int32_t* out);

/* ---------------------------------------------------------------- host-side, bit-exact, no GPU needed */
/* SplitMix64 stream (rng.hpp:14-19). */
int lsgd_b200_splitmix(uint64_t seed, int64_t n, uint64_t* out);
/* generate_synthetic (dataset.hpp:40, dataset.cpp:32-70): x [n*d] row-major float64, y [n]. */
int lsgd_b200_generate_synthetic(uint64_t seed, int64_t n, int32_t d, int32_t c, double spread, double* x, int32_t* y);
/* init_params (mlp.hpp:37, mlp.cpp:174-186): w [P]. */
int lsgd_b200_init_params(int32_t n_layers, const int32_t* layer_sizes, uint64_t seed, double scale, double* w);
int64_t lsgd_b200_n_params(int32_t n_layers, const int32_t* layer_sizes);
/* The exact minibatch index stream of a run: for iterations [t0, t0+n_steps), the global minibatch as drawn
 * by MinibatchSampler (sampler.cpp:15-43) from Rng(seed+2); worker i's shard is columns
 * [i*local_batch, (i+1)*local_batch) (partition_minibatch, sampler.cpp:45-57). out [n_steps * N*local_batch].
 * With shared_minibatch = 0, row t holds the N independent local draws of Rng(seed+3+i) (executors.cpp:73). */
int lsgd_b200_minibatch_indices(const lsgd_b200_config* cfg, int64_t t0, int64_t n_steps, int32_t* out);
/* learning_rate(hp, N, B_loc, epoch_float(t)) (optimizer.cpp:8-22, executors.cpp:441-444). */
int lsgd_b200_learning_rate(const lsgd_b200_config* cfg, int64_t t, double* out);
/* Topology (executors.cpp:389-433): for LSGD ranks 0..N+G-1 -> role (0 worker, 1 communicator) and group;
 * local_group(g) members and root; the B200 placement: device of worker i and of communicator slice j of g. */
int lsgd_b200_topology(const lsgd_b200_config* cfg, int32_t* role, int32_t* group, int32_t* device_of_worker);

/* ---------------------------------------------------------------- the step, in-process (executor seam) */
/* run_train with transport.backend = "b200": N workers on min(N, visible) GPUs, one host thread per GPU,
 * intra-group ordered peer reduce + NCCL (or ordered) global average on a side stream, broadcast fused with the
 * postponed update. Same result semantics as the reference (executors.hpp:106-133). */
int lsgd_b200_run_train(const lsgd_b200_config* cfg, lsgd_b200_result* out);

/* ---------------------------------------------------------------- the step, one process per GPU (run_rank seam) */
typedef struct lsgd_b200_rank lsgd_b200_rank;
/* Create worker `rank` (0..N-1) on CUDA device `device`; allocates its peer-visible payload/slice buffers. */
int lsgd_b200_rank_create(const lsgd_b200_config* cfg, int32_t rank, int32_t device, lsgd_b200_rank** out);
/* The caller's dataset for this rank (run_rank(cfg, const Dataset& data, ...), executors.hpp:143-144): x
 * [n_samples * n_features] row-major float64 (Dataset::features), y [n_samples] (Dataset::labels), replacing the
 * synthetic blobs the rank was created with. n_samples must equal cfg->n_samples (the sampler's range), n_features
 * cfg->n_features, labels in [0, n_classes): ConfigError otherwise. Call before the first step. */
int lsgd_b200_rank_upload_dataset(lsgd_b200_rank* r, const double* x, const int32_t* y, int64_t n_samples,
                                  int32_t n_features);
/* Bytes this rank must publish to every other rank (CUDA IPC handle + NCCL unique id for its slice comm). */
int lsgd_b200_rank_blob_size(int64_t* out);
int lsgd_b200_rank_export(lsgd_b200_rank* r, void* blob);
/* all_blobs: N blobs of rank_blob_size bytes each, in rank order (any host bootstrap may carry them). */
int lsgd_b200_rank_connect(lsgd_b200_rank* r, const void* all_blobs);
/* Issue `n_steps` further iterations asynchronously (io, postponed update, compute, reduce, global).
 * `host_indices` may be NULL (the rank's own sampler draws, like ShardSource::next, executors.cpp:75-79) or
 * [n_steps * local_batch] shard indices supplied by the caller (copied H2D inside the step). */
int lsgd_b200_rank_step(lsgd_b200_rank* r, int64_t n_steps, const int32_t* host_indices);
/* Data-loader form of the step (the e2e path): the caller supplies each step's shard ROWS in host memory
 * (pinned for full PCIe bandwidth) — x [n_steps * local_batch * n_features] in the config's dtype (float for fp32,
 * double for fp64), y [n_steps * local_batch] — copied H2D inside the step instead of the HBM gather. */
int lsgd_b200_rank_step_rows(lsgd_b200_rank* r, int64_t n_steps, const void* x, const int32_t* y);
/* Apply the pending update (the drain of executors.cpp:256) and wait for the device. */
int lsgd_b200_rank_drain(lsgd_b200_rank* r);
int lsgd_b200_rank_synchronize(lsgd_b200_rank* r);
/* Loss of the most recent applied round, read back from the device (D2H of one element). */
int lsgd_b200_rank_last_loss(lsgd_b200_rank* r, double* loss);
/* Non-blocking variant: enqueue the D2H copy of that loss (float for fp32, double for fp64; *elem_bytes says
 * which) into caller-owned pinned memory, ordered after the round's update; valid after the next synchronize. */
int lsgd_b200_rank_loss_async(lsgd_b200_rank* r, void* host_pinned, int32_t* elem_bytes);
int lsgd_b200_rank_get_params(lsgd_b200_rank* r, double* w, int64_t n);
int lsgd_b200_rank_set_params(lsgd_b200_rank* r, const double* w, int64_t n);
/* Losses / lrs of applied rounds [0, n) (device history, D2H). */
int lsgd_b200_rank_history(lsgd_b200_rank* r, double* loss, double* lr, int64_t n);
/* Kernels this rank has launched so far, and its CUDA stream (cudaStream_t) for event timing. */
int lsgd_b200_rank_launches(lsgd_b200_rank* r, int64_t* out);
int lsgd_b200_rank_stream(lsgd_b200_rank* r, void** stream);
/* Make that stream wait (device-side, no host sync) for all work issued so far on the rank's side streams
 * (communicator, update, host-row copies), so an event recorded on it after this call closes the issued steps. */
int lsgd_b200_rank_join(lsgd_b200_rank* r);
/* Device-timed average duration (ms) of the named kernel family over the launches since the last reset,
 * measured with CUDA events on the launching stream. family: "gemm", "reduce", "update", "global". */
int lsgd_b200_rank_kernel_time(lsgd_b200_rank* r, const char* family, double* avg_ms, int64_t* count);
int lsgd_b200_rank_timing(lsgd_b200_rank* r, int32_t enable);
int lsgd_b200_rank_destroy(lsgd_b200_rank* r);

/* ---------------------------------------------------------------- kernel seam (single GPU, for conformance) */
/* batch_gradient (mlp.hpp:54): grad [P], mean loss; x [n_rows*d] float64 host, y [n_rows], idx [b]. */
int lsgd_b200_batch_gradient(int32_t n_layers, const int32_t* layer_sizes, int32_t dtype, int32_t gemm,
                             const double* w, int64_t n_rows, const double* x, const int32_t* y,
                             const int32_t* idx, int64_t b, double* grad, double* mean_loss);
/* Ordered peer collectives on `world` ranks emulated on device 0 (transport.hpp:56-63, fixed ascending order):
 * op 0 reduce_to_root (result in row `root`), 1 broadcast of row root, 2 allreduce. */
int lsgd_b200_collective(int32_t op, int32_t dtype, int32_t world, int32_t root, int64_t n,
                         const double* contributions, double* out);
/* sgd_update (optimizer.cpp:24-42) on device; velocity may be NULL in plain mode. */
int lsgd_b200_sgd_update(int32_t dtype, int64_t n, double* w, const double* delta, double* velocity, int32_t mode,
                         double momentum, double weight_decay, double lr);

#ifdef __cplusplus
}
#endif
#endif /* LSGD_B200_H_ */
