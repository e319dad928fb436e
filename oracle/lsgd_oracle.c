/*
 * TEST INFRASTRUCTURE — CPU oracle for the LSGD synchronous-update step. NOT product code.
 *
 * A plain-C, single-threaded, float64 restatement of the reference's arithmetic for every function on
 * the hot path. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load it, and only as the checker.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against the golden vectors the
 * reference's own tests hold (tests/golden/reference_tests.json, transcribed from
 * proj/tests/test_*.cpp) AND against fixtures produced by the unmodified reference library built from
 * /root/reference (oracle/_ref/liblsgd_ref.so, tests/golden/make_golden.py). Every function cites the
 * reference file:line it restates. The build uses -ffp-contract=off so no a*b+c is fused, matching the
 * reference's x86-64 (no FMA) build, which makes the fp64 training history bit-identical.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- SplitMix64: proj/include/lsgd/rng.hpp:14-19 ------------------------------------------------ */
static uint64_t sm_next(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
/* rng.hpp:22-24: top 53 bits scaled by 2^-53. */
static double sm_double(uint64_t* s) { return (double)(sm_next(s) >> 11) * 0x1.0p-53; }
/* rng.hpp:27-29 */
static double sm_symmetric(uint64_t* s, double scale) { return scale * (2.0 * sm_double(s) - 1.0); }
/* rng.hpp:33: modulo draw. */
static uint64_t sm_below(uint64_t* s, uint64_t bound) { return sm_next(s) % bound; }
/* rng.hpp:44-51: Box-Muller, u1 in (0,1]. */
static void sm_gauss2(uint64_t* s, double* z0, double* z1) {
  const double two_pi = 6.283185307179586476925286766559;
  double u1 = 1.0 - sm_double(s);
  double u2 = sm_double(s);
  double r = sqrt(-2.0 * log(u1));
  *z0 = r * cos(two_pi * u2);
  *z1 = r * sin(two_pi * u2);
}

void lo_splitmix(uint64_t seed, int64_t n, uint64_t* out) {
  uint64_t s = seed;
  for (int64_t i = 0; i < n; ++i) out[i] = sm_next(&s);
}

uint64_t lo_fnv1a64(const void* data, int64_t n_bytes) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 1469598103934665603ULL;
  for (int64_t i = 0; i < n_bytes; ++i) {
    h ^= p[i];
    h *= 1099511628211ULL;
  }
  return h;
}

/* ---- synthetic blobs: proj/src/dataset.cpp:18-28 (fill) and :32-70 (generate) -------------------- */
static void gauss_fill(uint64_t* s, double* out, int n) {
  int i = 0;
  double a, b;
  while (i + 1 < n) {
    sm_gauss2(s, &out[i], &out[i + 1]);
    i += 2;
  }
  if (i < n) { /* odd tail: the sibling draw is discarded */
    sm_gauss2(s, &a, &b);
    out[i] = a;
  }
}

int lo_generate_synthetic(uint64_t seed, int64_t n, int d, int c, double spread, double* x, int32_t* y) {
  if (c < 2 || n < c || d < 1 || !(spread > 0.0)) return 2;
  uint64_t s = seed;
  double* centers = (double*)malloc(sizeof(double) * (size_t)c * (size_t)d);
  if (!centers) return 1;
  for (int k = 0; k < c; ++k) {
    double* ck = centers + (size_t)k * d;
    gauss_fill(&s, ck, d);
    double n2 = 0.0;
    for (int j = 0; j < d; ++j) n2 += ck[j] * ck[j];
    double r = sqrt(n2);
    if (r == 0.0) r = 1.0;
    for (int j = 0; j < d; ++j) ck[j] = spread * ck[j] / r;
  }
  for (int64_t i = 0; i < n; ++i) {
    int32_t lab = (int32_t)(i % c);
    y[i] = lab;
    double* xi = x + (size_t)i * d;
    gauss_fill(&s, xi, d);
    const double* ck = centers + (size_t)lab * d;
    for (int j = 0; j < d; ++j) xi[j] += ck[j];
  }
  free(centers);
  return 0;
}

/* ---- sampler: proj/src/sampler.cpp:9-43; partition :45-57 ----------------------------------------- */
typedef struct {
  int64_t n, cursor, epochs;
  uint64_t state;
  int with_replacement;
  int32_t* perm;
} lo_sampler_t;

static void sampler_refresh(lo_sampler_t* sp) {
  for (int64_t i = 0; i < sp->n; ++i) sp->perm[i] = (int32_t)i;
  for (int64_t i = sp->n - 1; i >= 1; --i) {
    uint64_t j = sm_below(&sp->state, (uint64_t)i + 1);
    int32_t t = sp->perm[i];
    sp->perm[i] = sp->perm[j];
    sp->perm[j] = t;
  }
  sp->cursor = 0;
  sp->epochs += 1;
}

static int sampler_init(lo_sampler_t* sp, int64_t n, uint64_t seed, int with_replacement) {
  memset(sp, 0, sizeof(*sp));
  if (n < 1) return 1;
  sp->n = n;
  sp->state = seed;
  sp->with_replacement = with_replacement;
  sp->perm = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  if (!sp->perm) return 1;
  if (!with_replacement) sampler_refresh(sp);
  return 0;
}

static int sampler_draw(lo_sampler_t* sp, int64_t size, int32_t* out) {
  if (size < 1 || size > sp->n) return 1;
  if (sp->with_replacement) {
    for (int64_t i = 0; i < size; ++i) out[i] = (int32_t)sm_below(&sp->state, (uint64_t)sp->n);
    return 0;
  }
  if (sp->cursor + size > sp->n) sampler_refresh(sp); /* drop-last */
  memcpy(out, sp->perm + sp->cursor, sizeof(int32_t) * (size_t)size);
  sp->cursor += size;
  return 0;
}

int lo_sampler(int64_t n, uint64_t seed, int64_t size, int64_t n_draws, int with_replacement, int32_t* out,
               int64_t* epochs_started) {
  lo_sampler_t sp;
  if (sampler_init(&sp, n, seed, with_replacement)) return 1;
  int rc = 0;
  for (int64_t k = 0; k < n_draws && rc == 0; ++k) rc = sampler_draw(&sp, size, out + k * size);
  if (epochs_started) *epochs_started = sp.epochs;
  free(sp.perm);
  return rc;
}

/* Contiguous equal split; the output is the shards concatenated, i.e. the input itself, once the
 * divisibility precondition (sampler.cpp:47-48) holds. */
int lo_partition(const int32_t* idx, int64_t size, int n_workers, int32_t* out) {
  if (n_workers < 1 || size % n_workers != 0) return 1;
  memcpy(out, idx, sizeof(int32_t) * (size_t)size);
  return 0;
}

/* ---- MLP: proj/include/lsgd/mlp.hpp:14-18 layout; proj/src/mlp.cpp -------------------------------- */
int64_t lo_n_params(int nl, const int* L) {
  int64_t p = 0;
  for (int k = 0; k + 1 < nl; ++k) p += (int64_t)L[k] * L[k + 1] + L[k + 1];
  return p;
}
static int64_t w_off(const int* L, int layer) {
  int64_t o = 0;
  for (int k = 0; k < layer; ++k) o += (int64_t)L[k] * L[k + 1] + L[k + 1];
  return o;
}
static int64_t b_off(const int* L, int layer) { return w_off(L, layer) + (int64_t)L[layer] * L[layer + 1]; }

/* mlp.cpp:174-186: weights in layout order, biases zero without consuming draws. */
int lo_init_params(int nl, const int* L, uint64_t seed, double scale, double* w) {
  if (!(scale >= 0.0)) return 1;
  uint64_t s = seed;
  memset(w, 0, sizeof(double) * (size_t)lo_n_params(nl, L));
  for (int k = 0; k + 1 < nl; ++k) {
    double* wk = w + w_off(L, k);
    int64_t nw = (int64_t)L[k] * L[k + 1];
    for (int64_t i = 0; i < nw; ++i) wk[i] = sm_symmetric(&s, scale);
  }
  return 0;
}

/* One sample: forward (mlp.cpp:60-92) into acts[k] (level-k+1 activations), returns the CE loss and
 * leaves softmax probabilities in the top level. */
static double sample_forward(int nl, const int* L, const double* w, const double* x, int32_t label,
                             double** acts) {
  int depth = nl - 1;
  const double* in = x;
  for (int k = 0; k < depth; ++k) {
    int ni = L[k], no = L[k + 1];
    const double* W = w + w_off(L, k);
    const double* b = w + b_off(L, k);
    double* out = acts[k];
    for (int j = 0; j < no; ++j) {
      double z = b[j];
      for (int i = 0; i < ni; ++i) z += W[(int64_t)j * ni + i] * in[i];
      out[j] = (k + 1 < depth && z < 0.0) ? 0.0 : z;
    }
    in = out;
  }
  double* lg = acts[depth - 1];
  int C = L[nl - 1];
  double zmax = lg[0];
  for (int c = 1; c < C; ++c)
    if (zmax < lg[c]) zmax = lg[c];
  double sum = 0.0;
  for (int c = 0; c < C; ++c) sum += exp(lg[c] - zmax);
  double lse = zmax + log(sum);
  double loss = lse - lg[label];
  for (int c = 0; c < C; ++c) lg[c] = exp(lg[c] - lse);
  return loss;
}

/* Backward (mlp.cpp:96-127): per-sample gradient written (not accumulated) into g. */
static void sample_backward(int nl, const int* L, const double* w, const double* x, int32_t label,
                            double** acts, double* d, double* dn, double* g) {
  int depth = nl - 1;
  int C = L[nl - 1];
  for (int c = 0; c < C; ++c) d[c] = acts[depth - 1][c];
  d[label] -= 1.0;
  for (int k = depth - 1; k >= 0; --k) {
    int ni = L[k], no = L[k + 1];
    const double* ap = (k == 0) ? x : acts[k - 1];
    double* gw = g + w_off(L, k);
    double* gb = g + b_off(L, k);
    for (int j = 0; j < no; ++j) {
      for (int i = 0; i < ni; ++i) gw[(int64_t)j * ni + i] = d[j] * ap[i];
      gb[j] = d[j];
    }
    if (k > 0) {
      const double* W = w + w_off(L, k);
      for (int i = 0; i < ni; ++i) {
        double s = 0.0;
        for (int j = 0; j < no; ++j) s += W[(int64_t)j * ni + i] * d[j];
        dn[i] = (acts[k - 1][i] > 0.0) ? s : 0.0;
      }
      double* t = d;
      d = dn;
      dn = t;
    }
  }
}

/* batch_gradient_serial (mlp.cpp:217-236): fold in batch order, then true division by B. */
int lo_batch_gradient(int nl, const int* L, const double* w, int64_t n_rows, const double* x, const int32_t* y,
                      const int32_t* idx, int64_t B, double* grad, double* mean_loss) {
  if (nl < 2 || B < 1) return 1;
  int C = L[nl - 1], d0 = L[0];
  int widest = 0;
  for (int k = 1; k < nl; ++k)
    if (L[k] > widest) widest = L[k];
  int64_t P = lo_n_params(nl, L);
  double** acts = (double**)malloc(sizeof(double*) * (size_t)(nl - 1));
  for (int k = 0; k + 1 < nl; ++k) acts[k] = (double*)malloc(sizeof(double) * (size_t)L[k + 1]);
  double* d = (double*)malloc(sizeof(double) * (size_t)widest);
  double* dn = (double*)malloc(sizeof(double) * (size_t)widest);
  double* g = (double*)malloc(sizeof(double) * (size_t)P);
  memset(grad, 0, sizeof(double) * (size_t)P);
  double lacc = 0.0;
  int rc = 0;
  for (int64_t s = 0; s < B; ++s) {
    int32_t r = idx[s];
    if (r < 0 || r >= n_rows || y[r] < 0 || y[r] >= C) {
      rc = 1;
      break;
    }
    const double* xs = x + (size_t)r * d0;
    lacc += sample_forward(nl, L, w, xs, y[r], acts);
    sample_backward(nl, L, w, xs, y[r], acts, d, dn, g);
    for (int64_t k = 0; k < P; ++k) grad[k] += g[k];
  }
  double inv = (double)B;
  for (int64_t k = 0; k < P; ++k) grad[k] /= inv;
  *mean_loss = lacc / inv;
  for (int k = 0; k + 1 < nl; ++k) free(acts[k]);
  free(acts);
  free(d);
  free(dn);
  free(g);
  return rc;
}

/* ---- optimizer: proj/src/optimizer.cpp:8-22 and :24-42 ------------------------------------------- */
double lo_learning_rate(double base_lr, double warmup_epochs, int decay_every, double decay_factor,
                        int n_workers, int local_batch, double epoch) {
  double gb = (double)n_workers * (double)local_batch;
  double target = base_lr * gb / 256.0;
  if (warmup_epochs > 0.0 && epoch < warmup_epochs) return base_lr + (target - base_lr) * (epoch / warmup_epochs);
  int64_t steps = (int64_t)floor(epoch / (double)decay_every);
  double lr = target;
  for (int64_t i = 0; i < steps; ++i) lr *= decay_factor;
  return lr;
}

void lo_sgd_update(int64_t n, double* w, const double* delta, double* v, int mode, double momentum,
                   double weight_decay, double lr) {
  if (mode == 0) {
    for (int64_t k = 0; k < n; ++k) w[k] -= lr * delta[k];
  } else {
    for (int64_t k = 0; k < n; ++k) {
      double g = delta[k] + weight_decay * w[k];
      v[k] = momentum * v[k] + g;
      w[k] -= lr * v[k];
    }
  }
}

/* ---- executors: the three training loops as one sequential simulation (executors.cpp:87-304) ------ */
typedef struct {
  int algorithm; /* 0 sequential, 1 csgd, 2 lsgd */
  int n_workers, n_groups, n_layers;
  const int* layer_sizes;
  int64_t n_samples;
  int n_features, n_classes;
  double spread;
  int mode;
  double base_lr, momentum, weight_decay, warmup_epochs;
  int decay_every_epochs;
  double decay_factor;
  int local_batch, epochs;
  int64_t iterations;
  uint64_t seed;
  double init_scale;
  double io_delay_s, global_link_delay_s; /* timing knobs only; no effect on arithmetic */
  int shared_minibatch;
} lo_config;

typedef struct {
  double* final_params; /* [P] */
  double* loss;         /* [T] */
  double* lr;           /* [T] */
  double* history;      /* [(T+1)*P] */
  double* worker_finals;
  int64_t* version_at_compute;
  double* phase_spans;
  double total_wall_s, throughput_sps;
} lo_result;

int64_t lo_resolve_iterations(const lo_config* c) {
  if (c->iterations > 0) return c->iterations;
  int64_t gb = (int64_t)c->local_batch * c->n_workers;
  return (int64_t)c->epochs * (c->n_samples / gb);
}

/* The payload rides [grad | mean_loss] (executors.cpp:59-63). Communicator sums its members in
 * ascending id, its own zero vector last (transport.cpp:27-48, executors.cpp:278), divides by N
 * (executors.cpp:287); communicators allreduce at the lowest id (transport.cpp:92-96). CSGD sums at
 * rank 0 then every worker divides by N (executors.cpp:166-170). Arithmetic is identical on every
 * replica, so one copy of w stands for all of them. */
int lo_run_train(const lo_config* c, lo_result* r) {
  int nl = c->n_layers;
  const int* L = c->layer_sizes;
  int N = c->n_workers, G = c->n_groups, B = c->local_batch;
  if (c->algorithm == 0 && N != 1) return 2;
  if (c->algorithm == 2 && (G < 1 || N % G != 0)) return 2;
  int64_t P = lo_n_params(nl, L), P1 = P + 1;
  int64_t T = lo_resolve_iterations(c);
  int64_t gbatch = (int64_t)B * N;
  int64_t n = c->n_samples;
  if (gbatch > n) return 2;

  double* x = (double*)malloc(sizeof(double) * (size_t)n * (size_t)c->n_features);
  int32_t* y = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  if (lo_generate_synthetic(c->seed, n, c->n_features, c->n_classes, c->spread, x, y)) return 2;
  double* w = (double*)malloc(sizeof(double) * (size_t)P);
  double* v = (double*)calloc((size_t)P, sizeof(double));
  lo_init_params(nl, L, c->seed + 1, c->init_scale, w);
  if (r->history) memcpy(r->history, w, sizeof(double) * (size_t)P);

  int n_samplers = c->shared_minibatch ? 1 : N;
  lo_sampler_t* samplers = (lo_sampler_t*)malloc(sizeof(lo_sampler_t) * (size_t)n_samplers);
  for (int i = 0; i < n_samplers; ++i)
    sampler_init(&samplers[i], n, c->shared_minibatch ? c->seed + 2 : c->seed + 3 + (uint64_t)i, 0);
  int32_t* mb = (int32_t*)malloc(sizeof(int32_t) * (size_t)gbatch);
  double* pay = (double*)malloc(sizeof(double) * (size_t)P1 * (size_t)N); /* per-worker payloads */
  double* acc = (double*)malloc(sizeof(double) * (size_t)P1);
  double* sg = (double*)malloc(sizeof(double) * (size_t)P1 * (size_t)G); /* communicator sums */
  int rc = 0;

  for (int64_t t = 0; t < T && rc == 0; ++t) {
    /* io: draw the shared global minibatch (or one local minibatch per worker) */
    if (c->shared_minibatch) {
      rc |= sampler_draw(&samplers[0], c->algorithm == 0 ? gbatch : gbatch, mb);
    } else {
      for (int i = 0; i < N; ++i) rc |= sampler_draw(&samplers[i], B, mb + (int64_t)i * B);
    }
    double epoch = (double)t * (double)gbatch / (double)n; /* executors.cpp:441-444 */
    double lr = lo_learning_rate(c->base_lr, c->warmup_epochs, c->decay_every_epochs, c->decay_factor, N, B, epoch);
    const double* delta;
    double loss;
    if (c->algorithm == 0) {
      rc |= lo_batch_gradient(nl, L, w, n, x, y, mb, gbatch, pay, &pay[P]);
      delta = pay;
      loss = pay[P];
    } else {
      for (int i = 0; i < N; ++i) {
        double* pi = pay + (int64_t)i * P1;
        rc |= lo_batch_gradient(nl, L, w, n, x, y, mb + (int64_t)i * B, B, pi, &pi[P]);
      }
      if (c->algorithm == 1) {
        memcpy(acc, pay, sizeof(double) * (size_t)P1);
        for (int i = 1; i < N; ++i)
          for (int64_t k = 0; k < P1; ++k) acc[k] += pay[(int64_t)i * P1 + k];
        for (int64_t k = 0; k < P1; ++k) acc[k] /= (double)N;
      } else {
        int per = N / G;
        for (int g = 0; g < G; ++g) {
          double* s = sg + (int64_t)g * P1;
          memcpy(s, pay + (int64_t)(g * per) * P1, sizeof(double) * (size_t)P1);
          for (int i = g * per + 1; i < (g + 1) * per; ++i)
            for (int64_t k = 0; k < P1; ++k) s[k] += pay[(int64_t)i * P1 + k];
          for (int64_t k = 0; k < P1; ++k) s[k] += 0.0; /* the communicator's zero contribution */
          for (int64_t k = 0; k < P1; ++k) s[k] /= (double)N;
        }
        memcpy(acc, sg, sizeof(double) * (size_t)P1);
        for (int g = 1; g < G; ++g)
          for (int64_t k = 0; k < P1; ++k) acc[k] += sg[(int64_t)g * P1 + k];
      }
      delta = acc;
      loss = acc[P];
    }
    if (!(lr > 0.0)) rc |= 1;
    lo_sgd_update(P, w, delta, v, c->mode, c->momentum, c->weight_decay, lr);
    for (int64_t k = 0; k < P; ++k)
      if (!isfinite(w[k])) rc |= 1;
    if (r->loss) r->loss[t] = loss;
    if (r->lr) r->lr[t] = lr;
    if (r->history) memcpy(r->history + (t + 1) * P, w, sizeof(double) * (size_t)P);
    if (r->version_at_compute)
      for (int i = 0; i < N; ++i) r->version_at_compute[(int64_t)i * T + t] = t;
  }
  if (r->final_params) memcpy(r->final_params, w, sizeof(double) * (size_t)P);
  if (r->worker_finals)
    for (int i = 0; i < N; ++i) memcpy(r->worker_finals + (int64_t)i * P, w, sizeof(double) * (size_t)P);
  for (int i = 0; i < n_samplers; ++i) free(samplers[i].perm);
  free(samplers);
  free(x);
  free(y);
  free(w);
  free(v);
  free(mb);
  free(pay);
  free(acc);
  free(sg);
  return rc;
}

/* Ordered collectives over in-memory rows (transport.cpp:17-96): op 0 reduce at root, 1 broadcast of
 * root's row, 2 allreduce (reduce at lowest id, then broadcast). */
int lo_collective(int op, int world, int root, int64_t n, const double* contrib, double* out) {
  if (world < 1 || root < 0 || root >= world) return 1;
  if (op == 1) {
    for (int r = 0; r < world; ++r) memcpy(out + (int64_t)r * n, contrib + (int64_t)root * n, sizeof(double) * (size_t)n);
    return 0;
  }
  double* acc = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(acc, contrib, sizeof(double) * (size_t)n);
  for (int r = 1; r < world; ++r)
    for (int64_t k = 0; k < n; ++k) acc[k] += contrib[(int64_t)r * n + k];
  if (op == 0) {
    memcpy(out + (int64_t)root * n, acc, sizeof(double) * (size_t)n);
  } else {
    for (int r = 0; r < world; ++r) memcpy(out + (int64_t)r * n, acc, sizeof(double) * (size_t)n);
  }
  free(acc);
  return 0;
}
