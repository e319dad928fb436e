// SIMT kernels of the LSGD step for sm_100a: shard gather (K1), the bit-faithful sequential-k GEMM used for the
// fp64 parity mode and as the fp32 fallback (K2/K4/K5), the softmax-CE head (K3), the ordered peer sums
// (K6/K7), the fused broadcast-pull + SGD/momentum update (K8) and the flag primitives that order them across
// GPUs. Rounding: in EXACT mode every multiply and add rounds separately (no FMA contraction), reproducing the
// reference's x86-64 build operation for operation (mlp.cpp:70-75, 110-123, 262-271; transport.cpp:27-48;
// optimizer.cpp:30-38).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "kernels.cuh"

namespace lsgd_b200 {

namespace {

template <typename T>
struct Rn;
template <>
struct Rn<float> {
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
  static __device__ __forceinline__ float fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
};
template <>
struct Rn<double> {
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double fma(double a, double b, double c) { return __fma_rn(a, b, c); }
};

// 16-byte vector of T.
template <typename T>
struct alignas(16) Vec {
  static constexpr int kN = 16 / sizeof(T);
  T v[kN];
};

template <typename T>
__device__ __forceinline__ Vec<T> ld16(const T* p) {
  return *reinterpret_cast<const Vec<T>*>(p);
}
template <typename T>
__device__ __forceinline__ void st16(T* p, const Vec<T>& v) {
  *reinterpret_cast<Vec<T>*>(p) = v;
}

// Dynamic shared memory requested by the update / exchange kernels (LSGD_B200_SIDE_SMEM, bytes; unused by the
// kernels): > 227 KB - the GEMM's 209 KB keeps them off SMs that hold a GEMM CTA (tuning knob).
inline size_t side_smem() {
  static const size_t n = [] {
    const char* e = std::getenv("LSGD_B200_SIDE_SMEM");
    return static_cast<size_t>(e ? std::atol(e) : 0);
  }();
  return n;
}

inline int grid_for(int64_t work, int threads, int cap = 148 * 8) {
  int64_t g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  return static_cast<int>(g < cap ? g : cap);
}

// ------------------------------------------------------------------------------------------------ K1 gather
template <typename T>
__global__ void gather_kernel(const T* __restrict__ rows, const int32_t* __restrict__ labels,
                              const int32_t* __restrict__ idx, int d, T* __restrict__ x, int32_t* __restrict__ y) {
  const int s = blockIdx.x;
  const int64_t r = idx[s];
  if (threadIdx.x == 0) y[s] = labels[r];
  const T* src = rows + r * d;
  T* dst = x + static_cast<int64_t>(s) * d;
  constexpr int V = Vec<T>::kN;
  if (d % V == 0) {
    for (int i = threadIdx.x; i < d / V; i += blockDim.x) st16(dst + i * V, ld16(src + i * V));
  } else {
    for (int i = threadIdx.x; i < d; i += blockDim.x) dst[i] = src[i];
  }
}

// ------------------------------------------------------------------------------------------------ K2/K4/K5
constexpr int kBM = 64, kBN = 64, kBK = 16;

template <typename T, bool EXACT, int EPI>
__global__ void __launch_bounds__(256) gemm_simt_kernel(int M, int N, int K, const T* __restrict__ A, int64_t lda_m,
                                                        int64_t lda_k, const T* __restrict__ B, int64_t ldb_k,
                                                        int64_t ldb_n, T* __restrict__ C, int64_t ldc,
                                                        const T* __restrict__ bias, int relu, T divisor,
                                                        const T* __restrict__ mask) {
  __shared__ T As[kBK][kBM + 1];
  __shared__ T Bs[kBK][kBN + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * kBN;
  T acc[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    int n = n0 + tx + 16 * j;
    T init = (EPI == kEpiForward && n < N) ? bias[n] : T(0);
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][j] = init;
  }
  const bool a_kfast = (lda_k == 1);
  const bool b_nfast = (ldb_n == 1);
  for (int k0 = 0; k0 < K; k0 += kBK) {
    for (int e = threadIdx.x; e < kBM * kBK; e += 256) {
      int kk, mm;
      if (a_kfast) { kk = e % kBK; mm = e / kBK; } else { mm = e % kBM; kk = e / kBM; }
      int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < M && k < K) ? A[m * lda_m + k * lda_k] : T(0);
    }
    for (int e = threadIdx.x; e < kBN * kBK; e += 256) {
      int kk, nn;
      if (b_nfast) { nn = e % kBN; kk = e / kBN; } else { kk = e % kBK; nn = e / kBK; }
      int n = n0 + nn, k = k0 + kk;
      Bs[kk][nn] = (n < N && k < K) ? B[k * ldb_k + n * ldb_n] : T(0);
    }
    __syncthreads();
    const int kmax = (K - k0) < kBK ? (K - k0) : kBK;  // never fold padding into the ordered sum
    for (int kk = 0; kk < kmax; ++kk) {
      T a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (EXACT) acc[i][j] = Rn<T>::add(acc[i][j], Rn<T>::mul(a[i], b[j]));
          else acc[i][j] = Rn<T>::fma(a[i], b[j], acc[i][j]);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int m = m0 + ty + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tx + 16 * j;
      if (n >= N) continue;
      T v = acc[i][j];
      if (EPI == kEpiForward) {
        if (relu && v < T(0)) v = T(0);
      } else if (EPI == kEpiWeightGrad) {
        v = Rn<T>::div(v, divisor);
      } else {
        if (!(mask[m * ldc + n] > T(0))) v = T(0);
      }
      C[m * ldc + n] = v;
    }
  }
}

// ------------------------------------------------------------------------------------------------ K3 head
template <typename T>
__device__ __forceinline__ T dexp(T x);
template <>
__device__ __forceinline__ float dexp<float>(float x) { return expf(x); }
template <>
__device__ __forceinline__ double dexp<double>(double x) { return exp(x); }
template <typename T>
__device__ __forceinline__ T dlog(T x);
template <>
__device__ __forceinline__ float dlog<float>(float x) { return logf(x); }
template <>
__device__ __forceinline__ double dlog<double>(double x) { return log(x); }

template <typename T>
__global__ void softmax_xent_kernel(const T* __restrict__ logits, const int32_t* __restrict__ labels, int b, int c,
                                    T* __restrict__ delta, T* __restrict__ sample_loss) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= b) return;
  const T* z = logits + static_cast<int64_t>(s) * c;
  T* dz = delta + static_cast<int64_t>(s) * c;
  T zmax = z[0];
  for (int k = 1; k < c; ++k) zmax = (zmax < z[k]) ? z[k] : zmax;
  T sum = T(0);
  for (int k = 0; k < c; ++k) sum = Rn<T>::add(sum, dexp<T>(Rn<T>::sub(z[k], zmax)));
  T lse = Rn<T>::add(zmax, dlog<T>(sum));
  int lab = labels[s];
  sample_loss[s] = Rn<T>::sub(lse, z[lab]);
  for (int k = 0; k < c; ++k) {
    T p = dexp<T>(Rn<T>::sub(z[k], lse));
    dz[k] = (k == lab) ? Rn<T>::sub(p, T(1)) : p;
  }
}

template <typename T>
__global__ void mean_loss_kernel(const T* __restrict__ sample_loss, int b, T* __restrict__ out) {
  T acc = T(0);
  for (int s = 0; s < b; ++s) acc = Rn<T>::add(acc, sample_loss[s]);
  *out = Rn<T>::div(acc, static_cast<T>(b));
}

template <typename T>
__global__ void bias_grad_kernel(const T* __restrict__ delta, int b, int n_out, T* __restrict__ db) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_out) return;
  T acc = T(0);
  for (int s = 0; s < b; ++s) acc = Rn<T>::add(acc, delta[static_cast<int64_t>(s) * n_out + j]);
  db[j] = Rn<T>::div(acc, static_cast<T>(b));
}

// ------------------------------------------------------------------------------------------------ K6/K7
// 2 vectors per thread per trip, every source load of both issued before the first add (NVLink latency is
// ~2 us; the loads of all peers for a vector are independent).
template <typename T>
__global__ void __launch_bounds__(256) ordered_sum_kernel(SrcList<T> src, int n_src, int64_t len, T* __restrict__ dst,
                                                          bool add_zero, T divisor, bool scalar_only) {
  constexpr int V = Vec<T>::kN;
  const int64_t nvec = scalar_only ? 0 : len / V;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nvec; i += 2 * stride) {
    const int64_t i1 = i + stride;
    const bool two = i1 < nvec;
    Vec<T> acc0 = ld16(src.p[0] + i * V), acc1;
    if (two) acc1 = ld16(src.p[0] + i1 * V);
    for (int s = 1; s < n_src; ++s) {
      Vec<T> x0 = ld16(src.p[s] + i * V), x1;
      if (two) x1 = ld16(src.p[s] + i1 * V);
#pragma unroll
      for (int q = 0; q < V; ++q) acc0.v[q] = Rn<T>::add(acc0.v[q], x0.v[q]);
      if (two) {
#pragma unroll
        for (int q = 0; q < V; ++q) acc1.v[q] = Rn<T>::add(acc1.v[q], x1.v[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < V; ++q) {
      if (add_zero) {
        acc0.v[q] = Rn<T>::add(acc0.v[q], T(0));
        acc1.v[q] = Rn<T>::add(acc1.v[q], T(0));
      }
      if (divisor != T(0)) {
        acc0.v[q] = Rn<T>::div(acc0.v[q], divisor);
        acc1.v[q] = Rn<T>::div(acc1.v[q], divisor);
      }
    }
    st16(dst + i * V, acc0);
    if (two) st16(dst + i1 * V, acc1);
  }
  // scalar tail (len is padded to a vector multiple by the engine; kept for standalone callers)
  for (int64_t e = nvec * V + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < len; e += stride) {
    T a = src.p[0][e];
    for (int s = 1; s < n_src; ++s) a = Rn<T>::add(a, src.p[s][e]);
    if (add_zero) a = Rn<T>::add(a, T(0));
    if (divisor != T(0)) a = Rn<T>::div(a, divisor);
    dst[e] = a;
  }
}

// ------------------------------------------------------------------------------------------------ K8
template <typename T, bool EXACT>
__device__ __forceinline__ void sgd_one(T& w, T& v, T d, const UpdateArgs<T>& a) {
  if (a.mode == 0) {
    w = EXACT ? Rn<T>::sub(w, Rn<T>::mul(a.lr, d)) : Rn<T>::fma(-a.lr, d, w);
  } else {
    if (EXACT) {
      T g = Rn<T>::add(d, Rn<T>::mul(a.weight_decay, w));
      v = Rn<T>::add(Rn<T>::mul(a.momentum, v), g);
      w = Rn<T>::sub(w, Rn<T>::mul(a.lr, v));
    } else {
      T g = Rn<T>::fma(a.weight_decay, w, d);
      v = Rn<T>::fma(a.momentum, v, g);
      w = Rn<T>::fma(-a.lr, v, w);
    }
  }
}

template <typename T>
__device__ __forceinline__ T pre_delta(T d, const UpdateArgs<T>& a) {
  if (a.add_zero) d = Rn<T>::add(d, T(0));  // the communicator's zero contribution (executors.cpp:278)
  if (a.post_div != T(0)) d = Rn<T>::div(d, a.post_div);
  return d;
}

__device__ __forceinline__ float tf32_round(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
template <typename T>
__device__ __forceinline__ void store_split(const UpdateArgs<T>&, int64_t, const T*, int) {}
template <>
__device__ __forceinline__ void store_split<float>(const UpdateArgs<float>& a, int64_t e, const float* w, int n) {
  if (!a.w_hi) return;
  if (n == 4) {
    float4 h = make_float4(tf32_round(w[0]), tf32_round(w[1]), tf32_round(w[2]), tf32_round(w[3]));
    *reinterpret_cast<float4*>(a.w_hi + e) = h;
    *reinterpret_cast<float4*>(a.w_lo + e) = make_float4(tf32_round(w[0] - h.x), tf32_round(w[1] - h.y),
                                                         tf32_round(w[2] - h.z), tf32_round(w[3] - h.w));
    return;
  }
  for (int q = 0; q < n; ++q) {
    float h = tf32_round(w[q]);
    a.w_hi[e + q] = h;
    a.w_lo[e + q] = tf32_round(w[q] - h);
  }
}

template <typename T, bool EXACT, int U>
__global__ void __launch_bounds__(256) update_kernel(UpdateArgs<T> a) {
  constexpr int V = Vec<T>::kN;
  const int64_t nvec = a.scalar_only ? 0 : a.n_params / V;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  bool bad = false;
  const bool mom = a.mode != 0;
  // U vectors per thread per trip, all loads issued before the math (memory-level parallelism with few CTAs)
  for (int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < nvec; i0 += U * stride) {
    Vec<T> d[U], w[U], v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < nvec && !(i * V >= a.skip_lo && i * V < a.skip_hi)) {
        const int64_t e = i * V;
        const int64_t j = e / a.slice_len;  // slice_len is a multiple of V: a vector never straddles slices
        d[u] = ld16(a.slices.p[j] + (e - j * a.slice_len));
        w[u] = ld16(a.w + e);
        if (mom) v[u] = ld16(a.v + e);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= nvec || (i * V >= a.skip_lo && i * V < a.skip_hi)) continue;
      const int64_t e = i * V;
#pragma unroll
      for (int q = 0; q < V; ++q) {
        T dq = pre_delta(d[u].v[q], a);
        T vq = mom ? v[u].v[q] : T(0);
        sgd_one<T, EXACT>(w[u].v[q], vq, dq, a);
        if (mom) v[u].v[q] = vq;
        bad |= !isfinite(w[u].v[q]);
      }
      st16(a.w + e, w[u]);
      if (mom) st16(a.v + e, v[u]);
      store_split<T>(a, e, w[u].v, V);
    }
  }
  const int64_t end = a.n_params + (a.loss_out ? 1 : 0);
  for (int64_t e = nvec * V + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < end; e += stride) {
    if (e >= a.skip_lo && e < a.skip_hi) continue;
    const int64_t j = e / a.slice_len;
    T d = pre_delta(a.slices.p[j][e - j * a.slice_len], a);
    if (e == a.n_params) {  // the loss slot rides the same reduction (executors.cpp:59-63, 226)
      *a.loss_out = d;
      continue;
    }
    T w = a.w[e], v = mom ? a.v[e] : T(0);
    sgd_one<T, EXACT>(w, v, d, a);
    a.w[e] = w;
    if (mom) a.v[e] = v;
    store_split<T>(a, e, &w, 1);
    bad |= !isfinite(w);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x % 32) == 0) atomicOr(a.bad, 1u);
}

// ------------------------------------------------------------------------------------------------ flags
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spin (one thread per flag) until every flag reaches `target`. Protocol check: a flag above target + max_lead
// means its producer has already written a LATER round into a buffer this consumer has not read yet (a WAR
// violation of the round-counter protocol); that is reported as code 2 through `timed_out` (TransportError on the
// host) instead of silently consuming overwritten data.
__global__ void wait_flags_kernel(FlagList fl, int n, unsigned long long target, unsigned long long max_lead,
                                  unsigned long long timeout_ns, volatile int* timed_out) {
  const int i = threadIdx.x;
  if (i < n) {
    const unsigned long long t0 = globaltimer();
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(fl.f[i]) : "memory");
      if (v >= target) {
        if (v - target > max_lead) {  // (no overflow for max_lead = ~0: check disabled)
          *timed_out = 2;
          __threadfence_system();
        }
        break;
      }
      if (*timed_out) break;  // another waiter (or the host, to abort) already gave up
      if (globaltimer() - t0 > timeout_ns) {
        *timed_out = 1;
        __threadfence_system();
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
}

template <typename T>
__global__ void __launch_bounds__(256) push_kernel(const T* __restrict__ src, int64_t len, DstList<T> dst, int n_dst) {
  constexpr int V = Vec<T>::kN;
  const int64_t nvec = len / V;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nvec; i += stride) {
    const Vec<T> v = ld16(src + i * V);
    for (int d = 0; d < n_dst; ++d) st16(dst.p[d] + i * V, v);
  }
  for (int64_t e = nvec * V + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < len; e += stride)
    for (int d = 0; d < n_dst; ++d) dst.p[d][e] = src[e];
}

// Push-based exchange (all reads local, all cross-GPU traffic as NVLink stores, which need no round trip):
// dst_d[e] = ((src_0[e] + src_1[e]) + ... [+ 0.0]) [/ divisor] for every destination d (ordered sum, K6/K7), and
// the pairwise copies of the member -> owner scatter. Grid-capped (they co-run with the GEMMs), so each thread
// keeps U vectors of every source in flight (NS = source count, 0 = runtime count) to cover HBM latency.
template <typename T, int NS, int U>
__global__ void __launch_bounds__(256) reduce_push_kernel(const __grid_constant__ SrcList<T> src, int n_src, int64_t len,
                                                          const __grid_constant__ DstList<T> dst, int n_dst,
                                                          bool add_zero, T divisor) {
  constexpr int V = Vec<T>::kN;
  constexpr int NSX = NS > 0 ? NS : 1;
  const int ns = NS > 0 ? NS : n_src;
  const int64_t nvec = len / V;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < nvec; i0 += U * stride) {
    Vec<T> acc[U];
    if (NS > 0) {
      Vec<T> x[NSX][U];
#pragma unroll
      for (int s = 0; s < NSX; ++s)
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (i0 + u * stride < nvec) x[s][u] = ld16(src.p[s] + (i0 + u * stride) * V);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc[u] = x[0][u];
#pragma unroll
        for (int s = 1; s < NSX; ++s)
#pragma unroll
          for (int q = 0; q < V; ++q) acc[u].v[q] = Rn<T>::add(acc[u].v[q], x[s][u].v[q]);
      }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i0 + u * stride < nvec) acc[u] = ld16(src.p[0] + (i0 + u * stride) * V);
      for (int s = 1; s < ns; ++s) {
        Vec<T> x[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (i0 + u * stride < nvec) x[u] = ld16(src.p[s] + (i0 + u * stride) * V);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int q = 0; q < V; ++q) acc[u].v[q] = Rn<T>::add(acc[u].v[q], x[u].v[q]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int q = 0; q < V; ++q) {
        if (add_zero) acc[u].v[q] = Rn<T>::add(acc[u].v[q], T(0));
        if (divisor != T(0)) acc[u].v[q] = Rn<T>::div(acc[u].v[q], divisor);
      }
    }
    for (int d = 0; d < n_dst; ++d)
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i0 + u * stride < nvec) st16(dst.p[d] + (i0 + u * stride) * V, acc[u]);
  }
  for (int64_t e = nvec * V + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < len; e += stride) {
    T a = src.p[0][e];
    for (int s = 1; s < ns; ++s) a = Rn<T>::add(a, src.p[s][e]);
    if (add_zero) a = Rn<T>::add(a, T(0));
    if (divisor != T(0)) a = Rn<T>::div(a, divisor);
    for (int d = 0; d < n_dst; ++d) dst.p[d][e] = a;
  }
}

template <typename T, int U>
__global__ void __launch_bounds__(256) copy_pairs_kernel(const __grid_constant__ SrcList<T> src,
                                                         const __grid_constant__ DstList<T> dst, int n_pairs,
                                                         int64_t len) {
  constexpr int V = Vec<T>::kN;
  const int64_t nvec = len / V;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int p = 0; p < n_pairs; ++p) {
    const T* __restrict__ sp = src.p[p];
    T* dp = dst.p[p];
    for (int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < nvec; i0 += U * stride) {
      Vec<T> x[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i0 + u * stride < nvec) x[u] = ld16(sp + (i0 + u * stride) * V);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i0 + u * stride < nvec) st16(dp + (i0 + u * stride) * V, x[u]);
    }
    for (int64_t e = nvec * V + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < len; e += stride)
      dp[e] = sp[e];
  }
}

template <typename T>
__device__ __forceinline__ UpdateArgs<T> gu_split_args(const GlobalUpdateArgs<T>&) {
  return UpdateArgs<T>{};
}
template <>
__device__ __forceinline__ UpdateArgs<float> gu_split_args<float>(const GlobalUpdateArgs<float>& a) {
  UpdateArgs<float> u{};
  u.w_hi = a.w_hi;
  u.w_lo = a.w_lo;
  return u;
}

template <typename T, bool EXACT>
__device__ __forceinline__ void gu_update_one(const GlobalUpdateArgs<T>& a, int64_t idx, T d, bool& bad) {
  if (idx < a.n_params) {
    T w = a.w[idx], v = a.mode ? a.v[idx] : T(0);
    UpdateArgs<T> u = gu_split_args<T>(a);
    u.mode = a.mode;
    u.lr = a.lr;
    u.momentum = a.momentum;
    u.weight_decay = a.weight_decay;
    sgd_one<T, EXACT>(w, v, d, u);
    a.w[idx] = w;
    if (a.mode) a.v[idx] = v;
    store_split<T>(u, idx, &w, 1);
    bad |= !isfinite(w);
  } else if (idx == a.n_params && a.loss_out) {
    *a.loss_out = d;
  }
}

// One 16-byte store through an NVLS multicast address: the NVSwitch writes it into every bound member's memory.
__device__ __forceinline__ void multimem_st(float* p, const Vec<float>& v) {
  asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.v[0]), "f"(v.v[1]), "f"(v.v[2]),
               "f"(v.v[3])
               : "memory");
}
__device__ __forceinline__ void multimem_st(double* p, const Vec<double>& v) {
  asm volatile("multimem.st.global.f64 [%0], %1;" ::"l"(p), "d"(v.v[0]) : "memory");  // (no .v2.f64 form)
  asm volatile("multimem.st.global.f64 [%0], %1;" ::"l"(p + 1), "d"(v.v[1]) : "memory");
}

template <typename T, bool EXACT>
__global__ void __launch_bounds__(256) global_update_kernel(const __grid_constant__ GlobalUpdateArgs<T> a,
                                                            bool vec_params) {
  constexpr int V = Vec<T>::kN;
  const int64_t nvec = a.len / V;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  UpdateArgs<T> u = gu_split_args<T>(a);  // carries w_hi / w_lo for store_split
  u.mode = a.mode;
  u.lr = a.lr;
  u.momentum = a.momentum;
  u.weight_decay = a.weight_decay;
  bool bad = false;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nvec; i += stride) {
    const int64_t e = i * V;
    auto member_sum = [&](int base) {  // a group's slot sum from its k member sub-slices (K6 order, + 0.0, / N)
      Vec<T> s = ld16(a.src.p[base] + e);
      for (int m = 1; m < a.k; ++m) {
        const Vec<T> x = ld16(a.src.p[base + m] + e);
#pragma unroll
        for (int q = 0; q < V; ++q) s.v[q] = Rn<T>::add(s.v[q], x.v[q]);
      }
#pragma unroll
      for (int q = 0; q < V; ++q) {
        if (a.add_zero) s.v[q] = Rn<T>::add(s.v[q], T(0));
        if (a.divisor != T(0)) s.v[q] = Rn<T>::div(s.v[q], a.divisor);
      }
      return s;
    };
    const Vec<T> s = member_sum(a.direct ? a.g * a.k : 0);  // this group's slot sum, recomputed
    auto group_sum = [&](int gg) {  // the other groups' K6 results (recomputed from raw payloads when k = 1)
      if (a.direct) return member_sum(gg * a.k);
      Vec<T> x = ld16(a.gsum.p[gg] + e);
      if (a.gsum_raw) {
#pragma unroll
        for (int q = 0; q < V; ++q) {
          if (a.add_zero) x.v[q] = Rn<T>::add(x.v[q], T(0));
          if (a.divisor != T(0)) x.v[q] = Rn<T>::div(x.v[q], a.divisor);
        }
      }
      return x;
    };
    Vec<T> r = a.g == 0 ? s : group_sum(0);  // K7: ascending group order
    for (int gg = 1; gg < a.G; ++gg) {
      const Vec<T> x = gg == a.g ? s : group_sum(gg);
#pragma unroll
      for (int q = 0; q < V; ++q) r.v[q] = Rn<T>::add(r.v[q], x.v[q]);
    }
    if (a.mc) multimem_st(a.mc + e, r);  // NVLS: one store, replicated by the switch to every member
    for (int d = 0; d < a.n_push; ++d) st16(a.push.p[d] + e, r);  // broadcast to the other members
    if (a.out_local) st16(a.out_local + e, r);
    const int64_t i0 = a.first + e;
    if (vec_params && i0 + V <= a.n_params) {  // K8 on the owner's own parameters
      Vec<T> w = ld16(a.w + i0), v;
      if (a.mode) v = ld16(a.v + i0);
#pragma unroll
      for (int q = 0; q < V; ++q) {
        T vq = a.mode ? v.v[q] : T(0);
        sgd_one<T, EXACT>(w.v[q], vq, r.v[q], u);
        if (a.mode) v.v[q] = vq;
        bad |= !isfinite(w.v[q]);
      }
      st16(a.w + i0, w);
      if (a.mode) st16(a.v + i0, v);
      store_split<T>(u, i0, w.v, V);
    } else {
#pragma unroll
      for (int q = 0; q < V; ++q) gu_update_one<T, EXACT>(a, i0 + q, r.v[q], bad);
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x % 32) == 0) atomicOr(a.bad, 1u);
}

__global__ void store_u64_kernel(unsigned long long* p, unsigned long long v) { *p = v; }
__global__ void min_u64_kernel(const unsigned long long* ver, int b0, int b1, long long* dst) {
  unsigned long long m = ~0ull;
  for (int b = b0; b < b1; ++b) m = min(m, ver[b]);
  *dst = static_cast<long long>(m);
}

__global__ void signal_many_kernel(SignalList fl, int n, unsigned long long v) {
  __threadfence_system();
  if (threadIdx.x < n) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(fl.f[threadIdx.x]), "l"(v) : "memory");
}

__global__ void signal_flag_kernel(unsigned long long* f, unsigned long long v) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(v) : "memory");
}

__global__ void sleep_kernel(unsigned long long ns) {
  const unsigned long long t0 = globaltimer();
  while (globaltimer() - t0 < ns) __nanosleep(1000);
}

template <typename T>
__global__ void from_f64_kernel(const double* __restrict__ s, int64_t n, T* __restrict__ d) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    d[i] = static_cast<T>(s[i]);
}
template <typename T>
__global__ void to_f64_kernel(const T* __restrict__ s, int64_t n, double* __restrict__ d) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    d[i] = static_cast<double>(s[i]);
}

}  // namespace

// ------------------------------------------------------------------------------------------------ launchers
template <typename T>
void launch_gather(const T* rows, const int32_t* labels, const int32_t* idx, int b, int d, T* x, int32_t* y,
                   cudaStream_t st, LaunchCounter& lc) {
  gather_kernel<T><<<b, 256, 0, st>>>(rows, labels, idx, d, x, y);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

template <typename T>
void launch_gemm_simt(int epi, bool exact, int M, int N, int K, const T* A, int64_t lda_m, int64_t lda_k, const T* B,
                      int64_t ldb_k, int64_t ldb_n, T* C, int64_t ldc, const T* bias, int relu, T divisor,
                      const T* mask, cudaStream_t st, LaunchCounter& lc) {
  dim3 grid((N + kBN - 1) / kBN, (M + kBM - 1) / kBM);
#define LSGD_GEMM_CASE(E, X)                                                                                    \
  gemm_simt_kernel<T, X, E><<<grid, 256, 0, st>>>(M, N, K, A, lda_m, lda_k, B, ldb_k, ldb_n, C, ldc, bias, relu, \
                                                  divisor, mask)
  if (exact) {
    if (epi == kEpiForward) LSGD_GEMM_CASE(kEpiForward, true);
    else if (epi == kEpiWeightGrad) LSGD_GEMM_CASE(kEpiWeightGrad, true);
    else LSGD_GEMM_CASE(kEpiInputGrad, true);
  } else {
    if (epi == kEpiForward) LSGD_GEMM_CASE(kEpiForward, false);
    else if (epi == kEpiWeightGrad) LSGD_GEMM_CASE(kEpiWeightGrad, false);
    else LSGD_GEMM_CASE(kEpiInputGrad, false);
  }
#undef LSGD_GEMM_CASE
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

template <typename T>
void launch_softmax_xent(const T* logits, const int32_t* labels, int b, int c, T* delta, T* sample_loss,
                         cudaStream_t st, LaunchCounter& lc) {
  softmax_xent_kernel<T><<<(b + 127) / 128, 128, 0, st>>>(logits, labels, b, c, delta, sample_loss);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

template <typename T>
void launch_mean_loss(const T* sample_loss, int b, T* out, cudaStream_t st, LaunchCounter& lc) {
  mean_loss_kernel<T><<<1, 1, 0, st>>>(sample_loss, b, out);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

template <typename T>
void launch_bias_grad(const T* delta, int b, int n_out, T* db, cudaStream_t st, LaunchCounter& lc) {
  bias_grad_kernel<T><<<(n_out + 127) / 128, 128, 0, st>>>(delta, b, n_out, db);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

template <typename T>
void launch_ordered_sum(SrcList<T> src, int n_src, int64_t len, T* dst, bool add_zero, T divisor, cudaStream_t st,
                        LaunchCounter& lc) {
  int64_t work = (len / Vec<T>::kN + 1) / 2 + 1;
  bool scalar = (reinterpret_cast<uintptr_t>(dst) & 15u) != 0;
  for (int i = 0; i < n_src; ++i) scalar = scalar || (reinterpret_cast<uintptr_t>(src.p[i]) & 15u) != 0;
  if (scalar) work = len;
  ordered_sum_kernel<T><<<grid_for(work, 256), 256, 0, st>>>(src, n_src, len, dst, add_zero, divisor, scalar);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

template <typename T>
void launch_update(const UpdateArgs<T>& a_in, bool exact, cudaStream_t st, LaunchCounter& lc) {
  UpdateArgs<T> a = a_in;
  auto misaligned = [](const void* p) { return p != nullptr && (reinterpret_cast<uintptr_t>(p) & 15u) != 0; };
  bool slices_ok = a.slice_len % Vec<T>::kN == 0;
  for (int j = 0; j < kMaxPeers && a.slices.p[j]; ++j) slices_ok = slices_ok && !misaligned(a.slices.p[j]);
  a.scalar_only = (misaligned(a.w) || misaligned(a.v) || misaligned(a.w_hi) || misaligned(a.w_lo) || !slices_ok) ? 1 : 0;
  static const int unroll = [] {
    const char* e = std::getenv("LSGD_B200_UPD_UNROLL");
    const int v = e ? std::atoi(e) : 1;
    return (v == 2 || v == 4) ? v : 1;
  }();
  int64_t work = a.scalar_only ? a.n_params + 1 : a.n_params / Vec<T>::kN / unroll + 1;
  static const int cap = [] {
    const char* e = std::getenv("LSGD_B200_UPD_CTAS");
    const int v = e ? std::atoi(e) : 148 * 8;
    return v > 0 ? v : 148 * 8;
  }();
  int g = grid_for(work, 256, cap);
#define LSGD_UPD(X, UU) update_kernel<T, X, UU><<<g, 256, side_smem(), st>>>(a)
  if (exact) {
    if (unroll == 1) LSGD_UPD(true, 1);
    else if (unroll == 4) LSGD_UPD(true, 4);
    else LSGD_UPD(true, 2);
  } else {
    if (unroll == 1) LSGD_UPD(false, 1);
    else if (unroll == 4) LSGD_UPD(false, 4);
    else LSGD_UPD(false, 2);
  }
#undef LSGD_UPD
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

void launch_store_u64(unsigned long long* ver, unsigned long long value, cudaStream_t st, LaunchCounter& lc) {
  store_u64_kernel<<<1, 1, 0, st>>>(ver, value);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}
void launch_min_u64(const unsigned long long* ver, int b0, int b1, long long* dst, cudaStream_t st,
                    LaunchCounter& lc) {
  min_u64_kernel<<<1, 1, 0, st>>>(ver, b0, b1, dst);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

// Experimental (LSGD_B200_WAIT_MEMOP=1, A/B only): the wait as cuStreamWaitValue64 (GEQ) stream memory operations —
// no SM slot — at the price of the device-side timeout and protocol check.
using StreamWaitValue64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
StreamWaitValue64 stream_wait_value64() {
  static StreamWaitValue64 fn = [] {
    const char* e = std::getenv("LSGD_B200_WAIT_MEMOP");
    if (!(e && std::atoi(e) != 0)) return static_cast<StreamWaitValue64>(nullptr);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<StreamWaitValue64>(nullptr);
    }
    return reinterpret_cast<StreamWaitValue64>(p);
  }();
  return fn;
}

void launch_wait_flags(FlagList flags, int n, unsigned long long target, unsigned long long timeout_ns,
                       volatile int* timed_out, cudaStream_t st, LaunchCounter& lc, unsigned long long max_lead) {
  if (StreamWaitValue64 wv = max_lead != ~0ull ? stream_wait_value64() : nullptr) {
    for (int i = 0; i < n; ++i) {
      const CUresult r = wv(reinterpret_cast<CUstream>(st),
                            reinterpret_cast<CUdeviceptr>(const_cast<unsigned long long*>(flags.f[i])), target,
                            CU_STREAM_WAIT_VALUE_GEQ);
      check<Error>(r == CUDA_SUCCESS, "cuStreamWaitValue64 failed (", static_cast<int>(r), ")");
    }
    return;
  }
  wait_flags_kernel<<<1, 32, 0, st>>>(flags, n, target, max_lead, timeout_ns, timed_out);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

void launch_signal_flag(unsigned long long* flag, unsigned long long value, cudaStream_t st, LaunchCounter& lc) {
  signal_flag_kernel<<<1, 1, 0, st>>>(flag, value);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

template <typename T>
void launch_push(const T* src, int64_t len, DstList<T> dst, int n_dst, cudaStream_t st, LaunchCounter& lc) {
  push_kernel<T><<<grid_for(len / Vec<T>::kN + 1, 256, 148 * 2), 256, 0, st>>>(src, len, dst, n_dst);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

int comm_ctas() {
  static const int n = [] {
    const char* e = std::getenv("LSGD_B200_COMM_CTAS");
    const int v = e ? std::atoi(e) : 148;
    return v > 0 ? v : 148;
  }();
  return n;
}

template <typename T>
void launch_reduce_push(SrcList<T> src, int n_src, int64_t len, DstList<T> dst, int n_dst, bool add_zero, T divisor,
                        cudaStream_t st, LaunchCounter& lc) {
  bool aligned = true;
  for (int i = 0; i < n_src; ++i) aligned = aligned && (reinterpret_cast<uintptr_t>(src.p[i]) & 15u) == 0;
  for (int i = 0; i < n_dst; ++i) aligned = aligned && (reinterpret_cast<uintptr_t>(dst.p[i]) & 15u) == 0;
  check<Error>(aligned && len % Vec<T>::kN == 0, "reduce_push: slices must be 16-byte aligned vectors");
  check<Error>(n_src >= 1 && n_src <= kMaxPeers && n_dst >= 1 && n_dst <= kMaxPeers, "reduce_push: bad fan-in/out");
  constexpr int U = 4;
  const int g = grid_for(len / Vec<T>::kN / U + 1, 256, comm_ctas());
  switch (n_src) {
    case 1: reduce_push_kernel<T, 1, U><<<g, 256, side_smem(), st>>>(src, n_src, len, dst, n_dst, add_zero, divisor); break;
    case 2: reduce_push_kernel<T, 2, U><<<g, 256, side_smem(), st>>>(src, n_src, len, dst, n_dst, add_zero, divisor); break;
    case 4: reduce_push_kernel<T, 4, U><<<g, 256, side_smem(), st>>>(src, n_src, len, dst, n_dst, add_zero, divisor); break;
    default: reduce_push_kernel<T, 0, U><<<g, 256, side_smem(), st>>>(src, n_src, len, dst, n_dst, add_zero, divisor); break;
  }
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

template <typename T>
void launch_copy_pairs(SrcList<T> src, DstList<T> dst, int n_pairs, int64_t len, cudaStream_t st, LaunchCounter& lc) {
  if (n_pairs == 0) return;
  copy_pairs_kernel<T, 4><<<grid_for(len / Vec<T>::kN / 4 + 1, 256, comm_ctas()), 256, side_smem(), st>>>(src, dst, n_pairs,
                                                                                                  len);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

template <typename T>
void launch_global_update(const GlobalUpdateArgs<T>& a, bool exact, cudaStream_t st, LaunchCounter& lc) {
  bool aligned = a.len % Vec<T>::kN == 0;
  const int n_src = a.direct ? a.k * a.G : a.k;
  for (int i = 0; i < n_src; ++i) aligned = aligned && (reinterpret_cast<uintptr_t>(a.src.p[i]) & 15u) == 0;
  for (int g = 0; g < a.G && !a.direct; ++g)
    if (g != a.g) aligned = aligned && (reinterpret_cast<uintptr_t>(a.gsum.p[g]) & 15u) == 0;
  for (int d = 0; d < a.n_push; ++d) aligned = aligned && (reinterpret_cast<uintptr_t>(a.push.p[d]) & 15u) == 0;
  if (a.out_local) aligned = aligned && (reinterpret_cast<uintptr_t>(a.out_local) & 15u) == 0;
  if (a.mc) aligned = aligned && (reinterpret_cast<uintptr_t>(a.mc) & 15u) == 0;
  check<Error>(aligned, "global_update: slices must be 16-byte aligned vectors");
  const bool vec_params = (reinterpret_cast<uintptr_t>(a.w + a.first) & 15u) == 0 &&
                          (a.v == nullptr || (reinterpret_cast<uintptr_t>(a.v + a.first) & 15u) == 0);
  static const int cap = [] {  // LSGD_B200_GLOBAL_CTAS (A/B knob)
    const char* e = std::getenv("LSGD_B200_GLOBAL_CTAS");
    const int v = e ? std::atoi(e) : 148 * 8;
    return v > 0 ? v : 148 * 8;
  }();
  const int g = grid_for(a.len / Vec<T>::kN + 1, 256, cap);
  if (exact) global_update_kernel<T, true><<<g, 256, side_smem(), st>>>(a, vec_params);
  else global_update_kernel<T, false><<<g, 256, side_smem(), st>>>(a, vec_params);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

// Release of cross-GPU round counters after the prior work of the stream. By default a stream memory operation
// (cuStreamWriteValue64, executed by the GPU front end with a system-wide fence before the write): it needs no SM,
// so a flag is released as soon as its copy or kernel ends even when long-running kernels hold every SM's thread
// slots (a 1-CTA signal kernel then waits for them — up to ~200 us per hop, profiles/r2_timeline_n4_waits.txt).
// LSGD_B200_SIGNAL_MEMOP=0: the signal kernel.
using StreamWriteValue64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
StreamWriteValue64 stream_write_value64() {
  static StreamWriteValue64 fn = [] {
    const char* e = std::getenv("LSGD_B200_SIGNAL_MEMOP");
    if (e && std::atoi(e) == 0) return static_cast<StreamWriteValue64>(nullptr);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<StreamWriteValue64>(nullptr);
    }
    return reinterpret_cast<StreamWriteValue64>(p);
  }();
  return fn;
}

void launch_signal_many(SignalList flags, int n, unsigned long long value, cudaStream_t st, LaunchCounter& lc) {
  // One destination: the memop. Several: one kernel (one fence, n stores) — each fenced memop costs more than the
  // kernel saves there, and dropping the fence on the later writes is not safe (A/B: 1x4 / 4x1 -4..5% with a memop
  // per flag, 2x2 +1.4% with memops; profiles/r2_signal_memop_ab.log).
  StreamWriteValue64 wv = n == 1 ? stream_write_value64() : nullptr;
  if (wv) {
    const CUresult r = wv(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(flags.f[0]), value, 0);
    check<Error>(r == CUDA_SUCCESS, "cuStreamWriteValue64 failed (", static_cast<int>(r), ")");
    return;
  }
  signal_many_kernel<<<1, 32, 0, st>>>(flags, n, value);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

void launch_sleep(double seconds, cudaStream_t st, LaunchCounter& lc) {
  if (seconds <= 0.0) return;
  sleep_kernel<<<1, 1, 0, st>>>(static_cast<unsigned long long>(seconds * 1e9));
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

template <typename T>
void launch_from_f64(const double* src, int64_t n, T* dst, cudaStream_t st, LaunchCounter& lc) {
  from_f64_kernel<T><<<grid_for(n, 256), 256, 0, st>>>(src, n, dst);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}
template <typename T>
void launch_to_f64(const T* src, int64_t n, double* dst, cudaStream_t st, LaunchCounter& lc) {
  to_f64_kernel<T><<<grid_for(n, 256), 256, 0, st>>>(src, n, dst);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

#define LSGD_INSTANTIATE(T)                                                                                        \
  template void launch_gather<T>(const T*, const int32_t*, const int32_t*, int, int, T*, int32_t*, cudaStream_t,    \
                                 LaunchCounter&);                                                                  \
  template void launch_gemm_simt<T>(int, bool, int, int, int, const T*, int64_t, int64_t, const T*, int64_t,       \
                                    int64_t, T*, int64_t, const T*, int, T, const T*, cudaStream_t, LaunchCounter&); \
  template void launch_softmax_xent<T>(const T*, const int32_t*, int, int, T*, T*, cudaStream_t, LaunchCounter&);  \
  template void launch_mean_loss<T>(const T*, int, T*, cudaStream_t, LaunchCounter&);                              \
  template void launch_bias_grad<T>(const T*, int, int, T*, cudaStream_t, LaunchCounter&);                         \
  template void launch_ordered_sum<T>(SrcList<T>, int, int64_t, T*, bool, T, cudaStream_t, LaunchCounter&);        \
  template void launch_update<T>(const UpdateArgs<T>&, bool, cudaStream_t, LaunchCounter&);                        \
  template void launch_from_f64<T>(const double*, int64_t, T*, cudaStream_t, LaunchCounter&);                      \
  template void launch_to_f64<T>(const T*, int64_t, double*, cudaStream_t, LaunchCounter&);                       \
  template void launch_push<T>(const T*, int64_t, DstList<T>, int, cudaStream_t, LaunchCounter&);                 \
  template void launch_reduce_push<T>(SrcList<T>, int, int64_t, DstList<T>, int, bool, T, cudaStream_t,              \
                                      LaunchCounter&);                                                             \
  template void launch_copy_pairs<T>(SrcList<T>, DstList<T>, int, int64_t, cudaStream_t, LaunchCounter&);         \
  template void launch_global_update<T>(const GlobalUpdateArgs<T>&, bool, cudaStream_t, LaunchCounter&);

LSGD_INSTANTIATE(float)
LSGD_INSTANTIATE(double)

}  // namespace lsgd_b200
