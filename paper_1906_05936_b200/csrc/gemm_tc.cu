// tcgen05 split-TF32 GEMM for sm_100a. See gemm_tc.cuh for the numerics.
//
// Persistent kernel, one CTA per SM, 128 x 256 fp32 tiles D = A * B^T (TN form: A is M x K, B is N x K) in TMEM:
//   warp 0      TMA producer: per 16-wide K block, A_hi, A_lo, B_hi, B_lo -> one 48 KB smem stage (4-stage ring)
//   warp 1      TMEM allocator + single-thread MMA issuer: per 8-wide K step three tcgen05.mma.kind::tf32
//               (hi*lo, lo*hi, hi*hi) accumulate into one of two 256-column TMEM accumulators, K in chunks of
//               512 (chunk 0 -> the tile's sum S, later chunks -> the other accumulator X); tcgen05.commit frees
//               the stage / hands a finished chunk to the epilogue warps
//   warps 2..5  fold each later chunk into S (S + X, round to nearest: the tensor pipe's own fp32 accumulation
//               does not round, its error grows with K), then the epilogue (overlapping the next tile's first
//               chunk): tcgen05.ld 32x32b -> registers -> fused bias/ReLU | /B | ReLU-mask, fp32 output plus the
//               hi/lo split the next GEMM consumes; with WS they also split the raw weight k-blocks into hi/lo
// Operands may be K-major ([rows][K], TMA SWIZZLE_64B / UMMA SWIZZLE_64B) or MN-major ([K][rows], TMA
// SWIZZLE_128B_ATOM_32B / UMMA SWIZZLE_128B_BASE32B, the only MN-major layout tf32 supports), so dX (W read
// MN-major) and dW (delta and activations read MN-major) need no transposed copies.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "gemm_tc.cuh"

namespace lsgd_b200 {

namespace {

// BK = 16. PAIR = 1: one CTA per 128 x 256 tile, 48 KB stages x 4. PAIR = 2 (cta_group::2): a CTA pair computes a
// 256 x 256 tile, each CTA staging its 128 rows of A and half (128 rows) of B -> 32 KB stages x 6; per MMA flop the
// pair moves 1/3 fewer bytes from L2 than two single CTAs (the 1-CTA kernel is L2-throughput bound).
constexpr int BM = 128, BN = 256, BK = 16, THREADS = 192;
constexpr int MN_CHUNK_BYTES = BK * 128;  // one 32-wide MN chunk of an MN-major tile: BK rows of 128 B
constexpr int A_BYTES = BM * BK * 4;      // 8 KB
constexpr int STAGE_RING_BYTES = 192 * 1024;
constexpr int EPI_STAGE_BYTES = 32 * 32 * 4;  // per epilogue warp: one 32 x 32 fp32 chunk (4 KB)
// fused update: per epilogue warp, w and v of one 32 x 32 chunk (8 KB), double-buffered (cp.async one chunk ahead)
constexpr int UPD_PREF_BYTES = 2 * 2 * EPI_STAGE_BYTES;
// kWgradUpd: dW + fused update; kWgradScat: dW scattered to the sub-slice owners (each its own instantiation, so the
// plain weight-gradient kernel carries neither path)
enum : int { kFwd = 0, kWgrad = 1, kIgrad = 2, kRaw = 3, kWgradUpd = 4, kWgradScat = 5 };
template <int PAIR, int EPI = kFwd, bool WS = false>
struct Cfg {
  static constexpr int B_ROWS = BN / PAIR;                          // B rows staged by one CTA
  static constexpr int B_BYTES = B_ROWS * BK * 4;                   // 16 KB | 8 KB
  // WS: B (the weights) arrives as raw fp32 and is split into hi / lo in shared memory (no w_hi / w_lo in HBM)
  static constexpr int RAW_BYTES = WS ? B_BYTES : 0;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES + RAW_BYTES;  // 48 | 32 KB (+16 | 8 KB raw)
  // the fused-update epilogue trades mainloop stages (K = B is short) for its w/v staging
  static constexpr int STAGES = EPI == kWgradUpd ? (PAIR == 2 ? 4 : 3)
                                : (WS ? (208 * 1024) / STAGE_BYTES : STAGE_RING_BYTES / STAGE_BYTES);  // 4 | 6 (WS: 3 | 5)
  static constexpr int RING = STAGES * STAGE_BYTES;
  static constexpr int PREF = EPI == kWgradUpd ? 4 * UPD_PREF_BYTES : 0;
  static constexpr int SMEM = RING + 4 * EPI_STAGE_BYTES + PREF + 1024;  // + alignment slack
  static_assert(SMEM <= 232448, "dynamic shared memory over the sm_100 limit");
};
constexpr uint32_t TMEM_COLS = 256;
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // clears the CTA-rank bit of a shared::cluster address -> leader CTA

struct EpiParams {
  float* out;
  int64_t ldo;
  float* out_hi;
  float* out_lo;
  const float* bias;
  const float* mask;
  int64_t ldm;
  int relu;
  float div;
  float* partial;  // split-K raw partial sums [splits][M][N]
  int M, N;
  uint32_t mn_lbo, mn_sbo, mn_layout;  // MN-major descriptor geometry (see op_desc)
  uint32_t prefetch;                   // prefetch.tensormap the four operand maps
  int div_pow2;                        // div is a power of two: multiply by the exact reciprocal
  float div_inv;
  uint32_t probe;  // bring-up/tuning only (LSGD_TC_PROBE): 1 skip epilogue stores, 2 skip MMAs, 4 skip TMA loads
  int kcb;         // K blocks per accumulation chunk (>= the K extent: one chunk; see the kernel comment)
  BucketScatter scat;  // weight-gradient output routed to the sub-slice owners (n = 0: plain ep.out)
  int fuse_upd;        // weight gradient: apply the update (upd) instead of storing the gradient
  FusedUpdate upd;
};



// Destination of bucket-local element e (a float4 never straddles sub-slices: S is a multiple of 64).
__device__ __forceinline__ float* scatter_at(const BucketScatter& sc, int64_t e) {
  int j = 0;
  while (j + 1 < sc.n && e >= (j + 1) * sc.S) ++j;
  return sc.dst[j] + (e - j * sc.S);
}

// ------------------------------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(su32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {  // non-blocking probe
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(su32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  while (!mbar_try(b, parity)) {
  }
}
__device__ __forceinline__ void tma_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_3d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// cta_group::2 TMA: data lands in the issuing CTA's smem, the byte count completes on the leader's barrier.
__device__ __forceinline__ void tma_2d_pair(const CUtensorMap* map, uint32_t bar, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_3d_pair(const CUtensorMap* map, uint32_t bar, void* dst, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(smem_dst)), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 32 lanes x 32 columns of fp32 between TMEM and registers (one warp, its lane quadrant)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accum) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accum) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
// Arrive on the barrier at this offset in both CTAs of the pair once the issued MMAs complete.
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n .reg .b16 m;\n mov.b16 m, 3;\n"
      " tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}\n" ::"r"(
          su32(bar))
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}

// Shared-memory matrix descriptor, sm_100 version 1. layout: 2 = SWIZZLE_128B (K-major operands),
// 1 = SWIZZLE_128B_BASE32B (the only MN-major layout tf32 operands support: 32-byte chunks of each 128 B MN row
// XOR-swizzled over 4-row K atoms; written by TMA's SWIZZLE_128B_ATOM_32B).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint64_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;
  d |= layout << 61;
  return d;
}

// Instruction descriptor: D f32, A/B tf32, majors, N>>3, M>>4.
__host__ __device__ constexpr uint32_t idesc_tf32(bool a_mn, bool b_mn, int m) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         (static_cast<uint32_t>(BN >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

// Descriptor of operand tile `base` (R rows/cols of MN, 32 K) for the kk-th 8-wide K step.
template <bool MN>
__device__ __forceinline__ uint64_t op_desc(uint32_t base, int kk, const EpiParams& ep) {
  // MN-major: 32-col MN chunks BK*128 B apart (LBO), 4-row K atoms 512 B apart (SBO), +8 K rows = +1 KB per K step
  if (MN) return sdesc(base + kk * 1024, ep.mn_lbo, ep.mn_sbo, ep.mn_layout);
  // K-major: one 64 B row of BK = 16 tf32 per M/N row (written by TMA SWIZZLE_64B)
  static_assert(BK == 16, "K-major descriptors assume 64 B rows (SWIZZLE_64B)");
  return sdesc(base + kk * 32, 16, 512, 4);  // SWIZZLE_64B: 64 B K rows, 8-row atoms 512 B apart, +32 B per K step
}

// TMA of one operand tile (R along M/N) for K block starting at k.
template <bool MN, int PAIR>
__device__ __forceinline__ void load_op(const CUtensorMap* map, uint64_t* bar, uint8_t* dst, int r0, int k) {
  if (PAIR == 2) {
    const uint32_t lead = su32(bar) & kPeerMask;
    if (MN) tma_3d_pair(map, lead, dst, 0, k, r0 / 32);
    else tma_2d_pair(map, lead, dst, k, r0);
  } else if (MN) {
    tma_3d(map, bar, dst, 0, k, r0 / 32);  // all R/32 chunks in one box (see make_map)
  } else {
    tma_2d(map, bar, dst, k, r0);
  }
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// K8 on 4 consecutive parameters (same operations as update_kernel<float, false>), w4/v4 already loaded: stores
// w, v and the TF32 split; returns true if a result is non-finite.
__device__ __forceinline__ bool fused_update4(const FusedUpdate& u, int64_t at, const float* g, float4 w4, float4 v4) {
  float w[4] = {w4.x, w4.y, w4.z, w4.w}, v[4] = {v4.x, v4.y, v4.z, v4.w};
  bool bad = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float d = g[i];
    if (u.add_zero) d = __fadd_rn(d, 0.f);
    if (u.post_div != 0.f) d = __fdiv_rn(d, u.post_div);
    if (u.mode == 0) {
      w[i] = __fmaf_rn(-u.lr, d, w[i]);
    } else {
      const float gg = __fmaf_rn(u.weight_decay, w[i], d);
      v[i] = __fmaf_rn(u.momentum, v[i], gg);
      w[i] = __fmaf_rn(-u.lr, v[i], w[i]);
    }
    bad |= !isfinite(w[i]);
  }
  *reinterpret_cast<float4*>(u.w + at) = make_float4(w[0], w[1], w[2], w[3]);
  if (u.mode) *reinterpret_cast<float4*>(u.v + at) = make_float4(v[0], v[1], v[2], v[3]);
  float h[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = tf32_rna(w[i]);
  *reinterpret_cast<float4*>(u.hi + at) = make_float4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<float4*>(u.lo + at) =
      make_float4(tf32_rna(w[0] - h[0]), tf32_rna(w[1] - h[1]), tf32_rna(w[2] - h[2]), tf32_rna(w[3] - h[3]));
  return bad;
}
__device__ __forceinline__ float4 upd_w4(const FusedUpdate& u, int64_t at) {
  return *reinterpret_cast<const float4*>(u.w + at);
}
__device__ __forceinline__ float4 upd_v4(const FusedUpdate& u, int64_t at) {
  return u.mode ? *reinterpret_cast<const float4*>(u.v + at) : make_float4(0.f, 0.f, 0.f, 0.f);
}

// Epilogue on 4 consecutive columns [col, col + 4) of one row (coalesced: the lanes of a warp cover whole 128 B
// rows). aux = b[col..col+3] (forward) or the ReLU mask source act[row][col..col+3] (input gradient), loaded by the
// caller ahead of time (epi_aux) so its latency overlaps the previous chunk.
// EPI is a template parameter throughout: each kernel instantiation carries one epilogue only (a single kernel
// with every epilogue inlined stalled on instruction fetch).
template <int EPI>
__device__ __forceinline__ float4 epi_aux(const EpiParams& ep, int row, int col) {
  if (EPI == kFwd) return __ldg(reinterpret_cast<const float4*>(ep.bias + col));
  if (EPI == kIgrad) return __ldg(reinterpret_cast<const float4*>(ep.mask + static_cast<int64_t>(row) * ep.ldm + col));
  return make_float4(0.f, 0.f, 0.f, 0.f);
}
template <int EPI>
__device__ __forceinline__ void epi_vec4(const EpiParams& ep, int row, int col, float4 v, float4 aux,
                                         const BucketScatter& scat_table) {
  constexpr int epi = EPI;
  const float4 bias4 = aux;
  float o[4] = {v.x, v.y, v.z, v.w};
  if (epi == kFwd) {
    const float b[4] = {bias4.x, bias4.y, bias4.z, bias4.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      o[i] = __fadd_rn(o[i], b[i]);
      if (ep.relu && o[i] < 0.f) o[i] = 0.f;
    }
  } else if (epi == kWgrad || epi == kWgradUpd || epi == kWgradScat) {
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = ep.div_pow2 ? o[i] * ep.div_inv : __fdiv_rn(o[i], ep.div);  // x*2^-k == x/2^k
  } else {
    const float mk[4] = {aux.x, aux.y, aux.z, aux.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (!(mk[i] > 0.f)) o[i] = 0.f;
  }
  const int64_t at = static_cast<int64_t>(row) * ep.ldo + col;
  if (epi == kWgradUpd) {
    if (fused_update4(ep.upd, at, o, upd_w4(ep.upd, at), upd_v4(ep.upd, at))) atomicOr(ep.upd.bad, 1u);
    return;
  }
  float* outp = epi == kWgradScat ? scatter_at(scat_table, ep.scat.e0 + at) : ep.out + at;
  *reinterpret_cast<float4*>(outp) = make_float4(o[0], o[1], o[2], o[3]);
  if (ep.out_hi) {
    const float h0 = tf32_rna(o[0]), h1 = tf32_rna(o[1]), h2 = tf32_rna(o[2]), h3 = tf32_rna(o[3]);
    *reinterpret_cast<float4*>(ep.out_hi + at) = make_float4(h0, h1, h2, h3);
    *reinterpret_cast<float4*>(ep.out_lo + at) =
        make_float4(tf32_rna(o[0] - h0), tf32_rna(o[1] - h1), tf32_rna(o[2] - h2), tf32_rna(o[3] - h3));
  }
}

// Persistent: one CTA (PAIR = 1) or CTA pair (PAIR = 2, a 2-CTA cluster) per tile slot; slot c takes tiles c,
// c + slots, ... (m fastest, so the slots working at the same time share B tiles in L2). Two TMEM accumulators
// (2 x 256 columns) let the epilogue of tile i overlap the MMAs of tile i+1; the smem stage ring runs continuously
// across tiles. In pair mode the leader CTA (rank 0) issues the cta_group::2 MMAs and owns the full/tmem-empty
// barriers; both CTAs load their halves, and the MMA commits multicast to both CTAs' empty/tmem-full barriers.
template <bool A_MN, bool B_MN, int PAIR, int EPI, bool WS>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap ta_hi, const __grid_constant__ CUtensorMap ta_lo,
                       const __grid_constant__ CUtensorMap tb_hi, const __grid_constant__ CUtensorMap tb_lo,
                       int k_per_split, int splits, const __grid_constant__ EpiParams ep) {
  using C = Cfg<PAIR, EPI, WS>;
  // tile order: m fastest (concurrent slots share B tiles in L2), except for the fused update, whose epilogue
  // streams w / v / w_hi / w_lo rows: n fastest keeps concurrent tiles on the same rows (DRAM page locality)
  constexpr bool kNFast = EPI == kWgradUpd;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ alignas(8) uint64_t full_bar[STAGES];
  __shared__ alignas(8) uint64_t empty_bar[STAGES];
  __shared__ alignas(8) uint64_t tfull_bar[2];
  __shared__ alignas(8) uint64_t tempty_bar[2];
  __shared__ alignas(8) uint64_t xform_bar[WS ? STAGES : 1];  // WS: stage s split into hi / lo (both CTAs)
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = PAIR == 2 ? cluster_rank() : 0u;
  const int slot = blockIdx.x / PAIR, nslots = gridDim.x / PAIR;
  const int mt = ep.M / (BM * PAIR), nt = ep.N / BN;
  const int tiles = mt * nt * splits;
  const int nkb = k_per_split / BK;
  // K chunks: the tensor pipe's fp32 accumulation does not round to nearest, so its error grows with the number of
  // MMAs folded into one accumulator (linearly in K: 5.7e-5 norm-wise at K = 8192 against 1.1e-6 for an fp32 FMA
  // GEMM). A tile's K runs as chunks of kcb k-blocks: chunk 0 accumulates into the tile's accumulator S, each later
  // chunk into the other one (X), which the epilogue warps fold into S (S + X, round-to-nearest fp32, chunk order)
  // while the next chunk's MMAs wait only for that fold. With one chunk this is the plain double-buffered tile loop.
  const int kcb = ep.kcb > 0 && ep.kcb < nkb ? ep.kcb : nkb;
  const int nch = (nkb + kcb - 1) / kcb;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 4 * PAIR);  // one arrival per epilogue warp of each CTA
    }
    if (WS)
      for (int s = 0; s < STAGES; ++s) mbar_init(&xform_bar[s], 4 * PAIR);  // one per transform warp per CTA
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (ep.prefetch) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta_hi)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta_lo)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb_hi)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb_lo)) : "memory");
    }
  }
  if (warp == 1) {
    if (PAIR == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_slot)),
                   "r"(2 * TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_slot)),
                   "r"(2 * TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if (PAIR == 2) cluster_sync_all();  // the peer's barriers are initialised before any remote arrive / TMA
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;  // k-blocks issued by this CTA across all its tiles (stage ring position)
      for (int t = slot; t < tiles; t += nslots) {
        const int z = t / (mt * nt), r = t % (mt * nt);
        const int tm = kNFast ? r / nt : r % mt, tn = kNFast ? r % nt : r / mt;
        const int m0 = tm * BM * PAIR + static_cast<int>(rank) * BM;
        const int n0 = tn * BN + static_cast<int>(rank) * C::B_ROWS, k0 = z * k_per_split;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const uint32_t s = it % STAGES, ph = (it / STAGES) & 1u;
          if (it >= STAGES) mbar_wait(&empty_bar[s], ph ^ 1u);
          uint8_t* st = smem + s * C::STAGE_BYTES;
          if (ep.probe & 4u) {
            if (rank == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full_bar[s])) : "memory");
            continue;
          }
          const int k = k0 + kb * BK;
          if (WS) {
            // every CTA completes its own barrier (its transform warps wait on it); the raw weights land behind
            // the hi / lo slots the transform fills
            mbar_expect_tx(&full_bar[s], 2 * A_BYTES + C::RAW_BYTES);
            load_op<A_MN, 1>(&ta_hi, &full_bar[s], st, m0, k);
            load_op<A_MN, 1>(&ta_lo, &full_bar[s], st + A_BYTES, m0, k);
            load_op<B_MN, 1>(&tb_hi, &full_bar[s], st + 2 * A_BYTES + 2 * C::B_BYTES, n0, k);
            continue;
          }
          if (rank == 0) mbar_expect_tx(&full_bar[s], C::STAGE_BYTES * PAIR);  // the leader counts both halves
          load_op<A_MN, PAIR>(&ta_hi, &full_bar[s], st, m0, k);
          load_op<A_MN, PAIR>(&ta_lo, &full_bar[s], st + A_BYTES, m0, k);
          load_op<B_MN, PAIR>(&tb_hi, &full_bar[s], st + 2 * A_BYTES, n0, k);
          load_op<B_MN, PAIR>(&tb_lo, &full_bar[s], st + 2 * A_BYTES + C::B_BYTES, n0, k);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = idesc_tf32(A_MN, B_MN, BM * PAIR);
      uint32_t it = 0, local = 0, sess0 = 0, sess1 = 0;  // MMA sessions issued into accumulator 0 / 1
      for (int t = slot; t < tiles; t += nslots, ++local) {
        const uint32_t P = local & 1u;
        for (int ch = 0; ch < nch; ++ch) {
          // chunk 0 -> accumulator P (the tile's running sum S), chunks >= 1 -> the other one (X, folded into S)
          const uint32_t b = ch == 0 ? P : P ^ 1u;
          const uint32_t sess = b ? sess1 : sess0;
          if (sess > 0) mbar_wait(&tempty_bar[b], (sess - 1u) & 1u);  // its previous contents consumed
          tc_fence_after();
          const uint32_t acc_tmem = tmem + b * TMEM_COLS;
          const int kb0 = ch * kcb, kb1 = kb0 + kcb < nkb ? kb0 + kcb : nkb;
          for (int kb = kb0; kb < kb1; ++kb, ++it) {
            const uint32_t s = it % STAGES, ph = (it / STAGES) & 1u;
            mbar_wait(WS ? &xform_bar[s] : &full_bar[s], ph);
            tc_fence_after();
            const uint32_t st = su32(smem + s * C::STAGE_BYTES);
            const uint32_t a_hi = st, a_lo = st + A_BYTES, b_hi = st + 2 * A_BYTES, b_lo = b_hi + C::B_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              if (ep.probe & 2u) break;
              const uint32_t accum = (kb > kb0 || kk > 0) ? 1u : 0u;
              const uint64_t dah = op_desc<A_MN>(a_hi, kk, ep), dal = op_desc<A_MN>(a_lo, kk, ep);
              const uint64_t dbh = op_desc<B_MN>(b_hi, kk, ep), dbl = op_desc<B_MN>(b_lo, kk, ep);
              if (PAIR == 2) {
                mma_tf32_pair(acc_tmem, dah, dbl, idesc, accum);
                mma_tf32_pair(acc_tmem, dal, dbh, idesc, 1u);
                mma_tf32_pair(acc_tmem, dah, dbh, idesc, 1u);
              } else {
                mma_tf32(acc_tmem, dah, dbl, idesc, accum);
                mma_tf32(acc_tmem, dal, dbh, idesc, 1u);
                mma_tf32(acc_tmem, dah, dbh, idesc, 1u);
              }
            }
            if (PAIR == 2) mma_commit_pair(&empty_bar[s]);  // stage s is free (in both CTAs) once these MMAs read it
            else mma_commit(&empty_bar[s]);
          }
          if (PAIR == 2) mma_commit_pair(&tfull_bar[b]);  // accumulator b holds the finished chunk
          else mma_commit(&tfull_bar[b]);
          if (b) ++sess1;
          else ++sess0;
        }
      }
    }
  } else {
    // epilogue warps 2..5 -> TMEM lane quadrant warp % 4 (this CTA's 128 rows of the tile)
    const int q = warp & 3;
    uint32_t local = 0, es0 = 0, es1 = 0;  // accumulator 0 / 1 sessions waited for
    uint32_t xit = 0, kb_end = 0;              // WS: k-blocks transformed / k-blocks up to the current chunk's end
    // WS: split raw weight k-blocks into the hi / lo operand slots as they land, up to flat k-block `target`:
    // elementwise, so the TMA swizzle (a 16 B-chunk permutation shared by all three tiles) needs no index math
    auto transform_to = [&](uint32_t target) {
      const int tid = threadIdx.x - 64;
      for (; xit < target; ++xit) {
        const uint32_t s = xit % STAGES, ph = (xit / STAGES) & 1u;
        mbar_wait(&full_bar[s], ph);
        uint8_t* st = smem + s * C::STAGE_BYTES;
        const uint32_t raw = su32(st + 2 * A_BYTES + 2 * C::B_BYTES);
        const uint32_t hi = su32(st + 2 * A_BYTES), lo = su32(st + 2 * A_BYTES + C::B_BYTES);
        constexpr int N4 = C::B_BYTES / 16;
        float4 v[N4 / 128];
#pragma unroll
        for (int j = 0; j < N4 / 128; ++j) v[j] = lds128(raw + 16u * (tid + 128 * j));  // all loads first
#pragma unroll
        for (int j = 0; j < N4 / 128; ++j) {
          const uint32_t o = 16u * (tid + 128 * j);
          const float4 h = make_float4(tf32_rna(v[j].x), tf32_rna(v[j].y), tf32_rna(v[j].z), tf32_rna(v[j].w));
          sts128(hi + o, h);
          sts128(lo + o, make_float4(tf32_rna(v[j].x - h.x), tf32_rna(v[j].y - h.y), tf32_rna(v[j].z - h.z),
                                     tf32_rna(v[j].w - h.w)));
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core reads
        __syncwarp();
        if (lane == 0) {
          const uint32_t bar = PAIR == 2 ? (su32(&xform_bar[s]) & kPeerMask) : su32(&xform_bar[s]);
          asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar) : "memory");
        }
      }
    };
    auto release = [&](uint32_t b) {  // this warp is done with accumulator b (leader's barrier)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        const uint32_t bar = PAIR == 2 ? (su32(&tempty_bar[b]) & kPeerMask) : su32(&tempty_bar[b]);
        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar) : "memory");
      }
    };
    // wait for accumulator b; WS: meanwhile split the next k-blocks (up to `ahead`) as soon as each one lands, so
    // the MMA warp finds transformed stages the moment it may continue (warp-uniform polls)
    auto wait_full = [&](uint32_t b, uint32_t ahead) {
      uint32_t& es = b ? es1 : es0;
      if (WS) {
        while (!__shfl_sync(0xffffffffu, mbar_test(&tfull_bar[b], es & 1u), 0)) {
          if (xit < ahead && __shfl_sync(0xffffffffu, mbar_test(&full_bar[xit % STAGES], (xit / STAGES) & 1u), 0))
            transform_to(xit + 1);
        }
      } else {
        mbar_wait(&tfull_bar[b], es & 1u);
      }
      ++es;
      tc_fence_after();
    };
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    for (int t = slot; t < tiles; t += nslots, ++local) {
      const uint32_t P = local & 1u, Q = P ^ 1u;
      uint32_t ahead = 0;
      for (int ch = 0; ch < nch; ++ch) {
        const int len = kcb < nkb - ch * kcb ? kcb : nkb - ch * kcb;
        kb_end += static_cast<uint32_t>(len);
        const bool last = ch == nch - 1;
        // WS: this chunk's k-blocks now; up to a ring's worth of the next chunk's (or next tile's) while its
        // accumulator drains (their slots free up as this chunk's MMAs retire)
        const int nl = !last ? (kcb < nkb - (ch + 1) * kcb ? kcb : nkb - (ch + 1) * kcb)
                             : (t + nslots < tiles ? (kcb < nkb ? kcb : nkb) : 0);
        ahead = kb_end + static_cast<uint32_t>(nl < STAGES ? nl : STAGES);
        if (WS) transform_to(kb_end);
        if (ch == 0) continue;
        // fold chunk ch (accumulator Q) into the running sum S (accumulator P): S = S + X, in chunk order; the
        // last chunk folds too, so Q is free for the next tile's first chunk while this tile's epilogue runs
        if (ch == 1) wait_full(P, 0u);
        wait_full(Q, ahead);
#pragma unroll 1
        for (int c = 0; c < BN; c += 64) {  // 64 columns per TMEM round trip
          uint32_t x0[32], s0[32], x1[32], s1[32];
          const uint32_t xa = tmem + Q * TMEM_COLS + lane_off + static_cast<uint32_t>(c);
          const uint32_t sa = tmem + P * TMEM_COLS + lane_off + static_cast<uint32_t>(c);
          tmem_ld32(xa, x0);
          tmem_ld32(sa, s0);
          tmem_ld32(xa + 32, x1);
          tmem_ld32(sa + 32, s1);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            s0[j] = __float_as_uint(__fadd_rn(__uint_as_float(s0[j]), __uint_as_float(x0[j])));
            s1[j] = __float_as_uint(__fadd_rn(__uint_as_float(s1[j]), __uint_as_float(x1[j])));
          }
          tmem_st32(sa, s0);
          tmem_st32(sa + 32, s1);
        }
        tmem_wait_st();
        release(Q);
      }
      const int z = t / (mt * nt), r = t % (mt * nt);
      const int tm = kNFast ? r / nt : r % mt, tn = kNFast ? r % nt : r / mt;
      const int m0 = tm * BM * PAIR + static_cast<int>(rank) * BM, n0 = tn * BN;
      // scalar fields in registers; the scatter table stays in (grid-constant) param space, where it is indexed
      const EpiParams e = ep;
      const bool raw = splits > 1;  // split-K: raw partial planes, the epilogue runs in splitk_reduce
      float* partial = raw ? ep.partial + static_cast<int64_t>(z) * ep.M * ep.N : nullptr;
      // TMEM gives lane = row; the chunk goes through a swizzled 4 KB smem tile (16 B chunk j of row r at
      // j ^ (r & 7): conflict-free both ways) so each global access of the warp covers 4 whole 128 B rows.
      float4* stg = reinterpret_cast<float4*>(smem + C::RING + q * EPI_STAGE_BYTES);
      const int ch = lane & 7;
      float4 aux[8];  // bias / mask operands of the current chunk, prefetched one chunk ahead
#pragma unroll
      for (int i = 0; i < 8; ++i)
        aux[i] = raw ? make_float4(0.f, 0.f, 0.f, 0.f) : epi_aux<EPI>(e, m0 + q * 32 + 4 * i + (lane >> 3), n0 + ch * 4);
      // fused update: w / v of the lane's 8 rows x 4 columns stream into a per-warp smem double buffer with
      // cp.async one chunk ahead (chunk 0 before the accumulator is even ready), so the epilogue keeps a chunk of
      // loads in flight instead of one round trip per chunk
      const bool fu = EPI == kWgradUpd && !raw;
      float4* pref = reinterpret_cast<float4*>(smem + C::RING + 4 * EPI_STAGE_BYTES + q * UPD_PREF_BYTES);
      auto prefetch_wv = [&](int cc) {
        float4* buf = pref + ((cc / 32) & 1) * 512;  // [w: 8 x 32 | v: 8 x 32] float4 per buffer
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int64_t at = static_cast<int64_t>(m0 + q * 32 + 4 * i + (lane >> 3)) * e.ldo + n0 + cc + ch * 4;
          cp_async16(buf + i * 32 + lane, e.upd.w + at);
          if (e.upd.mode) cp_async16(buf + 256 + i * 32 + lane, e.upd.v + at);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      if (fu) prefetch_wv(0);
      if (nch == 1) wait_full(P, ahead);
      else tc_fence_after();  // S was last written by this warp's own fold (tcgen05.st, waited)
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        float4 nxt[8];
        if (fu && c + 32 < BN) prefetch_wv(c + 32);
        uint32_t rr[32];
        tmem_ld32(tmem + P * TMEM_COLS + lane_off + static_cast<uint32_t>(c), rr);
        const int cn = c + 32 < BN ? c + 32 : c;
        if (!fu && !raw) {
#pragma unroll
          for (int i = 0; i < 8; ++i) nxt[i] = epi_aux<EPI>(e, m0 + q * 32 + 4 * i + (lane >> 3), n0 + cn + ch * 4);
        }
        tmem_wait_ld();
        if (ep.probe & 1u) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          stg[lane * 8 + (j ^ (lane & 7))] = make_float4(__uint_as_float(rr[4 * j]), __uint_as_float(rr[4 * j + 1]),
                                                         __uint_as_float(rr[4 * j + 2]), __uint_as_float(rr[4 * j + 3]));
        __syncwarp();
        const int col = n0 + c + ch * 4;
        if (fu) {
          // this chunk's w / v group has landed (the next chunk's may still be in flight)
          if (c + 32 < BN) asm volatile("cp.async.wait_group 1;" ::: "memory");
          else asm volatile("cp.async.wait_group 0;" ::: "memory");
          const float4* buf = pref + ((c / 32) & 1) * 512;
          bool bad = false;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rw = 4 * i + (lane >> 3);
            const float4 acc = stg[rw * 8 + (ch ^ (rw & 7))];
            float g[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) g[u] = e.div_pow2 ? g[u] * e.div_inv : __fdiv_rn(g[u], e.div);
            const float4 v4 = e.upd.mode ? buf[256 + i * 32 + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
            bad |= fused_update4(e.upd, static_cast<int64_t>(m0 + q * 32 + rw) * e.ldo + col, g, buf[i * 32 + lane],
                                 v4);
          }
          if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(e.upd.bad, 1u);
        } else if (raw) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rw = 4 * i + (lane >> 3);
            *reinterpret_cast<float4*>(partial + static_cast<int64_t>(m0 + q * 32 + rw) * e.N + col) =
                stg[rw * 8 + (ch ^ (rw & 7))];
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rw = 4 * i + (lane >> 3);
            epi_vec4<EPI>(e, m0 + q * 32 + rw, col, stg[rw * 8 + (ch ^ (rw & 7))], aux[i], ep.scat);
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) aux[i] = nxt[i];
        }
        __syncwarp();
      }
      release(P);
    }
  }
  tc_fence_before();
  if (PAIR == 2) cluster_sync_all();  // both CTAs are done with the pair's TMEM and barriers
  else __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    if (PAIR == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * TMEM_COLS) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * TMEM_COLS) : "memory");
  }
}

// Split-K: sum the partial tiles in ascending split order, then the epilogue (deterministic, no atomics).
template <int EPI>
__global__ void splitk_reduce_kernel(int splits, const __grid_constant__ EpiParams ep) {
  const int64_t total = static_cast<int64_t>(ep.M) * ep.N / 4;
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < total;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t e0 = g * 4;
    const int row = static_cast<int>(e0 / ep.N), col = static_cast<int>(e0 % ep.N);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < splits; ++s) {
      const float4 q = *reinterpret_cast<const float4*>(ep.partial + static_cast<int64_t>(s) * ep.M * ep.N + e0);
      v.x += q.x;
      v.y += q.y;
      v.z += q.z;
      v.w += q.w;
    }
    epi_vec4<EPI>(ep, row, col, v, epi_aux<EPI>(ep, row, col), ep.scat);
  }
}

__global__ void split_tf32_kernel(const float* __restrict__ x, int64_t n, float* __restrict__ hi,
                                  float* __restrict__ lo) {
  const int64_t n4 = n / 4;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 v = reinterpret_cast<const float4*>(x)[i];
    float4 h = make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
    reinterpret_cast<float4*>(hi)[i] = h;
    reinterpret_cast<float4*>(lo)[i] =
        make_float4(tf32_rna(v.x - h.x), tf32_rna(v.y - h.y), tf32_rna(v.z - h.z), tf32_rna(v.w - h.w));
  }
  for (int64_t i = n4 * 4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float h = tf32_rna(x[i]);
    hi[i] = h;
    lo[i] = tf32_rna(x[i] - h);
  }
}

// Mean of the per-sample losses for the fp32 path: one warp, lanes own a fixed strided subset, fixed shuffle tree
// (deterministic; the fp64 parity path keeps the reference's sequential fold, mlp.cpp:262-271).
__global__ void mean_loss_warp_kernel(const float* __restrict__ sample_loss, int b, float* __restrict__ out) {
  float acc = 0.f;
  for (int s = threadIdx.x; s < b; s += 32) acc += sample_loss[s];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (threadIdx.x == 0) *out = __fdiv_rn(acc, static_cast<float>(b));
}

// Softmax-CE head for the tensor-core path: one warp per sample, lanes striding the classes (coalesced), max and
// sum by warp shuffles; writes delta = softmax - onehot and its hi/lo split for the backward GEMMs.
__global__ void softmax_xent_split_kernel(const float* __restrict__ logits, const int32_t* __restrict__ labels, int b,
                                          int c, float* __restrict__ delta, float* __restrict__ dhi,
                                          float* __restrict__ dlo, float* __restrict__ sample_loss) {
  const int s = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (s >= b) return;
  const float* z = logits + static_cast<int64_t>(s) * c;
  const int lab = labels[s];
  if (c <= 32 * 32) {  // the sample's logits stay in registers (one global read instead of three)
    float zr[32];
    float zmax = -INFINITY;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int k = lane + 32 * q;
      zr[q] = k < c ? z[k] : -INFINITY;
      zmax = fmaxf(zmax, zr[q]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) zmax = fmaxf(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
    float sum = 0.f;
#pragma unroll
    for (int q = 0; q < 32; ++q)
      if (lane + 32 * q < c) sum += expf(zr[q] - zmax);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float lse = zmax + logf(sum);
    float zl = 0.f;  // the label's logit, selected without dynamic register indexing
#pragma unroll
    for (int q = 0; q < 32; ++q)
      if (q == lab / 32) zl = zr[q];
    if (lane == lab % 32) sample_loss[s] = lse - zl;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int k = lane + 32 * q;
      if (k >= c) break;
      const float p = expf(zr[q] - lse);
      const float d = (k == lab) ? p - 1.f : p;
      const int64_t at = static_cast<int64_t>(s) * c + k;
      delta[at] = d;
      const float h = tf32_rna(d);
      dhi[at] = h;
      dlo[at] = tf32_rna(d - h);
    }
    return;
  }
  float zmax = -INFINITY;
  for (int k = lane; k < c; k += 32) zmax = fmaxf(zmax, z[k]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) zmax = fmaxf(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
  float sum = 0.f;
  for (int k = lane; k < c; k += 32) sum += expf(z[k] - zmax);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float lse = zmax + logf(sum);
  if (lane == 0) sample_loss[s] = lse - z[lab];
  for (int k = lane; k < c; k += 32) {
    const float p = expf(z[k] - lse);
    const float d = (k == lab) ? p - 1.f : p;
    const int64_t at = static_cast<int64_t>(s) * c + k;
    delta[at] = d;
    const float h = tf32_rna(d);
    dhi[at] = h;
    dlo[at] = tf32_rna(d - h);
  }
}

// Bias gradient for the fp32 path: db[j] = (sum_s delta[s, j]) / B. 32 columns x 8 row-partitions per block,
// partials combined in a fixed order (deterministic, no atomics).
__global__ void bias_grad_f32_kernel(const float* __restrict__ delta, int b, int n, float* __restrict__ db,
                                     const __grid_constant__ BucketScatter scat, const __grid_constant__ FusedUpdate upd) {
  // 32 columns x 32 row partitions per block (each thread: rows y, y+32, ..., 4 loads in flight per trip), the
  // partials combined in a fixed order: deterministic, no atomics
  __shared__ float part[32][33];
  const int j = blockIdx.x * 32 + threadIdx.x;
  float acc = 0.f;
  if (j < n) {
    int r = threadIdx.y;
    for (; r + 96 < b; r += 128) {
      const float a0 = delta[static_cast<int64_t>(r) * n + j], a1 = delta[static_cast<int64_t>(r + 32) * n + j];
      const float a2 = delta[static_cast<int64_t>(r + 64) * n + j], a3 = delta[static_cast<int64_t>(r + 96) * n + j];
      acc += a0;
      acc += a1;
      acc += a2;
      acc += a3;
    }
    for (; r < b; r += 32) acc += delta[static_cast<int64_t>(r) * n + j];
  }
  part[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && j < n) {
    float t = part[0][threadIdx.x];
#pragma unroll
    for (int q = 1; q < 32; ++q) t += part[q][threadIdx.x];
    t = __fdiv_rn(t, static_cast<float>(b));
    if (upd.w) {
      float d = t;
      if (upd.add_zero) d = __fadd_rn(d, 0.f);
      if (upd.post_div != 0.f) d = __fdiv_rn(d, upd.post_div);
      float w = upd.w[j], v = upd.mode ? upd.v[j] : 0.f;
      if (upd.mode == 0) {
        w = __fmaf_rn(-upd.lr, d, w);
      } else {
        v = __fmaf_rn(upd.momentum, v, __fmaf_rn(upd.weight_decay, w, d));
        w = __fmaf_rn(-upd.lr, v, w);
      }
      upd.w[j] = w;
      if (upd.mode) upd.v[j] = v;
      const float h = tf32_rna(w);
      upd.hi[j] = h;
      upd.lo[j] = tf32_rna(w - h);
      if (!isfinite(w)) atomicOr(upd.bad, 1u);
    } else if (scat.n) {
      *scatter_at(scat, scat.e0 + j) = t;
    } else {
      db[j] = t;
    }
  }
  if (upd.loss_out && blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0) {  // the folded loss slot
    float d = *upd.loss_in;
    if (upd.add_zero) d = __fadd_rn(d, 0.f);
    if (upd.post_div != 0.f) d = __fdiv_rn(d, upd.post_div);
    *upd.loss_out = d;
  }
}

// ------------------------------------------------------------------------------------------ host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    LSGD_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    check<Error>(p != nullptr && q == cudaDriverEntryPointSuccess, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

// MN-major operand geometry: TMA swizzle SWIZZLE_128B_ATOM_32B + UMMA layout SWIZZLE_128B_BASE32B, LBO = MN chunk
// stride, SBO = 4-row K atom stride.
struct MnGeometry {
  uint32_t lbo = MN_CHUNK_BYTES, sbo = 512, layout = 1, tma_swizzle = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
};
const MnGeometry& mn_geometry() {
  static const MnGeometry g;
  return g;
}

// Operand view: `rows` along M or N, `k` along K, stored K-major ([rows][ld]) or MN-major ([k][ld]).
struct OpView {
  const float* ptr;
  int64_t rows, k, ld;
  bool mn;
};

// K-major operand: 2D map {K, rows}, box {BK, tile_rows}, SWIZZLE_64B.
// MN-major operand: 3D view {32 (MN within a chunk), K, rows/32 (chunks)} with strides {ld*4 B, 128 B}, box
// {32, BK, tile_rows/32}: one TMA brings the whole tile, chunk c landing at c * BK*128 B (the LBO of op_desc).
CUtensorMap make_map(const OpView& v, int tile_rows) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  cuuint64_t dims[3], strides[2];
  cuuint32_t box[3], estr[3] = {1, 1, 1};
  cuuint32_t rank = 2;
  if (v.mn) {
    rank = 3;
    dims[0] = 32;
    dims[1] = static_cast<cuuint64_t>(v.k);
    dims[2] = static_cast<cuuint64_t>(v.rows / 32);
    strides[0] = static_cast<cuuint64_t>(v.ld) * 4;
    strides[1] = 128;
    box[0] = 32;
    box[1] = BK;
    box[2] = static_cast<cuuint32_t>(tile_rows / 32);
  } else {
    dims[0] = static_cast<cuuint64_t>(v.k);
    dims[1] = static_cast<cuuint64_t>(v.rows);
    strides[0] = static_cast<cuuint64_t>(v.ld) * 4;
    box[0] = BK;
    box[1] = static_cast<cuuint32_t>(tile_rows);
  }
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<float*>(v.ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           v.mn ? static_cast<CUtensorMapSwizzle>(mn_geometry().tma_swizzle) : CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  check<Error>(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (", static_cast<int>(r), ")");
  return m;
}

struct GemmPlan {
  CUtensorMap a_hi, a_lo, b_hi, b_lo;  // ws: b_hi maps the raw fp32 weights (b_lo unused)
  bool a_mn = false, b_mn = false, ws = false;
  int M = 0, N = 0, K = 0, splits = 1, epi = 0, pair = 1;
  EpiParams ep{};
};

// SMs the persistent GEMM may occupy (LSGD_TC_MAX_SMS caps it: the rest stay free for the update / exchange
// kernels, which are kept off GEMM SMs by their shared-memory request; tuning knob)
int sm_count() {
  static int sms = [] {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, 0);
    if (v <= 0) v = 148;
    if (const char* e = std::getenv("LSGD_TC_MAX_SMS")) {
      const int cap = std::atoi(e);
        if (cap >= 2 && cap < v) v = cap;
    } else if (v == 148) {
      v = 128;  // 64 CTA pairs: every cfg3 GEMM has a multiple of 64 pair tiles, the other 20 SMs run side work
    }
    return v;
  }();
  return sms;
}

template <bool A_MN, bool B_MN, int PAIR, int EPI, bool WS = false>
void launch_variant(const GemmPlan& p, cudaStream_t st) {
  // the dynamic-smem opt-in is per device: remember which devices this instantiation was configured on
  static std::mutex mu;
  static uint64_t configured = 0;
  int dev = 0;
  LSGD_CUDA(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!(configured >> dev & 1ull)) {
      LSGD_CUDA(cudaFuncSetAttribute(gemm_tf32x3_kernel<A_MN, B_MN, PAIR, EPI, WS>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<PAIR, EPI, WS>::SMEM));
      configured |= 1ull << dev;
    }
  }
  const int tiles = (p.N / BN) * (p.M / (BM * PAIR)) * p.splits;
  const int slots = sm_count() / PAIR;
  const int grid = (tiles < slots ? tiles : slots) * PAIR;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = Cfg<PAIR, EPI, WS>::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PAIR;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  LSGD_CUDA(cudaLaunchKernelEx(&cfg, gemm_tf32x3_kernel<A_MN, B_MN, PAIR, EPI, WS>, p.a_hi, p.a_lo, p.b_hi, p.b_lo,
                               p.K / p.splits, p.splits, p.ep));
}

template <int PAIR, int EPI>
void launch_pair_epi(const GemmPlan& p, cudaStream_t st) {
  if (!p.a_mn && !p.b_mn) launch_variant<false, false, PAIR, EPI>(p, st);
  else if (!p.a_mn && p.b_mn) launch_variant<false, true, PAIR, EPI>(p, st);
  else if (p.a_mn && p.b_mn) launch_variant<true, true, PAIR, EPI>(p, st);
  else launch_variant<true, false, PAIR, EPI>(p, st);
}
template <int PAIR>
void launch_pair(const GemmPlan& p, cudaStream_t st) {
  if (p.ws) {  // the two weight-reading GEMMs: forward (W K-major) and input gradient (W MN-major)
    check<Error>(!p.a_mn && ((p.epi == kFwd && !p.b_mn) || (p.epi == kIgrad && p.b_mn)), "gemm: unsupported WS form");
    if (p.epi == kFwd) launch_variant<false, false, PAIR, kFwd, true>(p, st);
    else launch_variant<false, true, PAIR, kIgrad, true>(p, st);
    return;
  }
  if (p.epi == kFwd) launch_pair_epi<PAIR, kFwd>(p, st);
  else if (p.epi == kWgrad && p.ep.fuse_upd) launch_pair_epi<PAIR, kWgradUpd>(p, st);
  else if (p.epi == kWgrad && p.ep.scat.n) launch_pair_epi<PAIR, kWgradScat>(p, st);
  else if (p.epi == kWgrad) launch_pair_epi<PAIR, kWgrad>(p, st);
  else launch_pair_epi<PAIR, kIgrad>(p, st);
}

void run_plan(const GemmPlan& p, cudaStream_t st, LaunchCounter& lc) {
  if (p.pair == 2) launch_pair<2>(p, st);
  else launch_pair<1>(p, st);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
  if (p.splits > 1) {
    int64_t work = static_cast<int64_t>(p.M) * p.N / 4;
    int grid = static_cast<int>(std::min<int64_t>((work + 255) / 256, 148 * 8));
    if (p.epi == kFwd) splitk_reduce_kernel<kFwd><<<grid, 256, 0, st>>>(p.splits, p.ep);
    else if (p.epi == kWgrad && p.ep.fuse_upd) splitk_reduce_kernel<kWgradUpd><<<grid, 256, 0, st>>>(p.splits, p.ep);
    else if (p.epi == kWgrad && p.ep.scat.n) splitk_reduce_kernel<kWgradScat><<<grid, 256, 0, st>>>(p.splits, p.ep);
    else if (p.epi == kWgrad) splitk_reduce_kernel<kWgrad><<<grid, 256, 0, st>>>(p.splits, p.ep);
    else splitk_reduce_kernel<kIgrad><<<grid, 256, 0, st>>>(p.splits, p.ep);
    ++lc.n;
    LSGD_CUDA(cudaGetLastError());
  }
}

// Split K (ordered partial reduction) only when the tiles alone leave most SMs idle.
int choose_splits(int M, int N, int K, int pair) {
  const int tiles = (M / (BM * pair)) * (N / BN);
  const int slots = 160 / pair;
  int s = 1;
  while (tiles * s * 2 <= slots && K % (BK * s * 2) == 0 && K / (s * 2) >= 4 * BK) s *= 2;
  return s;
}

GemmPlan make_plan(const OpView& a_hi, const float* a_lo, const OpView& b_hi, const float* b_lo, int epi,
                   const EpiParams& ep, float* partial, size_t partial_elems, const float* b_raw = nullptr) {
  GemmPlan p;
  p.a_mn = a_hi.mn;
  p.b_mn = b_hi.mn;
  p.M = static_cast<int>(a_hi.rows);
  p.N = static_cast<int>(b_hi.rows);
  p.K = static_cast<int>(a_hi.k);
  check<Error>(a_hi.k == b_hi.k, "gemm: K mismatch");
  check<Error>(p.M % BM == 0 && p.N % BN == 0 && p.K % BK == 0, "gemm: shape ", p.M, "x", p.N, "x", p.K,
               " is not a multiple of the 128x256x16 tile");
  // CTA pairs whenever the M extent allows 256-row tiles (LSGD_TC_PAIR=0 forces single CTAs: tuning only)
  static const bool no_pair = std::getenv("LSGD_TC_PAIR") && std::atoi(std::getenv("LSGD_TC_PAIR")) == 0;
  p.pair = (!no_pair && p.M % (2 * BM) == 0) ? 2 : 1;
  p.a_hi = make_map(a_hi, BM);
  OpView al = a_hi;
  al.ptr = a_lo;
  p.a_lo = make_map(al, BM);
  p.b_hi = make_map(b_hi, BN / p.pair);
  OpView bl = b_hi;
  bl.ptr = b_lo;
  p.b_lo = make_map(bl, BN / p.pair);
  if (b_raw) {  // split the weights in shared memory: B is read once, as fp32
    OpView br = b_hi;
    br.ptr = b_raw;
    p.b_hi = make_map(br, BN / p.pair);
    p.b_lo = p.b_hi;
    p.ws = true;
  }
  p.epi = epi;
  p.ep = ep;
  const MnGeometry& g = mn_geometry();
  p.ep.mn_lbo = g.lbo;
  p.ep.mn_sbo = g.sbo;
  p.ep.mn_layout = g.layout;
  p.ep.prefetch = 1u;
  static const uint32_t probe = std::getenv("LSGD_TC_PROBE") ? std::atoi(std::getenv("LSGD_TC_PROBE")) : 0;
  p.ep.probe = probe;
  // accumulation chunk (K elements; LSGD_TC_KCHUNK, 0 = the whole K in one accumulator)
  static const int kchunk = std::getenv("LSGD_TC_KCHUNK") ? std::atoi(std::getenv("LSGD_TC_KCHUNK")) : 512;
  p.ep.kcb = kchunk > 0 ? (kchunk + BK - 1) / BK : 0;
  int ex = 0;
  p.ep.div_pow2 = (ep.div > 0.f && std::frexp(ep.div, &ex) == 0.5f) ? 1 : 0;
  p.ep.div_inv = p.ep.div_pow2 ? 1.0f / ep.div : 0.f;
  p.ep.M = p.M;
  p.ep.N = p.N;
  p.splits = std::getenv("LSGD_TC_NOSPLIT") ? 1 : choose_splits(p.M, p.N, p.K, p.pair);
  if (static_cast<size_t>(p.splits) * p.M * p.N > partial_elems) p.splits = 1;
  p.ep.partial = partial;
  return p;
}

}  // namespace

// Per-layer plans of one worker's step (built once; the buffers they point at never move).
struct TcLayer {
  GemmPlan fwd, wgrad, igrad;
  bool has_igrad = false;
  // weight-gradient plans of row blocks [row0, row0 + rows) of dW_k (the engine's gradient buckets), built lazily
  std::map<std::pair<int, int>, GemmPlan> wgrad_rows;
  OpView dw_a, dw_b;
  const float *dw_a_lo = nullptr, *dw_b_lo = nullptr;
  EpiParams dw_ep{};
};

bool tc_shapes_supported(const std::vector<int32_t>& layers, int batch) {
  if (batch % BM != 0 || batch < BM) return false;
  for (int32_t s : layers)
    if (s % BN != 0) return false;
  return layers.size() >= 2;
}

bool tc_weight_split_in_smem() {
  static const bool on = [] {
    const char* e = std::getenv("LSGD_TC_WSPLIT");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

void tc_alloc(TcWorkspace& ws, const Layout& L, int batch, int n_features, const float* w_master) {
  const float* w_raw = (w_master && tc_weight_split_in_smem()) ? w_master : nullptr;
  ws.weights_split_in_smem = w_raw != nullptr;
  auto dalloc = [&](size_t elems) {
    void* p = nullptr;
    LSGD_CUDA(cudaMalloc(&p, elems * sizeof(float)));
    ws.bufs.push_back(p);
    return static_cast<float*>(p);
  };
  const int B = batch;
  ws.batch = B;
  ws.w_hi = dalloc(static_cast<size_t>(L.n_params));
  ws.w_lo = dalloc(static_cast<size_t>(L.n_params));
  ws.x_hi = dalloc(static_cast<size_t>(B) * n_features);
  ws.x_lo = dalloc(static_cast<size_t>(B) * n_features);
  for (int k = 0; k < L.depth(); ++k) {
    ws.act.push_back(dalloc(static_cast<size_t>(B) * L.out(k)));
    ws.act_hi.push_back(dalloc(static_cast<size_t>(B) * L.out(k)));
    ws.act_lo.push_back(dalloc(static_cast<size_t>(B) * L.out(k)));
  }
  for (int k = 0; k < L.depth(); ++k) {
    ws.dlt.push_back(dalloc(static_cast<size_t>(B) * L.out(k)));
    ws.dlt_hi.push_back(dalloc(static_cast<size_t>(B) * L.out(k)));
    ws.dlt_lo.push_back(dalloc(static_cast<size_t>(B) * L.out(k)));
  }
  ws.partial_elems = static_cast<size_t>(16) << 20;  // 64 MB of split-K partials
  ws.partial = dalloc(ws.partial_elems);
  const int depth = L.depth();
  for (int k = 0; k < depth; ++k) {
    auto* tl = new TcLayer;
    const int ni = L.in(k), no = L.out(k);
    const float* in = k == 0 ? nullptr : ws.act[static_cast<size_t>(k - 1)];
    (void)in;
    const float* in_hi = k == 0 ? ws.x_hi : ws.act_hi[static_cast<size_t>(k - 1)];
    const float* in_lo = k == 0 ? ws.x_lo : ws.act_lo[static_cast<size_t>(k - 1)];
    const float* wk_hi = ws.w_hi + L.w_off[static_cast<size_t>(k)];
    const float* wk_lo = ws.w_lo + L.w_off[static_cast<size_t>(k)];
    const size_t di = static_cast<size_t>(k);  // delta of layer k
    // forward: act_k[B, no] = in[B, ni] . W_k[no, ni]^T + b_k
    {
      EpiParams ep{};
      ep.out = ws.act[static_cast<size_t>(k)];
      ep.ldo = no;
      const bool last = k + 1 == depth;
      ep.out_hi = last ? nullptr : ws.act_hi[static_cast<size_t>(k)];
      ep.out_lo = last ? nullptr : ws.act_lo[static_cast<size_t>(k)];
      ep.relu = last ? 0 : 1;
      tl->fwd = make_plan(OpView{in_hi, B, ni, ni, false}, in_lo, OpView{wk_hi, no, ni, ni, false}, wk_lo, kFwd, ep,
                          ws.partial, ws.partial_elems, w_raw ? w_raw + L.w_off[static_cast<size_t>(k)] : nullptr);
    }
    // weight grad: dW_k[no, ni] = delta_k^T[no, B] . in[B, ni] / B  (both operands read MN-major)
    {
      EpiParams ep{};
      ep.ldo = ni;  // out pointer (payload) bound per step
      ep.div = static_cast<float>(B);
      tl->wgrad = make_plan(OpView{ws.dlt_hi[di], no, B, no, true}, ws.dlt_lo[di], OpView{in_hi, ni, B, ni, true},
                            in_lo, kWgrad, ep, ws.partial, ws.partial_elems);
      tl->dw_a = OpView{ws.dlt_hi[di], no, B, no, true};
      tl->dw_a_lo = ws.dlt_lo[di];
      tl->dw_b = OpView{in_hi, ni, B, ni, true};
      tl->dw_b_lo = in_lo;
      tl->dw_ep = ep;
    }
    // input grad: delta_{k-1}[B, ni] = (delta_k[B, no] . W_k[no, ni]) * [act_{k-1} > 0]  (W read MN-major)
    if (k > 0) {
      EpiParams ep{};
      ep.out = ws.dlt[di - 1];
      ep.ldo = ni;
      ep.out_hi = ws.dlt_hi[di - 1];
      ep.out_lo = ws.dlt_lo[di - 1];
      ep.mask = ws.act[static_cast<size_t>(k - 1)];
      ep.ldm = ni;
      tl->igrad = make_plan(OpView{ws.dlt_hi[di], B, no, no, false}, ws.dlt_lo[di], OpView{wk_hi, ni, no, ni, true},
                            wk_lo, kIgrad, ep, ws.partial, ws.partial_elems,
                            w_raw ? w_raw + L.w_off[static_cast<size_t>(k)] : nullptr);
      tl->has_igrad = true;
    }
    ws.layers.push_back(tl);
  }
  ws.ready = true;
}

void tc_free(TcWorkspace& ws) {
  for (void* p : ws.bufs) cudaFree(p);
  ws.bufs.clear();
  for (TcLayer* l : ws.layers) delete l;
  ws.layers.clear();
  ws.ready = false;
}

static void split(const float* x, int64_t n, float* hi, float* lo, cudaStream_t st, LaunchCounter& lc) {
  int64_t work = (n / 4) + 1;
  int grid = static_cast<int>(std::min<int64_t>((work + 255) / 256, 148 * 8));
  split_tf32_kernel<<<grid, 256, 0, st>>>(x, n, hi, lo);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

void tc_split_weights(TcWorkspace& ws, const Layout& L, const float* w, cudaStream_t st, LaunchCounter& lc) {
  // one pass over the whole parameter vector (biases split too; they are never read from the split copies)
  split(w, L.n_params, ws.w_hi, ws.w_lo, st, lc);
}

// Gather of the shard rows straight into the TF32 split the first GEMM reads (x in fp32 is never materialised).
__global__ void gather_split_kernel(const float* __restrict__ rows, const int32_t* __restrict__ labels,
                                    const int32_t* __restrict__ idx, int d, float* __restrict__ hi,
                                    float* __restrict__ lo, int32_t* __restrict__ y) {
  const int s = blockIdx.x;
  const int64_t r = idx[s];
  if (threadIdx.x == 0) y[s] = labels[r];
  const float4* src = reinterpret_cast<const float4*>(rows + r * d);
  float4* h4 = reinterpret_cast<float4*>(hi + static_cast<int64_t>(s) * d);
  float4* l4 = reinterpret_cast<float4*>(lo + static_cast<int64_t>(s) * d);
#pragma unroll 4
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) {
    const float4 v = src[i];
    const float4 h = make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
    h4[i] = h;
    l4[i] = make_float4(tf32_rna(v.x - h.x), tf32_rna(v.y - h.y), tf32_rna(v.z - h.z), tf32_rna(v.w - h.w));
  }
}

void tc_gather_split(TcWorkspace& ws, const Layout& L, const float* rows, const int32_t* labels, const int32_t* idx,
                     int32_t* y, cudaStream_t st, LaunchCounter& lc) {
  gather_split_kernel<<<ws.batch, 256, 0, st>>>(rows, labels, idx, L.in(0), ws.x_hi, ws.x_lo, y);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

void tc_split_input(TcWorkspace& ws, const Layout& L, const float* x, cudaStream_t st, LaunchCounter& lc) {
  split(x, static_cast<int64_t>(ws.batch) * L.in(0), ws.x_hi, ws.x_lo, st, lc);
}

void tc_forward_layer(TcWorkspace& ws, const Layout& L, int k, const float* w, cudaStream_t st, LaunchCounter& lc) {
  GemmPlan p = ws.layers[static_cast<size_t>(k)]->fwd;
  p.ep.bias = w + L.b_off[static_cast<size_t>(k)];
  run_plan(p, st, lc);
}

void tc_head(TcWorkspace& ws, const Layout& L, const int32_t* y, float* sample_loss, float* loss_out, cudaStream_t st,
             LaunchCounter& lc) {
  const int depth = L.depth();
  const int B = ws.batch;
  const int C = L.out(depth - 1);
  const size_t top = static_cast<size_t>(depth - 1);
  softmax_xent_split_kernel<<<(B + 7) / 8, 256, 0, st>>>(ws.act[static_cast<size_t>(depth - 1)], y, B, C,
                                                             ws.dlt[top], ws.dlt_hi[top], ws.dlt_lo[top], sample_loss);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
  mean_loss_warp_kernel<<<1, 32, 0, st>>>(sample_loss, B, loss_out);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

void tc_backward_dw(TcWorkspace& ws, const Layout& L, int k, int row0, int rows, float* gW, cudaStream_t st,
                    LaunchCounter& lc, const BucketScatter* scat, const FusedUpdate* upd) {
  (void)L;
  TcLayer* tl = ws.layers[static_cast<size_t>(k)];
  auto key = std::make_pair(row0, rows);
  auto it = tl->wgrad_rows.find(key);
  if (it == tl->wgrad_rows.end()) {
    OpView a = tl->dw_a;  // rows of dW_k are the MN (out) index of delta_k
    a.ptr += row0;
    a.rows = rows;
    OpView alo = a;
    alo.ptr = tl->dw_a_lo + row0;
    it = tl->wgrad_rows.emplace(key, make_plan(a, alo.ptr, tl->dw_b, tl->dw_b_lo, kWgrad, tl->dw_ep, ws.partial,
                                               ws.partial_elems)).first;
  }
  GemmPlan pw = it->second;
  pw.ep.out = gW;
  if (scat) pw.ep.scat = *scat;
  if (upd) {
    pw.ep.fuse_upd = 1;
    pw.ep.upd = *upd;
  }
  run_plan(pw, st, lc);
}

void tc_backward_bias(TcWorkspace& ws, const Layout& L, int k, float* gb, cudaStream_t st, LaunchCounter& lc,
                      const BucketScatter* scat, const FusedUpdate* upd) {
  const size_t di = static_cast<size_t>(k);
  BucketScatter sc = scat ? *scat : BucketScatter{};
  FusedUpdate fu = upd ? *upd : FusedUpdate{};
  bias_grad_f32_kernel<<<(L.out(k) + 31) / 32, dim3(32, 32), 0, st>>>(ws.dlt[di], ws.batch, L.out(k), gb, sc, fu);
  ++lc.n;
  LSGD_CUDA(cudaGetLastError());
}

void tc_backward_dx(TcWorkspace& ws, const Layout& L, int k, cudaStream_t st, LaunchCounter& lc) {
  (void)L;
  TcLayer* tl = ws.layers[static_cast<size_t>(k)];
  if (tl->has_igrad) run_plan(tl->igrad, st, lc);
}

void tc_backward_layer(TcWorkspace& ws, const Layout& L, int k, float* gW, float* gb, cudaStream_t st,
                       LaunchCounter& lc) {
  tc_backward_dw(ws, L, k, 0, L.out(k), gW, st, lc);
  tc_backward_bias(ws, L, k, gb, st, lc);
  tc_backward_dx(ws, L, k, st, lc);
}

void tc_test_gemm(int a_mn, int b_mn, int epi, int M, int N, int K, int reps, const float* A, const float* Bm,
                  const float* bias, const float* mask, float div, int relu, float* out, double* avg_ms) {
  LSGD_CUDA(cudaSetDevice(0));
  TcWorkspace ws;
  auto dalloc = [&](size_t elems) {
    void* p = nullptr;
    LSGD_CUDA(cudaMalloc(&p, elems * sizeof(float)));
    ws.bufs.push_back(p);
    return static_cast<float*>(p);
  };
  const size_t na = static_cast<size_t>(M) * K, nb = static_cast<size_t>(N) * K, no = static_cast<size_t>(M) * N;
  float *a = dalloc(na), *ah = dalloc(na), *al = dalloc(na), *b = dalloc(nb), *bh = dalloc(nb), *bl = dalloc(nb);
  float *o = dalloc(no), *oh = dalloc(no), *ol = dalloc(no), *bs = dalloc(N), *mk = dalloc(no);
  const size_t pe = static_cast<size_t>(16) << 20;
  float* part = dalloc(pe);
  LSGD_CUDA(cudaMemcpy(a, A, na * 4, cudaMemcpyHostToDevice));
  LSGD_CUDA(cudaMemcpy(b, Bm, nb * 4, cudaMemcpyHostToDevice));
  if (bias) LSGD_CUDA(cudaMemcpy(bs, bias, static_cast<size_t>(N) * 4, cudaMemcpyHostToDevice));
  if (mask) LSGD_CUDA(cudaMemcpy(mk, mask, no * 4, cudaMemcpyHostToDevice));
  LaunchCounter lc;
  split(a, static_cast<int64_t>(na), ah, al, 0, lc);
  split(b, static_cast<int64_t>(nb), bh, bl, 0, lc);
  EpiParams ep{};
  ep.out = o;
  ep.ldo = N;
  ep.out_hi = oh;
  ep.out_lo = ol;
  ep.bias = bs;
  ep.mask = mk;
  ep.ldm = N;
  ep.relu = relu;
  ep.div = div;
  OpView va{ah, M, K, a_mn ? M : K, a_mn != 0}, vb{bh, N, K, b_mn ? N : K, b_mn != 0};
  // LSGD_TC_TEST_WS=1: the weight-reading forms (forward K-major B, input-gradient MN-major B) split B in SMEM
  static const bool test_ws = std::getenv("LSGD_TC_TEST_WS") && std::atoi(std::getenv("LSGD_TC_TEST_WS")) != 0;
  const bool ws_form = !a_mn && ((epi == kFwd && !b_mn) || (epi == kIgrad && b_mn));
  GemmPlan p = make_plan(va, al, vb, bl, epi, ep, part, pe, test_ws && ws_form ? b : nullptr);
  run_plan(p, 0, lc);
  if (reps > 1 && avg_ms) {  // device-timed repetitions (bring-up / tuning)
    cudaEvent_t e0, e1;
    LSGD_CUDA(cudaEventCreate(&e0));
    LSGD_CUDA(cudaEventCreate(&e1));
    LSGD_CUDA(cudaEventRecord(e0, 0));
    for (int r = 0; r < reps; ++r) run_plan(p, 0, lc);
    LSGD_CUDA(cudaEventRecord(e1, 0));
    LSGD_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    LSGD_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *avg_ms = ms / reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  LSGD_CUDA(cudaDeviceSynchronize());
  LSGD_CUDA(cudaMemcpy(out, o, no * 4, cudaMemcpyDeviceToHost));
  tc_free(ws);
}

}  // namespace lsgd_b200

namespace lsgd_b200 {
// Bring-up probe: one forward/backward of the tensor-core path on host buffers, dumping the intermediates.
// outs: act (sum_k B*out_k, per layer in order), top delta (B*C), grad (P, reference layout), loss (1).
void tc_debug_step(const std::vector<int32_t>& layers, int batch, const float* w_host, const float* x_host,
                   const int32_t* y_host, float* act_out, float* delta_out, float* grad_out, float* loss_out) {
  LSGD_CUDA(cudaSetDevice(0));
  Layout L(layers);
  TcWorkspace ws;
  float *w = nullptr, *x = nullptr, *grad = nullptr, *sl = nullptr, *loss = nullptr;
  int32_t* y = nullptr;
  LSGD_CUDA(cudaMalloc(&w, sizeof(float) * L.n_params));
  tc_alloc(ws, L, batch, layers[0], w);
  LSGD_CUDA(cudaMalloc(&grad, sizeof(float) * L.n_params));
  LSGD_CUDA(cudaMalloc(&x, sizeof(float) * batch * layers[0]));
  LSGD_CUDA(cudaMalloc(&y, sizeof(int32_t) * batch));
  LSGD_CUDA(cudaMalloc(&sl, sizeof(float) * batch));
  LSGD_CUDA(cudaMalloc(&loss, sizeof(float)));
  LSGD_CUDA(cudaMemcpy(w, w_host, sizeof(float) * L.n_params, cudaMemcpyHostToDevice));
  LSGD_CUDA(cudaMemcpy(x, x_host, sizeof(float) * batch * layers[0], cudaMemcpyHostToDevice));
  LSGD_CUDA(cudaMemcpy(y, y_host, sizeof(int32_t) * batch, cudaMemcpyHostToDevice));
  LaunchCounter lc;
  cudaStream_t st = 0;
  tc_split_weights(ws, L, w, st, lc);
  tc_split_input(ws, L, x, st, lc);
  for (int k = 0; k < L.depth(); ++k) tc_forward_layer(ws, L, k, w, st, lc);
  tc_head(ws, L, y, sl, loss, st, lc);
  LSGD_CUDA(cudaDeviceSynchronize());
  int64_t off = 0;
  for (int k = 0; k < L.depth(); ++k) {
    LSGD_CUDA(cudaMemcpy(act_out + off, ws.act[static_cast<size_t>(k)], sizeof(float) * batch * L.out(k),
                         cudaMemcpyDeviceToHost));
    off += static_cast<int64_t>(batch) * L.out(k);
  }
  LSGD_CUDA(cudaMemcpy(delta_out, ws.dlt[static_cast<size_t>(L.depth() - 1)], sizeof(float) * batch * L.out(L.depth() - 1),
                       cudaMemcpyDeviceToHost));
  for (int k = L.depth() - 1; k >= 0; --k)
    tc_backward_layer(ws, L, k, grad + L.w_off[static_cast<size_t>(k)], grad + L.b_off[static_cast<size_t>(k)], st, lc);
  LSGD_CUDA(cudaDeviceSynchronize());
  LSGD_CUDA(cudaMemcpy(grad_out, grad, sizeof(float) * L.n_params, cudaMemcpyDeviceToHost));
  LSGD_CUDA(cudaMemcpy(loss_out, loss, sizeof(float), cudaMemcpyDeviceToHost));
  cudaFree(w);
  cudaFree(grad);
  cudaFree(x);
  cudaFree(y);
  cudaFree(sl);
  cudaFree(loss);
  tc_free(ws);
}
}  // namespace lsgd_b200
