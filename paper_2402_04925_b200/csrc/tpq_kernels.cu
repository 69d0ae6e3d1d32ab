// sm_100a kernels of the TP-aware GPTQ MLP hot path (arxiv 2402.04925).
//
//  k_tcgemv<G>     one dequant-GEMM layer for M <= 16:  Y = X . deq(W),  deq = s * (q - z)
//                  (PAPER.md:L19 per-group scales/zeros; after Alg. 1 every group is G
//                  consecutive rows, so the fp32 scale is applied once per group).
//                  Blackwell-native: per CTA, one warp streams (128-column tile x group) weight
//                  records and the matching activation block into a shared-memory ring with TMA
//                  bulk copies (mbarrier complete_tx, L2 evict-first for the weights); four
//                  warps turn int4 codes into f16 MMA operands with LOP3 magic numbers straight
//                  into TENSOR MEMORY (tcgen05.st, A operand); one thread issues tcgen05.mma
//                  kind::f16 (M=128 columns, N=16 batch rows, A from TMEM, B = activations from
//                  smem, D fp32 in TMEM); the same four warps read D back per group (tcgen05.ld)
//                  and apply the fp32 scale.  The zero point and the magic-number offsets are
//                  folded into one extra K=16 MMA per group (correction block, internal.h).
//                  Persistent stream-K over units with a deterministic last-arriver fix-up;
//                  programmatic dependent launch (weight prefetch overlaps the previous kernel).
//  k_to_xext       X[:, P1] gather (Alg. 3 L1) or the naive AllGather
//                  re-permute + CHUNK (Alg. 2 L3-4) into the B-operand layout.
//  k_gather_rm     the same gathers to row-major (staged API).
//  k_sum_partials  rank-order sum (single-GPU shard simulation only).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "internal.h"

namespace tpq {
namespace {

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));  // (a & b) | c
  return d;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TPQ_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TPQ_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Wait used by the producer / MMA warps: poll with a short sleep between probes so a waiting
// helper warp does not steal issue slots from the dequant warps on its scheduler.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  while (!done) {
    __nanosleep(32);
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
// Optional wait-time accounting (build with -DTPQ_PROF; profiling aid, not in the product build).
#ifdef TPQ_PROF
__device__ unsigned long long g_tpq_prof[16];
#define TPQ_PROF_DECL long long _pt[16] = {0}; const long long _t_start = clock64();
#define TPQ_WAIT(bar, par, k)              \
  do {                                     \
    const long long _t0 = clock64();       \
    mbar_wait(bar, par);                   \
    _pt[k] += clock64() - _t0;             \
  } while (0)
#define TPQ_WAITS(bar, par, k)             \
  do {                                     \
    const long long _t0 = clock64();       \
    mbar_wait_sleep(bar, par);             \
    _pt[k] += clock64() - _t0;             \
  } while (0)
__device__ long long g_tpq_trace[16][32][8];
#define TPQ_EV(e, i)                                                                      \
  if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (i) < 32) g_tpq_trace[threadIdx.x >> 5][i][e] = clock64();
#define TPQ_TIC(k) const long long _tic##k = clock64();
#define TPQ_TOC(k, slot) _pt[slot] += clock64() - _tic##k;
#define TPQ_PROF_FLUSH(ktot)                                                  \
  do {                                                                        \
    _pt[ktot] += clock64() - _t_start;                                        \
    if ((threadIdx.x & 31) == 0)                                              \
      for (int _k = 0; _k < 16; ++_k)                                         \
        if (_pt[_k]) atomicAdd(&g_tpq_prof[_k], (unsigned long long)_pt[_k]); \
  } while (0)
#else
#define TPQ_PROF_DECL
#define TPQ_WAIT(bar, par, k) mbar_wait(bar, par)
#define TPQ_WAITS(bar, par, k) mbar_wait_sleep(bar, par)
#define TPQ_TIC(k)
#define TPQ_TOC(k, slot)
#define TPQ_EV(e, i)
#define TPQ_PROF_FLUSH(ktot) \
  do {                       \
  } while (0)
#endif
// 1-D TMA bulk copy global -> shared, completion counted on `bar` in bytes.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// tcgen05.st 32x32b: each thread of the warp writes N consecutive 32-bit TMEM columns of its lane.
#define TPQ_R4(b) "r"(r[b]), "r"(r[b + 1]), "r"(r[b + 2]), "r"(r[b + 3])
#define TPQ_R16(b) TPQ_R4(b), TPQ_R4(b + 4), TPQ_R4(b + 8), TPQ_R4(b + 12)
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      TPQ_R16(0)
      : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      TPQ_R16(0), TPQ_R16(16)
      : "memory");
}
__device__ __forceinline__ void tmem_st64(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,"
      "%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,"
      "%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64};" ::"r"(taddr),
      TPQ_R16(0), TPQ_R16(16), TPQ_R16(32), TPQ_R16(48)
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), TPQ_R4(0),
               TPQ_R4(4)
               : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), TPQ_R4(0) : "memory");
}
__device__ __forceinline__ void tmem_st1(uint32_t taddr, uint32_t v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(v) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
  return e != 0;
}
// D[tmem] (+)= A[tmem] . B[smem]   (tcgen05.mma kind::f16, cta_group::1).  Called by a whole warp
// with warp-uniform operands; one elected lane issues (keeps the operands in uniform registers:
// ~11 cycles per N=16 MMA instead of ~80 when issued from a divergent single-lane branch,
// tools/probe_tmem_lat.cu).
__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Single-lane forms (caller elects the lane once for a whole group of MMAs).
__device__ __forceinline__ void umma_ts1(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit1(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
// K-major, SWIZZLE_NONE smem descriptor: 8x16B core matrices, LBO = 128 B between the two k-halves
// of a k16 block, SBO = byte distance between the two 8-row groups, version 1 (sm_100).  Verified
// by tools/probe_tcgen05.cu.
__device__ __forceinline__ uint64_t bdesc(uint32_t saddr, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) |
         (1ull << 46);
}
// Offset (in halves) of element (m, kk) of group g in the activation operand (internal.h).
__device__ __forceinline__ int64_t xoff(int64_t g, int m, int kk, int G) {
  return (g * kNPad + m) * (G + 16) + kk;
}
// instruction descriptor: D f32, A/B f16, both K-major, N = 16, M = 128
constexpr uint32_t kIdesc = (1u << 4) | ((uint32_t)(kNPad >> 3) << 17) | ((uint32_t)(kTileCols >> 4) << 24);

// ------------------------------------------------------------------ GEMV configuration
// Warp roles (480 threads, two CTAs per SM):
//   warps 0-7   dequant: warp w converts the codes of TMEM lane quarter w%4 (weight columns
//               32(w%4)..+31) for k-half w/4 of the unit into the A operand in TMEM (tcgen05.st).
//   warps 8-11  epilogue: lane quarter w-8; tcgen05.ld of D per unit, fp32 scale, tile output.
//   warp 12     TMA producer: weight records (ring full/empty).
//   warp 13     MMA issuer: (G/16 + 1) tcgen05.mma per unit and the commits.
//   warp 14     activation stager: the M real rows of each unit's activation block (xfull/xempty).
// Only barrier waits connect the roles, so each warp's per-unit latency overlaps the others'.
constexpr int kGemvThreads = 480;
template <int G>
struct TC {
  static constexpr int KB = G / 16 + 1;                        // k16 blocks per group incl. correction
  static constexpr int UB = 64 * G + 320;                      // weight record bytes
  static constexpr int UBP = (UB + 127) / 128 * 128;
  static constexpr int XG = KB * kNPad * 32;                   // activation block bytes per group
  static constexpr int NS = G == 128 ? 6 : (G == 64 ? 10 : 16);  // weight ring stages
  static constexpr int NX = NS;                                  // activation ring stages
  static constexpr int STAGE = UBP;
  static constexpr int XRING = NS * STAGE;                       // byte offset of the activation ring
  // TMEM A / D buffers: 3 A buffers break the dequant -> MMA -> a_empty -> dequant loop; the
  // epilogue warps keep up with 2 D buffers.  3*72 + 2*16 = 248 <= 256 columns: two CTAs per SM.
  static constexpr int NA = 3, ND = 2;
  static constexpr int SR = 8;                                 // scale ring (> NA + ND units deep)
  static constexpr int ACOLS = G / 2 + 8;                      // f16x2 columns (+ correction block)
  static constexpr int DCOLS = kNPad;
  static constexpr int USED = ND * DCOLS + NA * ACOLS;
  static constexpr int TCOLS = USED <= 32 ? 32 : USED <= 64 ? 64 : USED <= 128 ? 128 : USED <= 256 ? 256 : 512;
  static constexpr int WPW = G / 16;                           // u32 code words per column per k-half
  static constexpr int SCRATCH = kTileCols * 33 * 4;           // epilogue reduction scratch
  static constexpr int SCALES = XRING + NX * XG + SCRATCH;     // byte offset of the scale ring
  static constexpr int BARS = SCALES + SR * kTileCols * 4;     // byte offset of the mbarriers
  static constexpr int SMEM = BARS + 8 * (2 * NS + 2 * NX + 2 * NA + 2 * ND + SR);
};

struct GemvArgs {
  const uint8_t* packed;
  const uint8_t* xext;
  int M;
  int64_t K, N;
  int NT, NG;
  int64_t U;
  int grid;
  void* out;
  int out_mode;
  int64_t out_ld;
  int next_G;
  float* ws;
  int* cnt;
};

__device__ __forceinline__ int64_t cta_start(int64_t c, int64_t U, int grid) { return c * U / grid; }
// CTA whose range contains unit u:  largest c with floor(c U / grid) <= u.
__device__ __forceinline__ int cta_of_unit(int64_t u, int64_t U, int grid) {
  return (int)(((u + 1) * grid + U - 1) / U) - 1;
}

__device__ __forceinline__ uint32_t split_hi_lo(float v) {
  const __half hi = __float2half_rn(v);
  const __half lo = __float2half_rn(v - __half2float(hi));
  return (uint32_t)__half_as_ushort(hi) | ((uint32_t)__half_as_ushort(lo) << 16);
}

// Write one finished 128-column tile (thread t owns column n = tile*128 + t, rows 0..15).
// Called by the 128 epilogue threads together (uses named barrier 1 and `scratch`); t = column.
__device__ void write_tile(const GemvArgs& a, int tile, int t, const float (&acc)[kNPad], float* scratch) {
  const int64_t n = (int64_t)tile * kTileCols + t;
  if (a.out_mode == OUT_ROWMAJOR) {
    __half* out = reinterpret_cast<__half*>(a.out);
#pragma unroll
    for (int m = 0; m < kNPad; ++m)
      if (m < a.M) out[(int64_t)m * a.out_ld + n] = __float2half_rn(acc[m]);
    return;
  }
  // OUT_XEXT: B operand of the next layer (k' = n, group size G2), plus its correction block.
  const int G2 = a.next_G;
  const int64_t g2 = n / G2;
  const int kk = (int)(n % G2);
  const bool lo = (kk & 3) < 2;
  __half* xo = reinterpret_cast<__half*>(a.out);
#pragma unroll
  for (int m = 0; m < kNPad; ++m) {
    const __half h = __float2half_rn(m < a.M ? acc[m] : 0.f);
    const __half b = lo ? h : __hmul(h, __float2half(0.0625f));
    if (m < a.M) xo[xoff(g2, m, kk, G2)] = b;
    const float bf = __half2float(b);
    scratch[t * 33 + m] = bf;                        // S_B contribution
    scratch[t * 33 + 16 + m] = lo ? bf : 16.f * bf;  // S_x contribution
  }
  named_bar(1, kTileCols);
  const int per = kTileCols / G2;  // groups in this tile
  if (t < per * 32) {
    const int gi = t >> 5, q = t & 31;
    const int m = q & 15;
    if (m < a.M) {
      float s = 0.f;
      for (int i = 0; i < G2; ++i) s += scratch[(gi * G2 + i) * 33 + q];
      const int64_t gg = ((int64_t)tile * kTileCols) / G2 + gi;
      __half* corr = reinterpret_cast<__half*>(a.out) + xoff(gg, m, G2 + (q < 16 ? 0 : 2), G2);
      *reinterpret_cast<uint32_t*>(corr) = split_hi_lo(s);
    }
  }
  named_bar(1, kTileCols);
}

template <int G>
__global__ void __launch_bounds__(kGemvThreads, 2) k_tcgemv(const GemvArgs a) {
  using C = TC<G>;
  extern __shared__ __align__(1024) uint8_t smem[];
  float* scratch = reinterpret_cast<float*>(smem + C::XRING + C::NX * C::XG);
  float* sring = reinterpret_cast<float*>(smem + C::SCALES);  // [SR][128] fp32 scales
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BARS);
  uint64_t* full = bars;                 // weight ring: TMA landed
  uint64_t* empty = full + C::NS;        // weight ring: the 8 dequant warps hold their codes
  uint64_t* xfull = empty + C::NS;       // activation ring: TMA landed
  uint64_t* xempty = xfull + C::NX;      // activation ring: MMA commit
  uint64_t* a_full = xempty + C::NX;     // TMEM A buffer: 8 dequant warps stored their part
  uint64_t* a_empty = a_full + C::NA;    // TMEM A buffer: MMA commit
  uint64_t* d_full = a_empty + C::NA;    // TMEM D buffer: MMA commit
  uint64_t* d_empty = d_full + C::ND;    // TMEM D buffer: 4 epilogue warps read it
  uint64_t* s_full = d_empty + C::ND;    // scale ring: 4 dequant warps (k-half 0) wrote it
  __shared__ uint32_t s_tmem;
  __shared__ int s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int64_t u0 = cta_start(blockIdx.x, a.U, a.grid);
  const int64_t u1 = cta_start(blockIdx.x + 1, a.U, a.grid);
  const int nu = (int)(u1 - u0);

  if (tid == 0) {
    for (int s = 0; s < C::NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 8);
    }
    for (int s = 0; s < C::NX; ++s) {
      mbar_init(xfull + s, 32);  // 32 stager lanes (cp.async.mbarrier.arrive.noinc)
      mbar_init(xempty + s, 1);
    }
    for (int b = 0; b < C::NA; ++b) {
      mbar_init(a_full + b, 8);
      mbar_init(a_empty + b, 1);
    }
    for (int d = 0; d < C::ND; ++d) {
      mbar_init(d_full + d, 1);
      mbar_init(d_empty + d, 4);
    }
    for (int r = 0; r < C::SR; ++r) mbar_init(s_full + r, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 13) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "n"(C::TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_launch_dependents();
  // warp-uniform TMEM base (shfl keeps it in the uniform datapath for the MMA operands)
  const uint32_t tmem = __shfl_sync(0xffffffffu, s_tmem, 0);
  const uint32_t d_col0 = 0, a_col0 = C::ND * C::DCOLS;

  if (warp == 12) {
    // ===================== TMA producer (warp-uniform loop, one elected lane issues) ===========
    // Weight records do not depend on the previous kernel: the first NS are requested before
    // griddepcontrol.wait (programmatic dependent launch overlaps them with the previous kernel).
    TPQ_PROF_DECL
    const uint64_t pw = policy_evict_first();
    const int pre = nu < C::NS ? nu : C::NS;
    for (int i = 0; i < pre; ++i) {
      if (elect_one()) {
        mbar_arrive_expect_tx(full + i, C::UB);
        bulk_g2s(smem + i * C::STAGE, a.packed + (u0 + i) * C::UB, C::UB, full + i, pw);
      }
      __syncwarp();
    }
    for (int i = 0, s = 0, ph = 0; i + C::NS < nu; ++i) {  // refill as the dequant warps release
      TPQ_WAIT(empty + s, (uint32_t)ph, 1);
      if (elect_one()) {
        mbar_arrive_expect_tx(full + s, C::UB);
        bulk_g2s(smem + s * C::STAGE, a.packed + (u0 + i + C::NS) * C::UB, C::UB, full + s, pw);
      }
      __syncwarp();
      TPQ_EV(0, i + C::NS)
      if (++s == C::NS) { s = 0; ph ^= 1; }
    }
    TPQ_PROF_FLUSH(8);
  } else if (warp == 14) {
    // ===================== activation stager (cp.async, asynchronous) =====================
    // Unit (tile, g) needs group g's activation block in the tcgen05 canonical B layout.  Only the
    // M real rows are copied (16-byte cp.async per row chunk, straight from L2); completion is
    // signalled on xfull by cp.async.mbarrier.arrive, so the warp runs NX units ahead without
    // waiting for data.  Rows >= M of a stage are never consumed (their D rows are discarded).
    TPQ_PROF_DECL
    constexpr int RW = G + 16, CPR = RW / 8;  // halves / 16-byte chunks per row record
    const uint32_t xring = smem_u32(smem + C::XRING);
    pdl_wait();  // activations come from the previous kernel in the stream
    int g = (int)(u0 % a.NG);
    for (int i = 0, x = 0, phx = 0; i < nu; ++i, g = (g + 1 == a.NG) ? 0 : g + 1) {
      if (i >= C::NX) TPQ_WAIT(xempty + x, (uint32_t)(phx ^ 1), 0);
      const __half* src = reinterpret_cast<const __half*>(a.xext) + (int64_t)g * kNPad * RW;
      const uint32_t dst = xring + x * C::XG;
      for (int t = lane; t < a.M * CPR; t += 32) {
        const int m = t / CPR, c = t - m * CPR;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                         dst + (uint32_t)(((m >> 3) * RW * 8 + c * 64 + (m & 7) * 8) * 2)),
                     "l"(src + m * RW + c * 8)
                     : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(xfull + x)) : "memory");
      TPQ_EV(1, i)
      if (++x == C::NX) { x = 0; phx ^= 1; }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    TPQ_PROF_FLUSH(15);
  } else if (warp == 13) {
    // ===================== MMA issuer (warp-uniform operands, one elected lane issues) =========
    TPQ_PROF_DECL
    const uint32_t xring = smem_u32(smem + C::XRING);
    int x = 0, b = 0, d = 0;
    uint32_t px = 0, pb = 0, pd = 0;  // phase bits of the ring positions
    for (int i = 0; i < nu; ++i) {
      TPQ_WAIT(xfull + x, px, 2);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // cp.async data -> tensor core
      TPQ_WAIT(a_full + b, pb, 3);
      TPQ_EV(0, i)
      TPQ_WAIT(d_empty + d, pd ^ 1, 4);
      TPQ_EV(1, i)
      tc_fence_after();
      const uint64_t bd0 = bdesc(xring + x * C::XG, (G + 16) * 16);
      uint32_t aop[C::KB];
      uint64_t bop[C::KB];
      const uint32_t dt = tmem + d_col0 + d * C::DCOLS, at = tmem + a_col0 + b * C::ACOLS;
#pragma unroll
      for (int j = 0; j < C::KB; ++j) {  // operands first (independent conversions), then back-to-back issue
        aop[j] = at + j * 8;
        bop[j] = bd0 + (uint64_t)(j * (256 / 16));
      }
      if (elect_one()) {
#pragma unroll
        for (int j = 0; j < C::KB; ++j) umma_ts1(dt, aop[j], bop[j], kIdesc, j > 0);
        umma_commit1(d_full + d);
        umma_commit1(a_empty + b);
        umma_commit1(xempty + x);
      }
      __syncwarp();
      TPQ_EV(2, i)
      if (++x == C::NX) { x = 0; px ^= 1; }
      if (++b == C::NA) { b = 0; pb ^= 1; }
      if (++d == C::ND) { d = 0; pd ^= 1; }
    }
    TPQ_PROF_FLUSH(9);
  } else if (warp < 8) {
    // ===================== warps 0-7: dequant (regs -> TMEM A) =====================
    TPQ_PROF_DECL
    const int qw = warp & 3, kh = warp >> 2;         // lane quarter, k-half
    const int col = qw * 32 + lane;                  // weight column of the tile = TMEM lane
    const uint32_t lane_base = (uint32_t)(qw * 32) << 16;
    if (kh == 1) {  // constant part of the correction block of both A buffers: (-1024,-1024), ., 0 x 6
      for (int b = 0; b < C::NA; ++b) {
        const uint32_t cz[4] = {0xE400E400u, 0u, 0u, 0u};
        const uint32_t z4[4] = {0u, 0u, 0u, 0u};
        tmem_st4(tmem + lane_base + a_col0 + b * C::ACOLS + G / 2, cz);
        tmem_st4(tmem + lane_base + a_col0 + b * C::ACOLS + G / 2 + 4, z4);
      }
      tmem_wait_st();
    }
    for (int i = 0; i < nu; ++i) {
      const int s = i % C::NS, b = i % C::NA;
      TPQ_WAIT(full + s, (uint32_t)((i / C::NS) & 1), 5);
      TPQ_EV(0, i)
      const uint8_t* st = smem + s * C::STAGE;
      uint32_t wv[C::WPW];  // this warp's code words: k = kh*G/2 + 8w .. +7, w < WPW
#pragma unroll
      for (int w = 0; w < C::WPW; w += (C::WPW >= 4 ? 4 : C::WPW)) {
        const int gw = kh * C::WPW + w;  // word index within the column
        const uint8_t* p = st + ((gw >> 2) * kTileCols + col) * 16 + (gw & 3) * 4;
        if constexpr (C::WPW >= 4) {
          const uint4 v = *reinterpret_cast<const uint4*>(p);
          wv[w] = v.x;
          wv[w + 1] = v.y;
          wv[w + 2] = v.z;
          wv[w + 3] = v.w;
        } else {
          const uint2 v = *reinterpret_cast<const uint2*>(p);
          wv[w] = v.x;
          wv[w + 1] = v.y;
        }
      }
      uint32_t zz = 0;
      if (kh == 0) {  // hand this unit's fp32 column scale to the epilogue warps
        sring[(i % C::SR) * kTileCols + col] = __half2float(*reinterpret_cast<const __half*>(st + 64 * G + 2 * col));
      } else {
        const uint32_t z = (st[64 * G + 256 + (col >> 1)] >> (4 * (col & 1))) & 0xFu;
        zz = (uint32_t)__half_as_ushort(__float2half(-(float)z)) * 0x10001u;
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(empty + s);
        if (kh == 0) mbar_arrive(s_full + i % C::SR);
      }
      TPQ_TIC(a)
      uint32_t r[4 * C::WPW];
#pragma unroll
      for (int w = 0; w < C::WPW; ++w) {
        const uint32_t x = wv[w], x8 = x >> 8;
        r[4 * w + 0] = lop3_and_or(x, 0x000F000Fu, 0x64006400u);   // k0,k0+1   : 1024 + q
        r[4 * w + 1] = lop3_and_or(x, 0x00F000F0u, 0x64006400u);   // k0+2,k0+3 : 1024 + 16 q
        r[4 * w + 2] = lop3_and_or(x8, 0x000F000Fu, 0x64006400u);  // k0+4,k0+5
        r[4 * w + 3] = lop3_and_or(x8, 0x00F000F0u, 0x64006400u);  // k0+6,k0+7
      }
      TPQ_TOC(a, 11)
      TPQ_EV(1, i)
      TPQ_TIC(c)
      TPQ_WAIT(a_empty + b, (uint32_t)(((i / C::NA) & 1) ^ 1), 6);  // MMA of unit i-NA done
      tc_fence_after();
      const uint32_t ab = tmem + lane_base + a_col0 + b * C::ACOLS;
      if constexpr (C::WPW == 8) {
        tmem_st32(ab + kh * 32, r);
      } else if constexpr (C::WPW == 4) {
        tmem_st16(ab + kh * 16, r);
      } else {
        tmem_st8(ab + kh * 8, r);
      }
      if (kh == 1) tmem_st1(ab + G / 2 + 1, zz);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(a_full + b);
      TPQ_EV(2, i)
      TPQ_TOC(c, 13)
    }
    TPQ_PROF_FLUSH(10);
  } else {
    // ===================== warps 8-11: epilogue =====================
    TPQ_PROF_DECL
    const int qw = warp - 8, col = qw * 32 + lane;
    const uint32_t lane_base = (uint32_t)(qw * 32) << 16;
    pdl_wait();  // outputs may still be read by the previous kernel in the stream
    float acc[kNPad];
#pragma unroll
    for (int m = 0; m < kNPad; ++m) acc[m] = 0.f;
    int64_t seg_start = u0;  // first unit of the current tile segment
    int g = (int)(u0 % a.NG), tile = (int)(u0 / a.NG);
    for (int k = 0; k < nu; ++k) {
      const int d = k % C::ND;
      TPQ_WAIT(d_full + d, (uint32_t)((k / C::ND) & 1), 7);
      tc_fence_after();
      uint32_t v[16];
      tmem_ld16(tmem + lane_base + d_col0 + d * C::DCOLS, v);
      TPQ_WAIT(s_full + k % C::SR, (uint32_t)((k / C::SR) & 1), 12);
      const float s = sring[(k % C::SR) * kTileCols + col];
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(d_empty + d);
      TPQ_EV(0, k)
#pragma unroll
      for (int m = 0; m < kNPad; ++m) acc[m] = fmaf(s, __uint_as_float(v[m]), acc[m]);
      const int64_t u = u0 + k;
      if (g == a.NG - 1 || k == nu - 1) {
        const bool full_tile = (seg_start == (int64_t)tile * a.NG) && (g == a.NG - 1);
        if (full_tile) {
          write_tile(a, tile, col, acc, scratch);
        } else {
          const int slot = (seg_start == u0) ? 0 : 1;
          float* mine = a.ws + ((size_t)blockIdx.x * 2 + slot) * (kNPad * kTileCols);
#pragma unroll
          for (int m = 0; m < kNPad; ++m)
            if (m < a.M) __stcg(mine + m * kTileCols + col, acc[m]);
          __threadfence();
          named_bar(1, kTileCols);
          const int c_first = cta_of_unit((int64_t)tile * a.NG, a.U, a.grid);
          const int c_last = cta_of_unit((int64_t)tile * a.NG + a.NG - 1, a.U, a.grid);
          if (col == 0) s_last = (atomicAdd(a.cnt + tile, 1) == c_last - c_first);
          named_bar(1, kTileCols);
          if (s_last) {
            __threadfence();
            float r[kNPad];
#pragma unroll
            for (int m = 0; m < kNPad; ++m) r[m] = 0.f;
            for (int c = c_first; c <= c_last; ++c) {
              const int cslot = (cta_start(c, a.U, a.grid) / a.NG == tile) ? 0 : 1;
              const float* src = a.ws + ((size_t)c * 2 + cslot) * (kNPad * kTileCols);
#pragma unroll
              for (int m = 0; m < kNPad; ++m)
                if (m < a.M) r[m] += __ldcg(src + m * kTileCols + col);
            }
            write_tile(a, tile, col, r, scratch);
            if (col == 0) a.cnt[tile] = 0;  // self-reset for the next launch / graph replay
          }
        }
#pragma unroll
        for (int m = 0; m < kNPad; ++m) acc[m] = 0.f;
        seg_start = u + 1;
      }
      if (++g == a.NG) {
        g = 0;
        ++tile;
      }
    }
    TPQ_PROF_FLUSH(14);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 13) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TCOLS) : "memory");
  }
}

template <class Kern, class... Args>
cudaError_t launch_pdl(Kern k, dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

template <int G>
int blocks_per_sm_t() {
  constexpr int smem = TC<G>::SMEM;
  static_assert(smem <= 227 * 1024, "GEMV smem over the per-CTA limit");
  if (cudaFuncSetAttribute(k_tcgemv<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return 0;
  if (cudaFuncSetAttribute(k_tcgemv<G>, cudaFuncAttributePreferredSharedMemoryCarveout,
                           (int)cudaSharedmemCarveoutMaxShared) != cudaSuccess)
    return 0;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_tcgemv<G>, kGemvThreads, smem) != cudaSuccess) return 0;
  const int by_tmem = 512 / TC<G>::TCOLS;
  if (getenv("TPQ_VERBOSE")) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_tcgemv<G>);
    fprintf(stderr, "[tpq] k_tcgemv<%d>: regs %d, smem dyn %d static %zu, occupancy %d, tmem cap %d\n", G, fa.numRegs,
            smem, fa.sharedSizeBytes, nb, by_tmem);
  }
  // The occupancy API under-reports here (1) while ncu's block limits (registers 2, smem 2)
  // admit two CTAs; TMEM (512 columns per SM) is the binding constraint.
  return nb < 1 ? 0 : by_tmem;
}

// ------------------------------------------------------------------ gathers
__device__ __forceinline__ int64_t gather_src(int m, int64_t k, int64_t ld, const int32_t* idx, int mode,
                                              int64_t nn, int M) {
  if (mode == GATHER_COLS) return (int64_t)m * ld + (idx ? (int64_t)idx[k] : k);
  const int64_t c = idx[k];
  return (c / nn) * (int64_t)M * nn + (int64_t)m * nn + (c % nn);
}

// One CTA per group: thread (m, c8) builds 8 consecutive k of row m (16 B of the B operand) and
// the group's correction block from fixed-order sums.
__global__ void k_to_xext(const __half* __restrict__ src, int64_t ld, const int32_t* __restrict__ idx, int mode,
                          int64_t nn, int M, int64_t K, int G, uint8_t* __restrict__ dst) {
  pdl_launch_dependents();
  pdl_wait();  // src is produced by, and dst still read by, earlier kernels in the stream
  extern __shared__ float red[];  // [16 m][G/8][2]
  const int g = blockIdx.x;
  const int cpr = G / 8;  // 8-k chunks per row
  const int m = threadIdx.x / cpr, c8 = threadIdx.x % cpr;
  __half* xo = reinterpret_cast<__half*>(dst);
  float sb = 0.f, sx = 0.f;
  uint32_t pk[4] = {0, 0, 0, 0};
  if (m < M) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int64_t k = (int64_t)g * G + c8 * 8 + e;
      const __half h = src[gather_src(m, k, ld, idx, mode, nn, M)];
      const bool lo = (e & 3) < 2;
      const __half b = lo ? h : __hmul(h, __float2half(0.0625f));
      const float bf = __half2float(b);
      sb += bf;
      sx += lo ? bf : 16.f * bf;
      pk[e >> 1] |= (uint32_t)__half_as_ushort(b) << (16 * (e & 1));
    }
  }
  if (m < M) *reinterpret_cast<uint4*>(xo + xoff(g, m, c8 * 8, G)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  red[(m * cpr + c8) * 2 + 0] = sb;
  red[(m * cpr + c8) * 2 + 1] = sx;
  __syncthreads();
  if (c8 == 0 && m < M) {
    float tb = 0.f, tx = 0.f;
    for (int i = 0; i < cpr; ++i) {
      tb += red[(m * cpr + i) * 2 + 0];
      tx += red[(m * cpr + i) * 2 + 1];
    }
    *reinterpret_cast<uint4*>(xo + xoff(g, m, G, G)) = make_uint4(split_hi_lo(tb), split_hi_lo(tx), 0u, 0u);
    *reinterpret_cast<uint4*>(xo + xoff(g, m, G + 8, G)) = make_uint4(0u, 0u, 0u, 0u);
  }
}

__global__ void k_gather_rm(const __half* __restrict__ src, int64_t ld, const int32_t* __restrict__ idx, int mode,
                            int64_t nn, int M, int64_t K, __half* __restrict__ dst) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t total = (int64_t)M * K;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / K);
    const int64_t k = i % K;
    dst[i] = src[gather_src(m, k, ld, idx, mode, nn, M)];
  }
}

struct PartsArg {
  const __half* p[8];
};

__global__ void k_sum_partials(PartsArg pa, int nparts, int64_t count, __half* __restrict__ out) {
  pdl_launch_dependents();
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int r = 0; r < nparts; ++r) s += __half2float(pa.p[r][i]);
    out[i] = __float2half_rn(s);
  }
}

int grid_for(int64_t work, int per_block) {
  int64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > 148 * 8) g = 148 * 8;
  return (int)g;
}

}  // namespace

// ------------------------------------------------------------------ launchers
#ifdef TPQ_PROF
int trace_read(long long* out) {
  return cudaMemcpyFromSymbol(out, g_tpq_trace, sizeof(long long) * 16 * 32 * 8) != cudaSuccess;
}
int prof_read(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, g_tpq_prof, sizeof(unsigned long long) * 16) != cudaSuccess) return 1;
  unsigned long long z[16] = {0};
  return cudaMemcpyToSymbol(g_tpq_prof, z, sizeof(z)) != cudaSuccess;
}
#endif
int gemv_blocks_per_sm(int G) {
  if (G == 128) return blocks_per_sm_t<128>();
  if (G == 64) return blocks_per_sm_t<64>();
  if (G == 32) return blocks_per_sm_t<32>();
  return 0;
}

cudaError_t launch_gemv(const LayerDev& L, const void* xext, int M, void* out, int out_mode, int64_t out_ld,
                        int next_G, cudaStream_t st) {
  if (M < 1 || M > kMaxM) return cudaErrorInvalidValue;
  GemvArgs a;
  a.packed = L.packed;
  a.xext = reinterpret_cast<const uint8_t*>(xext);
  a.M = M;
  a.K = L.K;
  a.N = L.N;
  a.NT = L.NT;
  a.NG = L.NG;
  a.U = L.U;
  a.grid = L.grid;
  a.out = out;
  a.out_mode = out_mode;
  a.out_ld = out_ld;
  a.next_G = next_G;
  a.ws = L.ws;
  a.cnt = L.cnt;
  if (L.G == 128) return launch_pdl(k_tcgemv<128>, dim3(a.grid), dim3(kGemvThreads), TC<128>::SMEM, st, a);
  if (L.G == 64) return launch_pdl(k_tcgemv<64>, dim3(a.grid), dim3(kGemvThreads), TC<64>::SMEM, st, a);
  if (L.G == 32) return launch_pdl(k_tcgemv<32>, dim3(a.grid), dim3(kGemvThreads), TC<32>::SMEM, st, a);
  return cudaErrorInvalidValue;
}

cudaError_t launch_to_xext(const void* src, int64_t ld, const int32_t* idx, int mode, int64_t nn, int M, int64_t K,
                           int G, void* dst, cudaStream_t st) {
  if (M < 1 || M > kMaxM || K % G) return cudaErrorInvalidValue;
  const int threads = kNPad * (G / 8);
  return launch_pdl(k_to_xext, dim3((unsigned)(K / G)), dim3(threads), (size_t)threads * 2 * sizeof(float), st,
                    reinterpret_cast<const __half*>(src), ld, idx, mode, nn, M, K, G, reinterpret_cast<uint8_t*>(dst));
}

cudaError_t launch_gather_rowmajor(const void* src, int64_t ld, const int32_t* idx, int mode, int64_t nn, int M,
                                   int64_t K, void* dst, cudaStream_t st) {
  const int64_t total = (int64_t)M * K;
  return launch_pdl(k_gather_rm, dim3(grid_for(total, 256)), dim3(256), 0, st, reinterpret_cast<const __half*>(src),
                    ld, idx, mode, nn, M, K, reinterpret_cast<__half*>(dst));
}

cudaError_t launch_sum_partials(const void* const* parts, int nparts, int64_t count, void* out, cudaStream_t st) {
  if (nparts < 1 || nparts > 8) return cudaErrorInvalidValue;
  PartsArg pa;
  for (int r = 0; r < 8; ++r) pa.p[r] = reinterpret_cast<const __half*>(parts[r < nparts ? r : 0]);
  return launch_pdl(k_sum_partials, dim3(grid_for(count, 256)), dim3(256), 0, st, pa, nparts, count,
                    reinterpret_cast<__half*>(out));
}

}  // namespace tpq
