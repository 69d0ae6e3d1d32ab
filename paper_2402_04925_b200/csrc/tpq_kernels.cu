// sm_100a kernels of the TP-aware GPTQ MLP hot path (arxiv 2402.04925).
//
//  k_dqgemv<G>     one dequant-GEMM layer for M <= 16:  Y = X . deq(W),  deq = s (q - z)
//                  (PAPER.md:L19 per-group scales/zeros; after Alg. 1 every group is G
//                  consecutive rows, so a 128-row k-block carries 128/G groups'
//                  metadata next to its codes).  Blackwell-native: per SM one persistent CTA;
//                  one warp streams (128-column tile x 128-row k-block) weight records into a
//                  shared-memory ring with TMA bulk copies (mbarrier complete_tx, L2 evict-first);
//                  12 warps turn int4 codes into fp16 s (q - z) with LOP3 magic numbers straight
//                  into TENSOR MEMORY (tcgen05.st, the MMA A operand); one warp stages the
//                  activation slice (tensor TMA); two warps issue tcgen05.mma kind::f16 (M = 128
//                  columns, N = 16 batch rows, A from TMEM, B = activations from smem); the
//                  accumulator of a tile segment stays in TMEM and four warps read it back once per
//                  segment.  Persistent stream-K over units with tiles split between CTAs
//                  reduced inside the kernel (per-tile release counters; the fix-up kernels
//                  k_split_fixup / k_mm_fixup only when a tile spans > 4 CTA ranges), or, for small
//                  TP shards, cluster split-K reduced through distributed shared memory; fixed sum
//                  order (deterministic); programmatic dependent launch (the weight prefetch
//                  overlaps the previous kernel).
//  k_dqgemm<G,NB>  A7 (17 <= M < 128): same records, weights as the TMEM A operand, N = 64..256.
//  k_dqgemm_ss<G>  A7 (M >= 128): mixed-input SS GEMM, activations as the reused smem A operand.
//  k_gather_rm     X[:, P1] gather (Alg. 3 L1) or the naive AllGather re-permute
//                  + CHUNK (Alg. 2 L3-4), row-major; k_gather_rows the
//                  staged-row variant.
//  k_sum_partials  rank-order sum (single-GPU shard simulation only).
#include <cuda.h>  // CUtensorMap; the map is encoded on the host through the runtime's driver entry point
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
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
// Wait with a suspend-time hint: the warp sleeps until the phase completes (or the hint, in ns,
// expires) instead of spinning try_wait / branch / yield through the issue slots of busy warps.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TPQ_WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra TPQ_WAITS_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000)
      : "memory");
}
// Wait for a phase expected to take many microseconds (e.g. a whole tile segment): back off with
// __nanosleep between try_waits.  A plain try_wait loop returns after a short hardware window whatever
// the suspend hint, and its retries compete for issue slots with the warps doing the work
// (profiles/r02_summary.md: the epilogue's d_full loop was 12 % of all issued instructions).
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity, unsigned ns) {
  if (ns == 0) {
    mbar_wait(bar, parity);
    return;
  }
  while (!mbar_try(bar, parity)) __nanosleep(ns);
}

// Per-CTA timeline (build with -DTPQ_PROF; profiling aid, not in the product build): entry,
// work start, end (globaltimer ns), SM id, split-tile publish, reducer wait start / end, reducer's own
// accumulator final, clock64 at entry and end, first pair's A operands stored, last MMA commit, and
// each epilogue warp's reduced tile stored, per CTA, per layer (slot 1: N > K, i.e. layer 1 of the MLP).
#ifdef TPQ_PROF
__device__ unsigned long long g_tpq_cta[2][1024][16];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TPQ_CTA(e, v) \
  if (blockIdx.x < 1024) g_tpq_cta[a.NT * kTileCols > a.NKB * kUnitK][blockIdx.x][e] = (v);
// per-unit event timeline of CTA 0 of the layer-2 launch: [warp][unit < 64][event]
__device__ long long g_tpq_trace[2][24][64][4];
#ifndef TPQ_TRACE_CTA
#define TPQ_TRACE_CTA 0  // traced CTA; TPQ_TRACE_N_GT_K=1 traces the launch with N > K (layer 1 of the MLP)
#endif
#ifndef TPQ_TRACE_N_GT_K
#define TPQ_TRACE_N_GT_K 0
#endif
#ifndef TPQ_TRACE_CTA2
#define TPQ_TRACE_CTA2 (-1)  // a second traced CTA (globaltimer in both when set)
#endif
#define TPQ_EV(e, i) \
  if ((blockIdx.x == TPQ_TRACE_CTA || (int)blockIdx.x == TPQ_TRACE_CTA2) && \
      (a.NT * kTileCols > a.NKB * kUnitK) == TPQ_TRACE_N_GT_K && lane == 0 && (i) < 64) \
    g_tpq_trace[blockIdx.x == TPQ_TRACE_CTA ? 0 : 1][warp][i][e] = TPQ_TRACE_CTA2 >= 0 ? (long long)gtime() : clock64();
// k-step event timeline of pair 0 of a k_dqgemm_ss2 launch: [row (+ 12 when N > K)][k-step < 64][event], clock64
// (SM-local: compare times within one CTA's rows only; globaltimer reads cost ~100 ns each)
#define TPQ_EV2(row, e, i) \
  if (blockIdx.x < 2 && lane == 0 && (i) < 64) g_tpq_trace[0][(row) + (a.NG * 256 > a.NKB * kUnitK ? 12 : 0)][i][e] = clock64();
#else
#define TPQ_CTA(e, v)
#define TPQ_EV(e, i)
#define TPQ_EV2(row, e, i)
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
// 3-D tensor TMA global -> shared (tensor map in kernel parameter space), completion on `bar`.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Stage release by lane 0 once every lane's shared-memory loads of the stage have returned: the
// warp reduction reads each lane's `dep` (an XOR over all registers loaded from the stage), which
// waits on those loads; the never-taken store keeps the reduction.  A plain __syncwarp + arrive
// right after the loads let the producer's TMA overwrite a stage whose loads were still in flight
// (run-to-run mismatches at M = 16, tools/stress_reg.py).
__device__ __forceinline__ void release_loaded(uint64_t* bar, uint32_t dep, int lane, float* sink, int never) {
  const uint32_t all = __reduce_or_sync(0xffffffffu, dep);
  if (all == 0x9e3779b9u && never < 0) sink[threadIdx.x] = 0.f;
  if (lane == 0) mbar_arrive(bar);
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// Prefetch part `part` of `parts` of [p, p + bytes) into L2 (bulk prefetch, 32 KB per instruction):
// the next layer's weights of a small shard, fetched while this kernel is latency-bound.
__device__ __forceinline__ void prefetch_l2_part(const uint8_t* p, int64_t bytes, int part, int parts) {
  if (!p || bytes <= 0) return;
  int64_t lo = bytes * part / parts, hi = bytes * (part + 1) / parts;
  lo &= ~(int64_t)15;
  hi &= ~(int64_t)15;
  for (int64_t o = lo; o < hi; o += 32768) {
    const uint32_t n = (uint32_t)(hi - o < 32768 ? hi - o : 32768);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + o), "r"(n) : "memory");
  }
}

// cluster helpers (also used by the A7 CTA-pair GEMM)
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 4-byte store into another CTA's shared memory, completion (bytes) counted on that CTA's barrier
__device__ __forceinline__ void st_async4(uint32_t dst, float v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(dst),
               "r"(__float_as_uint(v)), "r"(bar)
               : "memory");
}

// Split-tile hand-off between the CTAs of one GEMV launch, per epilogue warp (lane quarter qw, no
// cross-warp barrier): each contributor warp stores its 32 columns, then lane 0 adds 1 with release
// semantics to the tile's counter cnt[4 t + qw] (__syncwarp orders the warp's stores before it); the
// reducer's warp qw polls that counter with relaxed loads, acquires once it reaches the number of
// contributors, reads the partials and re-arms the counter to 0 for the next launch (stream order).
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void warp_publish(int* cnt, int lane) {
  __syncwarp();
  if (lane == 0) red_release_add(cnt, 1);
}
// non-blocking: true (with acquire) once *cnt >= n
__device__ __forceinline__ bool warp_poll(const int* cnt, int n, int lane) {
  int ok = 0;
  if (lane == 0 && ld_relaxed(cnt) >= n) ok = ld_acquire(cnt) >= n;
  ok = __shfl_sync(0xffffffffu, ok, 0);
  __syncwarp();
  return ok;
}
__device__ __forceinline__ void warp_wait(const int* cnt, int n, int lane) {
  if (lane == 0)
    while (ld_acquire(cnt) < n) __nanosleep(32);
  __syncwarp();
}
// acc[m] += p[m * 128] for rows m < M, all loads in flight together
template <int NR>
__device__ __forceinline__ void add_partial(const float* p, int M, float (&acc)[NR]) {
  float t[NR];
#pragma unroll
  for (int m = 0; m < NR; ++m) t[m] = m < M ? __ldcg(p + m * 128) : 0.f;
#pragma unroll
  for (int m = 0; m < NR; ++m) acc[m] += t[m];
}

// tcgen05.st 32x32b: each thread of the warp writes N consecutive 32-bit TMEM columns of its lane.
#define TPQ_R4(b) "r"(r[b]), "r"(r[b + 1]), "r"(r[b + 2]), "r"(r[b + 3])
#define TPQ_R16(b) TPQ_R4(b), TPQ_R4(b + 4), TPQ_R4(b + 8), TPQ_R4(b + 12)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      TPQ_R16(0), TPQ_R16(16)
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
// NP consecutive TMEM columns of this lane (NP / 16 loads)
template <int NP>
__device__ __forceinline__ void tmem_ld_np(uint32_t taddr, uint32_t* v) {
#pragma unroll
  for (int j = 0; j < NP / 16; ++j) tmem_ld16(taddr + 16 * j, v + 16 * j);
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
  return e != 0;
}
// D[tmem] (+)= A[tmem] . B[smem]  (tcgen05.mma kind::f16, cta_group::1), issued by one lane that
// the caller elects once for a whole group of MMAs; the operands are computed warp-uniformly
// beforehand so they stay in uniform registers (~11 cycles per N=16 MMA back to back,
// tools/probe_tmem_lat.cu).
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
// One GEMV unit: 8 x tcgen05.mma kind::f16 (M=128, N=16, K=16) into d, A from TMEM columns
// a + 8j, B from the SW128 activation slice at descriptor b: k16 block j at byte offset
// (j / 4) * 2048 + (j % 4) * 32, i.e. + (j / 4) * 128 + (j % 4) * 2 in descriptor units.  The
// first MMA accumulates iff acc0 != 0.  One asm block so the operands are formed with uniform adds
// right before the issue (a per-MMA C++ loop cost ~110 instructions per unit, most of them
// control flow, which the issuing warp could not afford among four dequant warps per SMSP).
template <int HB = 128>  // descriptor units (16 B) from a slice's k-half 0 to k-half 1: NP rows x 128 B / 16
__device__ __forceinline__ void umma_unit16(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 a1, a2, a3, a4, a5, a6, a7;\n\t"
      ".reg .b64 b1, b2, b3, b4, b5, b6, b7;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\tadd.u32 a4, %1, 32;\n\t"
      "add.u32 a5, %1, 40;\n\tadd.u32 a6, %1, 48;\n\tadd.u32 a7, %1, 56;\n\t"
      "add.u64 b1, %2, 2;\n\tadd.u64 b2, %2, 4;\n\tadd.u64 b3, %2, 6;\n\tadd.u64 b4, %2, %5;\n\t"
      "add.u64 b5, %2, %6;\n\tadd.u64 b6, %2, %7;\n\tadd.u64 b7, %2, %8;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], b2, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], b3, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [a4], b4, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [a5], b5, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [a6], b6, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [a7], b7, %3, 1;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc0), "n"(HB), "n"(HB + 2), "n"(HB + 4), "n"(HB + 6)
      : "memory");
}
// K-major SWIZZLE_128B smem descriptor (sm_100 version 1, layout type 2 in bits 61-63): rows of
// 128 B (64 f16 of K) in 8-row, 1024-byte swizzle atoms (16-byte chunk c of row r stored at chunk
// c ^ (r % 8)), SBO = 1024 B between 8-row groups, LBO unused (1).  The k16 block j of a row starts
// 32 j bytes into it: the start address advances by 32 B, the hardware applies the XOR.
__device__ __forceinline__ uint64_t bdesc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
         (2ull << 61);
}
// instruction descriptor: D f32, A/B f16, both K-major, N = 16, M = 128
constexpr uint32_t idesc_n(int n) { return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kTileCols >> 4) << 24); }

// ------------------------------------------------------------------ stream-K partition
// CTA c of `grid` owns units [c U / grid, (c + 1) U / grid) of a layer.
__device__ __forceinline__ int64_t cta_start(int64_t c, int64_t U, int grid) { return c * U / grid; }
// CTA owning unit u under cta_start (inverse of the floor partition).
__device__ __forceinline__ int cta_of_unit(int64_t u, int64_t U, int grid) {
  return (int)(((u + 1) * grid + U - 1) / U) - 1;
}

__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
// SiLU(x) = x / (1 + exp(-x)) in fp32 (the gate activation of the gate_proj variant, reading c23)
__device__ __forceinline__ float silu_f(float x) { return x / (1.f + expf(-x)); }
__device__ __forceinline__ __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }


struct GemvArgs {
  const uint8_t* packed;
  int M;
  int NT, NKB;      // tiles, k-blocks per tile
  int64_t U;        // NT * NKB units
  int grid;
  __half* out;      // [M][out_ld] row-major
  int64_t out_ld;
  float* ws;        // [grid][2 slots][16][128] fp32 split-tile partials (slot 0 = first segment, 1 = last)
  const float* colf;  // [N] 2^(24 - E_n): the records hold s' = s 2^E_n per column n
  const uint32_t* meta;  // unordered layers: [ng][ldm] {lo: fp16 s', hi: fp16 C = -z s' 2^-24}
  int64_t ldm;
  const uint8_t* pf;  // (small shards) the next layer's packed weights, prefetched into L2; else NULL
  int64_t pf_bytes;
  const uint8_t* pf_next;  // (full layers) the next layer's records: the first pf_units of each of its
  int64_t pf_U;            // pf_grid stream-K CTAs (c pf_U / pf_grid) are prefetched into L2; else NULL
  int pf_grid, pf_units;
  int pf_cs, pf_nkb;       // the next layer's cluster size (> 1: CTA c starts at (c / cs) NKB + (c % cs) NKB / cs)
  int csize;        // > 1: cluster split-K (grid = NT x csize, clusters of csize CTAs, one tile each)
  int* cnt;         // [NT] split-tile arrival counters (0 between launches); NULL: the fix-up kernel after
};

// ------------------------------------------------------------------ GEMV (M <= 16)
// Designed for issue: round 1's GEMV spent 1521 warp instructions per 128 x 128 unit, 380 per SMSP
// against the ~378 cycles one unit may take at HBM speed (profiles/r02_summary.md); this one:
//   * dequant in THREE sets of FOUR warps (one per SMSP / TMEM lane quarter); a warp converts its
//     32 columns of BOTH units of a pair per iteration, so waits, hand-offs and index arithmetic are
//     paid once per pair; set s owns TMEM A buffer s and the pairs p = s, s + 3, ...;
//   * a weight stage is released right after the warp's last tcgen05.st of the unit (every loaded
//     register has been consumed by then: no reduction guard);
//   * the epilogue walks tile segments, not units.
// Warps 0-3 epilogue, 4-15 dequant, 16 TMA producer, 17 activation stager, 18-19 MMA issuers: the
// SMSP arbiter prefers higher warp ids, so the warps that only wait sit lowest.
constexpr int kSets = 3, kDeq0 = 4, kProdWarp = 16, kStageWarp = 17, kMmaWarp = 18;
constexpr int kGemvThreads = 20 * 32;

// G = 0: the unordered-g_idx layer (TPQ_UNORDERED, the Fig. 1 formulation): a record
// holds the 128 rows' codes in checkpoint order plus their group ids (uint8), and the dequant warps
// look each row's {s', C} up in an L2-resident [ng][N] table instead of a per-block record header.
// GT: the gated layer 1 of the gate_proj variant (f2, readings c23-c25): records stream as gate(t, kb),
// up(t, kb) pairs, so a dequant pair IS one (tile, k-block) of both layers; gate and up accumulate in
// separate TMEM accumulators and the epilogue writes fp16(SiLU(gate) * up).
// NP: batch rows per MMA (N) and per activation slice: 16 for M <= 16, 32 for 17 <= M <= 32 (the same
// dequant-bound pipeline with twice the MMA N, accumulator columns and activation bytes).
template <int G, bool GT = false, int NP = kNPad>
struct TC {
  static_assert(NP == 16 || (NP == 32 && !GT), "N = 32 for the plain layer only (TMEM budget)");
  static constexpr bool UN = G == 0;
  static_assert(!(UN && GT), "the unordered baseline has no gated variant");
  static constexpr int KG = UN ? 1 : kUnitK / G;
  static constexpr int UB = UN ? kUnitK * kTileCols / 2 + kUnitK : (int)unit_bytes_c(G == 0 ? 128 : G);
  static constexpr int STAGE = (UB + 127) / 128 * 128;
  static constexpr int NS = NP == 16 ? 18 : 12;  // N = 32: 14-18 stages measured alike; 12 leaves a 48 KB landing zone                   // weight ring stages (units)
  static constexpr int XU = NP * kUnitK * 2;   // activation bytes per unit
  static constexpr int NX = NP == 16 ? 6 : 4;                    // activation pair slots
  static constexpr int AU = kUnitK / 2;           // TMEM columns per unit of A
  static constexpr int RD = 6;                    // done ring: pair p on p % 6
  // a_full(p) on barrier p % NAF: the previous completion there, pair p - 6, had the same MMA issuer
  // (p % 2) and dequant set (p % 3), so the waiter consumed it before; with 3 barriers the issuer of
  // pair p could find pair p - 3's phase (other issuer) still open and read the one before it.
  static constexpr int NAF = 6;
  // done(p) on barrier p % RD.  Dequant set p % 3 waits done(p - 3) before overwriting its buffer:
  // the next completion there, p + 3, needs this set's own a_full(p + 3).  The stager waits
  // done(p - NX) before reusing slot p % NX: the next one, p - NX + RD >= p, needs its own later load.
  static_assert(RD % kSets == 0 && RD >= NX, "done ring aliasing");
  static constexpr int TCOLS = 512;
  static constexpr uint32_t IDESC = idesc_n(NP);
  static constexpr int HB = NP * 128 / 16;  // k-half offset of a slice in descriptor units
  static constexpr int DC = (GT ? 8 : 4) * NP;  // [2 segment buffers][2 issuers][gate, up if GT] x 16 columns
  static_assert(DC + kSets * 2 * AU <= TCOLS, "TMEM budget");
  static constexpr int XRING = 0;
  static constexpr int WRING = NX * 2 * XU;
  static constexpr int BARS = WRING + NS * STAGE;
  static constexpr int SMEM = BARS + 8 * (2 * NS + NX + NAF + RD + 6);
  // cluster split-K (small shards, GemvArgs::csize > 1): rank 0 of a cluster receives the other ranks'
  // fp32 partials of its tile, [rank - 1][16 rows][128 columns], in a landing zone after the barriers
  static constexpr int LAND = (SMEM + 127) / 128 * 128;
  static constexpr int CSMAX = GT || UN ? 1 : (227 * 1024 - 1024 - LAND) / (NP * kTileCols * 4) + 1 >= 4 ? 4
                               : (227 * 1024 - 1024 - LAND) / (NP * kTileCols * 4) + 1 >= 2 ? 2 : 1;
  static constexpr int SMEM_CL = LAND + (CSMAX - 1) * NP * kTileCols * 4;
};

template <int G, bool GT, int NP>
__global__ void __launch_bounds__(kGemvThreads, 1)
    k_dqgemv(const GemvArgs a, const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap xmapu) {
  using C = TC<G, GT, NP>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BARS);
  uint64_t* full = bars;                // [NS] weight record landed
  uint64_t* empty = full + C::NS;       // [NS] the 4 warps converting the unit are done with it
  uint64_t* xfull = empty + C::NS;      // [NX] the pair's activation slices landed
  uint64_t* a_full = xfull + C::NX;     // [NAF] pair p's A operands stored (the 4 warps of set p % 3)
  uint64_t* done = a_full + C::NAF;     // [RD] pair p's MMAs completed (tcgen05.commit)
  uint64_t* d_full = done + C::RD;      // [2] segment accumulators final (both issuers)
  uint64_t* d_empty = d_full + 2;       // [2] epilogue read them (4 warps)
  uint64_t* land_full = d_empty + 2;    // [1] cluster split-K: the other ranks' partials landed (rank 0)
  uint64_t* red_full = land_full + 1;   // [1] stream-K reducer: the contributors' partials staged in smem
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // stream-K over a.U units; gated (GT): over a.U (tile, k-block) pairs of gate + up records.
  // Cluster split-K (a.csize > 1): cluster c = tile c, rank r takes k-blocks [r NKB / S, (r+1) NKB / S).
  const int crank = a.csize > 1 ? (int)(blockIdx.x % (unsigned)a.csize) : 0;
  const int64_t v0 = a.csize > 1 ? (int64_t)(blockIdx.x / a.csize) * a.NKB + crank * a.NKB / a.csize
                                  : cta_start(blockIdx.x, a.U, a.grid);
  const int nv = a.csize > 1 ? (crank + 1) * a.NKB / a.csize - crank * a.NKB / a.csize
                             : (int)(cta_start(blockIdx.x + 1, a.U, a.grid) - v0);
  const int64_t u0 = GT ? 2 * v0 : v0;  // first record of the CTA
  const int nu = GT ? 2 * nv : nv;      // records of the CTA
  const int np = (nu + 1) / 2;

  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    TPQ_CTA(0, gtime())
    TPQ_CTA(3, smid)
    TPQ_CTA(8, clock64())
    for (int s = 0; s < C::NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 4);
    }
    for (int s = 0; s < C::NX; ++s) mbar_init(xfull + s, 1);
    for (int s = 0; s < C::NAF; ++s) mbar_init(a_full + s, 4);
    for (int r = 0; r < C::RD; ++r) mbar_init(done + r, 1);
    for (int d = 0; d < 2; ++d) {
      mbar_init(d_full + d, 2);
      mbar_init(d_empty + d, 4);
    }
    mbar_init(land_full, 1);
    mbar_init(red_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "n"(C::TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (a.csize > 1) cluster_sync_all();  // rank 0's land_full initialised before any st.async to it
  tc_fence_after();
  pdl_launch_dependents();
  const uint32_t tmem = __shfl_sync(0xffffffffu, s_tmem, 0);
  constexpr uint32_t kA0 = C::DC;  // A buffer of set s at kA0 + s * 2AU (unit h of the pair at + h AU)

  if (warp >= kDeq0 && warp < kProdWarp) {
    // ===================== dequant: set = warp / 4 - 1 takes pairs p = set, set + 3, ... =========
    const int set = (warp - kDeq0) >> 2, qw = warp & 3;
    const int col = qw * 32 + lane;
    const uint32_t a_buf = tmem + ((uint32_t)(qw * 32) << 16) + kA0 + set * 2 * C::AU;
    const int zbyte = kUnitK * kTileCols / 2 + C::KG * 256 + (col >> 1), zsh = 4 * (col & 1);
    const int sbyte = kUnitK * kTileCols / 2 + 2 * col;
    const bool xw = qw == 0;
    // S = s' for the nibbles at bits 0-3 (q 2^-24) and s' / 16 for bits 4-7 (q 2^-20), C = -z s' 2^-24
    int st = (2 * set) % C::NS;                       // stage of unit 2p
    uint32_t ph = (uint32_t)(((2 * set) / C::NS) & 1);
    for (int p = set; p < np; p += kSets) {
      TPQ_EV(0, p)
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        const int i = 2 * p + h;
        const int sh_ = st + h >= C::NS ? st + h - C::NS : st + h;
        const uint32_t phh = st + h >= C::NS ? ph ^ 1u : ph;
        if (i >= nu) break;
        mbar_wait(full + sh_, phh);
        if (h == 0) { TPQ_EV(1, p) }
        if (p == 0 && h == 0 && warp == kDeq0 && lane == 0) { TPQ_CTA(14, gtime()) }  // unit 0's weights landed
        const uint8_t* sp = smem + C::WRING + sh_ * C::STAGE;
        if constexpr (C::UN) {
          // Fig. 1 formulation: every row k has its own group g(k); the pair (k, k+1) of a half2 gets
          // S2 = (s'_g(k), s'_g(k+1)) and C2 = (C_g(k), C_g(k+1)) from the table, 4 bytes per (row,
          // column) read from L2 (coalesced across the warp's 32 columns): 64 KB per 128 x 128 block
          // against the 320 B header an ordered record carries ("frequently reload").
          const uint32_t* gw = reinterpret_cast<const uint32_t*>(sp + kUnitK * kTileCols / 2);
          const uint32_t* tab = a.meta + ((u0 + i) / a.NKB) * kTileCols + col;
          uint4 cw[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) cw[c] = *reinterpret_cast<const uint4*>(sp + code_block(c, col) * 16);
          const __half2 k16 = __float2half2_rn(0.0625f);
#pragma unroll
          for (int kh = 0; kh < 2; ++kh) {
            uint32_t r[32];
#pragma unroll
            for (int hb = 0; hb < 2; ++hb) {  // 4 words (32 rows) per batch: 32 table loads in flight
              uint32_t t[32];
#pragma unroll
              for (int w = 0; w < 4; ++w) {
                const int k0 = 64 * kh + 32 * hb + 8 * w;
                const uint32_t ga = gw[k0 / 4], gb = gw[k0 / 4 + 1];
#pragma unroll
                for (int e = 0; e < 8; ++e)
                  t[8 * w + e] = __ldg(tab + (int64_t)(((e < 4 ? ga : gb) >> (8 * (e & 3))) & 0xFFu) * a.ldm);
              }
#pragma unroll
              for (int w = 0; w < 4; ++w) {
                const int ww = 4 * hb + w;
                const uint4 c4 = cw[2 * kh + ww / 4];
                const uint32_t x = (ww & 3) == 0 ? c4.x : (ww & 3) == 1 ? c4.y : (ww & 3) == 2 ? c4.z : c4.w;
                const uint32_t x8 = x >> 8;
                const uint32_t* tt = t + 8 * w;
                const __half2 s0 = u2h(__byte_perm(tt[0], tt[1], 0x5410)), c0 = u2h(__byte_perm(tt[0], tt[1], 0x7632));
                const __half2 s1 = __hmul2(u2h(__byte_perm(tt[2], tt[3], 0x5410)), k16), c1 = u2h(__byte_perm(tt[2], tt[3], 0x7632));
                const __half2 s2 = u2h(__byte_perm(tt[4], tt[5], 0x5410)), c2 = u2h(__byte_perm(tt[4], tt[5], 0x7632));
                const __half2 s3 = __hmul2(u2h(__byte_perm(tt[6], tt[7], 0x5410)), k16), c3 = u2h(__byte_perm(tt[6], tt[7], 0x7632));
                r[4 * ww + 0] = h2u(__hfma2(u2h(x & 0x000F000Fu), s0, c0));
                r[4 * ww + 1] = h2u(__hfma2(u2h(x & 0x00F000F0u), s1, c1));
                r[4 * ww + 2] = h2u(__hfma2(u2h(x8 & 0x000F000Fu), s2, c2));
                r[4 * ww + 3] = h2u(__hfma2(u2h(x8 & 0x00F000F0u), s3, c3));
              }
            }
            if (h == 0 && kh == 0 && p >= kSets) {
              const int q = p - kSets;
              mbar_wait_backoff(done + q % C::RD, (uint32_t)((q / C::RD) & 1), 0);
              tc_fence_after();
            }
            tmem_st32(a_buf + h * C::AU + kh * 32, r);
          }
        } else {
          __half2 sl[C::KG], shh[C::KG], zc[C::KG];
  #pragma unroll
          for (int g = 0; g < C::KG; ++g) {
            const float z = (float)((sp[zbyte + g * 64] >> zsh) & 0xFu);
            const float sf = __half2float(*reinterpret_cast<const __half*>(sp + sbyte + g * 256));
            sl[g] = __float2half2_rn(sf);
            shh[g] = __float2half2_rn(sf * 0.0625f);
            zc[g] = __float2half2_rn(-z * sf * 5.9604644775390625e-8f);
          }
          uint4 cw[4];
  #pragma unroll
          for (int c = 0; c < 4; ++c) cw[c] = *reinterpret_cast<const uint4*>(sp + code_block(c, col) * 16);
  #pragma unroll
          for (int kh = 0; kh < 2; ++kh) {
            uint32_t r[32];
  #pragma unroll
            for (int w = 0; w < 8; ++w) {
              const int j = (64 * kh + 8 * w) / G;
              const uint4 c4 = cw[2 * kh + w / 4];
              const uint32_t x = (w & 3) == 0 ? c4.x : (w & 3) == 1 ? c4.y : (w & 3) == 2 ? c4.z : c4.w;
              const uint32_t x8 = x >> 8;
              r[4 * w + 0] = h2u(__hfma2(u2h(x & 0x000F000Fu), sl[j], zc[j]));
              r[4 * w + 1] = h2u(__hfma2(u2h(x & 0x00F000F0u), shh[j], zc[j]));
              r[4 * w + 2] = h2u(__hfma2(u2h(x8 & 0x000F000Fu), sl[j], zc[j]));
              r[4 * w + 3] = h2u(__hfma2(u2h(x8 & 0x00F000F0u), shh[j], zc[j]));
            }
            if (h == 0 && kh == 0 && p >= kSets) {
              // own buffer free: pair p - 3's MMAs completed
              const int q = p - kSets;
              mbar_wait_backoff(done + q % C::RD, (uint32_t)((q / C::RD) & 1), 0);
              TPQ_EV(2, p)
              tc_fence_after();
            }
            tmem_st32(a_buf + h * C::AU + kh * 32, r);
          }
        }
        // every register loaded from the stage fed the tcgen05.st just issued (in-order issue)
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + sh_);
      }
      tmem_wait_st();
      if (xw) mbar_wait(xfull + p % C::NX, (uint32_t)((p / C::NX) & 1));
      if (p == 0 && warp == kDeq0 && lane == 0) { TPQ_CTA(13, gtime()) }  // pair 0's activations landed
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(a_full + p % C::NAF);
      if (p == 0 && warp == kDeq0 && lane == 0) { TPQ_CTA(10, gtime()) }
      TPQ_EV(3, p)
      st += 2 * kSets;
      if (st >= C::NS) {
        st -= C::NS;
        ph ^= 1u;
      }
    }
  } else if (warp < kDeq0) {
    // ===================== epilogue: once per tile segment =====================
    const int qw = warp, col = qw * 32 + lane;
    const uint32_t lane_base = (uint32_t)(qw * 32) << 16;
    pdl_wait();
    if constexpr (GT) {
      // segments over (tile, k-block) pairs; issuer w owns the pairs p % 2 == w of a segment
      int tile = (int)(v0 / a.NKB);
      int64_t seg_start = v0;
      const int64_t vend = v0 + nv;
      constexpr int SLOT = 2 * NP * kTileCols;  // gate then up partials
      for (int seg = 0; seg_start < vend; ++seg, ++tile) {
        const int64_t tile_start = (int64_t)tile * a.NKB, tile_end = tile_start + a.NKB;
        const int64_t seg_end = tile_end < vend ? tile_end : vend;
        const int lo = (int)(seg_start - v0), hi = (int)(seg_end - 1 - v0);
        const int d = seg & 1;
        const bool reduce = a.cnt && seg_start == tile_start && seg_end < tile_end;  // as in the plain epilogue
        const bool publish = a.cnt && seg_start > tile_start;
        int* cnt = a.cnt ? a.cnt + 4 * tile + qw : nullptr;
        const float up = __ldg(a.colf + (int64_t)tile * kTileCols + col);
        mbar_wait_backoff(d_full + d, (uint32_t)((seg >> 1) & 1), 256);
        tc_fence_after();
        const bool w0 = hi > lo || (lo & 1) == 0, w1 = hi > lo || (lo & 1) == 1;
        float gu[2][NP];
#pragma unroll
        for (int kind = 0; kind < 2; ++kind) {  // 0 gate, 1 up: accumulator ((2 d + w) 2 + kind) x 16
          uint32_t v[NP], v1[NP];
          const uint32_t base = tmem + lane_base + (4 * d + kind) * NP;
          if (w0) tmem_ld_np<NP>(base, v);
          if (w1) tmem_ld_np<NP>(base + 2 * NP, v1);
          tmem_wait_ld();
#pragma unroll
          for (int m = 0; m < NP; ++m)
            gu[kind][m] = up * (w0 ? (w1 ? __uint_as_float(v[m]) + __uint_as_float(v1[m]) : __uint_as_float(v[m]))
                                   : __uint_as_float(v1[m]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(d_empty + d);
        const int64_t n = (int64_t)tile * kTileCols + col;
        if (publish) {
          float* mine = a.ws + (size_t)blockIdx.x * 2 * SLOT + col;
#pragma unroll
          for (int kind = 0; kind < 2; ++kind)
#pragma unroll
            for (int m = 0; m < NP; ++m)
              if (m < a.M) __stcg(mine + (kind * NP + m) * kTileCols, gu[kind][m]);
          warp_publish(cnt, lane);
        } else if (reduce) {
          const int nother = cta_of_unit(tile_end - 1, a.U, a.grid) - (int)blockIdx.x;
          warp_wait(cnt, nother, lane);
          for (int q = 0; q < nother; ++q) {  // CTA order after the own partial
            const float* src = a.ws + (size_t)(blockIdx.x + 1 + q) * 2 * SLOT + col;
#pragma unroll
            for (int kind = 0; kind < 2; ++kind) add_partial(src + kind * NP * kTileCols, a.M, gu[kind]);
          }
          if (lane == 0) *cnt = 0;
#pragma unroll
          for (int m = 0; m < NP; ++m)
            if (m < a.M) a.out[m * a.out_ld + n] = __float2half_rn(silu_f(gu[0][m]) * gu[1][m]);
        } else if (seg_start == tile_start && seg_end == tile_end) {
#pragma unroll
          for (int m = 0; m < NP; ++m)
            if (m < a.M) a.out[m * a.out_ld + n] = __float2half_rn(silu_f(gu[0][m]) * gu[1][m]);
        } else {
          // (cnt == NULL) split tile: gate and up partials into this CTA's slot; k_mm_fixup (gated) finishes them
          float* mine = a.ws + ((size_t)blockIdx.x * 2 + (seg_start == v0 ? 0 : 1)) * SLOT;
#pragma unroll
          for (int kind = 0; kind < 2; ++kind)
#pragma unroll
            for (int m = 0; m < NP; ++m)
              if (m < a.M) __stcg(mine + (kind * NP + m) * kTileCols + col, gu[kind][m]);
        }
        seg_start = seg_end;
      }
    } else if (a.csize > 1) {
      // cluster split-K: one segment, this rank's k-range of tile u0 / NKB.  Ranks > 0 send their
      // scaled fp32 partial into rank 0's landing zone (st.async, bytes counted on its land_full);
      // rank 0 adds them in rank order to its own and writes the fp16 tile: no global partials, no
      // counters, one distributed-shared-memory hop at the end of the layer.
      const int tile = (int)(u0 / a.NKB);
      const float up = __ldg(a.colf + (int64_t)tile * kTileCols + col);
      if (crank == 0 && threadIdx.x == 0)
        mbar_arrive_expect_tx(land_full, (uint32_t)((a.csize - 1) * a.M * kTileCols * 4));
      mbar_wait_backoff(d_full, 0u, 256);
      tc_fence_after();
      const int hi = nu - 1;  // units 0 .. hi: issuer 0 has pair 0, issuer 1 any pair 1
      const bool w0 = true, w1 = hi >= 3 || ((hi >> 1) & 1) == 1;
      uint32_t v[NP], v1[NP];
      if (w0) tmem_ld_np<NP>(tmem + lane_base, v);
      if (w1) tmem_ld_np<NP>(tmem + lane_base + NP, v1);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(d_empty);
      float acc[NP];
  #pragma unroll
      for (int m = 0; m < NP; ++m)
        acc[m] = up * (w0 ? (w1 ? __uint_as_float(v[m]) + __uint_as_float(v1[m]) : __uint_as_float(v[m]))
                          : __uint_as_float(v1[m]));
      if (crank > 0) {
        const uint32_t dst = mapa_shared(smem + C::LAND, 0) + (uint32_t)(((crank - 1) * NP * kTileCols + col) * 4);
        const uint32_t bar = mapa_shared(land_full, 0);
  #pragma unroll
        for (int m = 0; m < NP; ++m)
          if (m < a.M) st_async4(dst + m * kTileCols * 4, acc[m], bar);
      } else {
        mbar_wait_backoff(land_full, 0u, 64);
        const float* land = reinterpret_cast<const float*>(smem + C::LAND) + col;
        for (int r = 1; r < a.csize; ++r)
  #pragma unroll
          for (int m = 0; m < NP; ++m)
            if (m < a.M) acc[m] += land[((r - 1) * NP + m) * kTileCols];
        const int64_t n = (int64_t)tile * kTileCols + col;
  #pragma unroll
        for (int m = 0; m < NP; ++m)
          if (m < a.M) a.out[m * a.out_ld + n] = __float2half_rn(acc[m]);
      }
    } else {
      int tile = (int)(u0 / a.NKB);
      int64_t seg_start = u0;
      const int64_t uend = u0 + nu;
      constexpr int SLOT = NP * kTileCols;
      // split tile t (contributors c_first < ... < c_last): c_first holds its first units as its LAST
      // segment and reduces; every later contributor holds it as its FIRST segment and publishes
      // slot 0 -- early in its run, except the middle CTAs of a tile longer than a CTA's range.
      // The reducer takes the next contributor's partial as soon as it is there (polled while waiting
      // for its own accumulators), so a layer whose tiles are shorter than a range has no cross-CTA
      // wait at its end.
      const int64_t lt = (uend - 1) / a.NKB;  // tile of the CTA's last unit
      const bool red_last = a.cnt && lt * a.NKB >= u0 && uend < (lt + 1) * a.NKB;
      const int nother = red_last ? cta_of_unit((lt + 1) * a.NKB - 1, a.U, a.grid) - (int)blockIdx.x : 0;
      int* cnt_last = red_last ? a.cnt + 4 * lt + qw : nullptr;
      float pre[NP] = {};  // contributor c_first + 1's partial
      // the early take is for a single contributor of an N = 16 pass only (registers)
      bool have = !red_last || nother != 1 || NP != kNPad;
      for (int seg = 0; seg_start < uend; ++seg, ++tile) {
        const int64_t tile_start = (int64_t)tile * a.NKB, tile_end = tile_start + a.NKB;
        const int64_t seg_end = tile_end < uend ? tile_end : uend;  // exclusive
        const int lo = (int)(seg_start - u0), hi = (int)(seg_end - 1 - u0);
        const int d = seg & 1;
        const uint32_t par = (uint32_t)((seg >> 1) & 1);
        const bool reduce = red_last && seg_end == uend;
        const bool publish = a.cnt && seg_start > tile_start;
        if (!have) {
          if (reduce && threadIdx.x == 0) { TPQ_CTA(5, gtime()) }
          for (;;) {  // wait for the accumulators, taking the partial if it arrives first
            int ok = 0;
            if (lane == 0) ok = mbar_try(d_full + d, par);
            if (__shfl_sync(0xffffffffu, ok, 0)) break;
            if (warp_poll(cnt_last, nother, lane)) {
              add_partial(a.ws + (size_t)(blockIdx.x + 1) * 2 * SLOT + col, a.M, pre);
              have = true;
              if (threadIdx.x == 0) { TPQ_CTA(6, gtime()) }
              break;
            }
            __nanosleep(256);
          }
        }
        const float up = __ldg(a.colf + (int64_t)tile * kTileCols + col);  // 2^(24 - E) of this column
        mbar_wait_backoff(d_full + d, par, 256);
        tc_fence_after();
        const bool w0 = hi - lo >= 3 || ((lo >> 1) & 1) == 0 || ((hi >> 1) & 1) == 0;
        const bool w1 = hi - lo >= 3 || ((lo >> 1) & 1) == 1 || ((hi >> 1) & 1) == 1;
        uint32_t v[NP], v1[NP];
        const uint32_t dcol = tmem + lane_base + 2 * d * NP;
        if (w0) tmem_ld_np<NP>(dcol, v);
        if (w1) tmem_ld_np<NP>(dcol + NP, v1);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(d_empty + d);
  #pragma unroll
        for (int m = 0; m < NP; ++m)
          v[m] = __float_as_uint(up * (w0 ? (w1 ? __uint_as_float(v[m]) + __uint_as_float(v1[m]) : __uint_as_float(v[m]))
                                          : __uint_as_float(v1[m])));
        const int64_t n = (int64_t)tile * kTileCols + col;
        if (publish) {
          float* mine = a.ws + (size_t)blockIdx.x * 2 * SLOT + col;
  #pragma unroll
          for (int m = 0; m < NP; ++m)
            if (m < a.M) __stcg(mine + m * kTileCols, __uint_as_float(v[m]));
          warp_publish(a.cnt + 4 * tile + qw, lane);
          if (threadIdx.x == 0) { TPQ_CTA(4, gtime()) }
        } else if (reduce) {
          // CTA order: own partial, then c_first + 1, ..., c_last (deterministic)
          if (threadIdx.x == 0) { TPQ_CTA(7, gtime()) }
          float acc[NP];
  #pragma unroll
          for (int m = 0; m < NP; ++m) acc[m] = __uint_as_float(v[m]);
          if (NP == kNPad && nother == 1) {  // (tiles shorter than a CTA range: the partial was usually taken early)
            if (!have) {
              warp_wait(cnt_last, 1, lane);
              add_partial(a.ws + (size_t)(blockIdx.x + 1) * 2 * SLOT + col, a.M, pre);
              if (threadIdx.x == 0) { TPQ_CTA(6, gtime()) }
            }
  #pragma unroll
            for (int m = 0; m < NP; ++m) acc[m] += pre[m];
          } else {
            // Several contributors (middle CTAs finish with this one): once all four warps' counters
            // are complete, thread 0 bulk-copies every partial (M rows) into the activation ring --
            // free, every MMA of this CTA has completed -- so all of them arrive in one round trip
            // whatever the register budget, then each warp adds its columns in CTA order.
            float* stage = reinterpret_cast<float*>(smem + C::XRING);
            const int nst = nother < C::WRING / (SLOT * 4) ? nother : C::WRING / (SLOT * 4);
            if (threadIdx.x == 0) {
              for (int w = 0; w < 4; ++w)
                while (ld_acquire(a.cnt + 4 * lt + w) < nother) __nanosleep(32);
              asm volatile("fence.proxy.async.global;" ::: "memory");  // generic stores -> bulk-copy reads
              mbar_arrive_expect_tx(red_full, (uint32_t)(nst * a.M * kTileCols * 4));
              for (int q = 0; q < nst; ++q)
                bulk_g2s(stage + q * SLOT, a.ws + (size_t)(blockIdx.x + 1 + q) * 2 * SLOT, (uint32_t)(a.M * kTileCols * 4),
                         red_full, policy_evict_first());
              TPQ_CTA(6, gtime())
            }
            mbar_wait(red_full, 0u);
            for (int q = 0; q < nst; ++q)
  #pragma unroll
              for (int m = 0; m < NP; ++m)
                if (m < a.M) acc[m] += stage[q * SLOT + m * kTileCols + col];
            for (int q = nst; q < nother; ++q) add_partial(a.ws + (size_t)(blockIdx.x + 1 + q) * 2 * SLOT + col, a.M, acc);
          }
  #pragma unroll
          for (int m = 0; m < NP; ++m)
            if (m < a.M) a.out[m * a.out_ld + n] = __float2half_rn(acc[m]);
          if (lane == 0) *cnt_last = 0;
          if (lane == 0) { TPQ_CTA(12 + qw, gtime()) }  // this warp's reduced tile stored
        } else if (seg_start == tile_start && seg_end == tile_end) {
  #pragma unroll
          for (int m = 0; m < NP; ++m)
            if (m < a.M) a.out[m * a.out_ld + n] = __float2half_rn(__uint_as_float(v[m]));
        } else {
          // (cnt == NULL) split tile: partial into this CTA's slot (0 = its first segment, 1 = its
          // last), summed by the fix-up kernel in CTA order after this kernel
          float* mine = a.ws + ((size_t)blockIdx.x * 2 + (seg_start == u0 ? 0 : 1)) * SLOT;
  #pragma unroll
          for (int m = 0; m < NP; ++m)
            if (m < a.M) __stcg(mine + m * kTileCols + col, __uint_as_float(v[m]));
        }
        seg_start = seg_end;
      }
    }
  } else if (warp == kProdWarp) {
    // ===================== TMA producer =====================
    const uint64_t pw = policy_evict_first();
    const int pre = nu < C::NS ? nu : C::NS;
    for (int i = 0; i < pre; ++i) {
      if (elect_one()) {
        mbar_arrive_expect_tx(full + i, C::UB);
        bulk_g2s(smem + C::WRING + i * C::STAGE, a.packed + (u0 + i) * C::UB, C::UB, full + i, pw);
      }
      __syncwarp();
    }
    // small shards: the next layer's weights into L2 behind this CTA's own ring fill
    if (a.pf && lane == 0) prefetch_l2_part(a.pf, a.pf_bytes, (int)blockIdx.x, (int)gridDim.x);
    for (int i = 0, s = 0, ph = 0; i + C::NS < nu; ++i) {
      TPQ_EV(0, i)
      mbar_wait_sleep(empty + s, (uint32_t)ph);
      TPQ_EV(1, i)
      if (elect_one()) {
        mbar_arrive_expect_tx(full + s, C::UB);
        bulk_g2s(smem + C::WRING + s * C::STAGE, a.packed + (u0 + i + C::NS) * C::UB, C::UB, full + s, pw);
      }
      __syncwarp();
      if (++s == C::NS) {
        s = 0;
        ph ^= 1;
      }
    }
    // full layers: the first units of the next layer's CTA of the same index into L2 once this CTA's
    // own records are all requested, so that CTA's ring fill (it becomes resident when a CTA of this
    // layer exits) hits L2 instead of waiting ~1.5 us on HBM
    if (a.pf_next && lane == 0)
      for (int c = (int)blockIdx.x; c < a.pf_grid; c += (int)gridDim.x) {
        const int64_t s0 = a.pf_cs > 1 ? (int64_t)(c / a.pf_cs) * a.pf_nkb + (c % a.pf_cs) * a.pf_nkb / a.pf_cs
                                       : (int64_t)c * a.pf_U / a.pf_grid;
        prefetch_l2_part(a.pf_next + s0 * C::UB, (int64_t)a.pf_units * C::UB, 0, 1);
      }
  } else if (warp == kStageWarp) {
    // ===================== activation stager =====================
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
    pdl_wait();
    if (lane == 0) { TPQ_CTA(1, gtime()) }
    if constexpr (GT) {
      // pair p = (tile, k-block) v0 + p: the gate record's slice from X[:, P1g] (xmap), the up
      // record's from X[:, P1u] (xmapu), both at k-block kb
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmapu)) : "memory");
      int kb = (int)(v0 % a.NKB);
      for (int p = 0; p < np; ++p) {
        const int x = p % C::NX;
        if (p >= C::NX) mbar_wait_sleep(done + (p - C::NX) % C::RD, (uint32_t)(((p - C::NX) / C::RD) & 1));
        if (elect_one()) {
          mbar_arrive_expect_tx(xfull + x, 2 * C::XU);
          tma_load_3d(smem + C::XRING + 2 * x * C::XU, &xmap, 0, 0, 2 * kb, xfull + x);
          tma_load_3d(smem + C::XRING + (2 * x + 1) * C::XU, &xmapu, 0, 0, 2 * kb, xfull + x);
        }
        __syncwarp();
        kb = kb + 1 == a.NKB ? 0 : kb + 1;
      }
    } else {
      int kb = (int)(u0 % a.NKB);
      for (int p = 0; p < np; ++p) {
        const int x = p % C::NX, nh = (2 * p + 1 < nu) ? 2 : 1;
        const int kb1 = kb + 1 == a.NKB ? 0 : kb + 1;
        if (p >= C::NX) mbar_wait_sleep(done + (p - C::NX) % C::RD, (uint32_t)(((p - C::NX) / C::RD) & 1));
        if (elect_one()) {
          mbar_arrive_expect_tx(xfull + x, nh * C::XU);
          tma_load_3d(smem + C::XRING + 2 * x * C::XU, &xmap, 0, 0, 2 * kb, xfull + x);
          if (nh == 2) tma_load_3d(smem + C::XRING + (2 * x + 1) * C::XU, &xmap, 0, 0, 2 * kb1, xfull + x);
        }
        __syncwarp();
        kb = nh == 2 ? (kb1 + 1 == a.NKB ? 0 : kb1 + 1) : kb1;
      }
    }
  } else {
    // ===================== MMA issuers: warp kMmaWarp + w takes the pairs p % 2 == w ===============
    const int w = warp - kMmaWarp;
    const uint32_t xring = smem_u32(smem + C::XRING);
    const int kb0 = (int)(u0 % a.NKB);
    const int nseg = (kb0 + nu - 1) / a.NKB + 1;
    int sw = 0;
    auto skip_seg = [&]() {
      mbar_wait(d_empty + (sw & 1), (uint32_t)(((sw >> 1) & 1) ^ 1));
      if (lane == 0) mbar_arrive(d_full + (sw & 1));
      __syncwarp();
      ++sw;
    };
    static_assert(C::AU == 64, "umma_unit16 A offsets");
    if constexpr (GT) {
      // one pair = one (tile, k-block): gate record -> gate accumulator, up record -> up accumulator
      const int kbv = (int)(v0 % a.NKB);
      const int nsegv = nv > 0 ? (kbv + nv - 1) / a.NKB + 1 : 0;
      // k-block and segment of pair p tracked incrementally (no division per pair: the segment
      // boundaries must not slow the issue)
      int kbq = kbv + w, sg = 0;
      while (kbq >= a.NKB) {
        kbq -= a.NKB;
        ++sg;
      }
      for (int p = w; p < np; p += 2) {
        while (sw < sg) skip_seg();
        const bool first = kbq < 2 || p < 2;                  // this issuer's previous pair, p - 2, is outside the segment
        const bool last = kbq + 2 > a.NKB - 1 || p + 2 > nv - 1;  // so is its next, p + 2
        const int x = p % C::NX, b = p % kSets, d = sg & 1;
        const uint64_t bd0 = bdesc_sw128(xring + 2 * x * C::XU);
        const uint32_t at = tmem + kA0 + b * 2 * C::AU;
        mbar_wait_backoff(a_full + p % C::NAF, (uint32_t)((p / C::NAF) & 1), 0);
        tc_fence_after();
        if (first) {
          mbar_wait(d_empty + d, (uint32_t)(((sg >> 1) & 1) ^ 1));
          tc_fence_after();
        }
        const uint32_t dg = tmem + (4 * d + 2 * w) * NP;  // gate; up at + NP
        if (elect_one()) {
          umma_unit16<C::HB>(dg, at, bd0, C::IDESC, first ? 0u : 1u);
          umma_unit16<C::HB>(dg + NP, at + C::AU, bd0 + (C::XU >> 4), C::IDESC, first ? 0u : 1u);
          if (last) umma_commit1(d_full + d);
          umma_commit1(done + p % C::RD);
        }
        __syncwarp();
        if (last) ++sw;
        for (kbq += 2; kbq >= a.NKB; kbq -= a.NKB) ++sg;
      }
      while (sw < nsegv) skip_seg();
    } else {
    // k-block (kbp) and segment (sgp) of unit 2p tracked incrementally: a division per unit in
    // the segment-boundary path cost ~0.3 us per unit of issue there, which stalled the pipeline
    // ~1 us at every boundary (tools/trace_pair.py)
    int kbp = kb0 + 2 * w, sgp = 0;
    while (kbp >= a.NKB) {
      kbp -= a.NKB;
      ++sgp;
    }
    for (int p = w; p < np; p += 2) {
      const int x = p % C::NX, b = p % kSets;
      const uint64_t bd0 = bdesc_sw128(xring + 2 * x * C::XU);
      const int i0 = 2 * p;
      while (sw < sgp) skip_seg();  // before the a_full wait: a segment's d_full never waits for the next pair's dequant
      // units i0 - 3 .. i0 + 4 (this issuer's previous and next) all inside the segment
      const bool fast = sgp == sw && kbp >= 3 && kbp + 4 <= a.NKB - 1 && i0 >= 3 && i0 + 4 <= nu - 1;
      const uint32_t at = tmem + kA0 + b * 2 * C::AU;
      TPQ_EV(0, p)
      mbar_wait_backoff(a_full + p % C::NAF, (uint32_t)((p / C::NAF) & 1), 0);
      TPQ_EV(1, p)
      tc_fence_after();
      if (fast) {
        const uint32_t dt = tmem + (2 * (sgp & 1) + w) * NP;
        if (elect_one()) {
          umma_unit16<C::HB>(dt, at, bd0, C::IDESC, 1u);
          umma_unit16<C::HB>(dt, at + C::AU, bd0 + (C::XU >> 4), C::IDESC, 1u);
          umma_commit1(done + p % C::RD);
        }
        __syncwarp();
        TPQ_EV(3, p)
      } else {
        // a pair at a segment boundary (or the CTA's first / last pairs): per-unit accumulate and
        // commit flags, both units still under one elected issue.  This issuer's units around the
        // pair are i0 - 3, (i0, i0 + 1), i0 + 4, so unit 0 is first if i0 - 3 is outside its segment
        // and last if i0 + 1 is; unit 1 is first if i0 is outside its segment and last if i0 + 4 is.
        // A unit 1 in the next segment makes unit 0 last, so no segment is skipped between them.
        while (sw < sgp) skip_seg();
        const bool has1 = i0 + 1 < nu;
        int kb1 = kbp + 1, sg1 = sgp;
        if (kb1 >= a.NKB) {
          kb1 -= a.NKB;
          ++sg1;
        }
        const bool f0 = kbp < 3 || i0 < 3, l0 = kbp + 1 > a.NKB - 1 || i0 + 1 > nu - 1;
        const bool f1 = has1 && kb1 < 1, l1 = has1 && (kb1 + 3 > a.NKB - 1 || i0 + 4 > nu - 1);
        const int d0 = sgp & 1, d1 = sg1 & 1;
        if (f0) {
          mbar_wait(d_empty + d0, (uint32_t)(((sgp >> 1) & 1) ^ 1));
          tc_fence_after();
        }
        if (f1) {
          mbar_wait(d_empty + d1, (uint32_t)(((sg1 >> 1) & 1) ^ 1));
          tc_fence_after();
        }
        if (elect_one()) {
          umma_unit16<C::HB>(tmem + (2 * d0 + w) * NP, at, bd0, C::IDESC, f0 ? 0u : 1u);
          if (l0) umma_commit1(d_full + d0);
          if (has1) {
            umma_unit16<C::HB>(tmem + (2 * d1 + w) * NP, at + C::AU, bd0 + (C::XU >> 4), C::IDESC, f1 ? 0u : 1u);
            if (l1) umma_commit1(d_full + d1);
          }
          umma_commit1(done + p % C::RD);
        }
        __syncwarp();
        sw += (int)l0 + (int)l1;
        TPQ_EV(3, p)
      }
      for (kbp += 4; kbp >= a.NKB; kbp -= a.NKB) ++sgp;
    }
    while (sw < nseg) skip_seg();
    if (lane == 0) { TPQ_CTA(11, gtime()) }  // (both issuers write; the later one stays)
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    TPQ_CTA(2, gtime())
    TPQ_CTA(9, clock64())
  }
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TCOLS) : "memory");
  }
}

// ------------------------------------------------------------------ A7: tensor-core path, M > 16
// k_dqgemm<G, NB>: the same product for NB (64 / 128 / 256) activation rows per launch, where the
// tensor pipe, not HBM, is the limit.  Same weight records and stream-K split
// as the GEMV; differences:
//   * the fp16 scale is folded into the A operand, A = fp16(s (q - z)) (one rounding of the exact
//     (q - z) times s), so a tile segment accumulates entirely in one TMEM accumulator of NB
//     columns and the epilogue runs once per segment instead of once per unit;
//   * N = NB per tcgen05.mma (M = 128, K = 16); the activation slice of a unit is NB rows x 128 k,
//     one 3-D tensor TMA (box 64 k x NB rows x 2, 128B swizzle);
//   * hand-offs per unit (a unit carries 8 MMAs of N = NB: the tensor pipe, not the barriers,
//     paces it);
//   * a tile split between CTAs leaves fp32 partials (NB x 128 per segment) for k_mm_fixup, a
//     separate fully parallel kernel that sums them in CTA order (deterministic): one last-arriving
//     CTA summing up to NB x 128 x 6 values with 128 threads took longer than the GEMM itself.
// Warps: 0-7 dequant (lane quarter w%4, k-half w/4), 8-11 epilogue, 12 producer, 13 stager,
// 14 MMA issuer.
constexpr int kMmWarps = 15;
template <int G, int NB>
struct TM {
  static constexpr int KG = kUnitK / G, GPH = G >= kUnitK / 2 ? 1 : (kUnitK / 2) / G;
  static constexpr int UB = (int)unit_bytes_c(G), STAGE = (UB + 127) / 128 * 128;
  static constexpr int XU = NB * kUnitK * 2;  // activation slice bytes per unit
  static constexpr int NX = 2;                // activation slots
  static constexpr int NS = NB == 256 ? 8 : 12;
  static constexpr int NA = 2, AU = kUnitK / 2;  // A buffers (units), columns per unit
  static constexpr int RD = 2;                   // unit-done ring (>= NA, NX; single in-order issuer)
  static_assert(NB + NA * AU <= 512, "TMEM budget");
  static constexpr int XRING = 0, WRING = NX * XU, BARS = WRING + NS * STAGE;
  static constexpr int SMEM = BARS + 8 * (2 * NS + NX + NA + RD + 2);
  static constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(NB >> 3) << 17) | ((uint32_t)(kTileCols >> 4) << 24);
};

struct GemmArgs {
  const uint8_t* packed;
  int M;            // rows of this launch (<= NB)
  int NT, NKB;
  int64_t U;
  int grid;
  __half* out;      // [M][out_ld]
  int64_t out_ld;
  float* ws;        // [grid][2][NB][128]
  const float* colf;  // [N] 2^(24 - E_n) (records hold s' = s 2^E_n); the operand is fp16(s' 2^-12 (q - z))
};

template <int G, int NB>
__global__ void __launch_bounds__(kMmWarps * 32, 1) k_dqgemm(const GemmArgs a, const __grid_constant__ CUtensorMap xmap) {
  using C = TM<G, NB>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BARS);
  uint64_t* full = bars;              // [NS] weight record landed
  uint64_t* empty = full + C::NS;     // [NS] dequant warps hold their codes (8)
  uint64_t* xfull = empty + C::NS;    // [NX] activation slice landed
  uint64_t* a_full = xfull + C::NX;   // [NA] A operand stored (8)
  uint64_t* done = a_full + C::NA;    // [RD] unit's MMAs completed (frees A buffer and activation slot)
  uint64_t* d_full = done + C::RD;    // segment accumulator final
  uint64_t* d_empty = d_full + 1;     // epilogue read it (4)
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t u0 = cta_start(blockIdx.x, a.U, a.grid);
  const int nu = (int)(cta_start(blockIdx.x + 1, a.U, a.grid) - u0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 8);
    }
    for (int s = 0; s < C::NX; ++s) mbar_init(xfull + s, 1);
    for (int b = 0; b < C::NA; ++b) mbar_init(a_full + b, 8);
    for (int r = 0; r < C::RD; ++r) mbar_init(done + r, 1);
    mbar_init(d_full, 1);
    mbar_init(d_empty, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 14) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_launch_dependents();
  const uint32_t tmem = __shfl_sync(0xffffffffu, s_tmem, 0);
  constexpr uint32_t kA0 = NB;  // TMEM: accumulator columns [0, NB), A buffer b at NB + b * AU

  if (warp < 8) {
    // ===================== dequant: A = fp16(s (q - z)) -> TMEM =====================
    const int qw = warp & 3, kh = warp >> 2, col = qw * 32 + lane;
    const uint32_t lane_base = (uint32_t)(qw * 32) << 16;
    const __half2 k16 = __float2half2_rn(0.0625f);
    for (int i = 0; i < nu; ++i) {
      const int s = i % C::NS, b = i % C::NA;
      mbar_wait(full + s, (uint32_t)((i / C::NS) & 1));
      const uint8_t* st = smem + C::WRING + s * C::STAGE;
      const uint4 c0 = *reinterpret_cast<const uint4*>(st + code_block(kh * 2 + 0, col) * 16);
      const uint4 c1 = *reinterpret_cast<const uint4*>(st + code_block(kh * 2 + 1, col) * 16);
      const uint32_t wv[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
      __half2 zl[C::GPH], zh[C::GPH], sc[C::GPH];
#pragma unroll
      for (int j = 0; j < C::GPH; ++j) {
        const int gi = (kh * (kUnitK / 2)) / G + j;
        const uint8_t* meta = st + kUnitK * kTileCols / 2;
        const int z = (meta[C::KG * 256 + gi * 64 + (col >> 1)] >> (4 * (col & 1))) & 0xF;
        const __half sv = *reinterpret_cast<const __half*>(meta + gi * 256 + 2 * col);
        zl[j] = __float2half2_rn((float)(1024 + z));
        zh[j] = __float2half2_rn((float)(-64 - z));
        sc[j] = __float2half2_rn(__half2float(sv) * 2.44140625e-4f);  // s' 2^-12 (exact: power of two)
      }
      {
        uint32_t dep = c0.x ^ c0.w ^ c1.x ^ c1.w;
#pragma unroll
        for (int j = 0; j < C::GPH; ++j) dep ^= h2u(zl[j]) ^ h2u(sc[j]);
        release_loaded(empty + s, dep, lane, a.ws, a.M);
      }
      uint32_t r[32];
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const int j = C::GPH == 1 ? 0 : (w * 8) / G;
        const uint32_t x = wv[w], x8 = x >> 8;
        r[4 * w + 0] = h2u(__hmul2(__hsub2(u2h(lop3_and_or(x, 0x000F000Fu, 0x64006400u)), zl[j]), sc[j]));
        r[4 * w + 1] = h2u(__hmul2(__hfma2(u2h(lop3_and_or(x, 0x00F000F0u, 0x64006400u)), k16, zh[j]), sc[j]));
        r[4 * w + 2] = h2u(__hmul2(__hsub2(u2h(lop3_and_or(x8, 0x000F000Fu, 0x64006400u)), zl[j]), sc[j]));
        r[4 * w + 3] = h2u(__hmul2(__hfma2(u2h(lop3_and_or(x8, 0x00F000F0u, 0x64006400u)), k16, zh[j]), sc[j]));
      }
      if (i >= C::NA) mbar_wait(done + (i - C::NA) % C::RD, (uint32_t)(((i - C::NA) / C::RD) & 1));  // A free
      tc_fence_after();
      tmem_st32(tmem + lane_base + kA0 + b * C::AU + kh * 32, r);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(a_full + b);
    }
  } else if (warp < 12) {
    // ===================== epilogue: once per tile segment =====================
    const int qw = warp - 8, col = qw * 32 + lane;
    const uint32_t lane_base = (uint32_t)(qw * 32) << 16;
    pdl_wait();
    int64_t seg_start = u0;
    int kb = (int)(u0 % a.NKB), tile = (int)(u0 / a.NKB), seg = 0;
    for (int i = 0; i < nu; ++i) {
      if (kb == a.NKB - 1 || i == nu - 1) {  // unit i closes a segment
        const int64_t n = (int64_t)tile * kTileCols + col;
        const bool full_tile = seg_start == (int64_t)tile * a.NKB && kb == a.NKB - 1;
        mbar_wait(d_full, (uint32_t)(seg & 1));
        tc_fence_after();
        const int slot = (seg_start == u0) ? 0 : 1;
        float* mine = a.ws + ((size_t)blockIdx.x * 2 + slot) * ((size_t)NB * kTileCols);
        const float up = __ldg(a.colf + n) * 2.44140625e-4f;  // 2^(12 - E): undo s' 2^-12 (exact)
        for (int m0 = 0; m0 < a.M; m0 += 16) {  // 16 rows per tcgen05.ld
          uint32_t v[16];
          tmem_ld16(tmem + lane_base + m0, v);
          tmem_wait_ld();
#pragma unroll
          for (int m = 0; m < 16; ++m) {
            if (m0 + m >= a.M) break;
            const float y = up * __uint_as_float(v[m]);
            if (full_tile) a.out[(int64_t)(m0 + m) * a.out_ld + n] = __float2half_rn(y);
            else __stcg(mine + (size_t)(m0 + m) * kTileCols + col, y);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(d_empty);
        ++seg;
        seg_start = u0 + i + 1;
      }
      if (++kb == a.NKB) {
        kb = 0;
        ++tile;
      }
    }
  } else if (warp == 12) {
    // ===================== weight producer =====================
    const uint64_t pw = policy_evict_first();
    for (int i = 0; i < nu; ++i) {
      const int s = i % C::NS;
      if (i >= C::NS) mbar_wait(empty + s, (uint32_t)(((i / C::NS) & 1) ^ 1));
      if (elect_one()) {
        mbar_arrive_expect_tx(full + s, C::UB);
        bulk_g2s(smem + C::WRING + s * C::STAGE, a.packed + (u0 + i) * C::UB, C::UB, full + s, pw);
      }
      __syncwarp();
    }
  } else if (warp == 13) {
    // ===================== activation stager (one 3-D tensor TMA per unit) =====================
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
    pdl_wait();
    int kb = (int)(u0 % a.NKB);
    for (int i = 0; i < nu; ++i) {
      const int x = i % C::NX;
      if (i >= C::NX) mbar_wait(done + (i - C::NX) % C::RD, (uint32_t)(((i - C::NX) / C::RD) & 1));
      if (elect_one()) {
        mbar_arrive_expect_tx(xfull + x, C::XU);
        tma_load_3d(smem + C::XRING + x * C::XU, &xmap, 0, 0, 2 * kb, xfull + x);
      }
      __syncwarp();
      if (++kb == a.NKB) kb = 0;
    }
  } else {
    // ===================== MMA issuer =====================
    const uint32_t xring = smem_u32(smem + C::XRING);
    int kb = (int)(u0 % a.NKB), seg = 0;
    for (int i = 0; i < nu; ++i) {
      const bool first = i == 0 || kb == 0, last = i == nu - 1 || kb == a.NKB - 1;
      const int b = i % C::NA, x = i % C::NX;
      if (first) mbar_wait(d_empty, (uint32_t)((seg & 1) ^ 1));
      mbar_wait(a_full + b, (uint32_t)((i / C::NA) & 1));
      mbar_wait(xfull + x, (uint32_t)((i / C::NX) & 1));
      tc_fence_after();
      const uint64_t bd0 = bdesc_sw128(xring + x * C::XU);
      const uint32_t at = tmem + kA0 + b * C::AU;
      uint32_t aop[8];
      uint64_t bop[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        aop[j] = at + j * 8;
        bop[j] = bd0 + (uint64_t)(((j / 4) * (C::XU / 2) + (j % 4) * 32) >> 4);
      }
      if (elect_one()) {
#pragma unroll
        for (int j = 0; j < 8; ++j) umma_ts1(tmem, aop[j], bop[j], C::IDESC, (first && j == 0) ? 0u : 1u);
        umma_commit1(done + i % C::RD);
        if (last) umma_commit1(d_full);
      }
      __syncwarp();
      if (last) ++seg;
      if (++kb == a.NKB) kb = 0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 14) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// ------------------------------------------------------------------ A7, large M: mixed-input SS GEMM
// k_dqgemm_ss<G, BN>: for M >= 128 the activations are the A operand (MMA M = 128 batch rows, TMA
// from L2, reused across BN weight columns) and the dequantized weights the B operand (N = BN
// columns = BN / 128 tiles), written by warps into shared memory as fp16 s (q - z) in the K-major
// SWIZZLE_128B layout (fence.proxy.async before the hand-off).  K in 128-row records (8 MMAs of
// K = 16 per k-step), fp32 accumulator in TMEM (double-buffered across work items).  BN = 256 halves
// the activation traffic per MMA (the activation TMA, not the tensor pipe, paces BN = 128).
// Work items (m-block, n-group, k-split) round-robin over one wave; with k-splits the fp32 partials
// are summed by k_ss_fixup in split order (deterministic).
// Warps: 0 .. 8 BN/128 - 1 dequant, then 4 epilogue (TMEM lane quarter = 32 batch rows), producer, MMA.
template <int G, int BN>
struct TS {
  static constexpr int TPW = BN / kTileCols;  // weight tiles per item
  static constexpr int DW = 8 * TPW;          // dequant warps (16 columns x 2 k-halves each)
  static constexpr int EPI0 = DW, PROD = DW + 4, MMAW = DW + 5, WARPS = DW + 6;
  static constexpr int KG = kUnitK / G, GPH = G >= kUnitK / 2 ? 1 : (kUnitK / 2) / G;
  static constexpr int UB = (int)unit_bytes_c(G), STAGE = (UB + 127) / 128 * 128;
  static constexpr int BM = 128;
  static constexpr int XT = BM * kUnitK * 2;  // A tile (activations) per k-step: 32 KB
  static constexpr int WT = BN * kUnitK * 2;  // B tile (dequantized weights) per k-step
  static constexpr int NW = TPW == 1 ? 4 : 2;  // raw-weight k-steps in flight (TPW records each)
  static constexpr int NA = TPW == 1 ? 3 : 2, NB = 2;  // A (activation) and B (weight) stages
  static constexpr int KR = 6;  // k-step done ring: A slot reuse waits t - NA, B slot t - NB; the next
                                // k-step on either barrier needs its own A / B first (KR >= NA + NB)
  static constexpr int AR = 0, BR = AR + NA * XT, WR = BR + NB * WT;  // A, B 1024-aligned
  static constexpr int BARS = WR + NW * TPW * STAGE;
  static constexpr int SMEM = BARS + 8 * (2 * NW + NA + NB + KR + 4);
  static constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  static_assert(KR >= NA + NB, "done ring");
};

struct SsArgs {
  const uint8_t* packed;
  int M;              // rows of this pass (<= 512)
  int MB, NG, NKB, S; // m-blocks, column groups of BN, k-blocks, k-splits
  int items;          // NG * MB * S: item = (ng * MB + mb) * S + ks
  int grid;
  __half* out;        // [M][out_ld]
  int64_t out_ld;
  float* ws;          // [items][128][BN] k-split partials (S > 1)
  const float* colf;  // [N] 2^(24 - E_n) (records hold s' = s 2^E_n); the operand is fp16(s' 2^-12 (q - z))
};

template <int G, int BN>
__global__ void __launch_bounds__(TS<G, BN>::WARPS * 32, 1) k_dqgemm_ss(const SsArgs a, const __grid_constant__ CUtensorMap xmap) {
  using C = TS<G, BN>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BARS);
  uint64_t* w_full = bars;              // [NW] the k-step's raw weight records landed
  uint64_t* w_empty = w_full + C::NW;   // [NW] dequant warps read them (DW)
  uint64_t* a_full = w_empty + C::NW;   // [NA] activation tile landed
  uint64_t* b_full = a_full + C::NA;    // [NB] dequantized weight tile written (DW)
  uint64_t* k_done = b_full + C::NB;    // [KR] MMAs of k-step t completed: frees its A and B slot
  uint64_t* d_full = k_done + C::KR;    // [2] item's accumulator final
  uint64_t* d_empty = d_full + 2;       // [2] epilogue read it (4)
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NW; ++s) {
      mbar_init(w_full + s, 1);
      mbar_init(w_empty + s, C::DW);
    }
    for (int s = 0; s < C::NA; ++s) mbar_init(a_full + s, 1);
    for (int s = 0; s < C::NB; ++s) mbar_init(b_full + s, C::DW);
    for (int s = 0; s < C::KR; ++s) mbar_init(k_done + s, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(d_full + s, 1);
      mbar_init(d_empty + s, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == C::MMAW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "n"(2 * BN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_launch_dependents();
  const uint32_t tmem = __shfl_sync(0xffffffffu, s_tmem, 0);
  auto krange = [&](int ks, int& k0, int& k1) {  // k-block range of split ks
    k0 = (int)((int64_t)ks * a.NKB / a.S);
    k1 = (int)((int64_t)(ks + 1) * a.NKB / a.S);
  };

  if (warp < C::DW) {
    // ===================== dequant: records -> fp16 s (q - z) B tile (SW128) =====================
    const int jj = warp * 16 + (lane & 15), kh = lane >> 4;  // B row (column of the item), k-half
    const int h = jj / kTileCols, j = jj % kTileCols;          // weight tile of the item, its column
    const __half2 k16 = __float2half2_rn(0.0625f);
    int t = 0;  // k-step counter of this CTA
    for (int it = blockIdx.x; it < a.items; it += a.grid) {
      int k0, k1;
      krange(it % a.S, k0, k1);
      for (int kb = k0; kb < k1; ++kb, ++t) {
        const int ws = t % C::NW, ks = t % C::NB;
        mbar_wait(w_full + ws, (uint32_t)((t / C::NW) & 1));
        const uint8_t* st = smem + C::WR + (ws * C::TPW + h) * C::STAGE;
        const uint4 c0 = *reinterpret_cast<const uint4*>(st + code_block(kh * 2 + 0, j) * 16);
        const uint4 c1 = *reinterpret_cast<const uint4*>(st + code_block(kh * 2 + 1, j) * 16);
        const uint32_t wv[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
        __half2 zl[C::GPH], zh[C::GPH], sc[C::GPH];
#pragma unroll
        for (int g = 0; g < C::GPH; ++g) {
          const int gi = (kh * (kUnitK / 2)) / G + g;
          const uint8_t* meta = st + kUnitK * kTileCols / 2;
          const int z = (meta[C::KG * 256 + gi * 64 + (j >> 1)] >> (4 * (j & 1))) & 0xF;
          const __half sv = *reinterpret_cast<const __half*>(meta + gi * 256 + 2 * j);
          zl[g] = __float2half2_rn((float)(1024 + z));
          zh[g] = __float2half2_rn((float)(-64 - z));
          sc[g] = __float2half2_rn(__half2float(sv) * 2.44140625e-4f);  // s' 2^-12
        }
        {
          uint32_t dep = c0.x ^ c0.w ^ c1.x ^ c1.w;
#pragma unroll
          for (int g = 0; g < C::GPH; ++g) dep ^= h2u(zl[g]) ^ h2u(sc[g]);
          release_loaded(w_empty + ws, dep, lane, a.ws, a.M);
        }
        if (t >= C::NB) mbar_wait(k_done + (t - C::NB) % C::KR, (uint32_t)(((t - C::NB) / C::KR) & 1));  // B slot free
        uint8_t* brow = smem + C::BR + ks * C::WT + kh * (BN * 128) + jj * 128;
#pragma unroll
        for (int w = 0; w < 8; ++w) {  // word w = k 64 kh + 8w .. +7 = 16-byte chunk w of the row
          const int g = C::GPH == 1 ? 0 : (w * 8) / G;
          const uint32_t x = wv[w], x8 = x >> 8;
          uint4 o;
          o.x = h2u(__hmul2(__hsub2(u2h(lop3_and_or(x, 0x000F000Fu, 0x64006400u)), zl[g]), sc[g]));
          o.y = h2u(__hmul2(__hfma2(u2h(lop3_and_or(x, 0x00F000F0u, 0x64006400u)), k16, zh[g]), sc[g]));
          o.z = h2u(__hmul2(__hsub2(u2h(lop3_and_or(x8, 0x000F000Fu, 0x64006400u)), zl[g]), sc[g]));
          o.w = h2u(__hmul2(__hfma2(u2h(lop3_and_or(x8, 0x00F000F0u, 0x64006400u)), k16, zh[g]), sc[g]));
          *reinterpret_cast<uint4*>(brow + ((w ^ (jj & 7)) << 4)) = o;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
        __syncwarp();
        if (lane == 0) mbar_arrive(b_full + ks);
      }
    }
  } else if (warp < C::PROD) {
    // ===================== epilogue: one item at a time =====================
    const int qw = warp - C::EPI0;
    pdl_wait();
    int n_it = 0;
    for (int it = blockIdx.x; it < a.items; it += a.grid, ++n_it) {
      const int db = n_it & 1, mb = (it / a.S) % a.MB, ng = it / (a.S * a.MB);
      float cfv[BN / 32];  // column factors 2^(12 - E_n), lane = column within each 32: loaded under the MMAs
#pragma unroll
      for (int i = 0; i < BN / 32; ++i) cfv[i] = __ldg(a.colf + (int64_t)ng * BN + 32 * i + lane) * 2.44140625e-4f;
      mbar_wait(d_full + db, (uint32_t)((n_it >> 1) & 1));
      tc_fence_after();
      const int m = mb * C::BM + qw * 32 + lane;  // batch row of this thread (TMEM lane)
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t v[32];
        tmem_ld16(tmem + ((uint32_t)(qw * 32) << 16) + db * BN + c0, v);
        tmem_ld16(tmem + ((uint32_t)(qw * 32) << 16) + db * BN + c0 + 16, v + 16);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 32; ++q)
          v[q] = __float_as_uint(__uint_as_float(v[q]) * __shfl_sync(0xffffffffu, cfv[c0 / 32], q));
        if (m < a.M) {
          if (a.S == 1) {
            __half* o = a.out + (int64_t)m * a.out_ld + (int64_t)ng * BN + c0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint4 pk;
              uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
              for (int e = 0; e < 4; ++e)
                pw[e] = h2u(__floats2half2_rn(__uint_as_float(v[8 * q + 2 * e]), __uint_as_float(v[8 * q + 2 * e + 1])));
              *reinterpret_cast<uint4*>(o + 8 * q) = pk;
            }
          } else {
            float* o = a.ws + ((size_t)it * C::BM + (m - mb * C::BM)) * BN + c0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              __stcg(reinterpret_cast<float4*>(o + 4 * q),
                     make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                                 __uint_as_float(v[4 * q + 3])));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(d_empty + db);
    }
  } else if (warp == C::PROD) {
    // ===================== producer: weight records (bulk) + activation tiles (tensor TMA) =====
    const uint64_t pw = policy_evict_first();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
    pdl_wait();  // the activations come from the previous kernel in the stream
    int t = 0;
    for (int it = blockIdx.x; it < a.items; it += a.grid) {
      const int mb = (it / a.S) % a.MB, ng = it / (a.S * a.MB);
      int k0, k1;
      krange(it % a.S, k0, k1);
      for (int kb = k0; kb < k1; ++kb, ++t) {
        const int ws = t % C::NW, sa = t % C::NA;
        if (t >= C::NW) mbar_wait(w_empty + ws, (uint32_t)(((t - C::NW) / C::NW) & 1));
        if (elect_one()) {
          mbar_arrive_expect_tx(w_full + ws, C::TPW * C::UB);
          for (int h = 0; h < C::TPW; ++h)
            bulk_g2s(smem + C::WR + (ws * C::TPW + h) * C::STAGE,
                     a.packed + ((int64_t)(ng * C::TPW + h) * a.NKB + kb) * C::UB, C::UB, w_full + ws, pw);
        }
        __syncwarp();
        if (t >= C::NA) mbar_wait(k_done + (t - C::NA) % C::KR, (uint32_t)(((t - C::NA) / C::KR) & 1));  // A slot free
        if (elect_one()) {
          mbar_arrive_expect_tx(a_full + sa, C::XT);
          tma_load_3d(smem + C::AR + sa * C::XT, &xmap, 0, mb * C::BM, 2 * kb, a_full + sa);
        }
        __syncwarp();
      }
    }
  } else {
    // ===================== MMA issuer =====================
    int t = 0, n_it = 0;
    for (int it = blockIdx.x; it < a.items; it += a.grid, ++n_it) {
      const int db = n_it & 1;
      int k0, k1;
      krange(it % a.S, k0, k1);
      mbar_wait(d_empty + db, (uint32_t)(((n_it >> 1) & 1) ^ 1));
      for (int kb = k0; kb < k1; ++kb, ++t) {
        const int sa = t % C::NA, sb = t % C::NB;
        mbar_wait(a_full + sa, (uint32_t)((t / C::NA) & 1));
        mbar_wait(b_full + sb, (uint32_t)((t / C::NB) & 1));
        tc_fence_after();
        const uint32_t abase = smem_u32(smem + C::AR + sa * C::XT), bbase = smem_u32(smem + C::BR + sb * C::WT);
        uint64_t ad[8], bd[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {  // k16 block q: k-half q / 4, 32-byte step within the 128-byte row
          ad[q] = bdesc_sw128(abase + (q / 4) * (C::BM * 128) + (q % 4) * 32);
          bd[q] = bdesc_sw128(bbase + (q / 4) * (BN * 128) + (q % 4) * 32);
        }
        if (elect_one()) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + db * BN),
                "l"(ad[q]), "l"(bd[q]), "r"(C::IDESC), "r"((kb == k0 && q == 0) ? 0u : 1u)
                : "memory");
          umma_commit1(k_done + t % C::KR);
          if (kb == k1 - 1) umma_commit1(d_full + db);
        }
        __syncwarp();
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == C::MMAW) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * BN) : "memory");
  }
}

// ------------------------------------------------------------------ A7, CTA pair: k_dqgemm_ss2<G>
// The SS GEMM of k_dqgemm_ss as a CTA pair (cta_group::2, cluster of 2 on one TPC): MMA M = 256 batch
// rows (CTA r supplies rows [128 r, +128) of the activation tile), N = 256 weight columns (CTA r
// dequantizes weight tile 2 ng + r = pair columns [128 r, +128)), and CTA r's TMEM receives D rows
// [128 r, +128) x all 256 columns (layout verified by tools/probe_2cta.cu).  Per CTA and 128-row
// k-step the shared memory moves 32 KB of activations (TMA), 32 KB of dequantized weights, 8.5 KB
// of records and 64 KB of operand reads for 2 x the work of a 1-CTA 128 x 128 k-step.
// Hand-offs: both CTAs' activation TMAs complete on the LEADER's a_full (cta_group::2 TMA, 64 KB
// expected); each CTA's dequant warps arrive on the leader's b_full (remote arrive); the leader's MMA
// warp issues and commits to both CTAs' k_done / d_full (multicast); each epilogue arrives on the
// leader's d_empty.  Weight records and activations have their own producer warps, so the weight
// ring runs ahead of the MMA by the HBM latency, not by the activation ring.
// k-split partials leave through shared memory: each epilogue warp stages its 32 rows x 32 columns
// (4 KB, 16-byte chunks XOR-swizzled by row: conflict-free) and one lane bulk-copies them to a
// contiguous 4 KB of the partial buffer [grp][ks][c / 32][128 rows][32] (same swizzle; k_ss_fixup
// swz = 1).  Per-lane row stores (16 B to 32 rows per instruction) took 9 us per item (trace).
template <int G>
struct TS2 {
  static constexpr int DW = 8, EPI0 = 8, EW = 8, WPROD = EPI0 + EW, APROD = WPROD + 1, MMAW = APROD + 1, WARPS = MMAW + 1;
  static constexpr int KG = kUnitK / G, GPH = G >= kUnitK / 2 ? 1 : (kUnitK / 2) / G;
  static constexpr int UB = (int)unit_bytes_c(G), STAGE = (UB + 127) / 128 * 128;
  static constexpr int BM = 128, BN = 128;        // per CTA: activation rows, weight columns
  static constexpr int XT = BM * kUnitK * 2;      // A tile per k-step: 32 KB
  static constexpr int WT = BN * kUnitK * 2;      // B half per k-step: 32 KB
  static constexpr int NW = 3, NA = 3, NB = 2, KR = 6;
  static constexpr int EST = 32 * 128;            // epilogue staging per warp: 32 rows x 32 fp32
  static constexpr int AR = 0, BR = AR + NA * XT, WR = BR + NB * WT, ER = WR + NW * STAGE;
  static constexpr int CF = ER + EW * EST;        // per epilogue warp: its item's 128 column factors
  static constexpr int BARS = CF + EW * 512;
  static constexpr int SMEM = BARS + 8 * (2 * NW + NA + NB + KR + 6);
  // pair MMA: D f32, A/B f16 K-major, N = 256, M = 256
  static constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  static_assert(KR >= NA + NB, "done ring");
};

// Arrive on an mbarrier of a CTA of the cluster with the default (.release.cta) semantics: the data
// it publishes is in shared memory read by the pair's tensor cores (after fence.proxy.async) or is
// TMEM read back by tcgen05.ld (ordered by tcgen05.fence), not generic loads of another CTA, and
// .release.cluster costs a MEMBAR.ALL.GPU + ERRBAR per arrive (ncu: the pair's top stall).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// arrive on the barrier in both CTAs of the pair (mask = the pair's two cluster ranks)
__device__ __forceinline__ void umma_commit2(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// 16-byte store into another CTA's shared memory, completion (bytes) counted on that CTA's barrier
__device__ __forceinline__ void st_async16(uint32_t dst, uint4 v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(dst),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(bar)
               : "memory");
}
// TMA tile into this CTA's shared memory, completion (bytes) signalled on the pair leader's barrier
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 uint32_t leader_bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(leader_bar)
      : "memory");
}
// X2 = true: clusters of 4 CTAs = the two k-splits (S = 2, one item per pair) of one 256 x 256 tile.
// Instead of fp32 partials and k_ss_fixup, the two pairs exchange halves through distributed shared
// memory once their MMAs are done: split ks finalises columns [128 ks, +128) = its own accumulator
// + the other split's (64 KB per CTA by st.async into the receiver's free activation ring), written
// as fp16.  p0 + p1 is the fix-up's sum (commutative, one rounding), so the results are identical.
template <int G, bool X2>
__global__ void __launch_bounds__(TS2<G>::WARPS * 32, 1) k_dqgemm_ss2(const SsArgs a, const __grid_constant__ CUtensorMap xmap) {
  using C = TS2<G>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BARS);
  uint64_t* w_full = bars;              // [NW] raw weight record landed
  uint64_t* w_empty = w_full + C::NW;   // [NW] dequant warps read it (DW)
  uint64_t* a_full = w_empty + C::NW;   // [NA] leader: both CTAs' activation tiles landed (2 XT bytes)
  uint64_t* b_full = a_full + C::NA;    // [NB] leader: both CTAs' dequantized weight halves written (2 DW)
  uint64_t* k_done = b_full + C::NB;    // [KR] k-step t's MMAs completed (multicast commit)
  uint64_t* d_full = k_done + C::KR;    // [2] item's accumulator final (multicast commit)
  uint64_t* d_empty = d_full + 2;       // [2] leader: both epilogues read it (2 x EW)
  uint64_t* x_free = d_empty + 2;       // X2: the other split's operands are done (remote arrive)
  uint64_t* x_full = x_free + 1;        // X2: the other split's half of this CTA's rows landed (64 KB)
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank(), rank = crank & 1u, lead = crank & ~1u;  // rank within the pair, its leader
  const uint16_t pmask = (uint16_t)(3u << lead);
  const int pair = blockIdx.x >> 1, npairs = a.grid >> 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NW; ++s) {
      mbar_init(w_full + s, 1);
      mbar_init(w_empty + s, C::DW);
    }
    for (int s = 0; s < C::NA; ++s) mbar_init(a_full + s, 1);
    for (int s = 0; s < C::NB; ++s) mbar_init(b_full + s, 2 * C::DW);
    for (int s = 0; s < C::KR; ++s) mbar_init(k_done + s, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(d_full + s, 1);
      mbar_init(d_empty + s, 2 * C::EW);
    }
    mbar_init(x_free, 1);
    mbar_init(x_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == C::MMAW) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in every CTA before any remote arrive
  tc_fence_after();
  pdl_launch_dependents();
  const uint32_t tmem = __shfl_sync(0xffffffffu, s_tmem, 0);
  auto krange = [&](int ks, int& k0, int& k1) {
    k0 = (int)((int64_t)ks * a.NKB / a.S);
    k1 = (int)((int64_t)(ks + 1) * a.NKB / a.S);
  };
  // pair item it = (ng * MB + mb) * S + ks: MB counts 256-row blocks, ng 256-column groups

  if (warp < C::DW) {
    // ===================== dequant: this CTA's weight tile 2 ng + rank -> B half (SW128) ==========
    const int jj = warp * 16 + (lane & 15), kh = lane >> 4, j = jj;
    const __half2 k16 = __float2half2_rn(0.0625f);
    const uint32_t bfull_leader = mapa_shared(b_full, lead);
    int t = 0;
    for (int it = pair; it < a.items; it += npairs) {
      int k0, k1;
      krange(it % a.S, k0, k1);
      for (int kb = k0; kb < k1; ++kb, ++t) {
        const int ws = t % C::NW, ks = t % C::NB;
        if (warp == 0) { TPQ_EV2(rank, 0, t) }
        mbar_wait(w_full + ws, (uint32_t)((t / C::NW) & 1));
        if (warp == 0) { TPQ_EV2(rank, 1, t) }
        const uint8_t* st = smem + C::WR + ws * C::STAGE;
        const uint4 c0 = *reinterpret_cast<const uint4*>(st + code_block(kh * 2 + 0, j) * 16);
        const uint4 c1 = *reinterpret_cast<const uint4*>(st + code_block(kh * 2 + 1, j) * 16);
        const uint32_t wv[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
        __half2 zl[C::GPH], zh[C::GPH], sc[C::GPH];
#pragma unroll
        for (int g = 0; g < C::GPH; ++g) {
          const int gi = (kh * (kUnitK / 2)) / G + g;
          const uint8_t* meta = st + kUnitK * kTileCols / 2;
          const int z = (meta[C::KG * 256 + gi * 64 + (j >> 1)] >> (4 * (j & 1))) & 0xF;
          const __half sv = *reinterpret_cast<const __half*>(meta + gi * 256 + 2 * j);
          zl[g] = __float2half2_rn((float)(1024 + z));
          zh[g] = __float2half2_rn((float)(-64 - z));
          sc[g] = __float2half2_rn(__half2float(sv) * 2.44140625e-4f);  // s' 2^-12
        }
        {
          uint32_t dep = c0.x ^ c0.w ^ c1.x ^ c1.w;
#pragma unroll
          for (int g = 0; g < C::GPH; ++g) dep ^= h2u(zl[g]) ^ h2u(sc[g]);
          release_loaded(w_empty + ws, dep, lane, a.ws, a.M);
        }
        // B slot free in BOTH CTAs: k-step t - NB's MMAs completed (multicast commit)
        if (t >= C::NB) mbar_wait(k_done + (t - C::NB) % C::KR, (uint32_t)(((t - C::NB) / C::KR) & 1));
        if (warp == 0) { TPQ_EV2(rank, 2, t) }
        uint8_t* brow = smem + C::BR + ks * C::WT + kh * (C::BN * 128) + jj * 128;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          const int g = C::GPH == 1 ? 0 : (w * 8) / G;
          const uint32_t x = wv[w], x8 = x >> 8;
          uint4 o;
          o.x = h2u(__hmul2(__hsub2(u2h(lop3_and_or(x, 0x000F000Fu, 0x64006400u)), zl[g]), sc[g]));
          o.y = h2u(__hmul2(__hfma2(u2h(lop3_and_or(x, 0x00F000F0u, 0x64006400u)), k16, zh[g]), sc[g]));
          o.z = h2u(__hmul2(__hsub2(u2h(lop3_and_or(x8, 0x000F000Fu, 0x64006400u)), zl[g]), sc[g]));
          o.w = h2u(__hmul2(__hfma2(u2h(lop3_and_or(x8, 0x00F000F0u, 0x64006400u)), k16, zh[g]), sc[g]));
          *reinterpret_cast<uint4*>(brow + ((w ^ (jj & 7)) << 4)) = o;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor cores
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(bfull_leader + ks * 8);
        if (warp == 0) { TPQ_EV2(rank, 3, t) }
      }
    }
  } else if (warp < C::WPROD) {
    // ===================== epilogue: this CTA's 128 rows x 256 columns of the item =================
    // 8 warps: TMEM lane quarter qw (32 batch rows) x column half hc (4 chunks of 32 columns).  Each
    // chunk is staged in this warp's 4 KB of shared memory: fp32 partials (S > 1) leave by one 4 KB
    // bulk copy, fp16 results (S = 1) by row-contiguous 64-byte stores (8 rows per instruction).
    const int ew = warp - C::EPI0, qw = ew & 3, hc = ew >> 2;
    const uint32_t dempty_leader = mapa_shared(d_empty, lead);
    uint8_t* stg = smem + C::ER + ew * C::EST;
    float* cfs = reinterpret_cast<float*>(smem + C::CF + ew * 512);
    pdl_wait();
    if constexpr (X2) {
      // ---- split exchange: one item per pair, it = pair, ks = pq ----
      const int pq = (int)(crank >> 1), it = pair, mb = (it / 2) % a.MB, ng = it / (2 * a.MB);
      const uint32_t partner = crank ^ 2u;  // same rows, other split
      const int ml = qw * 32 + lane;
      mbar_wait(d_full, 0);
      tc_fence_after();
      if (hc != pq) {
        // send this warp's 32 rows x 128 columns (the partner finalises them), fp32 unscaled
        mbar_wait(x_free, 0);
        const uint32_t dst = mapa_shared(smem + C::AR, partner) + ml * 512, bar = mapa_shared(x_full, partner);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t v[32];
          tmem_ld16(tmem + ((uint32_t)(qw * 32) << 16) + 128 * hc + 32 * i, v);
          tmem_ld16(tmem + ((uint32_t)(qw * 32) << 16) + 128 * hc + 32 * i + 16, v + 16);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 8; ++q)  // 16-byte chunk 8 i + q of the row, swizzled by row
            st_async16(dst + ((((8 * i + q) ^ (ml & 7))) << 4), make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]),
                       bar);
        }
      } else {
        float cfv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) cfv[i] = __ldg(a.colf + (int64_t)ng * 256 + 128 * hc + 32 * i + lane) * 2.44140625e-4f;
#pragma unroll
        for (int i = 0; i < 4; ++i) cfs[32 * i + lane] = cfv[i];
        if (ew == 4 * pq && lane == 0) {  // this CTA's operands are free: the partner may write its half here
          mbar_arrive_expect_tx(x_full, 4 * 32 * 4 * 8 * 16);
          mbar_arrive_cluster(mapa_shared(x_free, partner));
        }
        __syncwarp();
        mbar_wait(x_full, 0);
        const uint8_t* inc = smem + C::AR + ml * 512;
        const int mrow0 = mb * 256 + (int)rank * 128 + qw * 32;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int c0 = 128 * hc + 32 * i;
          uint32_t v[32];
          tmem_ld16(tmem + ((uint32_t)(qw * 32) << 16) + c0, v);
          tmem_ld16(tmem + ((uint32_t)(qw * 32) << 16) + c0 + 16, v + 16);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 f = *reinterpret_cast<const float4*>(cfs + 32 * i + 4 * q);
            const float4 o = *reinterpret_cast<const float4*>(inc + ((((8 * i + q) ^ (ml & 7))) << 4));
            v[4 * q] = __float_as_uint(__uint_as_float(v[4 * q]) * f.x + o.x * f.x);
            v[4 * q + 1] = __float_as_uint(__uint_as_float(v[4 * q + 1]) * f.y + o.y * f.y);
            v[4 * q + 2] = __float_as_uint(__uint_as_float(v[4 * q + 2]) * f.z + o.z * f.z);
            v[4 * q + 3] = __float_as_uint(__uint_as_float(v[4 * q + 3]) * f.w + o.w * f.w);
          }
          __syncwarp();
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 pk;
            uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
            for (int e = 0; e < 4; ++e)
              pw[e] = h2u(__floats2half2_rn(__uint_as_float(v[8 * q + 2 * e]), __uint_as_float(v[8 * q + 2 * e + 1])));
            *reinterpret_cast<uint4*>(stg + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4)) = pk;
          }
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int r = 8 * j + (lane >> 2), q = lane & 3, m = mrow0 + r;
            const uint4 pk = *reinterpret_cast<const uint4*>(stg + r * 64 + ((q ^ ((r >> 1) & 3)) << 4));
            if (m < a.M) *reinterpret_cast<uint4*>(a.out + (int64_t)m * a.out_ld + (int64_t)ng * 256 + c0 + 8 * q) = pk;
          }
        }
      }
      tc_fence_before();
    } else {
    int n_it = 0;
    for (int it = pair; it < a.items; it += npairs, ++n_it) {
      const int db = n_it & 1, mb = (it / a.S) % a.MB, ng = it / (a.S * a.MB);
      // column factors 2^(12 - E_n) of this warp's 128 columns, staged under the MMAs (read back as
      // broadcast float4: shuffles serialised on the 96-register budget)
      float cfv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) cfv[i] = __ldg(a.colf + (int64_t)ng * 256 + 128 * hc + 32 * i + lane) * 2.44140625e-4f;
      __syncwarp();  // previous item's factors read
#pragma unroll
      for (int i = 0; i < 4; ++i) cfs[32 * i + lane] = cfv[i];
      __syncwarp();
      mbar_wait(d_full + db, (uint32_t)((n_it >> 1) & 1));
      if (ew == 0) { TPQ_EV2(6 + rank, 0, n_it) }
      tc_fence_after();
      const int mrow0 = mb * 256 + (int)rank * 128 + qw * 32;  // batch row of lane 0 (TMEM lane qw 32)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int c0 = 128 * hc + 32 * i;
        uint32_t v[32];
        tmem_ld16(tmem + ((uint32_t)(qw * 32) << 16) + db * 256 + c0, v);
        tmem_ld16(tmem + ((uint32_t)(qw * 32) << 16) + db * 256 + c0 + 16, v + 16);
        tmem_wait_ld();
        if (ew == 0) { TPQ_EV2(9 + rank, 0, i + 8 * n_it) }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 f = *reinterpret_cast<const float4*>(cfs + 32 * i + 4 * q);
          v[4 * q] = __float_as_uint(__uint_as_float(v[4 * q]) * f.x);
          v[4 * q + 1] = __float_as_uint(__uint_as_float(v[4 * q + 1]) * f.y);
          v[4 * q + 2] = __float_as_uint(__uint_as_float(v[4 * q + 2]) * f.z);
          v[4 * q + 3] = __float_as_uint(__uint_as_float(v[4 * q + 3]) * f.w);
        }
        if (ew == 0) { TPQ_EV2(9 + rank, 1, i + 8 * n_it) }
        if (a.S == 1) {
          // fp16 [32 rows][32 cols] = 64 B per row, 16-byte chunks swizzled by (row >> 1) & 3
          __syncwarp();  // previous chunk's rows read back
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 pk;
            uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
            for (int e = 0; e < 4; ++e)
              pw[e] = h2u(__floats2half2_rn(__uint_as_float(v[8 * q + 2 * e]), __uint_as_float(v[8 * q + 2 * e + 1])));
            *reinterpret_cast<uint4*>(stg + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4)) = pk;
          }
          __syncwarp();
          if (ew == 0) { TPQ_EV2(9 + rank, 2, i + 8 * n_it) }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int r = 8 * j + (lane >> 2), q = lane & 3, m = mrow0 + r;
            const uint4 pk = *reinterpret_cast<const uint4*>(stg + r * 64 + ((q ^ ((r >> 1) & 3)) << 4));
            if (m < a.M) *reinterpret_cast<uint4*>(a.out + (int64_t)m * a.out_ld + (int64_t)ng * 256 + c0 + 8 * q) = pk;
          }
        } else {
          // partial block of group 2 (ng MB + mb) + rank, split ks, column chunk c0 / 32: this warp's 4 KB
          const int grp = ng * (2 * a.MB) + 2 * mb + (int)rank;
          float* o = a.ws + ((((size_t)grp * a.S + it % a.S) * 8 + c0 / 32) * 128 + qw * 32) * 32;
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // previous chunk read out
          __syncwarp();
          if (ew == 0) { TPQ_EV2(9 + rank, 2, i + 8 * n_it) }
#pragma unroll
          for (int q = 0; q < 8; ++q)
            *reinterpret_cast<uint4*>(stg + lane * 128 + ((q ^ (lane & 7)) << 4)) =
                make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(o), "r"(smem_u32(stg)),
                         "n"(C::EST)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
        if (ew == 0) { TPQ_EV2(9 + rank, 3, i + 8 * n_it) }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(dempty_leader + db * 8);
      if (ew == 0) { TPQ_EV2(6 + rank, 1, n_it) }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // partials written before exit
    }
  } else if (warp == C::WPROD) {
    // ===================== weight producer: this CTA's records, NW k-steps ahead ====================
    const uint64_t pw = policy_evict_first();
    int t = 0;
    for (int it = pair; it < a.items; it += npairs) {
      const int ng = it / (a.S * a.MB);
      int k0, k1;
      krange(it % a.S, k0, k1);
      for (int kb = k0; kb < k1; ++kb, ++t) {
        const int ws = t % C::NW;
        TPQ_EV2(4 + rank, 0, t)
        if (t >= C::NW) mbar_wait(w_empty + ws, (uint32_t)(((t / C::NW) & 1) ^ 1));
        TPQ_EV2(4 + rank, 1, t)
        if (elect_one()) {
          mbar_arrive_expect_tx(w_full + ws, C::UB);
          bulk_g2s(smem + C::WR + ws * C::STAGE, a.packed + ((int64_t)(ng * 2 + (int)rank) * a.NKB + kb) * C::UB, C::UB,
                   w_full + ws, pw);
        }
        __syncwarp();
      }
    }
  } else if (warp == C::APROD) {
    // ===================== activation producer: this CTA's 128 rows, onto the leader's a_full =======
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
    const uint32_t afull_leader = mapa_shared(a_full, lead);
    pdl_wait();  // activations come from the previous kernel in the stream
    int t = 0;
    for (int it = pair; it < a.items; it += npairs) {
      const int mb = (it / a.S) % a.MB;
      int k0, k1;
      krange(it % a.S, k0, k1);
      for (int kb = k0; kb < k1; ++kb, ++t) {
        const int sa = t % C::NA;
        TPQ_EV2(2 + rank, 0, t)
        if (t >= C::NA) mbar_wait(k_done + (t - C::NA) % C::KR, (uint32_t)(((t - C::NA) / C::KR) & 1));  // A slot free
        TPQ_EV2(2 + rank, 1, t)
        if (elect_one()) {
          if (rank == 0) mbar_arrive_expect_tx(a_full + sa, 2 * C::XT);
          tma_load_3d_pair(smem + C::AR + sa * C::XT, &xmap, 0, mb * 256 + (int)rank * C::BM, 2 * kb,
                           afull_leader + sa * 8);
        }
        __syncwarp();
      }
    }
  } else if (rank == 0) {
    // ===================== MMA issuer (leader) =====================
    int t = 0, n_it = 0;
    for (int it = pair; it < a.items; it += npairs, ++n_it) {
      const int db = n_it & 1;
      int k0, k1;
      krange(it % a.S, k0, k1);
      mbar_wait(d_empty + db, (uint32_t)(((n_it >> 1) & 1) ^ 1));
      for (int kb = k0; kb < k1; ++kb, ++t) {
        const int sa = t % C::NA, sb = t % C::NB;
        TPQ_EV2(8, 0, t)
        mbar_wait(a_full + sa, (uint32_t)((t / C::NA) & 1));
        TPQ_EV2(8, 1, t)
        mbar_wait(b_full + sb, (uint32_t)((t / C::NB) & 1));
        TPQ_EV2(8, 2, t)
        tc_fence_after();
        const uint32_t abase = smem_u32(smem + C::AR + sa * C::XT), bbase = smem_u32(smem + C::BR + sb * C::WT);
        uint64_t ad[8], bd[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {  // k16 block q: k-half q / 4, 32-byte step within the 128-byte row
          ad[q] = bdesc_sw128(abase + (q / 4) * (C::BM * 128) + (q % 4) * 32);
          bd[q] = bdesc_sw128(bbase + (q / 4) * (C::BN * 128) + (q % 4) * 32);
        }
        if (elect_one()) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + db * 256),
                "l"(ad[q]), "l"(bd[q]), "r"(C::IDESC), "r"((kb == k0 && q == 0) ? 0u : 1u)
                : "memory");
          umma_commit2(k_done + t % C::KR, pmask);
          if (kb == k1 - 1) umma_commit2(d_full + db, pmask);
        }
        __syncwarp();
        TPQ_EV2(8, 3, t)
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();  // every CTA of the cluster done with the pair's TMEM, its barriers and shared memory
  if (warp == C::MMAW) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// k-split fix-up of k_dqgemm_ss: out[m][ng BN + c] = sum over ks of the item's partial (split order).
// Block (ng * MB + mb, r): rows mb 128 + 4 r + warp, thread = 4 consecutive columns, bn / 128 passes.
// swz = 1 (k_dqgemm_ss2): partials in [grp][ks][c / 32][128 rows][32], 16-byte chunks XOR-swizzled by row.
__global__ void k_ss_fixup(const float* __restrict__ ws, int M, int MB, int S, int bn, __half* __restrict__ out,
                           int64_t out_ld, int swz) {
  pdl_launch_dependents();
  pdl_wait();
  const int grp = blockIdx.x, mb = grp % MB, ng = grp / MB;
  const int ml = blockIdx.y * 4 + (threadIdx.x >> 5), m = mb * 128 + ml;
  if (m >= M) return;
  for (int c = (threadIdx.x & 31) * 4; c < bn; c += 128) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const size_t off = swz ? ((size_t)(c >> 5) * 128 + ml) * 32 + ((((c & 31) >> 2) ^ (ml & 7)) << 2) : (size_t)ml * bn + c;
    for (int ks = 0; ks < S; ++ks) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(ws + ((size_t)grp * S + ks) * 128 * bn + off));
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    uint2 pk;
    pk.x = h2u(__floats2half2_rn(acc.x, acc.y));
    pk.y = h2u(__floats2half2_rn(acc.z, acc.w));
    *reinterpret_cast<uint2*>(out + (int64_t)m * out_ld + (int64_t)ng * bn + c) = pk;
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

// launch_pdl for a kernel run as clusters of `cx` CTAs along x
template <class Kern, class... Args>
cudaError_t launch_pdl_cluster(Kern k, int cx, dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = (unsigned)cx;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

// ------------------------------------------------------------------ gathers
__device__ __forceinline__ int64_t gather_src(int m, int64_t k, int64_t ld, const int32_t* idx, int mode,
                                              int64_t nn, int M) {
  if (mode == GATHER_COLS) return (int64_t)m * ld + (idx ? (int64_t)idx[k] : k);
  const int64_t c = idx[k];
  return (c / nn) * (int64_t)M * nn + (int64_t)m * nn + (c % nn);
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

// A7 stream-K fix-up: tile t split between CTAs c_first..c_last (same partition as k_dqgemm):
// out[m][t*128 + j] = sum over c of the partial of CTA c (its slot for tile t), in CTA order.
// Block (t, mb): rows 4 mb + warp, thread j: columns 4 lane .. +3 (float4 loads, 8-byte stores).
__global__ void k_mm_fixup(const float* __restrict__ ws, int nb, int M, int NKB, int64_t U, int grid,
                           __half* __restrict__ out, int64_t out_ld, int gated) {
  pdl_launch_dependents();
  pdl_wait();  // the partials come from the GEMM just before
  const int t = blockIdx.x;
  const int c_first = cta_of_unit((int64_t)t * NKB, U, grid), c_last = cta_of_unit((int64_t)(t + 1) * NKB - 1, U, grid);
  if (c_first == c_last) return;  // the tile lies inside one CTA's range: written by the GEMM
  const int m = blockIdx.y * 4 + (threadIdx.x >> 5), j = (threadIdx.x & 31) * 4;
  if (m >= M) return;
  // contributor c's slot: every CTA after c_first starts inside tile t (slot 0, its first segment);
  // c_first's slot is 0 only if its range starts exactly at the tile.  Gated (gate_proj layer 1):
  // each slot holds the gate partials then the up partials, and the output is SiLU(gate) * up.
  const int s_first = cta_start(c_first, U, grid) == (int64_t)t * NKB ? 0 : 1;
  const int kinds = gated ? 2 : 1;
  float4 acc[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
  for (int kind = 0; kind < kinds; ++kind) {
    // contributors in CTA order, eight loads in flight per batch (one L2 round trip per batch)
    for (int c0 = c_first; c0 <= c_last; c0 += 8) {
      float4 v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int c = c0 + q <= c_last ? c0 + q : c_last;
        const int slot = c > c_first ? 0 : s_first;
        v[q] = __ldcg(reinterpret_cast<const float4*>(ws + (((size_t)c * 2 + slot) * kinds * nb + kind * nb + m) * kTileCols + j));
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (c0 + q <= c_last) {
          acc[kind].x += v[q].x;
          acc[kind].y += v[q].y;
          acc[kind].z += v[q].z;
          acc[kind].w += v[q].w;
        }
    }
  }
  float4 y = acc[0];
  if (gated) {
    y.x = silu_f(acc[0].x) * acc[1].x;
    y.y = silu_f(acc[0].y) * acc[1].y;
    y.z = silu_f(acc[0].z) * acc[1].z;
    y.w = silu_f(acc[0].w) * acc[1].w;
  }
  const __half2 lo = __floats2half2_rn(y.x, y.y), hi = __floats2half2_rn(y.z, y.w);
  uint2 pk;
  pk.x = *reinterpret_cast<const uint32_t*>(&lo);
  pk.y = *reinterpret_cast<const uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(out + (int64_t)m * out_ld + (int64_t)t * kTileCols + j) = pk;
}

// Split-tile fix-up sized to sit beside a GEMV CTA (<= 32 registers x 128 threads, one block per split
// tile): block b sums split tile tiles[b]'s contributors in CTA order, one thread per column, 4 rows
// x 2 contributors in flight; gated: gate and up partials, then fp16(SiLU(gate) * up).
__global__ void __launch_bounds__(128, 16) k_split_fixup(const float* __restrict__ ws, const int* __restrict__ tiles, int M,
                                                         int NKB, int64_t U, int grid, __half* __restrict__ out,
                                                         int64_t out_ld, int gated) {
  pdl_launch_dependents();
  pdl_wait();  // the partials come from the GEMV just before
  const int t = __ldg(tiles + blockIdx.x), col = threadIdx.x;
  const int c_first = cta_of_unit((int64_t)t * NKB, U, grid), c_last = cta_of_unit((int64_t)(t + 1) * NKB - 1, U, grid);
  const int s_first = cta_start(c_first, U, grid) == (int64_t)t * NKB ? 0 : 1;
  const int kinds = gated ? 2 : 1;
  __half* o = out + (int64_t)t * kTileCols + col;
  for (int m0 = 0; m0 < M; m0 += 4) {
    float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    for (int kind = 0; kind < kinds; ++kind)
      for (int c = c_first; c <= c_last; c += 2) {
        float v[2][4];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int cc = c + q <= c_last ? c + q : c_last;
          const float* src = ws + (((size_t)cc * 2 + (cc > c_first ? 0 : s_first)) * kinds + kind) * (kNPad * kTileCols) + col;
#pragma unroll
          for (int i = 0; i < 4; ++i) v[q][i] = m0 + i < M ? __ldcg(src + (m0 + i) * kTileCols) : 0.f;
        }
#pragma unroll
        for (int q = 0; q < 2; ++q)
          if (c + q <= c_last)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[kind][i] += v[q][i];
      }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (m0 + i < M) o[(m0 + i) * out_ld] = __float2half_rn(gated ? silu_f(acc[0][i]) * acc[1][i] : acc[0][i]);
  }
}

// X[:, idx] for the layer-1 operand: CTA (m, part) reads row m into shared memory with coalesced
// 16-byte loads, then gathers part `part` of the k range from there (a direct gather reads a
// 32-byte sector per 2-byte element).  dst[m][k] = src[m ld + idx[k]].
// At most 32 registers x 128 threads (4096) and one block per SM: the block fits beside a GEMV CTA
// (96 x 640 registers), so the GEMV launched after it can become resident and stream weights at once.
// NT = 512 for passes of more than 16 rows (one block per row): each thread then has <= 2 chunks of
// a K = 8192 row.  The indices (P1 as uint16, constant) are fetched before griddepcontrol.wait, so
// after the producer of `src` completes only the row's bulk copy and the shared-memory gather remain.
template <int NT>
__global__ void __launch_bounds__(NT, NT == 128 ? 16 : 4) k_gather_rows(const __half* __restrict__ src, int ld,
                                                                      const uint16_t* __restrict__ idx, int K,
                                                                      __half* __restrict__ dst) {
  extern __shared__ __align__(16) uint8_t srow_raw[];
  __shared__ __align__(8) uint64_t row_full;
  __half* srow = reinterpret_cast<__half*>(srow_raw);
  constexpr int PER = NT == 128 ? 1 : 2;  // chunks of 8 indices (one uint4) per thread prefetched ahead of the wait
  if (threadIdx.x == 0) mbar_init(&row_full, 1);
  const int m = blockIdx.x;
  const int nc = K >> 3, c0 = nc * (int)blockIdx.y / (int)gridDim.y, c1 = nc * ((int)blockIdx.y + 1) / (int)gridDim.y;
  const uint4* idx8 = reinterpret_cast<const uint4*>(idx);
  uint4 ix[PER];
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const int c = c0 + (int)threadIdx.x + p * NT;
    if (c < c1) ix[p] = __ldg(idx8 + c);
  }
  pdl_launch_dependents();
  __syncthreads();  // row_full initialised
  pdl_wait();
  if (threadIdx.x == 0) {  // the whole row by one bulk copy: no registers, no per-thread latency chain
    mbar_arrive_expect_tx(&row_full, (uint32_t)K * 2);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(srow)),
                 "l"(src + (size_t)m * (unsigned)ld), "r"((uint32_t)K * 2), "r"(smem_u32(&row_full))
                 : "memory");
  }
  mbar_wait(&row_full, 0);
  uint4* out = reinterpret_cast<uint4*>(dst + (size_t)m * (unsigned)K);
  const uint16_t* sh = reinterpret_cast<const uint16_t*>(srow);
  auto pair = [&](uint32_t w) { return (uint32_t)sh[w & 0xFFFFu] | ((uint32_t)sh[w >> 16] << 16); };
  auto gather8 = [&](const uint4 i) { return make_uint4(pair(i.x), pair(i.y), pair(i.z), pair(i.w)); };
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const int c = c0 + (int)threadIdx.x + p * NT;
    if (c < c1) out[c] = gather8(ix[p]);
  }
  for (int c = c0 + (int)threadIdx.x + PER * NT; c < c1; c += NT)  // rows longer than PER chunks per thread
    out[c] = gather8(__ldg(idx8 + c));
}

// Naive Alg. 2 L3-4 for rank r: dst[m][i] = buf[slice(i)][m][off(i)], the AllGather
// buffer buf[tp][M][n] read through the precomputed (slice, offset) = (c / n, c % n), c = P2[r n + i]
// (reading c17).  One element per thread over many SMs: the element loads are scattered 2-byte
// sectors, bounded by per-SM sector throughput (an 8-column x 4-row per-thread version on few blocks
// was 1.6x slower) and by the row's spread over all tp slices (staging whole Y1_global rows in shared
// memory fetches tp x the needed bytes: slower at TP=8); the constant (slice, offset) is loaded
// before the grid dependency, so only the element load follows it.
__global__ void __launch_bounds__(256) k_gather_ag(const __half* __restrict__ buf, const int2* __restrict__ so, int n,
                                                  int M, __half* __restrict__ dst) {
  pdl_launch_dependents();
  const int i = blockIdx.x * 256 + (int)threadIdx.x, m = blockIdx.y;
  int2 t = make_int2(0, 0);
  if (i < n) t = __ldg(so + i);
  pdl_wait();
  if (i < n) dst[(int64_t)m * n + i] = buf[((int64_t)t.x * M + m) * n + t.y];
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
int cta_read(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_tpq_cta, sizeof(unsigned long long) * 2 * 1024 * 16) != cudaSuccess;
}
int trace_read(long long* out) {
  return cudaMemcpyFromSymbol(out, g_tpq_trace, sizeof(long long) * 2 * 24 * 64 * 4) != cudaSuccess;
}
#endif
bool make_xmap(CUtensorMap* map, const void* base, int64_t K, int rows, int box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !encode)
      return false;
  }
  // dims (64 k, rows, K/64 k-halves); box (64, rows, 2) = one unit's slice: k-half kq at kq * rows * 128
  const cuuint64_t dims[3] = {(cuuint64_t)(kUnitK / 2), (cuuint64_t)rows, (cuuint64_t)(K / (kUnitK / 2))};
  const cuuint64_t strides[2] = {(cuuint64_t)K * 2, (cuuint64_t)kUnitK};  // bytes: row, k-half
  const cuuint32_t box[3] = {(cuuint32_t)(kUnitK / 2), (cuuint32_t)(box_rows > 0 ? box_rows : rows), 2};
  const cuuint32_t es[3] = {1, 1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int G, int NB>
bool prepare_mm_t() {
  constexpr int smem = TM<G, NB>::SMEM;
  static_assert(smem <= 227 * 1024, "GEMM smem over the per-CTA limit");
  static_assert(2 * smem > 228 * 1024, "GEMM must be one CTA per SM (TMEM 512 columns)");
  return cudaFuncSetAttribute(k_dqgemm<G, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess;
}
template <int G, int BN>
bool prepare_ss_t() {
  static_assert(TS<G, BN>::SMEM + 1024 <= 227 * 1024, "SS GEMM smem (+ static) over the per-CTA limit");
  return cudaFuncSetAttribute(k_dqgemm_ss<G, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, TS<G, BN>::SMEM) ==
         cudaSuccess;
}
template <int G>
bool prepare_ss2_t() {
  static_assert(TS2<G>::SMEM + 1024 <= 227 * 1024, "SS pair GEMM smem (+ static) over the per-CTA limit");
  return cudaFuncSetAttribute(k_dqgemm_ss2<G, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, TS2<G>::SMEM) ==
             cudaSuccess &&
         cudaFuncSetAttribute(k_dqgemm_ss2<G, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TS2<G>::SMEM) ==
             cudaSuccess;
}
template <int G>
bool prepare_mm_g() {
  bool ok = prepare_mm_t<G, 64>() && prepare_mm_t<G, 128>() && prepare_mm_t<G, 256>() && prepare_ss_t<G, 128>() &&
            prepare_ss2_t<G>();
  if constexpr (G == 128) ok = ok && prepare_ss_t<G, 256>();
  return ok;
}

// Every kernel of the forward prefers the maximum shared-memory carveout: consecutive kernels with
// different L1/shared splits make the SM drain and reconfigure between them, which also defeats the
// programmatic-dependent-launch overlap (the GEMV / GEMM kernels need ~210 KB anyway).
template <class Kern>
bool max_carveout(Kern k) {
  return getenv("TPQ_NO_CARVEOUT") ||
         cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared) ==
             cudaSuccess;
}
template <int G>
bool carveout_g() {
  return max_carveout(k_dqgemv<G, false, kNPad>) && max_carveout(k_dqgemv<G, true, kNPad>) &&
         max_carveout(k_dqgemv<G, false, 2 * kNPad>) && max_carveout(k_dqgemm<G, 64>) && max_carveout(k_dqgemm<G, 128>) &&
         max_carveout(k_dqgemm<G, 256>) && max_carveout(k_dqgemm_ss<G, 128>) && max_carveout(k_dqgemm_ss2<G, false>) && max_carveout(k_dqgemm_ss2<G, true>);
}

template <int G, bool GT, int NP = kNPad>
bool prepare_gemv() {
  using C = TC<G, GT, NP>;
  static_assert(C::SMEM <= 227 * 1024 && 2 * C::SMEM > 228 * 1024, "GEMV: one CTA per SM (TMEM 512 columns)");
  static_assert(C::SMEM_CL <= 227 * 1024 - 1024, "GEMV: landing zone of the cluster split-K");
  if (cudaFuncSetAttribute(k_dqgemv<G, GT, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_CL) != cudaSuccess)
    return false;
  if (C::CSMAX > 1 &&
      cudaFuncSetAttribute(k_dqgemv<G, GT, NP>, cudaFuncAttributeNonPortableClusterSizeAllowed, 0) != cudaSuccess)
    return false;
  if (getenv("TPQ_VERBOSE")) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_dqgemv<G, GT, NP>);
    fprintf(stderr, "[tpq] k_dqgemv<%d,%d,%d>: regs %d, local %zu, smem dyn %d\n", G, (int)GT, NP, fa.numRegs,
            fa.localSizeBytes, C::SMEM);
  }
  return true;
}

bool gemv_prepare(int G) {
  if (!(max_carveout(k_gather_rm) && max_carveout(k_gather_rows<128>) && max_carveout(k_gather_rows<512>) && max_carveout(k_gather_ag) && max_carveout(k_split_fixup) && max_carveout(k_mm_fixup) &&
        max_carveout(k_ss_fixup) && max_carveout(k_sum_partials) && max_carveout(k_dqgemv<0, false, kNPad>)))
    return false;
  if (!prepare_gemv<0, false>()) return false;  // unordered-g_idx layers (any G)
  if (!(G == 128 ? carveout_g<128>() : G == 64 ? carveout_g<64>() : G == 32 ? carveout_g<32>() : false)) return false;
  if (G == 128)
    return prepare_gemv<128, false>() && prepare_gemv<128, true>() && prepare_gemv<128, false, 2 * kNPad>() &&
           prepare_mm_g<128>();
  if (G == 64)
    return prepare_gemv<64, false>() && prepare_gemv<64, true>() && prepare_gemv<64, false, 2 * kNPad>() && prepare_mm_g<64>();
  if (G == 32)
    return prepare_gemv<32, false>() && prepare_gemv<32, true>() && prepare_gemv<32, false, 2 * kNPad>() && prepare_mm_g<32>();
  return false;
}

template <int G, bool GT, int NP = kNPad>
cudaError_t launch_gemv_t(const GemvArgs& a, const CUtensorMap& xmap, const CUtensorMap& xmapu, cudaStream_t st) {
  if (a.csize > 1)
    return launch_pdl_cluster(k_dqgemv<G, GT, NP>, a.csize, dim3(a.grid), dim3(kGemvThreads), TC<G, GT, NP>::SMEM_CL, st, a,
                              xmap, xmapu);
  return launch_pdl(k_dqgemv<G, GT, NP>, dim3(a.grid), dim3(kGemvThreads), TC<G, GT, NP>::SMEM, st, a, xmap, xmapu);
}

int gemv_cluster_max(int G) {
  return G == 128 ? TC<128, false>::CSMAX : G == 64 ? TC<64, false>::CSMAX : G == 32 ? TC<32, false>::CSMAX : 1;
}
int gemv_cluster_max32(int G) {
  return G == 128 ? TC<128, false, 32>::CSMAX : G == 64 ? TC<64, false, 32>::CSMAX : G == 32 ? TC<32, false, 32>::CSMAX : 1;
}

cudaError_t launch_gemv(const LayerDev& L, const CUtensorMap& xmap, const CUtensorMap* xmapu, int M, void* out,
                        int64_t out_ld, cudaStream_t st, const void* pf, int64_t pf_bytes, const LayerDev* next) {
  // 17 <= M <= 32: the N = 32 pipeline (plain layers; xmap with 32-row boxes) in the layer's own partition
  // (stream-K with the in-kernel reduction, or clusters that fit the N = 32 landing zone)
  const bool n32 = M > kMaxM;
  if (M < 1 || M > 2 * kMaxM || (L.gated && !xmapu) || (n32 && (L.gated || L.unord))) return cudaErrorInvalidValue;
  GemvArgs a;
  a.packed = L.packed;
  a.M = M;
  a.NT = L.NT;
  a.NKB = L.NKB;
  a.U = L.U;  // gated: (tile, k-block) pairs of gate + up records
  a.grid = L.grid;
  a.out = reinterpret_cast<__half*>(out);
  a.out_ld = out_ld;
  a.ws = L.ws;
  a.colf = L.colf;
  a.meta = L.meta;
  a.ldm = L.N;
  a.csize = L.csize;
  if (n32 && L.csize > gemv_cluster_max32(L.G)) return cudaErrorInvalidValue;  // (run_layer sends these to A7)
  a.pf = (const uint8_t*)pf;
  a.pf_bytes = pf_bytes;
  // 0 / 6 / 12 units: Llama TP=1 M=1 51.7 / 50.5 / 50.5 us, M=16 53.4 / 52.1 / 52.2 (same box)
  static const int pf_units = getenv("TPQ_PF_NEXT") ? atoi(getenv("TPQ_PF_NEXT")) : 8;
  const bool pn = next && !pf && next->G == L.G && !next->gated && !next->unord && pf_units > 0;
  a.pf_next = pn ? next->packed : nullptr;
  a.pf_U = pn ? next->U : 0;
  a.pf_grid = pn ? next->grid : 0;
  a.pf_units = pf_units;
  a.pf_cs = pn ? next->csize : 1;
  a.pf_nkb = pn ? next->NKB : 0;
  a.cnt = (L.inred || n32) && a.csize == 1 ? L.cnt : nullptr;  // N = 32: never the fix-up kernel
  const CUtensorMap& xu = xmapu ? *xmapu : xmap;
  cudaError_t e = cudaErrorInvalidValue;
  if (L.unord) e = launch_gemv_t<0, false>(a, xmap, xu, st);
  else if (L.gated) e = L.G == 128 ? launch_gemv_t<128, true>(a, xmap, xu, st)
                      : L.G == 64 ? launch_gemv_t<64, true>(a, xmap, xu, st)
                      : L.G == 32 ? launch_gemv_t<32, true>(a, xmap, xu, st) : cudaErrorInvalidValue;
  else if (n32) e = L.G == 128 ? launch_gemv_t<128, false, 2 * kNPad>(a, xmap, xu, st)
                   : L.G == 64 ? launch_gemv_t<64, false, 2 * kNPad>(a, xmap, xu, st)
                   : L.G == 32 ? launch_gemv_t<32, false, 2 * kNPad>(a, xmap, xu, st) : cudaErrorInvalidValue;
  else e = L.G == 128 ? launch_gemv_t<128, false>(a, xmap, xu, st)
           : L.G == 64 ? launch_gemv_t<64, false>(a, xmap, xu, st)
           : L.G == 32 ? launch_gemv_t<32, false>(a, xmap, xu, st) : cudaErrorInvalidValue;
  if (e != cudaSuccess || a.cnt || a.csize > 1) return e;  // split tiles reduced inside the GEMV
  // (tiles spanning > 4 CTA ranges) split tiles summed in CTA order after the GEMV by a fix-up
  // kernel ordered by griddepcontrol.wait.  M <= 4: k_split_fixup, one <= 32-register block per split tile that sits beside the next GEMV's
  // CTA (same-box: Llama TP=1 M=1 59.3 -> 57.0 us); M > 4: k_mm_fixup (one warp per row, float4 per
  // lane, 8 contributors in flight), faster there than 32 registers allow.
  if (L.split_tiles && M <= 4) {
    if (L.nsplit == 0) return cudaSuccess;
    return launch_pdl(k_split_fixup, dim3((unsigned)L.nsplit), dim3(128), 0, st, (const float*)L.ws, L.split_tiles, M, L.NKB,
                      L.U, L.grid, reinterpret_cast<__half*>(out), out_ld, L.gated);
  }
  return launch_pdl(k_mm_fixup, dim3((unsigned)L.NT, (unsigned)((M + 3) / 4)), dim3(128), 0, st, (const float*)L.ws, kNPad,
                    M, L.NKB, L.U, L.grid, reinterpret_cast<__half*>(out), out_ld, L.gated);
}

template <int G>
cudaError_t launch_mm_g(int nb, const GemmArgs& a, const CUtensorMap& map, cudaStream_t st) {
  if (nb == 64) return launch_pdl(k_dqgemm<G, 64>, dim3(a.grid), dim3(kMmWarps * 32), TM<G, 64>::SMEM, st, a, map);
  if (nb == 128) return launch_pdl(k_dqgemm<G, 128>, dim3(a.grid), dim3(kMmWarps * 32), TM<G, 128>::SMEM, st, a, map);
  if (nb == 256) return launch_pdl(k_dqgemm<G, 256>, dim3(a.grid), dim3(kMmWarps * 32), TM<G, 256>::SMEM, st, a, map);
  return cudaErrorInvalidValue;
}

cudaError_t launch_gemm(const LayerDev& L, const CUtensorMap& xmap, int nb, int M, void* out, int64_t out_ld,
                        cudaStream_t st) {
  if (M < 1 || M > nb) return cudaErrorInvalidValue;
  GemmArgs a;
  a.packed = L.packed;
  a.M = M;
  a.NT = L.NT;
  a.NKB = L.NKB;
  a.U = L.U;
  a.grid = L.grid_mm;
  a.out = reinterpret_cast<__half*>(out);
  a.out_ld = out_ld;
  a.ws = L.ws_mm;
  a.colf = L.colf;
  cudaError_t e = L.G == 128 ? launch_mm_g<128>(nb, a, xmap, st)
                  : L.G == 64 ? launch_mm_g<64>(nb, a, xmap, st)
                  : L.G == 32 ? launch_mm_g<32>(nb, a, xmap, st)
                              : cudaErrorInvalidValue;
  if (e != cudaSuccess) return e;
  return launch_pdl(k_mm_fixup, dim3((unsigned)L.NT, (unsigned)((M + 3) / 4)), dim3(128), 0, st, (const float*)L.ws_mm,
                    nb, M, L.NKB, L.U, L.grid_mm, reinterpret_cast<__half*>(out), out_ld, 0);
}

template <int G, int BN>
cudaError_t launch_ss_t(const SsArgs& a, const CUtensorMap& xmap, cudaStream_t st) {
  return launch_pdl(k_dqgemm_ss<G, BN>, dim3(a.grid), dim3(TS<G, BN>::WARPS * 32), TS<G, BN>::SMEM, st, a, xmap);
}

// CTA-pair SS GEMM: pair items (256-column group, 256-row block, k-split); k-split partials in the
// k_ss_fixup swizzled layout with 128-row blocks (group = 2 (ng MB + mb) + rank) and bn = 256.
cudaError_t launch_gemm_ss2(const LayerDev& L, const CUtensorMap& xmap, int M, int sms, void* out, int64_t out_ld,
                            cudaStream_t st) {
  SsArgs a;
  a.packed = L.packed;
  a.M = M;
  a.MB = (M + 255) / 256;
  a.NG = L.NT / 2;
  a.NKB = L.NKB;
  const int S = L.ws_ss ? ss_splits(a.NG, L.NKB, a.MB, sms / 2) : 1;
  a.S = S;
  a.items = a.NG * a.MB * S;
  a.grid = 2 * std::min(a.items, sms / 2);
  a.out = reinterpret_cast<__half*>(out);
  a.out_ld = out_ld;
  a.ws = L.ws_ss;
  a.colf = L.colf;
  cudaError_t e = cudaErrorInvalidValue;
  const dim3 blk(TS2<128>::WARPS * 32);  // same warp layout for every G
  // two k-splits that fit one wave: clusters of 4 exchange halves in distributed shared memory
  static const bool no_x2 = getenv("TPQ_NO_X2") != nullptr;
  if (S == 2 && a.items <= sms / 2 && !no_x2) {
    a.grid = 2 * a.items;
    if (L.G == 128) return launch_pdl_cluster(k_dqgemm_ss2<128, true>, 4, dim3(a.grid), blk, TS2<128>::SMEM, st, a, xmap);
    if (L.G == 64) return launch_pdl_cluster(k_dqgemm_ss2<64, true>, 4, dim3(a.grid), blk, TS2<64>::SMEM, st, a, xmap);
    if (L.G == 32) return launch_pdl_cluster(k_dqgemm_ss2<32, true>, 4, dim3(a.grid), blk, TS2<32>::SMEM, st, a, xmap);
    return cudaErrorInvalidValue;
  }
  if (L.G == 128) e = launch_pdl_cluster(k_dqgemm_ss2<128, false>, 2, dim3(a.grid), blk, TS2<128>::SMEM, st, a, xmap);
  else if (L.G == 64) e = launch_pdl_cluster(k_dqgemm_ss2<64, false>, 2, dim3(a.grid), blk, TS2<64>::SMEM, st, a, xmap);
  else if (L.G == 32) e = launch_pdl_cluster(k_dqgemm_ss2<32, false>, 2, dim3(a.grid), blk, TS2<32>::SMEM, st, a, xmap);
  if (e != cudaSuccess || S == 1) return e;
  return launch_pdl(k_ss_fixup, dim3((unsigned)(2 * a.MB * a.NG), 32), dim3(128), 0, st, (const float*)L.ws_ss, M,
                    2 * a.MB, S, 256, reinterpret_cast<__half*>(out), out_ld, 1);
}

cudaError_t launch_gemm_ss(const LayerDev& L, const CUtensorMap& xmap, int M, int sms, void* out, int64_t out_ld,
                           cudaStream_t st) {
  if (M < 1 || M > 512) return cudaErrorInvalidValue;
  if (ss_pair(L.NT, M)) return launch_gemm_ss2(L, xmap, M, sms, out, out_ld, st);
  const int bn = ss_bn(L.NT, L.G);
  SsArgs a;
  a.packed = L.packed;
  a.M = M;
  a.MB = (M + 127) / 128;
  a.NG = L.NT * kTileCols / bn;
  a.NKB = L.NKB;
  const int base = a.MB * a.NG;
  const int S = L.ws_ss ? ss_splits(a.NG, L.NKB, a.MB, sms) : 1;
  a.S = S;
  a.items = base * S;
  a.grid = std::min(a.items, sms);
  a.out = reinterpret_cast<__half*>(out);
  a.out_ld = out_ld;
  a.ws = L.ws_ss;
  a.colf = L.colf;
  cudaError_t e = cudaErrorInvalidValue;
  if (bn == 256) {
    if (L.G == 128) e = launch_ss_t<128, 256>(a, xmap, st);
  } else {
    if (L.G == 128) e = launch_ss_t<128, 128>(a, xmap, st);
    else if (L.G == 64) e = launch_ss_t<64, 128>(a, xmap, st);
    else if (L.G == 32) e = launch_ss_t<32, 128>(a, xmap, st);
  }
  if (e != cudaSuccess || S == 1) return e;
  return launch_pdl(k_ss_fixup, dim3((unsigned)base, 32), dim3(128), 0, st, (const float*)L.ws_ss, M, a.MB, S, bn,
                    reinterpret_cast<__half*>(out), out_ld, 0);
}

cudaError_t launch_gather_rowmajor(const void* src, int64_t ld, const int32_t* idx, int mode, int64_t nn, int M,
                                   int64_t K, void* dst, cudaStream_t st) {
  // column gather of rows that fit in shared memory, 16-byte aligned rows: stage each row
  if (mode == GATHER_COLS && idx && K % 8 == 0 && K * 2 <= 48 * 1024 && ld % 8 == 0 && ld < (1ll << 31) &&
      reinterpret_cast<uintptr_t>(src) % 16 == 0 && reinterpret_cast<uintptr_t>(idx) % 16 == 0)
  {
    // up to 8 parts per row (each part's block copies the whole row): 4 / 8 / 16 / 32 / 148 parts
    // measured 51.2 / 50.9 / 51.1 / 51.1 / 51.3 us for Llama TP=1 M=1 (TP=8: 13.6 / 13.4 / 13.5 / 13.6 / 14.2)
    const dim3 grid((unsigned)M, (unsigned)std::max(1, std::min(8, 148 / M)));
    const uint16_t* idx16 = reinterpret_cast<const uint16_t*>(idx + K);
    if (M > kMaxM)
      return launch_pdl(k_gather_rows<512>, grid, dim3(512), (size_t)K * 2, st, reinterpret_cast<const __half*>(src),
                        (int)ld, idx16, (int)K, reinterpret_cast<__half*>(dst));
    return launch_pdl(k_gather_rows<128>, grid, dim3(128), (size_t)K * 2, st, reinterpret_cast<const __half*>(src),
                      (int)ld, idx16, (int)K, reinterpret_cast<__half*>(dst));
  }
  const int64_t total = (int64_t)M * K;
  return launch_pdl(k_gather_rm, dim3(grid_for(total, 256)), dim3(256), 0, st, reinterpret_cast<const __half*>(src),
                    ld, idx, mode, nn, M, K, reinterpret_cast<__half*>(dst));
}

cudaError_t launch_gather_allgather(const void* buf, const void* so, int n, int M, void* dst, cudaStream_t st) {
  return launch_pdl(k_gather_ag, dim3((unsigned)((n + 255) / 256), (unsigned)M), dim3(256), 0,
                    st, reinterpret_cast<const __half*>(buf), reinterpret_cast<const int2*>(so), n, M,
                    reinterpret_cast<__half*>(dst));
}

cudaError_t launch_sum_partials(const void* const* parts, int nparts, int64_t count, void* out, cudaStream_t st) {
  if (nparts < 1 || nparts > 8) return cudaErrorInvalidValue;
  PartsArg pa;
  for (int r = 0; r < 8; ++r) pa.p[r] = reinterpret_cast<const __half*>(parts[r < nparts ? r : 0]);
  return launch_pdl(k_sum_partials, dim3(grid_for(count, 256)), dim3(256), 0, st, pa, nparts, count,
                    reinterpret_cast<__half*>(out));
}

}  // namespace tpq
