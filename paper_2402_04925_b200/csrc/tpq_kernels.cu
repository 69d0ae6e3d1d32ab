// sm_100a kernels of the TP-aware GPTQ MLP hot path (arxiv 2402.04925).
//
//  k_gemv<S, MT>   layer GEMV for M <= 16: Y = Xf . deq(W), deq = s * (q - z)
//                  (PAPER.md:L19 per-group scales/zeros; ordered groups PAPER.md:L57 let the
//                  fp32 scale be applied once per group).  HBM-bound: the packed int4 shard is
//                  streamed exactly once by TMA bulk copies (cp.async.bulk, mbarrier
//                  complete_tx, L2 evict-first) into a per-warp shared-memory ring; dequant in
//                  registers (LOP3 magic numbers, exact (q - z) in fp16), warp-level tensor-core
//                  MMA (mma.sync m16n8k16, fp16 x fp16 -> fp32; swap-AB: 16 weight columns are the
//                  MMA M dimension, the batch is MMA N), persistent stream-K over
//                  (64-column block x group) units with a deterministic last-arriver fix-up.
//                  Programmatic dependent launch: the weight prefetch starts before
//                  griddepcontrol.wait, so it overlaps the previous kernel's tail.
//  k_to_frag       X[:, P1] gather (Alg. 3 L1) and the naive AllGather
//                  re-permute + CHUNK (Alg. 2 L3-4) into the MMA B-fragment
//                  layout.
//  k_gather_rm     the same gathers to row-major (staged API).
//  k_sum_partials  rank-order sum (single-GPU shard simulation only).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

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
__device__ __forceinline__ uint32_t hsub2_u(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("sub.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t hfma2_u(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
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
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }

// ------------------------------------------------------------------ GEMV
// OCC = resident CTAs per SM (register budget 255 / OCC=1, 128 / OCC=2); NS = TMA ring stages
// per warp, sized so OCC x 8 warps x NS units are in flight per SM.
template <int S, int MT>
struct Cfg {
  static constexpr int UNIT = 32 * 16 * S + kMetaBytes;        // bytes per (block, group) record
  static constexpr int OCC = MT == 1 ? 2 : 1;
  static constexpr int NS = (OCC == 2 ? 2 : 4) * (S == 8 ? 1 : (S == 4 ? 2 : 3)) / (S == 2 ? 1 : 1);
  static constexpr int CW = S >= 4 ? 4 : S;                     // u32 words per lane per chunk
  static constexpr int NC = S / CW;                             // chunks per tile
  static constexpr int RING = 8 * NS * UNIT;                    // ring bytes per CTA (8 warps)
};

template <int MT>
__host__ __device__ constexpr int red_bytes() { return 8 * MT * 8 * kBlockCols * 4; }
template <int S, int MT>
constexpr size_t gemv_smem() { return (size_t)Cfg<S, MT>::RING + red_bytes<MT>() + 8 * Cfg<S, MT>::NS * 8; }

template <int S, int MT>
struct Frag {
  uint32_t w[4][S];        // codes: tile t, k16 step s
  uint32_t sc[4];          // half2 (s[r0], s[r1]) per tile
  uint32_t zz;             // zero bytes per tile
};

template <int S, int MT>
__device__ __forceinline__ void read_unit(Frag<S, MT>& f, const uint8_t* unit, int lane) {
  using C = Cfg<S, MT>;
#pragma unroll
  for (int c = 0; c < C::NC; ++c)
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint8_t* p = unit + ((c * 4 + t) * 32 + lane) * C::CW * 4;
      if constexpr (C::CW == 4) {
        const uint4 v = *reinterpret_cast<const uint4*>(p);
        f.w[t][c * 4 + 0] = v.x;
        f.w[t][c * 4 + 1] = v.y;
        f.w[t][c * 4 + 2] = v.z;
        f.w[t][c * 4 + 3] = v.w;
      } else {
        const uint2 v = *reinterpret_cast<const uint2*>(p);
        f.w[t][c * 2 + 0] = v.x;
        f.w[t][c * 2 + 1] = v.y;
      }
    }
  const uint8_t* meta = unit + 32 * 16 * S;
  const uint4 sc = *reinterpret_cast<const uint4*>(meta + (lane >> 2) * 16);
  f.sc[0] = sc.x;
  f.sc[1] = sc.y;
  f.sc[2] = sc.z;
  f.sc[3] = sc.w;
  f.zz = *reinterpret_cast<const uint32_t*>(meta + 128 + (lane >> 2) * 4);
}

template <int S, int MT>
__device__ __forceinline__ void load_x(uint32_t (&x)[MT][S][2], const uint4* __restrict__ xf, int64_t kchunks,
                                       int g, int lane, int M) {
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const bool live = (mt * 8 + (lane >> 2)) < M;
#pragma unroll
    for (int j = 0; j < S / 2; ++j) {
      uint4 v = make_uint4(0, 0, 0, 0);
      if (live) v = __ldcg(xf + ((size_t)(mt * kchunks + (int64_t)g * (S / 2) + j) * 32 + lane));
      x[mt][2 * j][0] = v.x;
      x[mt][2 * j][1] = v.y;
      x[mt][2 * j + 1][0] = v.z;
      x[mt][2 * j + 1][1] = v.w;
    }
  }
}

template <int S, int MT>
__device__ __forceinline__ void compute_unit(const Frag<S, MT>& f, const uint32_t (&x)[MT][S][2],
                                             float (&acc)[4][MT][4]) {
  uint32_t zlo[4], zhi[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const uint32_t zb = (f.zz >> (8 * t)) & 0xFFu;
    zlo[t] = (0x6400u | (zb & 0xFu)) * 0x10001u;          // fp16 (1024 + z[r0]) x2
    zhi[t] = (0xD400u | ((zb >> 4) << 4)) * 0x10001u;     // fp16 -(64 + z[r1]) x2
  }
  // 4 x MT independent accumulation chains (one per tile x m8-tile), interleaved so that
  // consecutive MMAs never depend on each other.
  float gacc[4][MT][4];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int i = 0; i < 4; ++i) gacc[t][mt][i] = 0.f;
#pragma unroll
  for (int s = 0; s < S; ++s) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint32_t w = f.w[t][s];
      const uint32_t w8 = w >> 8;
      // exact (q - z) in fp16: 0x6400|q = 1024+q ; 0x6400|(q<<4) = 1024+16q
      const uint32_t a0 = hsub2_u(lop3_and_or(w, 0x000F000Fu, 0x64006400u), zlo[t]);
      const uint32_t a1 = hfma2_u(lop3_and_or(w, 0x00F000F0u, 0x64006400u), 0x2C002C00u, zhi[t]);
      const uint32_t a2 = hsub2_u(lop3_and_or(w8, 0x000F000Fu, 0x64006400u), zlo[t]);
      const uint32_t a3 = hfma2_u(lop3_and_or(w8, 0x00F000F0u, 0x64006400u), 0x2C002C00u, zhi[t]);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) mma16816(gacc[t][mt], a0, a1, a2, a3, x[mt][s][0], x[mt][s][1]);
    }
  }
  // fp32 scale once per group (rows r0 -> c0,c1 ; r1 -> c2,c3)
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const __half2 h2 = *reinterpret_cast<const __half2*>(&f.sc[t]);
    const float s0 = __low2float(h2), s1 = __high2float(h2);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      acc[t][mt][0] = fmaf(s0, gacc[t][mt][0], acc[t][mt][0]);
      acc[t][mt][1] = fmaf(s0, gacc[t][mt][1], acc[t][mt][1]);
      acc[t][mt][2] = fmaf(s1, gacc[t][mt][2], acc[t][mt][2]);
      acc[t][mt][3] = fmaf(s1, gacc[t][mt][3], acc[t][mt][3]);
    }
  }
}

// Index (in halves) of element (m, k) in the frag layout of a K-column activation.
__device__ __forceinline__ int64_t frag_index(int m, int64_t k, int64_t K) {
  const int mt = m >> 3, g = m & 7;
  const int64_t c = k >> 5;
  const int kk = (int)(k & 31);
  const int s2 = kk >> 4, kin = kk & 15, h = kin >> 3, cc = kin & 7;
  const int lane = g * 4 + (cc >> 1), e = cc & 1;
  return ((((int64_t)mt * (K >> 5) + c) * 32 + lane) * 4 + s2 * 2 + h) * 2 + e;
}

struct GemvArgs {
  const uint8_t* packed;
  const uint4* xf;
  int M;
  int64_t K, N;
  int NB, NG;
  int64_t U;
  int grid;
  void* out;
  int out_mode;
  int64_t out_ld;
  float* ws;
  int* cnt;
  int dbg;  // profiling aid (TPQ_GEMV_DEBUG): 1 = skip compute, 2 = skip HBM (compute on stale smem)
};

__device__ __forceinline__ int64_t cta_start(int64_t c, int64_t U, int grid) { return c * U / grid; }
// CTA whose range contains unit u:  largest c with floor(c U / grid) <= u.
__device__ __forceinline__ int cta_of_unit(int64_t u, int64_t U, int grid) {
  return (int)(((u + 1) * grid + U - 1) / U) - 1;
}

__device__ __forceinline__ void store_out(const GemvArgs& a, int b, int e, float v) {
  const int m = e >> 6, nl = e & 63;
  if (m >= a.M) return;
  const int64_t n = (int64_t)b * kBlockCols + nl;
  const __half hv = __float2half_rn(v);
  if (a.out_mode == OUT_ROWMAJOR) {
    reinterpret_cast<__half*>(a.out)[(int64_t)m * a.out_ld + n] = hv;
  } else {
    reinterpret_cast<__half*>(a.out)[frag_index(m, n, a.N)] = hv;
  }
}

// The flattened sequence of (block, group) units one warp processes inside its CTA's
// stream-K range [u1s, u1): segments = maximal runs inside one 64-column block; within a
// segment warp w takes groups gb+w, gb+w+8, ...
struct WarpSeq {
  int64_t u, u1;
  int NG, b, gb, ge, g, warp;
  bool valid;
  __device__ __forceinline__ void seg(int64_t uu) {
    u = uu;
    b = (int)(u / NG);
    gb = (int)(u % NG);
    ge = (int)((int64_t)gb + (u1 - u) < NG ? (int64_t)gb + (u1 - u) : NG);
  }
  __device__ __forceinline__ void init(int64_t u0, int64_t u1_, int NG_, int warp_) {
    u1 = u1_;
    NG = NG_;
    warp = warp_;
    valid = u0 < u1;
    if (!valid) return;
    seg(u0);
    g = gb + warp;
    while (g >= ge) {  // no unit for this warp in the first segment
      if (u + (ge - gb) >= u1) {
        valid = false;
        return;
      }
      seg(u + (ge - gb));
      g = gb + warp;
    }
  }
  __device__ __forceinline__ void next() {
    g += 8;
    while (g >= ge) {
      if (u + (ge - gb) >= u1) {
        valid = false;
        return;
      }
      seg(u + (ge - gb));
      g = gb + warp;
    }
  }
};

template <int S, int MT>
__global__ void __launch_bounds__(kThreads, Cfg<S, MT>::OCC) k_gemv(const GemvArgs a) {
  using C = Cfg<S, MT>;
  constexpr int E = MT * 8 * kBlockCols;  // outputs per block (padded rows)
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;                                              // [8 warps][NS][UNIT]
  float* red = reinterpret_cast<float*>(smem + C::RING);            // [8 warps][E]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::RING + red_bytes<MT>());  // [8][NS]
  __shared__ int s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int64_t u0 = cta_start(blockIdx.x, a.U, a.grid);
  const int64_t u1 = cta_start(blockIdx.x + 1, a.U, a.grid);
  const int64_t kchunks = a.K >> 5;
  uint8_t* my_ring = ring + warp * C::NS * C::UNIT;
  uint64_t* my_bars = bars + warp * C::NS;

  if (lane == 0)
    for (int i = 0; i < C::NS; ++i) mbar_init(my_bars + i, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  pdl_launch_dependents();

  // ---- producer: prefetch the first NS units of this warp (weights do not depend on the
  // previous kernel, so this runs before griddepcontrol.wait)
  const uint64_t policy = policy_evict_first();
  WarpSeq prod;
  prod.init(u0, u1, a.NG, warp);
  if (lane == 0) {
#pragma unroll 1
    for (int i = 0; i < C::NS && prod.valid; ++i) {
      mbar_arrive_expect_tx(my_bars + i, C::UNIT);
      bulk_g2s(my_ring + i * C::UNIT, a.packed + ((size_t)prod.b * a.NG + prod.g) * C::UNIT, C::UNIT,
               my_bars + i, policy);
      prod.next();
    }
  } else {
    for (int i = 0; i < C::NS && prod.valid; ++i) prod.next();
  }
  pdl_wait();  // X / Y1 of the previous kernel are visible from here on

  WarpSeq cons;
  cons.init(u0, u1, a.NG, warp);
  uint32_t x[MT][S][2];
  if (cons.valid) load_x<S, MT>(x, a.xf, kchunks, cons.g, lane, a.M);
  int idx = 0;  // units consumed by this warp

  int64_t u = u0;
  bool first_seg = true;
  while (u < u1) {
    const int b = (int)(u / a.NG);
    const int gb = (int)(u % a.NG);
    const int ge = (int)((int64_t)gb + (u1 - u) < a.NG ? (int64_t)gb + (u1 - u) : a.NG);
    float acc[4][MT][4];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[t][mt][i] = 0.f;

    // consume one unit: wait for its TMA stage, pull the fragments to registers, refill the
    // stage with the unit NS ahead, prefetch the next unit's X into `xn`, then compute.
    auto step = [&](const uint32_t(&xc)[MT][S][2], uint32_t(&xn)[MT][S][2]) {
      const int slot = idx % C::NS;
      if (a.dbg != 2) mbar_wait(my_bars + slot, (uint32_t)((idx / C::NS) & 1));
      Frag<S, MT> f;
      read_unit<S, MT>(f, my_ring + slot * C::UNIT, lane);
      __syncwarp();
      if (lane == 0 && prod.valid && a.dbg != 2) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_expect_tx(my_bars + slot, C::UNIT);
        bulk_g2s(my_ring + slot * C::UNIT, a.packed + ((size_t)prod.b * a.NG + prod.g) * C::UNIT, C::UNIT,
                 my_bars + slot, policy);
      }
      if (prod.valid) prod.next();
      ++idx;
      cons.next();
      if (cons.valid) load_x<S, MT>(xn, a.xf, kchunks, cons.g, lane, a.M);
      if (a.dbg != 1) {
        compute_unit<S, MT>(f, xc, acc);
      } else {
        acc[0][0][0] += __uint_as_float(f.w[0][0] ^ f.w[3][S - 1] ^ f.zz);
      }
    };
    uint32_t x2[MT][S][2];
#pragma unroll 1
    for (int g = gb + warp; g < ge; g += 16) {  // two units per trip: x -> x2 -> x, no copies
      step(x, x2);
      if (g + 8 >= ge) {
        if (cons.valid) {
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int s = 0; s < S; ++s) {
              x[mt][s][0] = x2[mt][s][0];
              x[mt][s][1] = x2[mt][s][1];
            }
        }
        break;
      }
      step(x2, x);
    }

    // ---- CTA reduction over the 8 warps (fixed order) ----
    float* my = red + warp * E;
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int m0 = mt * 8 + 2 * (lane & 3), n0 = 16 * t + (lane >> 2);
        my[m0 * 64 + n0] = acc[t][mt][0];
        my[(m0 + 1) * 64 + n0] = acc[t][mt][1];
        my[m0 * 64 + n0 + 8] = acc[t][mt][2];
        my[(m0 + 1) * 64 + n0 + 8] = acc[t][mt][3];
      }
    __syncthreads();
    constexpr int PER = E / kThreads;
    float v[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int e = tid + i * kThreads;
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) s += red[w * E + e];
      v[i] = s;
    }
    const bool full = (gb == 0 && ge == a.NG);
    if (full) {
#pragma unroll
      for (int i = 0; i < PER; ++i) store_out(a, b, tid + i * kThreads, v[i]);
    } else {
      // ---- stream-K fix-up: deterministic, last arriver sums slots in CTA order ----
      const int slot = first_seg ? 0 : 1;
      float* mine = a.ws + ((size_t)blockIdx.x * 2 + slot) * (16 * 64);
#pragma unroll
      for (int i = 0; i < PER; ++i) __stcg(mine + tid + i * kThreads, v[i]);
      __threadfence();
      __syncthreads();
      const int c_first = cta_of_unit((int64_t)b * a.NG, a.U, a.grid);
      const int c_last = cta_of_unit((int64_t)b * a.NG + a.NG - 1, a.U, a.grid);
      if (tid == 0) {
        const int prev = atomicAdd(a.cnt + b, 1);
        s_last = (prev == c_last - c_first);
      }
      __syncthreads();
      if (s_last) {
        __threadfence();
#pragma unroll
        for (int i = 0; i < PER; ++i) v[i] = 0.f;
        for (int c = c_first; c <= c_last; ++c) {
          const int cslot = (cta_start(c, a.U, a.grid) / a.NG == b) ? 0 : 1;
          const float* src = a.ws + ((size_t)c * 2 + cslot) * (16 * 64);
#pragma unroll
          for (int i = 0; i < PER; ++i) v[i] += __ldcg(src + tid + i * kThreads);
        }
#pragma unroll
        for (int i = 0; i < PER; ++i) store_out(a, b, tid + i * kThreads, v[i]);
        if (tid == 0) a.cnt[b] = 0;  // self-reset for the next launch / graph replay
      }
    }
    __syncthreads();  // red[] and s_last reuse
    u += ge - gb;
    first_seg = false;
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

template <int S, int MT>
cudaError_t launch_gemv_t(const GemvArgs& a, cudaStream_t st) {
  return launch_pdl(k_gemv<S, MT>, dim3(a.grid), dim3(kThreads), gemv_smem<S, MT>(), st, a);
}

template <int S, int MT>
int blocks_per_sm_t() {
  constexpr size_t smem = gemv_smem<S, MT>();
  static_assert(smem <= 227 * 1024, "GEMV smem over the per-CTA limit");
  if (cudaFuncSetAttribute(k_gemv<S, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return 0;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_gemv<S, MT>, kThreads, smem) != cudaSuccess) return 0;
  return nb;
}

// ------------------------------------------------------------------ gathers
__device__ __forceinline__ int64_t gather_src(int m, int64_t k, int64_t ld, const int32_t* idx, int mode,
                                              int64_t nn, int M) {
  if (mode == GATHER_COLS) return (int64_t)m * ld + (idx ? (int64_t)idx[k] : k);
  const int64_t c = idx[k];
  return (c / nn) * (int64_t)M * nn + (int64_t)m * nn + (c % nn);
}

__global__ void k_to_frag(const __half* __restrict__ src, int64_t ld, const int32_t* __restrict__ idx, int mode,
                          int64_t nn, int M, int MT, int64_t K, uint4* __restrict__ dst) {
  pdl_launch_dependents();
  pdl_wait();  // src is produced by, and dst still read by, earlier kernels in the stream
  const int64_t total = (int64_t)MT * (K >> 5) * 32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(i & 31);
    const int64_t c = (i >> 5) % (K >> 5);
    const int mt = (int)((i >> 5) / (K >> 5));
    const int m = mt * 8 + (lane >> 2), tg = lane & 3;
    uint32_t out[4] = {0, 0, 0, 0};
    if (m < M) {
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t k = 32 * c + 16 * s2 + 8 * h + 2 * tg;
          const __half lo = src[gather_src(m, k, ld, idx, mode, nn, M)];
          const __half hi = src[gather_src(m, k + 1, ld, idx, mode, nn, M)];
          out[s2 * 2 + h] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
        }
    }
    dst[i] = make_uint4(out[0], out[1], out[2], out[3]);
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
int gemv_blocks_per_sm(int G, int MT) {
  const int S = G / 16;
#define TPQ_BPS(SV, MTV) \
  if (S == SV && MT == MTV) return blocks_per_sm_t<SV, MTV>();
  TPQ_BPS(2, 1) TPQ_BPS(2, 2) TPQ_BPS(4, 1) TPQ_BPS(4, 2) TPQ_BPS(8, 1) TPQ_BPS(8, 2)
#undef TPQ_BPS
  return 0;
}

cudaError_t launch_gemv(const LayerDev& L, const void* xf, int M, void* out, int out_mode, int64_t out_ld,
                        cudaStream_t st) {
  if (M < 1 || M > 16) return cudaErrorInvalidValue;
  const int MT = M <= 8 ? 1 : 2;
  GemvArgs a;
  a.packed = L.packed;
  a.xf = reinterpret_cast<const uint4*>(xf);
  a.M = M;
  a.K = L.K;
  a.N = L.N;
  a.NB = L.NB;
  a.NG = L.NG;
  a.U = L.U;
  a.grid = L.grid[MT];
  a.out = out;
  a.out_mode = out_mode;
  a.out_ld = out_ld;
  a.ws = L.ws;
  a.cnt = L.cnt;
  a.dbg = L.dbg;
  const int S = L.G / 16;
#define TPQ_GEMV(SV, MTV) \
  if (S == SV && MT == MTV) return launch_gemv_t<SV, MTV>(a, st);
  TPQ_GEMV(2, 1) TPQ_GEMV(2, 2) TPQ_GEMV(4, 1) TPQ_GEMV(4, 2) TPQ_GEMV(8, 1) TPQ_GEMV(8, 2)
#undef TPQ_GEMV
  return cudaErrorInvalidValue;
}

cudaError_t launch_to_frag(const void* src, int64_t ld, const int32_t* idx, int mode, int64_t nn, int M, int64_t K,
                           void* dst, cudaStream_t st) {
  if (M < 1 || M > 16 || (K & 31)) return cudaErrorInvalidValue;
  const int MT = M <= 8 ? 1 : 2;
  const int64_t total = (int64_t)MT * (K >> 5) * 32;
  return launch_pdl(k_to_frag, dim3(grid_for(total, 256)), dim3(256), 0, st, reinterpret_cast<const __half*>(src),
                    ld, idx, mode, nn, M, MT, K, reinterpret_cast<uint4*>(dst));
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
