// Host half of libtpq: the C-ABI of include/tpq.h.
//   * gptq_reorder      -- Alg. 1 as a stable counting sort.
//   * tp_shard_mlp      -- offline TP-aware transform (Alg. 3 Require L137),
//                          Megatron column/row split, repack into the device
//                          fragment-native layout (csrc/internal.h), H2D upload, stream-K plan.
//   * tp_mlp_forward*   -- enqueue the per-rank kernels (tpq_kernels.cu) and the NCCL
//                          collectives (AllReduce PAPER.md:L142; AllGather L117 for Alg. 2).
#include "tpq.h"

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define TPQ_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) return fail(TPQ_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

#define TPQ_NCCL(call)                                                                   \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess) return fail(TPQ_ENCCL, "%s: %s", #call, ncclGetErrorString(r_)); \
  } while (0)

template <class F>
void parallel_for(int64_t n, F f) {
  unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (n < 4096 || nt == 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t)
    th.emplace_back([=, &f] {
      for (int64_t i = (int64_t)t * n / nt; i < (int64_t)(t + 1) * n / nt; ++i) f(i);
    });
  for (auto& x : th) x.join();
}

// Canonical (unpacked, reordered) shard of one layer: q[K][N] codes, s[ng][N] fp16 bits,
// z[ng][N] codes.
struct Canon {
  int64_t K = 0, N = 0;
  int G = 0;
  std::vector<uint8_t> q, z;
  std::vector<uint16_t> s;
};

// Per-column scale exponent of the device records (reading c22): E_n >= 0 is the largest
// shift with max_g |s[g][n]| 2^E_n < 2^16, so that the stored s' = s 2^E_n is exact in fp16 (a
// power-of-two scale-up of finite fp16 values below the range limit) and the column's largest
// scale lands in [2^14, 2^16).  The kernels multiply their fp32 accumulators by 2^(c - E_n).
std::vector<int> column_exponents(const Canon& c) {
  std::vector<int> E((size_t)c.N, 0);
  const int64_t ng = c.K / c.G;
  for (int64_t n = 0; n < c.N; ++n) {
    int emax = -100;  // binary exponent of the largest |s| of the column
    for (int64_t g = 0; g < ng; ++g) {
      const uint16_t h = c.s[(size_t)(g * c.N + n)] & 0x7FFF;
      if (h == 0) continue;
      const int be = (h >> 10) ? (int)(h >> 10) - 15 : 7 - __builtin_clz((unsigned)h);  // subnormal: m 2^-24
      emax = std::max(emax, be);
    }
    E[(size_t)n] = emax == -100 ? 0 : std::max(0, 14 - emax);
  }
  return E;
}

// fp16 bits times 2^e (e >= 0), exact: the result stays finite by the choice of E
uint16_t half_scale_up(uint16_t h, int e) {
  if ((h & 0x7FFF) == 0 || e == 0) return h;
  const uint16_t sign = h & 0x8000;
  uint32_t ex = (h >> 10) & 0x1F, m = h & 0x3FF;
  while (e > 0 && ex == 0) {  // subnormal: shift the mantissa until it normalises
    m <<= 1;
    --e;
    if (m & 0x400) {
      ex = 1;
      m &= 0x3FF;
    }
  }
  return (uint16_t)(sign | ((ex + e) << 10) | m);
}
uint16_t half_scale_down(uint16_t h, int e) {  // inverse of half_scale_up on its outputs
  if ((h & 0x7FFF) == 0 || e == 0) return h;
  const uint16_t sign = h & 0x8000;
  int ex = (h >> 10) & 0x1F;
  uint32_t m = h & 0x3FF;
  if (ex - e >= 1) return (uint16_t)(sign | ((ex - e) << 10) | m);
  m |= 0x400;  // becomes subnormal: shift right by 1 - (ex - e) (exact for values produced by scale-up)
  m >>= (1 - (ex - e));
  return (uint16_t)(sign | m);
}

// Pack a canonical shard into the device layout of internal.h.
// Nibble slot (0..7) of k0 + i inside a code word (internal.h): k0,k0+1 -> n0,n4; k0+2,k0+3 -> n1,n5;
// k0+4,k0+5 -> n2,n6; k0+6,k0+7 -> n3,n7.
constexpr int kNibbleOfK[8] = {0, 4, 1, 5, 2, 6, 3, 7};

std::vector<uint8_t> pack_layer(const Canon& c, const std::vector<int>& E) {
  const int G = c.G, KG = tpq::kUnitK / G;
  const int64_t NT = c.N / tpq::kTileCols, NKB = c.K / tpq::kUnitK, UB = tpq::unit_bytes(G);
  constexpr int64_t kCodes = tpq::kUnitK * tpq::kTileCols / 2;
  std::vector<uint8_t> out((size_t)(NT * NKB * UB), 0);
  parallel_for(NT * NKB, [&](int64_t u) {
    const int64_t t = u / NKB, kb = u % NKB;
    uint8_t* rec = out.data() + u * UB;
    uint32_t* words = reinterpret_cast<uint32_t*>(rec);
    for (int j = 0; j < tpq::kTileCols; ++j) {
      const int64_t n = t * tpq::kTileCols + j;
      for (int ch = 0; ch < tpq::kUnitK / 32; ++ch)
        for (int w = 0; w < 4; ++w) {
          const int64_t k0 = kb * tpq::kUnitK + 32 * ch + 8 * w;
          uint32_t word = 0;
          for (int i = 0; i < 8; ++i) word |= (uint32_t)c.q[(size_t)((k0 + i) * c.N + n)] << (4 * kNibbleOfK[i]);
          words[tpq::code_block(ch, j) * 4 + w] = word;
        }
      for (int gi = 0; gi < KG; ++gi) {
        const int64_t g = kb * KG + gi;
        const uint16_t sp = half_scale_up(c.s[(size_t)(g * c.N + n)], E[(size_t)n]);  // s' = s 2^E_n
        memcpy(rec + kCodes + 256 * gi + 2 * j, &sp, 2);
        rec[kCodes + 256 * KG + 64 * gi + j / 2] |= (uint8_t)(c.z[(size_t)(g * c.N + n)] << (4 * (j & 1)));
      }
    }
  });
  return out;
}

// Unordered-g_idx layer (TPQ_UNORDERED, the Fig. 1 formulation): records of the codes in checkpoint
// row order (same code layout as pack_layer) followed by the 128 rows' group ids (uint8), and the
// [ng][N] table {lo: fp16 s' = s 2^E_n, hi: fp16(-z s' 2^-24)} the kernel reads per row.
struct Unord {
  std::vector<uint8_t> rec;
  std::vector<uint32_t> table;
};
uint16_t half_rn(float f) {  // round-to-nearest-even, subnormals included (host _Float16)
  const _Float16 h = (_Float16)f;
  uint16_t b;
  memcpy(&b, &h, 2);
  return b;
}
float half_to_float(uint16_t b) {
  _Float16 h;
  memcpy(&h, &b, 2);
  return (float)h;
}
Unord pack_layer_unordered(const Canon& c, const std::vector<int>& E, const std::vector<int32_t>& gk) {
  const int64_t NT = c.N / tpq::kTileCols, NKB = c.K / tpq::kUnitK, ng = c.K / c.G;
  constexpr int64_t kCodes = tpq::kUnitK * tpq::kTileCols / 2, UB = kCodes + tpq::kUnitK;
  Unord u;
  u.rec.assign((size_t)(NT * NKB * UB), 0);
  parallel_for(NT * NKB, [&](int64_t un) {
    const int64_t t = un / NKB, kb = un % NKB;
    uint8_t* rec = u.rec.data() + un * UB;
    uint32_t* words = reinterpret_cast<uint32_t*>(rec);
    for (int j = 0; j < tpq::kTileCols; ++j) {
      const int64_t n = t * tpq::kTileCols + j;
      for (int ch = 0; ch < tpq::kUnitK / 32; ++ch)
        for (int w = 0; w < 4; ++w) {
          const int64_t k0 = kb * tpq::kUnitK + 32 * ch + 8 * w;
          uint32_t word = 0;
          for (int i = 0; i < 8; ++i) word |= (uint32_t)c.q[(size_t)((k0 + i) * c.N + n)] << (4 * kNibbleOfK[i]);
          words[tpq::code_block(ch, j) * 4 + w] = word;
        }
    }
    for (int r = 0; r < tpq::kUnitK; ++r) rec[kCodes + r] = (uint8_t)gk[(size_t)(kb * tpq::kUnitK + r)];
  });
  u.table.resize((size_t)(ng * c.N));
  for (int64_t g = 0; g < ng; ++g)
    for (int64_t n = 0; n < c.N; ++n) {
      const uint16_t sp = half_scale_up(c.s[(size_t)(g * c.N + n)], E[(size_t)n]);
      const uint16_t cc = half_rn(-(float)c.z[(size_t)(g * c.N + n)] * half_to_float(sp) * 5.9604644775390625e-8f);
      u.table[(size_t)(g * c.N + n)] = (uint32_t)sp | ((uint32_t)cc << 16);
    }
  return u;
}

// Inverse of pack_layer (test export).
void unpack_layer(const std::vector<uint8_t>& pk, const std::vector<int>& E, int64_t K, int64_t N, int G, uint8_t* q,
                  uint16_t* s, uint8_t* z) {
  const int KG = tpq::kUnitK / G;
  const int64_t NT = N / tpq::kTileCols, NKB = K / tpq::kUnitK, UB = tpq::unit_bytes(G);
  constexpr int64_t kCodes = tpq::kUnitK * tpq::kTileCols / 2;
  parallel_for(NT * NKB, [&](int64_t u) {
    const int64_t t = u / NKB, kb = u % NKB;
    const uint8_t* rec = pk.data() + u * UB;
    const uint32_t* words = reinterpret_cast<const uint32_t*>(rec);
    for (int j = 0; j < tpq::kTileCols; ++j) {
      const int64_t n = t * tpq::kTileCols + j;
      for (int ch = 0; ch < tpq::kUnitK / 32; ++ch)
        for (int w = 0; w < 4; ++w) {
          const uint32_t word = words[tpq::code_block(ch, j) * 4 + w];
          const int64_t k0 = kb * tpq::kUnitK + 32 * ch + 8 * w;
          for (int i = 0; i < 8; ++i) q[(k0 + i) * N + n] = (word >> (4 * kNibbleOfK[i])) & 0xF;
        }
      for (int gi = 0; gi < KG; ++gi) {
        const int64_t g = kb * KG + gi;
        uint16_t sp;
        memcpy(&sp, rec + kCodes + 256 * gi + 2 * j, 2);
        s[g * N + n] = half_scale_down(sp, E[(size_t)n]);
        z[g * N + n] = (rec[kCodes + 256 * KG + 64 * gi + j / 2] >> (4 * (j & 1))) & 0xF;
      }
    }
  });
}

inline uint32_t nib(uint32_t w, int i) { return (w >> (4 * i)) & 0xFu; }



}  // namespace

constexpr int kGemmRows = 512;  // A7: activation rows per GEMM pass (the SS GEMMs take up to 512)
constexpr int kMmRows = 256;    // A7 below 128 rows: k_dqgemm's largest N

// A column permutation on the device as the gathers read it: K int32 indices, then the same K as
// uint16 (the staged-row gather keeps 8 of them per 16-byte register quad; K <= 24576 there).
cudaError_t upload_perm(int32_t* d, const int32_t* P, int64_t K) {
  std::vector<uint16_t> p16((size_t)K);
  for (int64_t k = 0; k < K; ++k) p16[(size_t)k] = (uint16_t)P[k];
  cudaError_t e = cudaMemcpy(d, P, (size_t)K * 4, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return e;
  return cudaMemcpy(d + K, p16.data(), (size_t)K * 2, cudaMemcpyHostToDevice);
}

struct tpq_comm {
  ncclComm_t comm;
  int tp, rank, device;
};

struct tpq_mlp {
  int64_t K1 = 0, N1 = 0, N2 = 0, n = 0, M_max = 0;
  int G1 = 0, G2 = 0, tp = 1, rank = 0, variant = 1, device = -1;
  std::vector<int32_t> P1, P2, w1_cols, w2_rows, gather_cols;
  int32_t w2_group_lo = 0, w2_group_hi = 0;
  std::vector<uint8_t> pk1, pk2;  // packed host copies
  std::vector<uint32_t> tab1, tab2;  // unordered layers: [ng][N] {s', C} tables (TPQ_UNORDERED)
  std::vector<uint8_t> z1u, z2u;      // unordered layers: zeros [ng][N] (export only)
  std::vector<int32_t> g1u, g2u;      // unordered layers: per-row group (export only)
  void* d_tab = nullptr;
  std::vector<int> E1, E2;        // per-column scale exponents of the records (column_exponents)
  tpq::LayerDev L1, L2;
  // device buffers
  void* d_w1 = nullptr;
  void* d_w2 = nullptr;
  int32_t* d_P1 = nullptr;
  int32_t* d_gcols = nullptr;  // naive: int2 (c / n, c % n) of c = P2[r n + i] (k_gather_ag)
  void* d_x1 = nullptr;        // layer-1 input X[:, P1], row-major [16][K1]
  void* d_y1 = nullptr;        // layer-1 output = layer-2 input, row-major [16][n]
  void* d_buf = nullptr;       // AllGather buffer [tp][rows][n]
  void* d_xin = nullptr;       // host-forward staging [M_max][K1]
  void* d_yout = nullptr;      // host-forward staging [M_max][N2]
  float* d_ws = nullptr;
  float* d_colf = nullptr;     // per-column 2^(24 - E) of layer 1 [n] then layer 2 [N2]
  int* d_split = nullptr;      // split tiles of layer 1 then layer 2 (k_split_fixup)
  CUtensorMap xmap1 = {}, xmap2 = {};  // TMA views of d_x1 / d_y1 (GEMV activation operand, 16 rows)
  // gate_proj variant (f2): layer 1 = gate + up; the up layer's own P1u and gathered X[:, P1u]
  bool gated = false;
  std::vector<int32_t> P1u;
  int32_t* d_P1u = nullptr;
  void* d_x1u = nullptr;
  CUtensorMap xmap1u = {};
  CUtensorMap xmap1_32 = {}, xmap2_32 = {};  // 32-row boxes of d_x1 / d_y1 (the N = 32 GEMV, 17 <= M <= 32)
  CUtensorMap mm1[3] = {}, mm2[3] = {};  // A7 views of d_x1 / d_y1 with 64 / 128 / 256 rows
  CUtensorMap ss1 = {}, ss2 = {};        // A7 SS views: 256-row buffers, 128-row boxes
  int sms = 148;
  int rows = 16;                       // activation rows per pass: 16 (GEMV) or 256 (M_max > 16)
  ncclComm_t comm = nullptr;
};

namespace {

int validate_layer(const gptq_layer* w, const char* name) {
  if (!w) return fail(TPQ_EINVAL, "%s is NULL", name);
  if (!w->qweight || !w->scales || !w->qzeros || !w->g_idx)
    return fail(TPQ_EINVAL, "%s: NULL array", name);
  if (w->bits != 4) return fail(TPQ_EUNSUPPORTED, "%s: bits=%d (only 4 supported)", name, w->bits);
  if (w->K < 8 || w->N < 8 || w->K % 8 || w->N % 8)
    return fail(TPQ_EINVAL, "%s: K=%lld N=%lld must be positive multiples of 8 (GPTQ packing)", name,
                (long long)w->K, (long long)w->N);
  if (w->G < 1) return fail(TPQ_EINVAL, "%s: G=%d", name, w->G);
  return TPQ_OK;
}

int validate_perm(const int32_t* P, const gptq_layer* w, const char* name) {
  if (!P) return fail(TPQ_EINVAL, "%s is NULL", name);
  std::vector<uint8_t> seen((size_t)w->K, 0);
  for (int64_t i = 0; i < w->K; ++i) {
    const int32_t p = P[i];
    if (p < 0 || p >= w->K || seen[p]) return fail(TPQ_EINVAL, "%s is not a permutation (index %lld)", name, (long long)i);
    seen[p] = 1;
    if (w->g_idx[p] != (int32_t)(i / w->G))
      return fail(TPQ_EINVAL,
                  "%s does not order g_idx: g_idx[P[%lld]] = %d != floor(i/G) = %lld (use gptq_reorder, Alg. 1)",
                  name, (long long)i, w->g_idx[p], (long long)(i / w->G));
  }
  return TPQ_OK;
}

void free_dev(tpq_mlp* h) {
  if (h->device < 0) return;
  cudaSetDevice(h->device);
  void* ptrs[] = {h->d_w1, h->d_w2, h->d_P1, h->d_gcols, h->d_x1, h->d_y1, h->d_buf, h->d_xin, h->d_yout, h->d_ws, h->d_colf, h->d_tab, h->d_P1u, h->d_x1u, h->d_split};
  for (void* p : ptrs)
    if (p) cudaFree(p);
}

int dev_alloc(void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes ? bytes : 16);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? TPQ_ENOMEM : TPQ_ECUDA, "cudaMalloc(%zu): %s", bytes,
                cudaGetErrorString(e));
  }
  return TPQ_OK;
}

// Stream-K plan: a persistent grid of one CTA per SM, each CTA a contiguous range of
// (tile, k-block) units; at least 4 units per CTA so the TMA ring has work to overlap.
void plan_layer(tpq::LayerDev& L, int64_t K, int64_t N, int G, int device, bool cluster_ok) {
  L.K = K;
  L.N = N;
  L.G = G;
  L.NT = (int)(N / tpq::kTileCols);
  L.NKB = (int)(K / tpq::kUnitK);
  L.U = (int64_t)L.NT * L.NKB;
  int sms = 148;
  if (device >= 0) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int64_t cap = std::max<int64_t>(1, L.U / 4);
  // Small shards (< 56 units per SM: Llama / Granite at TP >= 2) are latency-bound, not
  // bandwidth-bound: 128 of 148 CTAs measured faster per forward there (the next kernel can start on
  // SMs the previous one has already left; Llama TP=2 31.5 vs 32.6 us at M=1), while full layers need
  // every SM (Granite TP=1, 62 units per SM: 37.5 with 148 CTAs vs 39.3 with 128).
  int g = sms;
  if (L.U < 56LL * sms) g = std::max(1, sms * 128 / 148);
  if (const char* e = getenv("TPQ_GRID")) g = std::max(1, std::min(sms, atoi(e)));  // tuning aid
  L.grid = (int)std::min<int64_t>((int64_t)g, cap);
  // Split tiles are reduced inside the GEMV (c_first waits for the later contributors' partials,
  // staged into shared memory in one round trip) unless a tile spans more than 6 CTA ranges; then
  // the separate fix-up kernel after the GEMV.  (Granite TP=1 layer 2, 5 contributors per tile:
  // in-kernel 36.8 / 38.6 us at M = 1 / 16 against 37.5 / 40.8 with the fix-up kernel.)
  {
    const int64_t per = std::max<int64_t>(1, L.U / L.grid);
    const int64_t most = (L.NKB - 1 + per - 1) / per + 1;  // contributors of a tile, at most
    const char* e = getenv("TPQ_INRED_MAX");  // tuning aid (A/B): most contributors reduced in-kernel
    L.inred = most <= (e ? atoi(e) : 6) && !getenv("TPQ_FIXUP_KERNEL");
  }
  // Cluster split-K for small shards: one tile per cluster of cs CTAs, each a 1/cs k-range of it,
  // reduced through distributed shared memory (no cross-CTA hand-off through L2 at the end of the
  // layer, no fix-up kernel) -- when the clusters fit on the SMs and a CTA gets at most 4 units more
  // than under stream-K (~0.8 us, less than the hand-off it removes).  Llama TP=8: layer 1 in
  // clusters of 4 (16 units vs 14), layer 2 of 2 (14 vs 14): 16.8 -> 13.8 us at M = 1 (same box);
  // TP=4: both layers of 2, 22.8 -> 19.8 us; TP=1 layer 2 (112 units vs 97) stays stream-K.
  L.csize = 1;
  if (cluster_ok && device >= 0) {
    const int64_t per = (L.U + L.grid - 1) / L.grid;
    const char* ce = getenv("TPQ_CLUSTER");  // tuning aid: force a cluster size (1 = stream-K)
    const int cmax = tpq::gemv_cluster_max(G);
    for (int cs : {4, 2}) {
      if (cs > cmax || (int64_t)L.NT * cs > sms || L.NKB < 2 * cs) continue;
      if (ce ? atoi(ce) == cs : (L.NKB + cs - 1) / cs <= per + 4) {
        L.csize = cs;
        break;
      }
    }
    if (L.csize > 1) {
      L.grid = L.NT * L.csize;
      L.inred = 0;
    }
  }
  L.grid_mm = (int)std::min<int64_t>((int64_t)sms, cap);
  if (getenv("TPQ_VERBOSE"))
    fprintf(stderr, "[tpq] layer K=%lld N=%lld G=%d: grid %d over %lld units, split tiles reduced %s\n", (long long)K,
            (long long)N, G, L.grid, (long long)L.U,
            L.csize > 1 ? "in clusters (split-K)" : L.inred ? "in-kernel" : "by the fix-up kernel");
}

}  // namespace

extern "C" {

const char* tpq_last_error(void) { return g_err.c_str(); }
int tpq_version(void) { return (1 << 16) | 0; }

int gptq_reorder(const int32_t* g_idx, int64_t K, int32_t G, int32_t* perm_out, int32_t* g_idx_sorted_out) {
  try {
    if (!g_idx || !perm_out) return fail(TPQ_EINVAL, "gptq_reorder: NULL pointer");
    if (K < 1 || G < 1) return fail(TPQ_EINVAL, "gptq_reorder: K=%lld G=%d must be >= 1", (long long)K, G);
    if (K > INT32_MAX) return fail(TPQ_EINVAL, "gptq_reorder: K too large");
    const int64_t ng = (K + G - 1) / G;
    std::vector<int64_t> cnt((size_t)ng + 1, 0);
    for (int64_t i = 0; i < K; ++i) {
      const int32_t g = g_idx[i];
      if (g < 0 || g >= ng)
        return fail(TPQ_EINVAL, "gptq_reorder: g_idx[%lld]=%d outside [0,%lld)", (long long)i, g, (long long)ng);
      cnt[(size_t)g + 1]++;
    }
    for (int64_t g = 0; g < ng; ++g) {
      const int64_t want = std::min<int64_t>(G, K - g * G);
      if (cnt[(size_t)g + 1] != want)
        return fail(TPQ_EINVAL, "gptq_reorder: group %lld has %lld rows, Eq. 3 requires %lld", (long long)g,
                    (long long)cnt[(size_t)g + 1], (long long)want);
    }
    for (int64_t g = 0; g < ng; ++g) cnt[(size_t)g + 1] += cnt[(size_t)g];
    // stable counting sort: visiting i in ascending order keeps ties in original order (c6)
    for (int64_t i = 0; i < K; ++i) perm_out[cnt[(size_t)g_idx[i]]++] = (int32_t)i;
    if (g_idx_sorted_out)
      for (int64_t i = 0; i < K; ++i) g_idx_sorted_out[i] = g_idx[perm_out[i]];
    return TPQ_OK;
  } catch (const std::bad_alloc&) {
    return fail(TPQ_ENOMEM, "gptq_reorder: out of host memory");
  } catch (...) {
    return fail(TPQ_EINVAL, "gptq_reorder: unexpected exception");
  }
}

}  // extern "C"

namespace {

// Shared body of tp_shard_mlp and tp_shard_gated_mlp (wu, P1u non-NULL: gate_proj variant, w1 = gate).
int shard_impl(const gptq_layer* w1, const gptq_layer* wu, const gptq_layer* w2, const int32_t* P1, const int32_t* P1u,
               const int32_t* P2, int tp, int rank, int variant, int64_t M_max, int device, tpq_mlp** out) {
  if (!out) return fail(TPQ_EINVAL, "tp_shard_mlp: out is NULL");
  *out = nullptr;
  int rc;
  const bool gated = wu != nullptr;
  if ((rc = validate_layer(w1, gated ? "wg" : "w1"))) return rc;
  if ((rc = validate_layer(w2, gated ? "wd" : "w2"))) return rc;
  if (gated) {
    if ((rc = validate_layer(wu, "wu"))) return rc;
    if (wu->K != w1->K || wu->N != w1->N || wu->G != w1->G)
      return fail(TPQ_EINVAL, "wu (K=%lld N=%lld G=%d) must match wg (K=%lld N=%lld G=%d)", (long long)wu->K,
                  (long long)wu->N, wu->G, (long long)w1->K, (long long)w1->N, w1->G);
    if (variant == TPQ_UNORDERED) return fail(TPQ_EINVAL, "the gate_proj variant has no TPQ_UNORDERED baseline");
    if (M_max > 16) return fail(TPQ_EUNSUPPORTED, "the gate_proj variant runs the M <= 16 GEMV only (M_max=%lld)", (long long)M_max);
  }
  if (w1->N != w2->K)
    return fail(TPQ_EINVAL, "w1->N=%lld != w2->K=%lld", (long long)w1->N, (long long)w2->K);
  if (tp != 1 && tp != 2 && tp != 4 && tp != 8) return fail(TPQ_EINVAL, "tp=%d not in {1,2,4,8}", tp);
  if (rank < 0 || rank >= tp) return fail(TPQ_EINVAL, "rank=%d not in [0,%d)", rank, tp);
  if (variant != TPQ_NAIVE && variant != TPQ_TP_AWARE && variant != TPQ_UNORDERED)
    return fail(TPQ_EINVAL, "variant=%d", variant);
  const bool unord = variant == TPQ_UNORDERED;
  if (unord && tp != 1) return fail(TPQ_EINVAL, "TPQ_UNORDERED is the single-rank locality baseline: tp=%d", tp);
  if (unord && M_max > 16) return fail(TPQ_EUNSUPPORTED, "TPQ_UNORDERED runs the M <= 16 GEMV only (M_max=%lld)", (long long)M_max);
  if (M_max < 1 || M_max > 512) return fail(TPQ_EINVAL, "M_max=%lld not in [1,512]", (long long)M_max);
  if (device < -1) return fail(TPQ_EINVAL, "device=%d", device);
  const int64_t K1 = w1->K, N1 = w1->N, N2 = w2->N;
  if (N1 % tp) return fail(TPQ_EINVAL, "N1=%lld not divisible by tp=%d (CHUNK)", (long long)N1, tp);
  const int64_t n = N1 / tp;
  for (int G : {w1->G, w2->G})
    if (G != 32 && G != 64 && G != 128) return fail(TPQ_EUNSUPPORTED, "G=%d not in {32,64,128}", G);
  if (K1 % w1->G) return fail(TPQ_EUNSUPPORTED, "K1=%lld not a multiple of G1=%d (ragged group, c13)", (long long)K1, w1->G);
  if (K1 % tpq::kUnitK)
    return fail(TPQ_EUNSUPPORTED, "K1=%lld not a multiple of 128 (device k-blocks)", (long long)K1);
  if (n % tpq::kTileCols || N2 % tpq::kTileCols)
    return fail(TPQ_EINVAL, "n=N1/tp=%lld and N2=%lld must be multiples of 128 (device tiles)", (long long)n,
                (long long)N2);
  if (n % w2->G) return fail(TPQ_EINVAL, "n=%lld not a multiple of G2=%d: W2 shard would split a group (c12)", (long long)n, w2->G);
  if (unord) {
    for (const gptq_layer* w : {w1, w2}) {
      if (w->K / w->G > 256) return fail(TPQ_EUNSUPPORTED, "TPQ_UNORDERED: %lld groups > 256 (uint8 group ids)", (long long)(w->K / w->G));
      for (int64_t k = 0; k < w->K; ++k)
        if (w->g_idx[k] < 0 || w->g_idx[k] >= w->K / w->G) return fail(TPQ_EINVAL, "g_idx[%lld]=%d out of range", (long long)k, w->g_idx[k]);
    }
  } else {
    if ((rc = validate_perm(P1, w1, gated ? "P1g" : "P1"))) return rc;
    if ((rc = validate_perm(P2, w2, "P2"))) return rc;
    if (gated && (rc = validate_perm(P1u, wu, "P1u"))) return rc;
  }

  tpq_mlp* h = nullptr;
  try {
    h = new tpq_mlp();
    h->K1 = K1; h->N1 = N1; h->N2 = N2; h->n = n; h->M_max = M_max;
    h->G1 = w1->G; h->G2 = w2->G; h->tp = tp; h->rank = rank; h->variant = variant; h->device = device;
    if (unord) {  // no reordering: identity maps (checkpoint order)
      h->P1.resize(K1);
      h->P2.resize(N1);
      for (int64_t k = 0; k < K1; ++k) h->P1[k] = (int32_t)k;
      for (int64_t k = 0; k < N1; ++k) h->P2[k] = (int32_t)k;
      P1 = h->P1.data();
      P2 = h->P2.data();
    } else {
      h->P1.assign(P1, P1 + K1);
      h->P2.assign(P2, P2 + N1);
    }
    h->w1_cols.resize(n);
    h->w2_rows.resize(n);
    for (int64_t j = 0; j < n; ++j) {
      h->w1_cols[j] = variant == TPQ_TP_AWARE ? P2[rank * n + j] : (int32_t)(rank * n + j);  // W1[P1,P2] vs W1[P1]
      h->w2_rows[j] = P2[rank * n + j];                                                         // W2[P2] row block r
    }
    h->gather_cols.assign(P2 + rank * n, P2 + (rank + 1) * n);
    h->w2_group_lo = (int32_t)(rank * n / w2->G);
    h->w2_group_hi = (int32_t)((rank + 1) * n / w2->G);

    // ---- canonical shards ----
    auto build_c1 = [&](const gptq_layer* w, const int32_t* P) {  // W[P][:, w1_cols] (rows by P, cols by P2 or identity)
      Canon c;
      c.K = K1; c.N = n; c.G = w->G;
      c.q.resize((size_t)(K1 * n));
      parallel_for(K1, [&](int64_t k) {  // row k of W[P] = original row P[k]
        const int32_t src = P[k];
        const uint32_t* row = w->qweight + (size_t)(src / 8) * N1;
        for (int64_t j = 0; j < n; ++j) c.q[(size_t)(k * n + j)] = (uint8_t)nib(row[h->w1_cols[j]], src % 8);
      });
      const int64_t ng1 = K1 / w->G;
      c.s.resize((size_t)(ng1 * n));
      c.z.resize((size_t)(ng1 * n));
      for (int64_t g = 0; g < ng1; ++g)
        for (int64_t j = 0; j < n; ++j) {
          const int32_t col = h->w1_cols[j];
          c.s[(size_t)(g * n + j)] = w->scales[(size_t)(g * N1 + col)];
          c.z[(size_t)(g * n + j)] = (uint8_t)nib(w->qzeros[(size_t)(g * (N1 / 8) + col / 8)], col % 8);
        }
      return c;
    };
    Canon c1 = build_c1(w1, P1), c2, c1u;
    if (gated) {
      h->gated = true;
      h->P1u.assign(P1u, P1u + K1);
      c1u = build_c1(wu, P1u);  // Wu[P1u, P2]: the SAME column permutation as Wg (reading c24)
    }
    c2.K = n; c2.N = N2; c2.G = w2->G;
    c2.q.resize((size_t)(n * N2));
    parallel_for(n, [&](int64_t i) {  // local row i of W2[P2] block r = original row P2[r n + i]
      const int32_t src = h->w2_rows[i];
      const uint32_t* row = w2->qweight + (size_t)(src / 8) * N2;
      for (int64_t j = 0; j < N2; ++j) c2.q[(size_t)(i * N2 + j)] = (uint8_t)nib(row[j], src % 8);
    });
    const int64_t ng2 = n / w2->G;
    c2.s.resize((size_t)(ng2 * N2));
    c2.z.resize((size_t)(ng2 * N2));
    for (int64_t lg = 0; lg < ng2; ++lg) {
      const int64_t g = h->w2_group_lo + lg;
      for (int64_t j = 0; j < N2; ++j) {
        c2.s[(size_t)(lg * N2 + j)] = w2->scales[(size_t)(g * N2 + j)];
        c2.z[(size_t)(lg * N2 + j)] = (uint8_t)nib(w2->qzeros[(size_t)(g * (N2 / 8) + j / 8)], j % 8);
      }
    }
    h->E1 = column_exponents(c1);
    h->E2 = column_exponents(c2);
    if (gated) {  // one exponent per column for gate and up: the smaller one keeps both exact
      const std::vector<int> Eu = column_exponents(c1u);
      for (size_t j = 0; j < h->E1.size(); ++j) h->E1[j] = std::min(h->E1[j], Eu[j]);
    }
    if (unord) {
      h->g1u.assign(w1->g_idx, w1->g_idx + K1);
      h->g2u.assign(w2->g_idx, w2->g_idx + N1);
      Unord u1 = pack_layer_unordered(c1, h->E1, h->g1u), u2 = pack_layer_unordered(c2, h->E2, h->g2u);
      h->pk1 = std::move(u1.rec);
      h->pk2 = std::move(u2.rec);
      h->tab1 = std::move(u1.table);
      h->tab2 = std::move(u2.table);
      h->z1u = c1.z;
      h->z2u = c2.z;
      h->L1.unord = h->L2.unord = 1;
    } else if (gated) {
      // records of (tile, k-block) u as the pair gate(u), up(u) (k_dqgemv<G, true>)
      const std::vector<uint8_t> pg = pack_layer(c1, h->E1), pu = pack_layer(c1u, h->E1);
      const size_t UB = (size_t)tpq::unit_bytes(w1->G), nun = pg.size() / UB;
      h->pk1.resize(2 * pg.size());
      for (size_t u = 0; u < nun; ++u) {
        memcpy(h->pk1.data() + (2 * u) * UB, pg.data() + u * UB, UB);
        memcpy(h->pk1.data() + (2 * u + 1) * UB, pu.data() + u * UB, UB);
      }
      h->pk2 = pack_layer(c2, h->E2);
    } else {
      h->pk1 = pack_layer(c1, h->E1);
      h->pk2 = pack_layer(c2, h->E2);
    }
    plan_layer(h->L1, K1, n, w1->G, device, !gated && !unord);
    h->L1.gated = gated ? 1 : 0;
    plan_layer(h->L2, n, N2, w2->G, device, !unord);

    if (device >= 0) {
      auto upload = [&]() -> int {
        TPQ_CUDA(cudaSetDevice(device));
        // kernel attributes (dynamic shared memory, carveout) are per device: set them on this one
        for (int G : {w1->G, w2->G})
          if (!tpq::gemv_prepare(G)) {
            cudaGetLastError();
            return fail(TPQ_ECUDA, "kernel attribute setup failed for G=%d on device %d", G, device);
          }
        int r;
        auto A = [&](void** p, size_t b) { return dev_alloc(p, b); };
        // [grid][2 slots][gate, up][16 rows][128]; 32 rows when passes of 17..32 rows run the N = 32 GEMV
        const size_t wr = M_max > tpq::kMaxM ? 2 * tpq::kNPad : tpq::kNPad;
        const size_t ws1 = (size_t)h->L1.grid * 2 * wr * tpq::kTileCols * (gated ? 2 : 1);
        const size_t ws2 = (size_t)h->L2.grid * 2 * wr * tpq::kTileCols;
        h->rows = M_max > tpq::kMaxM ? kGemmRows : tpq::kMaxM;
        const size_t wm1 = M_max > tpq::kMaxM ? (size_t)h->L1.grid_mm * 2 * kMmRows * tpq::kTileCols : 0;
        const size_t wm2 = M_max > tpq::kMaxM ? (size_t)h->L2.grid_mm * 2 * kMmRows * tpq::kTileCols : 0;
        cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, device);
        auto ss_ws = [&](const tpq::LayerDev& L) -> size_t {  // largest k-split partial set (M >= 128 passes)
          if (M_max < 128) return 0;
          size_t items = 0;
          const int bn = tpq::ss_bn(L.NT, L.G), NG = L.NT * tpq::kTileCols / bn;
          for (int mb = 1; mb <= kGemmRows / 128; ++mb) {
            const int S = tpq::ss_splits(NG, L.NKB, mb, h->sms);
            if (S > 1) items = std::max(items, (size_t)mb * NG * S);
          }
          size_t fl = items * 128 * bn;
          if (L.NT % 2 == 0)  // CTA-pair kernel: (NT / 2 groups x 2 MB row blocks x S) x 128 x 256
            for (int mb = 1; mb <= kGemmRows / 256; ++mb) {
              const int S2 = tpq::ss_splits(L.NT / 2, L.NKB, mb, h->sms / 2);
              if (S2 > 1) fl = std::max(fl, (size_t)L.NT * mb * S2 * 128 * 256);
            }
          return fl;
        };
        const size_t ws1s = ss_ws(h->L1), ws2s = ss_ws(h->L2);
        if ((r = A(&h->d_w1, h->pk1.size())) || (r = A(&h->d_w2, h->pk2.size())) ||
            (r = A((void**)&h->d_P1, K1 * 6)) || (r = A((void**)&h->d_gcols, n * 8)) || (r = A(&h->d_x1, (size_t)h->rows * K1 * 2)) ||
            (r = A(&h->d_y1, (size_t)h->rows * n * 2)) || (r = A(&h->d_buf, (size_t)tp * h->rows * n * 2)) ||
            (r = A(&h->d_xin, (size_t)M_max * K1 * 2)) || (r = A(&h->d_yout, (size_t)M_max * N2 * 2)) ||
            (r = A((void**)&h->d_ws, (ws1 + ws2 + wm1 + wm2 + ws1s + ws2s) * 4)) ||
            (r = A((void**)&h->d_colf, (size_t)(n + N2) * 4)) ||
            (r = A(&h->d_tab, (h->tab1.size() + h->tab2.size()) * 4)) ||
            (gated && (r = A((void**)&h->d_P1u, K1 * 6))) || (gated && (r = A(&h->d_x1u, (size_t)h->rows * K1 * 2))))
          return r;
        if (gated) {
          TPQ_CUDA(upload_perm(h->d_P1u, P1u, K1));
          if (!tpq::make_xmap(&h->xmap1u, h->d_x1u, K1, tpq::kNPad))
            return fail(TPQ_ECUDA, "cuTensorMapEncodeTiled failed for the up_proj activation buffer");
        }
        TPQ_CUDA(cudaMemcpy(h->d_w1, h->pk1.data(), h->pk1.size(), cudaMemcpyHostToDevice));
        TPQ_CUDA(cudaMemcpy(h->d_w2, h->pk2.data(), h->pk2.size(), cudaMemcpyHostToDevice));
        TPQ_CUDA(upload_perm(h->d_P1, P1, K1));
        {
          std::vector<float> cf((size_t)(n + N2));
          for (int64_t j = 0; j < n; ++j) cf[(size_t)j] = std::ldexp(1.f, 24 - h->E1[(size_t)j]);
          for (int64_t j = 0; j < N2; ++j) cf[(size_t)(n + j)] = std::ldexp(1.f, 24 - h->E2[(size_t)j]);
          TPQ_CUDA(cudaMemcpy(h->d_colf, cf.data(), cf.size() * 4, cudaMemcpyHostToDevice));
        }
        {
          std::vector<int32_t> so((size_t)(2 * n));
          for (int64_t i = 0; i < n; ++i) {
            so[(size_t)(2 * i)] = (int32_t)(h->gather_cols[(size_t)i] / n);
            so[(size_t)(2 * i + 1)] = (int32_t)(h->gather_cols[(size_t)i] % n);
          }
          TPQ_CUDA(cudaMemcpy(h->d_gcols, so.data(), n * 8, cudaMemcpyHostToDevice));
        }
        bool mok = tpq::make_xmap(&h->xmap1, h->d_x1, K1, tpq::kNPad) && tpq::make_xmap(&h->xmap2, h->d_y1, n, tpq::kNPad);
        if (h->rows > tpq::kMaxM) {
          mok = mok && tpq::make_xmap(&h->xmap1_32, h->d_x1, K1, 2 * tpq::kNPad) &&
                tpq::make_xmap(&h->xmap2_32, h->d_y1, n, 2 * tpq::kNPad);
          for (int v = 0; v < 3; ++v)
            mok = mok && tpq::make_xmap(&h->mm1[v], h->d_x1, K1, 64 << v) && tpq::make_xmap(&h->mm2[v], h->d_y1, n, 64 << v);
          mok = mok && tpq::make_xmap(&h->ss1, h->d_x1, K1, kGemmRows, 128) &&
                tpq::make_xmap(&h->ss2, h->d_y1, n, kGemmRows, 128);
        }
        if (!mok) return fail(TPQ_ECUDA, "cuTensorMapEncodeTiled failed for the activation buffers");
        if (unord) {
          TPQ_CUDA(cudaMemcpy(h->d_tab, h->tab1.data(), h->tab1.size() * 4, cudaMemcpyHostToDevice));
          TPQ_CUDA(cudaMemcpy((uint32_t*)h->d_tab + h->tab1.size(), h->tab2.data(), h->tab2.size() * 4,
                              cudaMemcpyHostToDevice));
          h->L1.meta = (const uint32_t*)h->d_tab;
          h->L2.meta = (const uint32_t*)h->d_tab + h->tab1.size();
        }
        h->L1.colf = h->d_colf;
        h->L2.colf = h->d_colf + n;
        {  // tiles split between CTAs by the stream-K partition (CTA c owns [c U / grid, (c+1) U / grid))
          std::vector<int> sp;
          int n1 = 0;
          for (int layer = 0; layer < 2; ++layer) {
            const tpq::LayerDev& L = layer ? h->L2 : h->L1;
            auto cta_of = [&](int64_t u) { return (int)(((u + 1) * L.grid + L.U - 1) / L.U) - 1; };
            for (int t = 0; t < L.NT && L.csize == 1; ++t)
              if (cta_of((int64_t)t * L.NKB) != cta_of((int64_t)(t + 1) * L.NKB - 1)) sp.push_back(t);
            if (layer == 0) n1 = (int)sp.size();
          }
          const size_t nsp = std::max<size_t>(1, sp.size()), ncnt = 4 * (size_t)(h->L1.NT + h->L2.NT);
          if ((r = A((void**)&h->d_split, (nsp + ncnt) * 4))) return r;
          TPQ_CUDA(cudaMemset(h->d_split + nsp, 0, ncnt * 4));
          h->L1.cnt = h->d_split + nsp;  // split-tile arrival counters of the in-kernel reduction
          h->L2.cnt = h->L1.cnt + 4 * h->L1.NT;  // [NT][4 epilogue warps] per layer
          if (!sp.empty()) TPQ_CUDA(cudaMemcpy(h->d_split, sp.data(), sp.size() * 4, cudaMemcpyHostToDevice));
          h->L1.split_tiles = h->d_split;
          h->L1.nsplit = n1;
          h->L2.split_tiles = h->d_split + n1;
          h->L2.nsplit = (int)sp.size() - n1;
        }
        h->L1.packed = (const uint8_t*)h->d_w1;
        h->L2.packed = (const uint8_t*)h->d_w2;
        h->L1.ws = h->d_ws;
        h->L2.ws = h->d_ws + ws1;  // separate partial slots per layer
        h->L1.ws_mm = wm1 ? h->d_ws + ws1 + ws2 : nullptr;
        h->L2.ws_mm = wm2 ? h->d_ws + ws1 + ws2 + wm1 : nullptr;
        h->L1.ws_ss = ws1s ? h->d_ws + ws1 + ws2 + wm1 + wm2 : nullptr;
        h->L2.ws_ss = ws2s ? h->d_ws + ws1 + ws2 + wm1 + wm2 + ws1s : nullptr;
        TPQ_CUDA(cudaDeviceSynchronize());
        return TPQ_OK;
      };
      if ((rc = upload())) {
        free_dev(h);
        delete h;
        return rc;
      }
    }
    *out = h;
    return TPQ_OK;
  } catch (const std::bad_alloc&) {
    if (h) { free_dev(h); delete h; }
    return fail(TPQ_ENOMEM, "tp_shard_mlp: out of host memory");
  } catch (...) {
    if (h) { free_dev(h); delete h; }
    return fail(TPQ_EINVAL, "tp_shard_mlp: unexpected exception");
  }
}

}  // namespace

extern "C" {

int tp_shard_mlp(const gptq_layer* w1, const gptq_layer* w2, const int32_t* P1, const int32_t* P2, int tp, int rank,
                 int variant, int64_t M_max, int device, tpq_mlp** out) {
  return shard_impl(w1, nullptr, w2, P1, nullptr, P2, tp, rank, variant, M_max, device, out);
}

int tp_shard_gated_mlp(const gptq_layer* wg, const gptq_layer* wu, const gptq_layer* wd, const int32_t* P1g,
                       const int32_t* P1u, const int32_t* P2, int tp, int rank, int variant, int64_t M_max, int device,
                       tpq_mlp** out) {
  if (!wu) return fail(TPQ_EINVAL, "tp_shard_gated_mlp: wu is NULL");
  return shard_impl(wg, wu, wd, P1g, P1u, P2, tp, rank, variant, M_max, device, out);
}

int tpq_mlp_destroy(tpq_mlp* h) {
  if (!h) return TPQ_OK;
  free_dev(h);  // the attached comm is not owned
  delete h;
  return TPQ_OK;
}

int tpq_comm_unique_id(uint8_t out[128]) {
  if (!out) return fail(TPQ_EINVAL, "NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  TPQ_NCCL(ncclGetUniqueId(&id));
  memcpy(out, &id, 128);
  return TPQ_OK;
}

int tpq_comm_create(const uint8_t id[128], int tp, int rank, int device, tpq_comm** out) {
  if (!id || !out) return fail(TPQ_EINVAL, "NULL");
  *out = nullptr;
  if (tp < 1 || rank < 0 || rank >= tp) return fail(TPQ_EINVAL, "tp=%d rank=%d", tp, rank);
  if (device < 0) return fail(TPQ_EINVAL, "device=%d", device);
  TPQ_CUDA(cudaSetDevice(device));
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  ncclComm_t c = nullptr;
  TPQ_NCCL(ncclCommInitRank(&c, tp, uid, rank));
  tpq_comm* tc = new (std::nothrow) tpq_comm{c, tp, rank, device};
  if (!tc) {
    ncclCommDestroy(c);
    return fail(TPQ_ENOMEM, "tpq_comm_create");
  }
  *out = tc;
  return TPQ_OK;
}

int tpq_comm_destroy(tpq_comm* c) {
  if (!c) return TPQ_OK;
  ncclResult_t r = ncclCommDestroy(c->comm);
  delete c;
  if (r != ncclSuccess) return fail(TPQ_ENCCL, "ncclCommDestroy: %s", ncclGetErrorString(r));
  return TPQ_OK;
}

int tpq_mlp_set_comm(tpq_mlp* h, tpq_comm* c) {
  if (!h) return fail(TPQ_EINVAL, "NULL handle");
  if (!c) {
    h->comm = nullptr;
    return TPQ_OK;
  }
  if (h->device < 0) return fail(TPQ_ESTATE, "host-only handle has no device");
  if (c->tp != h->tp || c->rank != h->rank || c->device != h->device)
    return fail(TPQ_EINVAL, "comm (tp=%d rank=%d dev=%d) does not match handle (tp=%d rank=%d dev=%d)", c->tp, c->rank,
                c->device, h->tp, h->rank, h->device);
  h->comm = c->comm;
  return TPQ_OK;
}

}  // extern "C"

namespace {

int check_fwd(tpq_mlp* h, const void* X, int64_t M, const void* Y) {
  if (!h || !X || !Y) return fail(TPQ_EINVAL, "NULL argument");
  if (h->device < 0) return fail(TPQ_ESTATE, "host-only handle (device=-1) cannot run the forward");
  if (M < 1 || M > h->M_max) return fail(TPQ_EINVAL, "M=%lld not in [1, M_max=%lld]", (long long)M, (long long)h->M_max);
  return TPQ_OK;
}

// Gather + layer 1 + (naive: AllGather + P2 gather) + layer 2 for one chunk of <= 16 rows.
// Writes the rank-local partial Y2 (row-major [mc][N2] at Y).  `collective` enables the naive
// AllGather (tp > 1); otherwise the naive path must be at tp == 1.


// Passes of 17..32 rows run the GEMV pipeline with N = 32 (dequant-bound like M <= 16, one weight
// pass instead of the A7 GEMM's) for the plain TP-aware / naive MLP.
bool gemv32(const tpq_mlp* h, int64_t mc) {
  return mc > tpq::kMaxM && mc <= 2 * tpq::kMaxM && h->rows > tpq::kMaxM && !h->gated && h->variant != TPQ_UNORDERED &&
         !getenv("TPQ_NO_GEMV32");
}

// One dequant-GEMM layer for mc rows: the GEMV (mc <= 16) or the A7 tensor-core GEMM (mc <= 512:
// k_dqgemm below 128 rows, the SS GEMMs from 128).
// Small shards (both layers' weights well inside L2) are latency-bound, not bandwidth-bound: layer 1
// prefetches layer 2's weights into L2 (Llama TP=8 M=1: 13.9 -> 13.5 us; prefetching layer 1's from
// the gather kernel as well gained nothing and stretched the gather).
constexpr int64_t kPrefetchMax = 48ll << 20;
const void* pf_layer2(const tpq_mlp* h, int64_t* bytes) {
  const int64_t b1 = h->L1.U * tpq::unit_bytes(h->L1.G) * (h->L1.gated ? 2 : 1), b2 = h->L2.U * tpq::unit_bytes(h->L2.G);
  *bytes = 0;
  if (b1 + b2 > kPrefetchMax || getenv("TPQ_NO_PF")) return nullptr;
  *bytes = b2;
  return h->L2.packed;
}

cudaError_t run_layer(tpq_mlp* h, int layer, int mc, void* out, int64_t out_ld, cudaStream_t st) {
  const tpq::LayerDev& L = layer == 1 ? h->L1 : h->L2;
  // N = 32 passes keep the layer's partition: stream-K, or clusters small enough for the N = 32 landing
  // zone (a layer planned in clusters of 4 -- Llama TP=8 layer 1 -- runs the A7 GEMM instead: its
  // stream-K fallback with ~6 contributors per tile measured 19.6 against 11.7 us)
  if (mc <= tpq::kMaxM || (gemv32(h, mc) && L.csize <= tpq::gemv_cluster_max32(L.G))) {
    int64_t pfb = 0;
    const void* pf = layer == 1 ? pf_layer2(h, &pfb) : nullptr;
    const bool w = mc > tpq::kMaxM;
    return tpq::launch_gemv(L, layer == 1 ? (w ? h->xmap1_32 : h->xmap1) : (w ? h->xmap2_32 : h->xmap2),
                            layer == 1 && L.gated ? &h->xmap1u : nullptr, mc, out, out_ld, st, pf, pfb,
                            layer == 1 ? &h->L2 : nullptr);
  }
  if (mc > kMmRows || (mc >= 128 && !getenv("TPQ_NO_SS")))  // compute-bound: activations as the reused A operand
    return tpq::launch_gemm_ss(L, layer == 1 ? h->ss1 : h->ss2, mc, h->sms, out, out_ld, st);
  const int v = mc <= 64 ? 0 : mc <= 128 ? 1 : 2;
  return tpq::launch_gemm(L, layer == 1 ? h->mm1[v] : h->mm2[v], 64 << v, mc, out, out_ld, st);
}

// Rows per pass of the forward: 16 (GEMV) while M <= 16, else up to 512 (A7).
int64_t pass_rows(const tpq_mlp* h, int64_t M) {
  return M <= tpq::kMaxM ? tpq::kMaxM : gemv32(h, M) ? 2 * tpq::kMaxM : h->rows;
}

int chunk_forward(tpq_mlp* h, const uint16_t* X, int mc, void* Y, cudaStream_t st, bool collective) {
  TPQ_CUDA(tpq::launch_gather_rowmajor(X, h->K1, h->d_P1, tpq::GATHER_COLS, 0, mc, h->K1, h->d_x1, st));  // X[:,P1]
  if (h->gated)  // gate_proj variant: the up layer's own act_order, X[:, P1u]
    TPQ_CUDA(tpq::launch_gather_rowmajor(X, h->K1, h->d_P1u, tpq::GATHER_COLS, 0, mc, h->K1, h->d_x1u, st));
  if (h->variant != TPQ_NAIVE) {
    // Alg. 3 L1 (TPQ_UNORDERED: P1 = identity, checkpoint order): Y1_local is already in the row order of this rank's W2[P2] block (no exchange)
    TPQ_CUDA(run_layer(h, 1, mc, h->d_y1, h->n, st));
  } else {
    // Alg. 2 L1 into this rank's slot of the AllGather buffer [tp][mc][n]
    uint8_t* slot = (uint8_t*)h->d_buf + (size_t)h->rank * mc * h->n * 2;
    TPQ_CUDA(run_layer(h, 1, mc, slot, h->n, st));
    if (h->tp > 1) {
      if (!collective) return fail(TPQ_ESTATE, "naive variant with tp > 1 needs the AllGather (use tp_mlp_forward)");
      TPQ_NCCL(ncclAllGather(slot, h->d_buf, (size_t)mc * h->n, ncclFloat16, h->comm, st));  // Alg. 2 L2
    }
    // Alg. 2 L3-4: Y1_global[:, P2] then CHUNK(rank), fused into one gather
    TPQ_CUDA(tpq::launch_gather_allgather(h->d_buf, h->d_gcols, (int)h->n, mc, h->d_y1, st));
  }
  TPQ_CUDA(run_layer(h, 2, mc, Y, h->N2, st));  // L2 GEMM
  return TPQ_OK;
}

int forward_impl(tpq_mlp* h, const void* X, int64_t M, void* Y, cudaStream_t st, bool collective) {
  if (collective && h->tp > 1 && !h->comm) return fail(TPQ_ESTATE, "tp=%d requires tpq_mlp_set_comm", h->tp);
  TPQ_CUDA(cudaSetDevice(h->device));
  const int64_t R = pass_rows(h, M);
  for (int64_t m0 = 0; m0 < M; m0 += R) {
    const int mc = (int)std::min<int64_t>(R, M - m0);
    int rc = chunk_forward(h, (const uint16_t*)X + m0 * h->K1, mc, (uint8_t*)Y + (size_t)m0 * h->N2 * 2, st,
                           collective);
    if (rc) return rc;
  }
  if (collective && h->tp > 1)  // Alg. 2 L6 / Alg. 3 L3
    TPQ_NCCL(ncclAllReduce(Y, Y, (size_t)M * h->N2, ncclFloat16, ncclSum, h->comm, st));
  return TPQ_OK;
}

}  // namespace

extern "C" {

int tp_mlp_forward(tpq_mlp* h, const void* X, int64_t M, void* Y, void* stream) {
  int rc = check_fwd(h, X, M, Y);
  if (rc) return rc;
  return forward_impl(h, X, M, Y, (cudaStream_t)stream, true);
}

int tp_mlp_forward_local(tpq_mlp* h, const void* X, int64_t M, void* Y2_local, void* stream) {
  int rc = check_fwd(h, X, M, Y2_local);
  if (rc) return rc;
  return forward_impl(h, X, M, Y2_local, (cudaStream_t)stream, false);
}

int tp_mlp_forward_host(tpq_mlp* h, const uint16_t* X_host, int64_t M, uint16_t* Y_host, void* stream) {
  int rc = check_fwd(h, X_host, M, Y_host);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  TPQ_CUDA(cudaSetDevice(h->device));
  TPQ_CUDA(cudaMemcpyAsync(h->d_xin, X_host, (size_t)M * h->K1 * 2, cudaMemcpyHostToDevice, st));
  if ((rc = forward_impl(h, h->d_xin, M, h->d_yout, st, true))) return rc;
  TPQ_CUDA(cudaMemcpyAsync(Y_host, h->d_yout, (size_t)M * h->N2 * 2, cudaMemcpyDeviceToHost, st));
  TPQ_CUDA(cudaStreamSynchronize(st));
  return TPQ_OK;
}

int tpq_layer1(tpq_mlp* h, const void* X, int64_t M, void* Y1_local, void* stream) {
  int rc = check_fwd(h, X, M, Y1_local);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  TPQ_CUDA(cudaSetDevice(h->device));
  const int64_t R = pass_rows(h, M);
  for (int64_t m0 = 0; m0 < M; m0 += R) {
    const int mc = (int)std::min<int64_t>(R, M - m0);
    TPQ_CUDA(tpq::launch_gather_rowmajor((const uint16_t*)X + m0 * h->K1, h->K1, h->d_P1, tpq::GATHER_COLS, 0, mc,
                                         h->K1, h->d_x1, st));
    if (h->gated)
      TPQ_CUDA(tpq::launch_gather_rowmajor((const uint16_t*)X + m0 * h->K1, h->K1, h->d_P1u, tpq::GATHER_COLS, 0, mc,
                                           h->K1, h->d_x1u, st));
    TPQ_CUDA(run_layer(h, 1, mc, (uint8_t*)Y1_local + (size_t)m0 * h->n * 2, h->n, st));
  }
  return TPQ_OK;
}

int tpq_naive_gather(tpq_mlp* h, const void* buf, int64_t M, void* Y1in, void* stream) {
  int rc = check_fwd(h, buf, M, Y1in);
  if (rc) return rc;
  if (h->variant != TPQ_NAIVE) return fail(TPQ_EINVAL, "tpq_naive_gather needs a TPQ_NAIVE handle");
  TPQ_CUDA(cudaSetDevice(h->device));
  TPQ_CUDA(tpq::launch_gather_allgather(buf, h->d_gcols, (int)h->n, (int)M, Y1in,
                                       (cudaStream_t)stream));
  return TPQ_OK;
}

int tpq_layer2(tpq_mlp* h, const void* Y1in, int64_t M, void* Y2_local, void* stream) {
  int rc = check_fwd(h, Y1in, M, Y2_local);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  TPQ_CUDA(cudaSetDevice(h->device));
  const int64_t R = pass_rows(h, M);
  for (int64_t m0 = 0; m0 < M; m0 += R) {
    const int mc = (int)std::min<int64_t>(R, M - m0);
    // the GEMV reads its activations through the TMA view of d_y1
    TPQ_CUDA(tpq::launch_gather_rowmajor((const uint16_t*)Y1in + m0 * h->n, h->n, nullptr, tpq::GATHER_COLS, 0, mc,
                                         h->n, h->d_y1, st));
    TPQ_CUDA(run_layer(h, 2, mc, (uint8_t*)Y2_local + (size_t)m0 * h->N2 * 2, h->N2, st));
  }
  return TPQ_OK;
}

int tpq_sum_partials(const void* const* parts, int nparts, int64_t count, void* out, void* stream) {
  if (!parts || !out || nparts < 1 || nparts > 8 || count < 0) return fail(TPQ_EINVAL, "bad arguments");
  for (int i = 0; i < nparts; ++i)
    if (!parts[i]) return fail(TPQ_EINVAL, "parts[%d] is NULL", i);
  if (count == 0) return TPQ_OK;
  TPQ_CUDA(tpq::launch_sum_partials(parts, nparts, count, out, (cudaStream_t)stream));
  return TPQ_OK;
}

#ifdef TPQ_PROF
// Profiling build only (libtpq_prof.so): per-CTA GEMV timeline of the last launches.
int tpq_debug_cta(unsigned long long* out) { return tpq::cta_read(out) ? TPQ_ECUDA : TPQ_OK; }
int tpq_debug_trace(long long* out) { return tpq::trace_read(out) ? TPQ_ECUDA : TPQ_OK; }
#endif

int tpq_mlp_run_step(tpq_mlp* h, int step, int64_t M, void* stream) {
  if (!h) return fail(TPQ_EINVAL, "NULL handle");
  if (h->device < 0) return fail(TPQ_ESTATE, "host-only handle (device=-1)");
  const int64_t mmax = std::min<int64_t>(h->rows, h->M_max);  // one pass: 16 rows (GEMV) or 512 (A7)
  if (M < 1 || M > mmax) return fail(TPQ_EINVAL, "M=%lld not in [1, %lld]", (long long)M, (long long)mmax);
  cudaStream_t st = (cudaStream_t)stream;
  TPQ_CUDA(cudaSetDevice(h->device));
  const int mc = (int)M;
  switch (step) {
    case TPQ_STEP_GATHER:
      TPQ_CUDA(tpq::launch_gather_rowmajor(h->d_xin, h->K1, h->d_P1, tpq::GATHER_COLS, 0, mc, h->K1, h->d_x1, st));
      if (h->gated)
        TPQ_CUDA(tpq::launch_gather_rowmajor(h->d_xin, h->K1, h->d_P1u, tpq::GATHER_COLS, 0, mc, h->K1, h->d_x1u, st));
      return TPQ_OK;
    case TPQ_STEP_LAYER1:
      TPQ_CUDA(run_layer(h, 1, mc, h->d_y1, h->n, st));
      return TPQ_OK;
    case TPQ_STEP_LAYER2:
      TPQ_CUDA(run_layer(h, 2, mc, h->d_yout, h->N2, st));
      return TPQ_OK;
    case TPQ_STEP_NAIVE_GATHER:
      if (h->variant != TPQ_NAIVE) return fail(TPQ_EINVAL, "TPQ_STEP_NAIVE_GATHER needs a TPQ_NAIVE handle");
      TPQ_CUDA(tpq::launch_gather_allgather(h->d_buf, h->d_gcols, (int)h->n, mc, h->d_y1, st));
      return TPQ_OK;
    case TPQ_STEP_ALLGATHER:
      if (h->variant != TPQ_NAIVE) return fail(TPQ_EINVAL, "TPQ_STEP_ALLGATHER needs a TPQ_NAIVE handle");
      if (!h->comm) return fail(TPQ_ESTATE, "no communicator attached");
      TPQ_NCCL(ncclAllGather((uint8_t*)h->d_buf + (size_t)h->rank * mc * h->n * 2, h->d_buf, (size_t)mc * h->n,
                             ncclFloat16, h->comm, st));
      return TPQ_OK;
    case TPQ_STEP_ALLREDUCE:
      if (!h->comm) return fail(TPQ_ESTATE, "no communicator attached");
      TPQ_NCCL(ncclAllReduce(h->d_yout, h->d_yout, (size_t)M * h->N2, ncclFloat16, ncclSum, h->comm, st));
      return TPQ_OK;
    default:
      return fail(TPQ_EINVAL, "unknown step %d", step);
  }
}


int tpq_mlp_info(const tpq_mlp* h, tpq_mlp_info_t* o) {
  if (!h || !o) return fail(TPQ_EINVAL, "NULL");
  o->K1 = h->K1; o->N1 = h->N1; o->N2 = h->N2; o->n = h->n; o->M_max = h->M_max;
  o->G1 = h->G1; o->G2 = h->G2; o->tp = h->tp; o->rank = h->rank; o->variant = h->variant; o->device = h->device;
  o->w1_bytes = (int64_t)h->pk1.size();
  o->w2_bytes = (int64_t)h->pk2.size();
  o->units1 = h->L1.U;
  o->units2 = h->L2.U;
  o->grid1 = h->L1.grid;
  o->grid2 = h->L2.grid;
  o->has_comm = h->comm != nullptr;
  auto split = [](const tpq::LayerDev& L) { return L.csize > 1 ? L.csize : L.inred ? 0 : 1; };
  o->split1 = split(h->L1);
  o->split2 = split(h->L2);
  return TPQ_OK;
}

int tpq_mlp_index_maps(const tpq_mlp* h, int32_t* w1_cols, int32_t* w2_rows, int32_t* lo, int32_t* hi) {
  if (!h) return fail(TPQ_EINVAL, "NULL handle");
  if (w1_cols) memcpy(w1_cols, h->w1_cols.data(), h->n * 4);
  if (w2_rows) memcpy(w2_rows, h->w2_rows.data(), h->n * 4);
  if (lo) *lo = h->w2_group_lo;
  if (hi) *hi = h->w2_group_hi;
  return TPQ_OK;
}

int tpq_mlp_export_canonical(const tpq_mlp* h, int layer, uint8_t* q, uint16_t* s, uint8_t* z) {
  if (!h || !q || !s || !z) return fail(TPQ_EINVAL, "NULL");
  if (h->variant == TPQ_UNORDERED) {
    // codes from the records (checkpoint row order), scales from the table, zeros as packed
    const std::vector<uint8_t>& pk = layer == 1 ? h->pk1 : h->pk2;
    const std::vector<uint32_t>& tab = layer == 1 ? h->tab1 : h->tab2;
    const std::vector<int>& E = layer == 1 ? h->E1 : h->E2;
    const int64_t K = layer == 1 ? h->K1 : h->n, N = layer == 1 ? h->n : h->N2, G = layer == 1 ? h->G1 : h->G2;
    if (layer != 1 && layer != 2) return fail(TPQ_EINVAL, "layer=%d", layer);
    const int64_t NKB = K / tpq::kUnitK, UB = tpq::kUnitK * tpq::kTileCols / 2 + tpq::kUnitK;
    for (int64_t un = 0; un < (N / tpq::kTileCols) * NKB; ++un) {
      const int64_t t = un / NKB, kb = un % NKB;
      const uint32_t* words = reinterpret_cast<const uint32_t*>(pk.data() + un * UB);
      for (int j = 0; j < tpq::kTileCols; ++j)
        for (int ch = 0; ch < tpq::kUnitK / 32; ++ch)
          for (int w = 0; w < 4; ++w) {
            const uint32_t word = words[tpq::code_block(ch, j) * 4 + w];
            const int64_t k0 = kb * tpq::kUnitK + 32 * ch + 8 * w;
            for (int i = 0; i < 8; ++i) q[(k0 + i) * N + t * tpq::kTileCols + j] = (word >> (4 * kNibbleOfK[i])) & 0xF;
          }
    }
    for (int64_t g = 0; g < K / G; ++g)
      for (int64_t c = 0; c < N; ++c) {
        s[g * N + c] = half_scale_down((uint16_t)(tab[(size_t)(g * N + c)] & 0xFFFF), E[(size_t)c]);
        z[g * N + c] = (layer == 1 ? h->z1u : h->z2u)[(size_t)(g * N + c)];
      }
    return TPQ_OK;
  }
  if (h->gated && (layer == 1 || layer == 3)) {  // gate (1) / up (3) records of the interleaved layer 1
    const size_t UB = (size_t)tpq::unit_bytes(h->G1), nun = h->pk1.size() / (2 * UB);
    std::vector<uint8_t> part(nun * UB);
    for (size_t u = 0; u < nun; ++u) memcpy(part.data() + u * UB, h->pk1.data() + (2 * u + (layer == 3)) * UB, UB);
    unpack_layer(part, h->E1, h->K1, h->n, h->G1, q, s, z);
    return TPQ_OK;
  }
  if (layer == 1) unpack_layer(h->pk1, h->E1, h->K1, h->n, h->G1, q, s, z);
  else if (layer == 2) unpack_layer(h->pk2, h->E2, h->n, h->N2, h->G2, q, s, z);
  else return fail(TPQ_EINVAL, "layer=%d", layer);
  return TPQ_OK;
}

}  // extern "C"
