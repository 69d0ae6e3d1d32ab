// Internal interface between the host half (tpq_host.cpp) and the sm_100a kernels
// (tpq_kernels.cu).  Not part of the C-ABI.
//
// Device data layout:
//
// Packed layer shard (K rows in Alg.-1 order, N columns): 128-column TILES x 128-row K-BLOCKS.
// Unit (t, kb) is one contiguous record of unit_bytes(G) = 8192 + 320 * (128 / G) bytes,
// tile-major at offset (t * NKB + kb) * unit_bytes(G):
//   [0, 8192)                 int4 codes: 16-byte block code_block(c, j) = c * 128 + (j ^ 2c) holds
//                             chunk c (k = 128 kb + 32c .. +31) of column j (0..127); u32 word w of a chunk holds k0 = 32c + 8w .. k0+7 as
//                             nibbles n0=q[k0] n4=q[k0+1] n1=q[k0+2] n5=q[k0+3] n2=q[k0+4]
//                             n6=q[k0+5] n3=q[k0+6] n7=q[k0+7]  (LOP3 magic-number extraction
//                             yields f16x2 pairs of consecutive k = one TMEM column of the MMA
//                             A operand)
//   [8192 + 256 gi, +256)     fp16 s' = s 2^E of column j, group gi of the block (gi < 128 / G);
//                             E >= 0 per column (tpq_host.cpp column_exponents, LayerDev::colf)
//   [8192 + 256 (128/G) + 64 gi, +64)   int4 zero of column j, group gi (byte j/2, nibble j%2)
//
// Activations (GEMV input) and outputs are plain row-major fp16 [M][ld]; the layer-1 input is the
// gathered X[:, P1], the layer-1 output is the layer-2 input (TP-aware: already in P2 order).
#pragma once
#include <cuda.h>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

namespace tpq {

constexpr int kTileCols = 128;      // weight columns per tile (= TMEM lanes = MMA M)
constexpr int kUnitK = 128;         // weight rows per unit (8 MMAs of K = 16)
constexpr int kNPad = 16;           // batch rows per MMA (tcgen05 M=128 needs N % 16 == 0)
constexpr int kMaxM = 16;           // rows per forward chunk
constexpr int64_t unit_bytes_c(int G) { return (int64_t)kUnitK * kTileCols / 2 + 320LL * (kUnitK / G); }
inline int64_t unit_bytes(int G) { return unit_bytes_c(G); }
#ifdef __CUDACC__
#define TPQ_HD __host__ __device__
#else
#define TPQ_HD
#endif
// 16-byte code block of (chunk c, column j) inside a record: column XOR-swizzled by 2c within its
// aligned group of 8 (a permutation inside each aligned 8-column group, so the dequant warps' lanes,
// reading 8 consecutive columns of one chunk per quarter-warp, stay conflict-free).
TPQ_HD constexpr int code_block(int c, int j) { return c * kTileCols + (j ^ (2 * c)); }

struct LayerDev {
  const uint8_t* packed = nullptr;  // device
  int64_t K = 0, N = 0;
  int G = 0, NT = 0, NKB = 0;
  int64_t U = 0;           // NT * NKB units
  int grid = 0;            // persistent CTAs of the M <= 16 GEMV (stream-K), at most one per SM
  int grid_mm = 0;         // persistent CTAs of the A7 k_dqgemm (every SM)
  float* ws = nullptr;     // [grid][2 slots][16][128] fp32 stream-K partials of the GEMV (slot 0 = first segment)
  int csize = 1;           // > 1: cluster split-K (grid = NT x csize, one tile per cluster, DSMEM reduction)
  int inred = 0;           // 1: split tiles reduced inside the GEMV (cnt); 0: by the fix-up kernel after it
  int* cnt = nullptr;      // [NT][4] split-tile arrival counters of the GEMV, one per epilogue warp (zeroed at upload,
                           // re-armed by each reducer)
  float* ws_mm = nullptr;  // [grid_mm][2 slots][256][128] fp32 stream-K partials (A7 GEMM)
  float* ws_ss = nullptr;  // [items][128][128] fp32 k-split partials (A7 SS GEMM, M >= 128)
  const float* colf = nullptr;  // [N] 2^(24 - E_n): records hold s' = s 2^E_n (tpq_host.cpp column_exponents)
  const uint32_t* meta = nullptr;  // unordered layer (TPQ_UNORDERED): [ng][N] {fp16 s', fp16 -z s' 2^-24}
  int unord = 0;                   // 1: records in checkpoint row order with per-row group ids (k_dqgemv<0>)
  const int* split_tiles = nullptr;  // [nsplit] tiles of this layer split between CTAs (k_split_fixup's grid)
  int nsplit = 0;
  int gated = 0;                   // 1: gate_proj layer 1: gate(t, kb), up(t, kb) record pairs; U counts the pairs
};

enum GatherMode { GATHER_COLS = 0, GATHER_ALLGATHER = 1 };

// Set the GEMV kernel attributes (dynamic shared memory) on the current device; false on failure.
bool gemv_prepare(int G);
// Largest cluster size of the GEMV's cluster split-K for group size G (shared-memory landing zone).
int gemv_cluster_max(int G);
int gemv_cluster_max32(int G);  // the same for the N = 32 pipeline (17 <= M <= 32)

// out[m][n] = sum_k x[m][k] deq(W)[k][n] for M <= 16 rows (k_dqgemv + its split-tile fix-up); x is
// a [16][K] fp16 row-major buffer described by `xmap` (make_xmap, 16-row boxes), out is [M][out_ld]
// fp16 row-major.
// Gated layer (L.gated): xmap = X[:, P1g] (gate records), xmapu = X[:, P1u] (up records), out =
// fp16(SiLU(gate) * up); otherwise xmapu may be NULL.
// pf / pf_bytes (optional): a weight range (the next layer of a small shard) each CTA prefetches a
// share of into L2 after its own ring fill.
cudaError_t launch_gemv(const LayerDev& L, const CUtensorMap& xmap, const CUtensorMap* xmapu, int M, void* out,
                        int64_t out_ld, cudaStream_t st, const void* pf = nullptr, int64_t pf_bytes = 0,
                        const LayerDev* next = nullptr);

// A7 (M > 16): out[m][n] = sum_k x[m][k] deq(W)[k][n] for M <= nb rows (nb in {64, 128, 256}), x a
// [nb][K] fp16 row-major buffer described by xmap (make_xmap with rows = nb), out [M][out_ld].
cudaError_t launch_gemm(const LayerDev& L, const CUtensorMap& xmap, int nb, int M, void* out, int64_t out_ld,
                        cudaStream_t st);

// Tensor map of a [16][K] fp16 row-major activation buffer for the GEMV's TMA: box (64 k, 16 rows)
// with 128-byte swizzle = half a unit's slice in the K-major SW128 operand layout.  Returns false
// if the driver entry point is unavailable or encoding fails.
bool make_xmap(CUtensorMap* map, const void* base, int64_t K, int rows, int box_rows = 0);

// Weight columns per SS GEMM work item.  256 (two tiles, G = 128 only: shared memory) measured
// slower than 128 on Llama TP=8 (M = 128: 48.0 vs 39.6 us; the 256-column variant has only two
// activation stages), so it is selectable for experiments only (TPQ_SS_BN=256).
inline int ss_bn(int NT, int G) {
  static const bool wide = [] {
    const char* e = getenv("TPQ_SS_BN");
    return e && e[0] == '2';
  }();
  return wide && NT % 2 == 0 && G == 128 ? 256 : 128;
}

// The CTA-pair SS GEMM (k_dqgemm_ss2, cta_group::2: 256 batch rows x 256 weight columns per pair)
// for passes of more than 128 rows over an even tile count.  TPQ_SS2=0 selects the 1-CTA kernel.
inline bool ss_pair(int NT, int M) {
  static const bool off = [] {
    const char* e = getenv("TPQ_SS2");
    return e && e[0] == '0';
  }();
  return !off && NT % 2 == 0 && M > 128;
}

// k-splits of the SS GEMM for `mb` 128-row blocks and NG column groups: as many as keep the work items within one wave
// of `sms` CTAs, at least 4 k-blocks per split, at most 16 splits.
inline int ss_splits(int NG, int NKB, int mb, int sms) {
  const int base = mb * NG;
  int S = sms / base;
  const int cap = NKB / 4 < 16 ? NKB / 4 : 16;
  if (S > cap) S = cap;
  return S < 1 ? 1 : S;
}

// A7 for M >= 128 (<= 512 rows per pass): mixed-input SS GEMM, xmap = the [512][K] buffer with
// 128-row boxes; k-splits chosen to cover `sms` SMs (partials in L.ws_ss, k_ss_fixup).
cudaError_t launch_gemm_ss(const LayerDev& L, const CUtensorMap& xmap, int M, int sms, void* out, int64_t out_ld,
                           cudaStream_t st);

// Row-major gather dst[m*K + k] = v(m, k):
//   GATHER_COLS:      v(m, k) = src[m*ld + (idx ? idx[k] : k)]; idx holds K int32 indices followed by
//                     the same K as uint16 (read by the staged-row kernel, K <= 24576 there)
//   GATHER_ALLGATHER: c = idx[k]; v(m, k) = src[(c / nn) * M * nn + m * nn + c % nn]
cudaError_t launch_gather_rowmajor(const void* src, int64_t ld, const int32_t* idx, int mode, int64_t nn, int M,
                                   int64_t K, void* dst, cudaStream_t st);

#ifdef TPQ_PROF
int cta_read(unsigned long long* out);
int trace_read(long long* out);
#endif

// Naive Alg. 2 L3-4: dst[m][i] = buf[so[i].x][m][so[i].y], buf = the AllGather buffer [tp][M][n], so =
// int2 (c / n, c % n) per local column i.
cudaError_t launch_gather_allgather(const void* buf, const void* so, int n, int M, void* dst, cudaStream_t st);

cudaError_t launch_sum_partials(const void* const* parts, int nparts, int64_t count, void* out, cudaStream_t st);

}  // namespace tpq
