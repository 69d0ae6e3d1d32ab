// Internal interface between the host half (tpq_host.cpp) and the sm_100a kernels
// (tpq_kernels.cu).  Not part of the C-ABI.
//
// Device data layout:
//   A layer shard (K rows in Alg.-1 order, N columns) is cut into 64-column BLOCKS and
//   G-row GROUPS.  Unit (b, g) = block b x group g is one contiguous record of
//   kUnitBytes(G) = 32*G + 160 bytes, stored block-major: offset (b*NG + g)*kUnitBytes(G).
//     [0, 32*G)        int4 codes in mma.sync m16n8k16 A-fragment order: for chunk c, tile t
//                      (16 columns), lane l: CW words (CW = min(4, G/16)), word s = the 8 codes
//                      lane l needs for k16-step s (nibbles n0..n7 = A elements
//                      (r0,k0) (r1,k0) (r0,k0+8) (r1,k0+8) (r0,k0+1) (r1,k0+1) (r0,k0+9) (r1,k0+9),
//                      r0 = 16t + l/4, r1 = r0 + 8, k0 = 16s + 2(l%4)).
//     [32G, 32G+128)   fp16 scales: [rr 0..7][t 0..3] half2 (s[r0], s[r1]) with r0 = 16t + rr
//     [32G+128, +160)  int4 zeros:  [rr 0..7][t 0..3] byte z[r0] | z[r1] << 4
//   Activations enter the GEMV in "frag" layout Xf[mt][K/32][lane][4 x u32]: the mma.sync
//   B fragments of rows m = 8mt + l/4 for two k16 steps.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tpq {

constexpr int kBlockCols = 64;
constexpr int kMetaBytes = 160;
constexpr int kThreads = 256;  // 8 warps per CTA
constexpr int kMaxMT = 2;      // GEMV path: M <= 16 (two m8 tiles)
inline int64_t unit_bytes(int G) { return 32LL * G + kMetaBytes; }

struct LayerDev {
  const uint8_t* packed = nullptr;  // device
  int64_t K = 0, N = 0;
  int G = 0, NB = 0, NG = 0;
  int64_t U = 0;           // NB * NG units
  int grid[kMaxMT + 1] = {0, 0, 0};  // CTAs for MT = 1, 2
  float* ws = nullptr;     // [max grid][2 slots][16 * 64] fp32 stream-K partials
  int* cnt = nullptr;      // [NB] arrival counters (self-resetting)
};

enum OutMode { OUT_ROWMAJOR = 0, OUT_FRAG = 1 };
enum GatherMode { GATHER_COLS = 0, GATHER_ALLGATHER = 1 };

// Max co-resident CTAs of the GEMV kernel per SM for (G, MT); 0 on failure.
int gemv_blocks_per_sm(int G, int MT);

// out = Xf @ W  for M <= 16 rows.  OUT_ROWMAJOR: fp16 out[m*out_ld + n];
// OUT_FRAG: fp16 frag layout for a following layer with K' = N.
cudaError_t launch_gemv(const LayerDev& L, const void* xf, int M, void* out, int out_mode,
                        int64_t out_ld, cudaStream_t st);

// dst (frag layout, M <= 16 rows, K columns) from row-major src:
//   GATHER_COLS:      v(m, k) = src[m*ld + (idx ? idx[k] : k)]
//   GATHER_ALLGATHER: c = idx[k]; v(m, k) = src[(c / nn) * M * nn + m * nn + c % nn]
cudaError_t launch_to_frag(const void* src, int64_t ld, const int32_t* idx, int mode, int64_t nn,
                           int M, int64_t K, void* dst, cudaStream_t st);

// Row-major variant of the gather (staged API): dst[m*K + k] = v(m, k), any M.
cudaError_t launch_gather_rowmajor(const void* src, int64_t ld, const int32_t* idx, int mode,
                                   int64_t nn, int M, int64_t K, void* dst, cudaStream_t st);

cudaError_t launch_sum_partials(const void* const* parts, int nparts, int64_t count, void* out,
                                cudaStream_t st);

}  // namespace tpq
