// Internal interface between the host half (tpq_host.cpp) and the sm_100a kernels
// (tpq_kernels.cu).  Not part of the C-ABI.
//
// Device data layout:
//
// Packed layer shard (K rows in Alg.-1 order, N columns): 128-column TILES x G-row GROUPS.
// Unit (t, g) is one contiguous record of unit_bytes(G) = 64*G + 320 bytes, tile-major at
// offset (t*NG + g)*unit_bytes(G):
//   [0, 64G)          int4 codes: chunk c (k = 32c..32c+31) x column j (0..127) x 16 bytes;
//                     u32 word w of a chunk holds k0 = 32c + 8w .. k0+7 as nibbles
//                     n0=q[k0] n4=q[k0+1] n1=q[k0+2] n5=q[k0+3] n2=q[k0+4] n6=q[k0+5]
//                     n3=q[k0+6] n7=q[k0+7]  (so LOP3 magic-number extraction yields f16x2
//                     pairs of consecutive k = one TMEM column of the MMA A operand)
//   [64G, 64G+256)    fp16 scale of column j
//   [64G+256, +64)    int4 zero of column j (byte j/2, nibble j%2)
//
// Activation operand ("xext", compact): per group g, 16 row records of G+16 halves; element
// (m, kk) at halves (g*16 + m)*(G+16) + kk.  Values: x[m][gG+kk] at "lo" slots (kk%4 in {0,1}),
// x[m][gG+kk]/16 at "hi" slots (the A operand holds 1024+q resp. 1024+16q there); correction slots
// kk = G, G+1: fp16 split of S_B = sum_kk B ; G+2, G+3: fp16 split of S_x = sum_lo B + 16 sum_hi B ;
// G+4..G+15: 0.  The A operand holds (-1024, -1024, -z, -z) at the correction slots, so
// D = sum_k (q - z) x exactly up to fp32 rounding.  Only rows m < M are written / read: the GEMV
// copies them (cp.async) into the tcgen05 K-major SWIZZLE_NONE canonical B layout in shared memory
// (8x16-byte core matrices, LBO 128 B between k-halves, SBO (G+16)*16 B between row groups).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tpq {

constexpr int kTileCols = 128;      // weight columns per CTA tile (= TMEM lanes)
constexpr int kNPad = 16;           // batch rows per MMA (tcgen05 M=128 needs N % 16 == 0)
constexpr int kMaxM = 16;           // rows per forward chunk
inline int64_t unit_bytes(int G) { return 64LL * G + 320; }
inline int64_t xext_group_bytes(int G) { return (int64_t)kNPad * (G + 16) * 2; }
inline int64_t xext_bytes(int64_t K, int G) { return (K / G) * xext_group_bytes(G); }

struct LayerDev {
  const uint8_t* packed = nullptr;  // device
  int64_t K = 0, N = 0;
  int G = 0, NT = 0, NG = 0;
  int64_t U = 0;           // NT * NG units
  int grid = 0;            // persistent CTAs (stream-K)
  float* ws = nullptr;     // [grid][2 slots][16][128] fp32 stream-K partials
  int* cnt = nullptr;      // [NT] arrival counters (self-resetting)
};

enum OutMode { OUT_ROWMAJOR = 0, OUT_XEXT = 1 };
enum GatherMode { GATHER_COLS = 0, GATHER_ALLGATHER = 1 };

// Max co-resident CTAs of the GEMV kernel per SM for group size G; 0 on failure.  Also
// raises the kernel's dynamic shared memory limit on the current device.
int gemv_blocks_per_sm(int G);

// out = X @ deq(W) for M <= 16 rows, X given as xext (B operand, see above).
//   OUT_ROWMAJOR: fp16 out[m*out_ld + n];  OUT_XEXT: xext of the next layer (K' = N, G' = next_G).
cudaError_t launch_gemv(const LayerDev& L, const void* xext, int M, void* out, int out_mode, int64_t out_ld,
                        int next_G, cudaStream_t st);

// xext (K columns, group size G) from row-major activations, M <= 16:
//   GATHER_COLS:      v(m, k) = src[m*ld + (idx ? idx[k] : k)]
//   GATHER_ALLGATHER: c = idx[k]; v(m, k) = src[(c / nn) * M * nn + m * nn + c % nn]
cudaError_t launch_to_xext(const void* src, int64_t ld, const int32_t* idx, int mode, int64_t nn, int M, int64_t K,
                           int G, void* dst, cudaStream_t st);

// Row-major variant of the gather (staged API): dst[m*K + k] = v(m, k), any M.
cudaError_t launch_gather_rowmajor(const void* src, int64_t ld, const int32_t* idx, int mode, int64_t nn, int M,
                                   int64_t K, void* dst, cudaStream_t st);

#ifdef TPQ_PROF
int prof_read(unsigned long long* out);
int trace_read(long long* out);
#endif

cudaError_t launch_sum_partials(const void* const* parts, int nparts, int64_t count, void* out, cudaStream_t st);

}  // namespace tpq
