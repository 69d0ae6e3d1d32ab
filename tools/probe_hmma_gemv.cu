// Probe: can a register-dequant mma.sync (HMMA m16n8k16, f32 accumulate) inner loop retire a
// 128 x 128 int4 unit in the ~383 cycles per SM that HBM speed leaves on B200?  No global
// memory: codes and activations come from shared memory, so this is the compute ceiling.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_hmma_gemv tools/probe_hmma_gemv.cu
// One warp-step = 64 weight columns (four 16-column A fragments) x k16, N = 8 * NB batch rows.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));  // (a & b) | c
  return d;
}
__device__ __forceinline__ void hmma(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int NB>
__global__ void k(int iters, long long* out, float* sink) {
  __shared__ __align__(16) uint32_t codes[64 * 32 * 4];
  __shared__ __align__(16) __half xs[16 * 16 * 8];
  for (int i = threadIdx.x; i < 64 * 32 * 4; i += blockDim.x) codes[i] = i * 2654435761u;
  for (int i = threadIdx.x; i < 16 * 16 * 8; i += blockDim.x) xs[i] = __float2half(0.01f * (i % 7));
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float acc[4][NB][4], tot[4][NB][4];
#pragma unroll
  for (int f = 0; f < 4; ++f)
#pragma unroll
    for (int n = 0; n < NB; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[f][n][e] = tot[f][n][e] = 0.f;
  const __half2 zl = __float2half2_rn(1024.f + 7.f);
  const uint32_t xbase = (uint32_t)__cvta_generic_to_shared(xs) + (lane % 16) * 32 + (lane / 16) * 16;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint4 cw = reinterpret_cast<const uint4*>(codes)[((it * 8 + warp) & 63) * 32 + lane];
    uint32_t b[4];
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3])
                 : "r"(xbase + (it & 7) * 512));
    const uint32_t w[4] = {cw.x, cw.y, cw.z, cw.w};
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const uint32_t x = w[f], x8 = x >> 8;
      uint32_t a[4];
      __half2 t;
      t = __hsub2(*reinterpret_cast<const __half2*>(&(a[0] = lop3(x, 0x000F000Fu, 0x64006400u))), zl);
      a[0] = *reinterpret_cast<uint32_t*>(&t);
      t = __hsub2(*reinterpret_cast<const __half2*>(&(a[1] = lop3(x8, 0x000F000Fu, 0x64006400u))), zl);
      a[1] = *reinterpret_cast<uint32_t*>(&t);
      t = __hfma2(*reinterpret_cast<const __half2*>(&(a[2] = lop3(x, 0x00F000F0u, 0x64006400u))),
                  __float2half2_rn(0.0625f), __float2half2_rn(-71.f));
      a[2] = *reinterpret_cast<uint32_t*>(&t);
      t = __hfma2(*reinterpret_cast<const __half2*>(&(a[3] = lop3(x8, 0x00F000F0u, 0x64006400u))),
                  __float2half2_rn(0.0625f), __float2half2_rn(-71.f));
      a[3] = *reinterpret_cast<uint32_t*>(&t);
#pragma unroll
      for (int n = 0; n < NB; ++n) hmma(acc[f][n], a, b[2 * n], b[2 * n + 1]);
    }
    if ((it & 7) == 7) {  // group end (G = 128): fp32 scale, fresh accumulators
      const float s = 0.001f * (it & 15);
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int n = 0; n < NB; ++n)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            tot[f][n][e] = fmaf(s, acc[f][n][e], tot[f][n][e]);
            acc[f][n][e] = 0.f;
          }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float r = 0.f;
#pragma unroll
  for (int f = 0; f < 4; ++f)
#pragma unroll
    for (int n = 0; n < NB; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) r += tot[f][n][e];
  if (r == 1234.5f) sink[threadIdx.x] = r;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  long long* out;
  float* sink;
  cudaMallocManaged(&out, 148 * 8);
  cudaMalloc(&sink, 4096 * 4);
  const int iters = 4096;
  for (int nb : {1, 2})
    for (int warps : {4, 8, 12, 16, 24, 32}) {
      if (nb == 1) k<1><<<148, warps * 32>>>(iters, out, sink);
      else k<2><<<148, warps * 32>>>(iters, out, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      long long mx = 0;
      for (int i = 0; i < 148; ++i) mx = out[i] > mx ? out[i] : mx;
      // a 128 x 128 unit = 2 column halves x 8 k16 steps = 16 warp-steps
      const double units = (double)warps * iters / 16;
      printf("N=%2d warps=%2d: %.1f cycles per warp-step per SMSP, %.0f cycles per 128x128 unit per SM (budget ~383)\n",
             8 * nb, warps, (double)mx / (iters * (warps / 4.0)), (double)mx / units);
    }
  return 0;
}
