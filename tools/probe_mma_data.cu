// Probe: does the tcgen05.mma (kind::f16, M=128, N=16, K=16, A from TMEM, B from smem) rate depend
// on the operand VALUES?  A patterns: zero, small integers (q - z in [-15, 15], the exact GEMV
// operand), random fp16 (s (q - z) with the scale folded in); B: zero or random fp16 (N(0,1)).
// One CTA, 4 warps store A, warp 0 issues 8 x 2000 MMAs back to back into one accumulator.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_mma_data tools/probe_mma_data.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}
__device__ __forceinline__ __half val(int pat, uint32_t seed) {
  const uint32_t h = hsh(seed);
  if (pat == 0) return __float2half(0.f);
  if (pat == 1) return __float2half((float)((int)(h % 31) - 15));                       // small integer
  if (pat == 2) return __float2half(((float)((int)(h % 31) - 15)) * 0.00173f);          // s (q - z)
  return __float2half(((float)(h & 0xFFFF) / 65536.f - 0.5f) * 3.4f);                   // ~N(0,1)-ish
}
__global__ void k(int apat, int bpat, int iters, long long* out) {
  __shared__ __align__(1024) __half bsm[16 * 128];  // 16 rows x 128 k, SW128 K-major (2 x 2 KB)
  __shared__ uint32_t tb_s;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 16 * 128; i += blockDim.x) bsm[i] = val(bpat, 7777 + i);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = __shfl_sync(~0u, tb_s, 0);
  // A: 64 columns (128 k as f16x2) at column 256, lane quarter = warp
  for (int c = 0; c < 64; ++c) {
    const __half2 v = __halves2half2(val(apat, (warp * 32 + lane) * 1000 + 2 * c), val(apat, (warp * 32 + lane) * 1000 + 2 * c + 1));
    const uint32_t u = *reinterpret_cast<const uint32_t*>(&v);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tb + ((uint32_t)(warp * 32) << 16) + 256 + c), "r"(u));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  long long t0 = clock64();
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(16 >> 3) << 17) | (8u << 24);
    const uint32_t sb = smem_u32(bsm);
    uint64_t bd[8];
    uint32_t aa[8];
    for (int j = 0; j < 8; ++j) {
      const uint32_t sa = sb + (j / 4) * 2048 + (j % 4) * 32;
      bd[j] = (uint64_t)((sa >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
      aa[j] = tb + 256 + j * 8;
    }
    for (int it = 0; it < iters; ++it) {
      uint32_t e;
      asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
      if (e) {
        for (int j = 0; j < 8; ++j)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tb),
                       "r"(aa[j]), "l"(bd[j]), "r"(idesc), "r"(it + j > 0 ? 1 : 0)
                       : "memory");
      }
      __syncwarp();
    }
    if (lane == 0)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(smem_u32(&bar)));
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}
int main() {
  long long* out;
  cudaMallocManaged(&out, 64);
  const int iters = 4000;
  const char* an[4] = {"zero", "int(q-z)", "s(q-z)", "rand"};
  const char* bn[4] = {"zero", "-", "-", "rand"};
  for (int ap : {0, 1, 2, 3})
    for (int bp : {0, 3}) {
      k<<<1, 128>>>(ap, bp, iters, out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      printf("A %-9s B %-5s: %.1f cycles per MMA\n", an[ap], bn[bp], (double)out[0] / (iters * 8));
    }
  return 0;
}
