// Probe of the tcgen05 CTA-pair MMA (cta_group::2) operand / accumulator split on sm_100a:
// one cluster of 2 CTAs, one tcgen05.mma.cta_group::2.kind::f16 with M = 256, N = 256, K = 16.
// Each CTA writes 128 rows of A (its batch rows) and 128 rows of B (N/2 columns of the MMA) into
// its shared memory in the K-major SWIZZLE_128B layout; the leader issues the MMA; each CTA reads
// its accumulator lanes back.  The host checks D against A_full . B_full^T for the hypothesis
// "CTA r holds A rows [128 r, 128 r + 128) and B columns [128 r, 128 r + 128); its TMEM holds D rows
// [128 r, +128) x all 256 columns".
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/probe_2cta tools/probe_2cta.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ float aval(int r, int k) { return (float)(((r * 3 + k * 5) % 7) - 3); }
__device__ __forceinline__ float bval(int n, int k) { return (float)(((n * 7 + k * 3) % 9) - 4); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe(float* out) {
  __shared__ __align__(1024) uint8_t sa[128 * 128];
  __shared__ __align__(1024) uint8_t sb[128 * 128];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t s_tmem;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // row r of this CTA's A (global row 128 rank + r) and of its B (global column 128 rank + r), k < 16
  for (int r = tid; r < 128; r += 128) {
    for (int k = 0; k < 64; ++k) {
      const int c = k / 8, off = (r / 8) * 1024 + (r % 8) * 128 + ((c ^ (r % 8)) * 16) + (k % 8) * 2;
      const float av = k < 16 ? aval(128 * rank + r, k) : 0.f, bv = k < 16 ? bval(128 * rank + r, k) : 0.f;
      *reinterpret_cast<__half*>(sa + off) = __float2half(av);
      *reinterpret_cast<__half*>(sb + off) = __float2half(bv);
    }
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&s_tmem)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  // instruction descriptor: D f32, A/B f16 K-major, N = 256 (bits 17-22: N >> 3), M = 256 (bits 24-28: M >> 4)
  const uint32_t idesc = (1u << 4) | ((256u >> 3) << 17) | ((256u >> 4) << 24);
  if (rank == 0 && tid == 0) {
    const uint64_t ad = desc_sw128(smem_u32(sa)), bd = desc_sw128(smem_u32(sb));
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(ad), "l"(bd), "r"(idesc)
        : "memory");
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)),
        "h"((uint16_t)3)
        : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
          smem_u32(&bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // lane quarter of warp w = TMEM lanes 32 w .. 32 w + 31 = this CTA's D rows
  for (int c0 = 0; c0 < 256; c0 += 16) {
    uint32_t v[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int q = 0; q < 16; ++q) out[(128 * rank + 32 * warp + lane) * 256 + c0 + q] = __uint_as_float(v[q]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

static float aval_h(int r, int k) { return (float)(((r * 3 + k * 5) % 7) - 3); }
static float bval_h(int n, int k) { return (float)(((n * 7 + k * 3) % 9) - 4); }

int main() {
  float* d;
  cudaMalloc(&d, 256 * 256 * 4);
  cudaMemset(d, 0xFF, 256 * 256 * 4);
  probe<<<2, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("kernel error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> h(256 * 256);
  cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0, bad_swapB = 0;
  for (int m = 0; m < 256; ++m)
    for (int n = 0; n < 256; ++n) {
      float ref = 0.f;
      for (int k = 0; k < 16; ++k) ref += aval_h(m, k) * bval_h(n, k);
      if (h[m * 256 + n] != ref) ++bad;
      // alternative hypothesis: each CTA's D uses only its own B half (columns duplicated)
      float ref2 = 0.f;
      for (int k = 0; k < 16; ++k) ref2 += aval_h(m, k) * bval_h((m / 128) * 128 + (n % 128), k);
      if (h[m * 256 + n] != ref2) ++bad_swapB;
    }
  printf("split hypothesis mismatches: %d / 65536; own-B-only hypothesis: %d\n", bad, bad_swapB);
  printf("D[0][0..3] = %g %g %g %g ; D[200][130..131] = %g %g\n", h[0], h[1], h[2], h[3], h[200 * 256 + 130], h[200 * 256 + 131]);
  return bad != 0;
}
