// Probe: TS-MMA (A from TMEM) issue rate vs number of independent accumulator chains and N.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probe_mma_rate tools/probe_mma_rate.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(int chains, int N, int iters, int commits, long long* out) {
  __shared__ __align__(1024) uint8_t bsm[8192];
  __shared__ uint32_t tb_s;
  __shared__ __align__(8) uint64_t bar, bar2;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) bsm[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = __shfl_sync(~0u, tb_s, 0);
  long long t0 = clock64();
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    const uint32_t sb = smem_u32(bsm);
    uint64_t bd[8];
    uint32_t aa[8], dd[8];
    for (int j = 0; j < 8; ++j) {
      const uint32_t sa = sb + j * 512;
      bd[j] = (uint64_t)((sa >> 4) & 0x3FFF) | ((uint64_t)16 << 16) | ((uint64_t)8 << 32) | (1ull << 46);
      aa[j] = tb + 256 + j * 8;
      dd[j] = tb + (j % chains) * N;
    }
    for (int it = 0; it < iters; ++it) {
      uint32_t e;
      asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
      if (e) {
        for (int j = 0; j < 8; ++j)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dd[j]),
                       "r"(aa[j]), "l"(bd[j]), "r"(idesc), "r"(j >= chains ? 1 : 0)
                       : "memory");
        for (int c = 0; c < commits; ++c)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2)));
      }
      __syncwarp();
    }
    if ((threadIdx.x & 31) == 0)
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
  const int iters = 2000;
  for (int N : {8, 16, 32})
    for (int chains : {1, 2, 4, 8})
      for (int commits : {0, 3}) {
        k<<<1, 64>>>(chains, N, iters, commits, out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        printf("N=%2d chains=%d commits/unit=%d: %.1f cyc per MMA, %.0f per unit of 8\n", N, chains, commits,
               (double)out[0] / (iters * 8), (double)out[0] / iters);
      }
  return 0;
}
