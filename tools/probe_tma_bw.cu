// Micro-benchmark: HBM streaming bandwidth with 1-D TMA bulk copies into a shared-memory ring
// (one producer lane, 4 consumer warps that wait full / arrive empty), vs ring depth and CTAs/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/probe_tma_bw tools/probe_tma_bw.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                   smem_u32(bar)),
               "r"(parity)
               : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int UNIT, int NS>
__global__ void __launch_bounds__(160) stream(const uint8_t* src, int64_t units, uint32_t* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * UNIT);
  uint64_t* empty = full + NS;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int64_t u0 = blockIdx.x * units / gridDim.x, u1 = (blockIdx.x + 1) * units / gridDim.x;
  const int nu = (int)(u1 - u0);
  if (warp == 4) {
    if (lane == 0)
      for (int i = 0; i < nu; ++i) {
        const int s = i % NS;
        if (i >= NS) mbar_wait(empty + s, ((i / NS) - 1) & 1);
        mbar_expect(full + s, UNIT);
        bulk(sm + s * UNIT, src + (u0 + i) * UNIT, UNIT, full + s);
      }
  } else {
    uint32_t acc = 0;
    for (int i = 0; i < nu; ++i) {
      const int s = i % NS;
      mbar_wait(full + s, (i / NS) & 1);
      acc ^= reinterpret_cast<const uint32_t*>(sm + s * UNIT)[threadIdx.x];
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
    }
    if (acc == 0x12345678) sink[0] = acc;
  }
}

template <int UNIT, int NS>
void run(const uint8_t* src, int64_t bytes, uint32_t* sink, int ctas_per_sm) {
  const int smem = NS * UNIT + 16 * NS;
  cudaFuncSetAttribute(stream<UNIT, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(stream<UNIT, NS>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  const int64_t units = bytes / UNIT;
  const int grid = 148 * ctas_per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  stream<UNIT, NS><<<grid, 160, smem>>>(src, units, sink);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) stream<UNIT, NS><<<grid, 160, smem>>>(src, units, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const cudaError_t e = cudaGetLastError();
  printf("unit %5d B, NS %2d, ctas/SM %d: %7.1f GB/s (in flight/SM %6d B) %s\n", UNIT, NS, ctas_per_sm,
         units * UNIT * 5 / (ms * 1e-3) / 1e9, NS * UNIT * ctas_per_sm, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  const int64_t bytes = 1ll << 30;
  uint8_t* src;
  uint32_t* sink;
  cudaMalloc(&src, bytes);
  cudaMalloc(&sink, 64);
  cudaMemset(src, 1, bytes);
  run<8576, 4>(src, bytes, sink, 1);
  run<8576, 4>(src, bytes, sink, 2);
  run<8576, 6>(src, bytes, sink, 2);
  run<8576, 8>(src, bytes, sink, 2);
  run<8576, 12>(src, bytes, sink, 1);
  run<8576, 20>(src, bytes, sink, 1);
  run<4288, 16>(src, bytes, sink, 2);
  run<17152, 6>(src, bytes, sink, 2);
  run<8512, 20>(src, bytes, sink, 1);
  run<8512, 24>(src, bytes, sink, 1);
  run<17024, 12>(src, bytes, sink, 1);
  run<32768, 6>(src, bytes, sink, 1);
  return 0;
}
