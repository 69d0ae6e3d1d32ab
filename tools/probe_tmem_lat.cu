// Micro-benchmark: latency of (a) 4 warps tcgen05.st 64 columns + wait::st, (b) 9 chained
// tcgen05.mma kind::f16 M=128 N=16 K=16 (A from TMEM) issue -> commit arrival, (c) tcgen05.ld x16.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probe_tmem_lat tools/probe_tmem_lat.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t clk() {
  uint64_t c;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(c));
  return c;
}
__device__ __forceinline__ long long cyc() { return clock64(); }

template <int nmma, int nchain, int N>
__global__ void bench(long long* out, int reps) {
  __shared__ __align__(1024) uint8_t bsm[9 * 512 * (N / 16)];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 9 * 512 * (N / 16); i += blockDim.x) bsm[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tmem_base;
  uint32_t r[64];
  for (int i = 0; i < 64; ++i) r[i] = 0x3C003C00u * (i & 1);
  long long t_st = 0, t_mma = 0, t_ld = 0;
  uint32_t phase = 0;
  for (int rep = 0; rep < reps; ++rep) {
    __syncthreads();
    long long a = cyc();
    const uint32_t taddr = tb + ((uint32_t)(warp * 32) << 16) + 32;
#define R4(b) "r"(r[b]), "r"(r[b + 1]), "r"(r[b + 2]), "r"(r[b + 3])
#define R16(b) R4(b), R4(b + 4), R4(b + 8), R4(b + 12)
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,"
        "%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,"
        "%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64};" ::"r"(taddr),
        R16(0), R16(16), R16(32), R16(48)
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    long long b = cyc();
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    long long c = cyc();
    if (warp == 0) {  // whole warp, warp-uniform operands; one elected lane issues
      const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
      const uint32_t sbase = smem_u32(bsm);
#pragma unroll
      for (int j = 0; j < nmma; ++j) {
        const uint32_t saddr = sbase + (j % 9) * 512;
        const uint64_t desc = (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)8 << 16) | ((uint64_t)16 << 32) | (1ull << 46);
        const uint32_t acc = j >= nchain;
        const uint32_t dcol = tb + 160 + (j % nchain) * N, acol = tb + 32 + (j % 8) * 8;
        asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dcol),
                     "r"(acol), "l"(desc), "r"(idesc), "r"(acc));
      }
      asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar)));
    }
    asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n}" ::"r"(smem_u32(&bar)),
                 "r"(phase));
    phase ^= 1;
    long long d = cyc();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t v[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
                   "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(tb + ((uint32_t)(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    long long e = cyc();
    r[0] += v[0] & 1;
    if (rep > 0) {
      t_st += b - a;
      t_mma += d - c;
      t_ld += e - d;
    }
  }
  if (tid == 0) {
    out[0] = t_st / (reps - 1);
    out[1] = t_mma / (reps - 1);
    out[2] = t_ld / (reps - 1);
    out[3] = r[0];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(512));
}

int main() {
  long long* out;
  cudaMallocManaged(&out, 64);
#define RUN(NM, NC, NN)                                                                                   \
  {                                                                                                       \
    bench<NM, NC, NN><<<1, 128>>>(out, 20);                                                               \
    cudaError_t e = cudaDeviceSynchronize();                                                              \
    if (e != cudaSuccess) {                                                                               \
      printf("error %s\n", cudaGetErrorString(e));                                                        \
      return 1;                                                                                           \
    }                                                                                                     \
    printf("N=%d nchain=%d nmma=%d: st64+wait %lld, mma->commit %lld cyc, ld16 %lld\n", NN, NC, NM, out[0], out[1], \
           out[2]);                                                                                       \
  }
  RUN(9, 1, 16) RUN(36, 1, 16) RUN(36, 4, 16) RUN(72, 4, 16) RUN(36, 1, 64) RUN(36, 4, 64) RUN(36, 1, 128)
  return 0;
}
