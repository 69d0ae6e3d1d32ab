// Probe: validate tcgen05.mma kind::f16 with A from TMEM (written by tcgen05.st, 32x32b),
// B from shared memory (K-major, SWIZZLE_NONE canonical layout), D fp32 in TMEM read back
// with tcgen05.ld 32x32b.  M=128 (A rows = TMEM lanes), N=16, K=16*KB.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/probe tools/probe_tcgen05.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>

constexpr int M = 128, N = 16, KB = 3, K = 16 * KB;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __half* A /*[M][K]*/, const __half* B /*[N][K] (B^T: row n holds k)*/, float* D /*[M][N]*/,
                      int variant) {
  __shared__ __align__(1024) uint8_t bsm[KB * 512 * (N / 16)];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  // B -> smem canonical K-major no-swizzle: for k16 block j, n-group ng (8 rows), k-half kg:
  // core matrix of 8 rows x 16 B at j*(N/8)*256 + ng*256 + kg*128 ; row r at +16r
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    const int j = k / 16, kg = (k % 16) / 8, e = k % 8, ng = n / 8, r = n % 8;
    reinterpret_cast<__half*>(bsm)[(j * (N / 8) * 256 + ng * 256 + kg * 128 + r * 16) / 2 + e] = B[n * K + k];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(128));
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
  const uint32_t a_col = 32, d_col = 0;  // A at columns [32, 32 + K/2), D at [0, N)
  // A row (lane) = 32*warp + lane ; K/2 columns of f16x2 (low half = even k)
  {
    const int row = warp * 32 + lane;
    uint32_t r[K / 2];
    for (int c = 0; c < K / 2; ++c) {
      __half2 h = __halves2half2(A[row * K + 2 * c], A[row * K + 2 * c + 1]);
      r[c] = *reinterpret_cast<uint32_t*>(&h);
    }
    const uint32_t taddr = tb + ((uint32_t)(warp * 32) << 16) + a_col;
    static_assert(K / 2 == 24, "x24 below");
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr + 16), "r"(r[16]),
                 "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    // idesc: c_format F32 (bit4), a/b F16 (0), K-major both, n_dim = N>>3 at bit 17, m_dim = M>>4 at bit 24
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int j = 0; j < KB; ++j) {
      const uint32_t saddr = smem_u32(bsm) + j * (N / 8) * 256;
      uint64_t desc = 0;
      desc |= (uint64_t)((saddr >> 4) & 0x3FFF);
      desc |= (uint64_t)((128 >> 4) & 0x3FFF) << 16;  // LBO: between the two k-halves
      desc |= (uint64_t)((256 >> 4) & 0x3FFF) << 32;  // SBO: between 8-row groups
      desc |= (uint64_t)1 << 46;                      // version (sm100)
      if (variant == 1) {                             // swapped LBO/SBO (diagnostic)
        desc = (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(256 >> 4) << 16) | ((uint64_t)(128 >> 4) << 32) | (1ull << 46);
      }
      const uint32_t acc = j > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tb + d_col),
          "r"(tb + a_col + j * 8), "l"(desc), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  // wait
  asm volatile(
      "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    uint32_t v[16];
    const uint32_t taddr = tb + ((uint32_t)(warp * 32) << 16) + d_col;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int row = warp * 32 + lane;
    for (int n = 0; n < 16; ++n) D[row * N + n] = __uint_as_float(v[n]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(128));
}

int main() {
  __half *A, *B;
  float* D;
  cudaMallocManaged(&A, M * K * 2);
  cudaMallocManaged(&B, N * K * 2);
  cudaMallocManaged(&D, M * N * 4);
  srand(1);
  for (int i = 0; i < M * K; ++i) A[i] = __float2half((float)(rand() % 17 - 8));
  for (int i = 0; i < N * K; ++i) B[i] = __float2half((float)(rand() % 9 - 4) * 0.25f);
  for (int variant = 0; variant < 2; ++variant) {
    probe<<<1, 128>>>(A, B, D, variant);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("variant %d: CUDA error %s\n", variant, cudaGetErrorString(e));
      return 1;
    }
    int bad = 0;
    double maxerr = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)__half2float(A[m * K + k]) * __half2float(B[n * K + k]);
        double err = fabs(ref - D[m * N + n]);
        maxerr = fmax(maxerr, err);
        if (err > 1e-3) ++bad;
      }
    printf("variant %d: bad=%d / %d maxerr=%g  D[0][0..3]=%g %g %g %g\n", variant, bad, M * N, maxerr, D[0], D[1], D[2], D[3]);
  }
  return 0;
}
