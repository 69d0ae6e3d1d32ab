// Probe: TMEM store throughput (tcgen05.st 32x32b.x32 from many warps) and TS-MMA rate while
// other warps store.  nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probe_tmem_bw tools/probe_tmem_bw.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
#define R4(b) "r"(r[b]), "r"(r[b + 1]), "r"(r[b + 2]), "r"(r[b + 3])
#define R16(b) R4(b), R4(b + 4), R4(b + 8), R4(b + 12)
__device__ __forceinline__ void st32(uint32_t t, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
               "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(t), R16(0), R16(16) : "memory");
}
// mode 0: NW store warps, each `iters` x (st32 + wait::st); mode 1: the same without waits (one wait at end);
// mode 2: MMA only (warp 0 issues iters x 8 MMAs); mode 3: stores (no wait) + MMAs concurrently
__global__ void k(int mode, int iters, long long* out) {
  __shared__ __align__(1024) uint8_t bsm[4096];
  __shared__ uint32_t tb_s;
  __shared__ __align__(8) uint64_t bar, bar2;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) bsm[i] = 0;
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
  uint32_t r[32];
  for (int i = 0; i < 32; ++i) r[i] = lane * i;
  __syncthreads();
  long long t0 = clock64();
  const bool storer = (mode == 0 || mode == 1 || mode == 3) && warp >= 1;
  if (storer) {
    const uint32_t taddr = tb + ((uint32_t)((warp & 3) * 32) << 16) + 128 + ((warp >> 2) & 7) * 32;
    for (int it = 0; it < iters; ++it) {
      st32(taddr, r);
      if (mode == 0) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  if ((mode == 2 || mode == 3 || mode == 4 || mode == 5) && warp == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 17) | (8u << 24);
    const uint32_t sb = smem_u32(bsm);
    uint64_t bd[8];
    uint32_t aa[8];
    for (int j = 0; j < 8; ++j) {
      const uint32_t sa = sb + j * 512;
      bd[j] = (uint64_t)((sa >> 4) & 0x3FFF) | ((uint64_t)16 << 16) | ((uint64_t)8 << 32) | (1ull << 46);
      aa[j] = tb + 128 + j * 8;
    }
    for (int it = 0; it < iters; ++it) {
      uint32_t e;
      asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
      if (e) {
        for (int j = 0; j < 8; ++j)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tb),
                       "r"(aa[j]), "l"(bd[j]), "r"(idesc), "r"(j)
                       : "memory");
        if (mode == 4)  // commit after every unit of 8 MMAs (to a second barrier nobody waits on)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2)));
        if (mode == 5)
          for (int c = 0; c < 3; ++c)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2)));
      }
      __syncwarp();
    }
    if (lane == 0) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(smem_u32(&bar)));
  }
  long long t1 = clock64();
  __syncthreads();
  if (lane == 0) out[warp] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}
int main() {
  long long* out;
  cudaMallocManaged(&out, 64 * 8);
  const int iters = 1000;
  for (int mode = 2; mode < 6; ++mode)
    for (int nw : {2, 5, 9, 17}) {
      if (mode != 3 && nw != 2) continue;
      k<<<1, nw * 32>>>(mode, iters, out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      long long mx = 0;
      for (int w = 0; w < nw; ++w) mx = out[w] > mx ? out[w] : mx;
      const int nst = (mode != 3) ? 0 : nw - 1;
      printf("mode %d store-warps %2d: %lld cyc total; per st32/warp %.1f cyc; aggregate %.1f B/cyc; mma-warp %lld cyc (%.1f per MMA)\n",
             mode, nst, mx, nst ? (double)mx / iters : 0.0, nst ? (double)nst * iters * 4096 / mx : 0.0, out[0],
             (mode >= 2) ? (double)out[0] / (iters * 8) : 0.0);
    }
  return 0;
}
