// Does tcgen05.commit -> mbarrier fire only when the MMAs complete, when the
// commit directly follows another commit (the executor's empty/tfull pattern)?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4); d |= (uint64_t)1 << 16; d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61; return d;
}
__device__ __forceinline__ void wait_bar(uint64_t* b, uint32_t par) {
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(smem_u32(b)), "r"(par));
}
__global__ void __launch_bounds__(160, 1) k(int n, int nkb, int pace, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t empty, tfull;
  __shared__ uint32_t tbase;
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  const int tid = threadIdx.x;
  for (int i = tid; i < (16384 + 32768) / 4; i += 160) ((uint32_t*)base)[i] = 0x3f803f80u;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tfull)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t a = smem_u32(base), b = smem_u32(base + 16384);
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  __shared__ long long t_issue_end;
  if (tid == 128) {   // MMA thread (warp 4)
    for (int kb = 0; kb < nkb; ++kb) {
      long long tw = clock64();
      while (clock64() - tw < pace) {}
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = make_sdesc(a + kk * 32), bd = make_sdesc(b + kk * 32);
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tbase), "l"(ad), "l"(bd), "r"(idesc), "r"((kb | kk) ? 1 : 0));
      }
      if (mode == 0)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&empty)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&tfull)));
    t_issue_end = clock64();
  }
  if (tid < 128) {   // epilogue warps 0-3
    long long t0 = clock64();
    wait_bar(&tfull, 0);
    long long t1 = clock64();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t taddr = tbase + ((uint32_t)((tid >> 5) * 32) << 16);
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    float s = 0; for (int j = 0; j < 16; ++j) s += __uint_as_float(r[j]);
    long long t2 = clock64();
    if (tid == 0) { out[0] = t1 - t0; out[1] = t2 - t0; out[3] = (long long)s; }
  }
  __syncthreads();
  if (tid == 0) out[2] = t_issue_end;
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}
int main() {
  long long* d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int mode : {0, 1})
    for (int n : {64, 256})
      for (int pace : {0, 600}) {
        const int nkb = 8;
        k<<<1, 160, 64 * 1024>>>(n, nkb, pace, mode, d);
        cudaDeviceSynchronize();
        long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
        // expected MMA busy time: nkb * 4 * (128*n*16*2/8192) clk
        printf("mode=%s N=%d pace=%d: tfull seen at %lld clk, tmem data at %lld clk (MMA work %d clk) sum=%lld %s\n",
               mode == 0 ? "empty+tfull commits" : "tfull commit only", n, pace, h[0], h[1], nkb * 4 * (128 * n * 16 * 2 / 8192),
               h[3], cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
