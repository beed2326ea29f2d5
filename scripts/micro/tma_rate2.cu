// Per-SM TMA throughput with the executor's stage shape: each stage = A
// (im2col 128 px x 64 ch, 16 KB) + B (tiled 128 rows x 64, 16 KB) on one
// mbarrier; NP producer threads (lane 0 of warps 0..NP-1) own stages
// round-robin (stage s -> producer s % NP), STAGES total.  A consumer thread
// frees stages in order (no MMA).  Reports B/clk per SM at grid 148.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4); d |= (uint64_t)1 << 16; d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61; return d;
}
__device__ __forceinline__ void wait_bar(uint64_t* b, uint32_t par) {
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(smem_u32(b)), "r"(par));
}
__global__ void __launch_bounds__(160, 1) k(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                                            int np, int stages, int iters, int C, int Mtiles, int HoWo, int Wo, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[8], empty[8];
  __shared__ uint32_t tbase;
  const int use_mma = out[6] > 0;
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  const int tid = threadIdx.x, w = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (tid >= 128) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int cb = C / 64;
  if ((tid & 31) == 0 && w < np) {
    for (int i = w; i < iters; i += np) {
      const int s = i % stages;
      if (i >= stages) wait_bar(&empty[s], ((i / stages) + 1) & 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(32768));
      const uint32_t da = smem_u32(base + s * 32768), db = da + 16384;
      const int mt = (blockIdx.x + gridDim.x * (i / (9 * cb))) % Mtiles;
      const int kb = i % (9 * cb);
      const int m0 = mt * 128, img = m0 / HoWo, rem = m0 - img * HoWo, ho = rem / Wo, wo = rem - ho * Wo;
      const int tap = kb / cb, c0 = (kb % cb) * 64;
      const uint16_t r = tap / 3, sx = tap % 3;
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
                   " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};\n" ::"r"(da), "l"(&ta), "r"(smem_u32(&full[s])),
                   "r"(c0), "r"(wo - 1), "r"(ho - 1), "r"(img), "h"(sx), "h"(r) : "memory");
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n"
                   ::"r"(db), "l"(&tb), "r"(smem_u32(&full[s])), "r"(kb * 64), "r"((blockIdx.x % 4) * 128) : "memory");
    }
  }
  if (tid == 128) {   // consumer
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int s = i % stages;
      wait_bar(&full[s], (i / stages) & 1);
      if (use_mma) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t a = smem_u32(base + s * 32768), b = a + 16384;
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        for (int kk = 0; kk < 4; ++kk)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tbase), "l"(make_sdesc(a + kk * 32)), "l"(make_sdesc(b + kk * 32)), "r"(idesc), "r"(1));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&empty[s])));
      } else {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])));
      }
    }
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid >= 128) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}
int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc_t; PFN_cuTensorMapEncodeIm2col_v12000 enc_i;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc_t, cudaEnableDefault, &q);
  cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", (void**)&enc_i, cudaEnableDefault, &q);
  long long* d; cudaMalloc(&d, 64);
  const int B = 8, hw = 28, C = 512;
  void* x; size_t bytes = (size_t)B * hw * hw * C * 2; cudaMalloc(&x, bytes); cudaMemset(x, 0, bytes);
  void* wt; size_t wb = (size_t)512 * 9 * C * 2; cudaMalloc(&wt, wb); cudaMemset(wt, 0, wb);
  const int M = B * hw * hw, Mtiles = (M + 127) / 128;
  CUtensorMap ti, tt;
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)hw, (cuuint64_t)hw, (cuuint64_t)B};
  cuuint64_t st[3] = {(cuuint64_t)C * 2, (cuuint64_t)C * 2 * hw, (cuuint64_t)C * 2 * hw * hw};
  int lo[2] = {-1, -1}, up[2] = {-1, -1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  enc_i(&ti, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, x, dims, st, lo, up, 64, 128, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t d2[2] = {(cuuint64_t)C * 9, 512};
  cuuint64_t s2[1] = {(cuuint64_t)C * 9 * 2};
  cuuint32_t box[2] = {64, 128};
  enc_t(&tt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, wt, d2, s2, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768 + 1024);
  for (int mma : {0, 1}) for (int grid : {148}) for (int stages : {4, 6}) for (int np : {1, 2, 4}) {
    if (np > stages) continue;
    long long hv[8] = {0, 0, 0, 0, 0, 0, mma, 0};
    cudaMemcpy(d, hv, 64, cudaMemcpyHostToDevice);
    const int iters = 1152;
    k<<<grid, 160, stages * 32768 + 1024>>>(ti, tt, np, stages, 72, C, Mtiles, hw * hw, hw, d);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<grid, 160, stages * 32768 + 1024>>>(ti, tt, np, stages, iters, C, Mtiles, hw * hw, hw, d);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("mma=%d grid=%d stages=%d np=%d: %.1f B/clk/SM, %.2f TB/s chip, %.0f clk per 32KB stage (%s)\n", mma, grid, stages, np,
           (double)iters * 32768 / h, (double)grid * iters * 32768 / ms / 1e9, (double)h / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
