// TMA load throughput: im2col (128 pixels x 64 ch of one tap) vs tiled 2D
// (128 rows x 64 cols) boxes, 148 CTAs streaming through a STAGES-deep ring,
// L2-resident source.  Reports GB/s chip-wide and per-box latency.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_bar(uint64_t* b, uint32_t par) {
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(smem_u32(b)), "r"(par));
}
template <int STAGES>
__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ CUtensorMap tm, int mode, int iters, int C, int Mtiles,
                                           int HoWo, int Wo, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t fullx[4][STAGES];
  uint8_t* base0 = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  const int np = out[7] > 0 ? (int)out[7] : 1;   // producers (warps) per CTA
  const int same = out[6] > 0;              // producers = lanes of warp 0 (else lane 0 of warps)
  const int w = same ? (threadIdx.x < 32 ? threadIdx.x : 99) : ((threadIdx.x & 31) ? 99 : threadIdx.x >> 5);
  if (w >= np) return;
  uint64_t* full = fullx[w];
  uint8_t* base = base0 + w * STAGES * 16384;
  for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  long long t0 = clock64();
  const int cb = C / 64;
  for (int i = 0; i < iters; ++i) {
    const int s = i % STAGES;
    if (i >= STAGES) wait_bar(&full[s], ((i / STAGES) - 1) & 1);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(16384));
    const uint32_t dst = smem_u32(base + s * 16384);
    const int mt = (blockIdx.x * np + w + gridDim.x * np * (i / (9 * cb))) % Mtiles;
    const int kb = i % (9 * cb);
    if (mode == 0) {
      const int m0 = mt * 128, img = m0 / HoWo, rem = m0 - img * HoWo, ho = rem / Wo, wo = rem - ho * Wo;
      const int tap = kb / cb, c0 = (kb % cb) * 64;
      const uint16_t r = tap / 3, sx = tap % 3;
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
                   " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};\n" ::"r"(dst), "l"(&tm), "r"(smem_u32(&full[s])),
                   "r"(c0), "r"(wo - 1), "r"(ho - 1), "r"(img), "h"(sx), "h"(r) : "memory");
    } else {
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n"
                   ::"r"(dst), "l"(&tm), "r"(smem_u32(&full[s])), "r"((kb % (9 * cb)) * 64 % (C * 9)), "r"(mt * 128) : "memory");
    }
  }
  for (int i = iters; i < iters + STAGES; ++i) { const int s = i % STAGES; wait_bar(&full[s], ((i / STAGES) - 1) & 1); }
  long long t1 = clock64();
  if (blockIdx.x == 0 && w == 0) out[0] = t1 - t0;
}
int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc_t; PFN_cuTensorMapEncodeIm2col_v12000 enc_i;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc_t, cudaEnableDefault, &q);
  cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", (void**)&enc_i, cudaEnableDefault, &q);
  long long* d; cudaMalloc(&d, 64);
  const int B = 8;
  for (int hw : {56}) for (int C : {256}) {
    void* x; size_t bytes = (size_t)B * hw * hw * C * 2; cudaMalloc(&x, bytes * 9); cudaMemset(x, 0, bytes * 9);
    const int M = B * hw * hw, Mtiles = (M + 127) / 128;
    CUtensorMap ti, tt;
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)hw, (cuuint64_t)hw, (cuuint64_t)B};
    cuuint64_t st[3] = {(cuuint64_t)C * 2, (cuuint64_t)C * 2 * hw, (cuuint64_t)C * 2 * hw * hw};
    int lo[2] = {-1, -1}, up[2] = {-1, -1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r1 = enc_i(&ti, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, x, dims, st, lo, up, 64, 128, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint64_t d2[2] = {(cuuint64_t)C * 9, (cuuint64_t)M};
    cuuint64_t s2[1] = {(cuuint64_t)C * 9 * 2};
    cuuint32_t box[2] = {64, 128};
    CUresult r2 = enc_t(&tt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, d2, s2, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int mode : {0, 1}) for (int grid : {148}) for (int np : {1, 2, 4}) for (int same : {0, 1}) {
      const int stages = 4;
      const int iters = 2000;
      auto kern = k<4>;
      long long npv[8] = {0, 0, 0, 0, 0, 0, same, np};
      cudaMemcpy(d, npv, 64, cudaMemcpyHostToDevice);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, np * stages * 16384 + 1024);
      kern<<<grid, 128, np * stages * 16384 + 1024>>>(mode ? tt : ti, mode, 50, C, Mtiles, hw * hw, hw, d);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      kern<<<grid, 128, np * stages * 16384 + 1024>>>(mode ? tt : ti, mode, iters, C, Mtiles, hw * hw, hw, d);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("hw=%d C=%d %s grid=%d np=%d same_warp=%d: %.2f TB/s chip, %.1f B/clk per SM (%s)\n", hw, C,
             mode ? "tiled2d" : "im2col ", grid, np, same, (double)grid * np * iters * 16384 / ms / 1e9,
             (double)np * iters * 16384 / h, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(x);
  }
  return 0;
}
