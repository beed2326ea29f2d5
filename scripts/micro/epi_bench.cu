// The executor's staged bf16 epilogue chunk loop (32 columns per step, shuffle
// scale/bias, clamp, RNE pack, swizzled STS, TMA store per 64 columns) run in
// isolation by 4 warps (one per SMSP) over a TMEM accumulator: cycles per
// 32-column chunk, to separate the code's own latency from interference.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) : "r"(taddr));
}

__device__ __forceinline__ void epi_chunk32(const uint32_t (&r)[32], const float* esc, const float* ebi, int cc0, int cin,
                                            uint32_t wbuf_s, int lane, float lo, float hi) {
#pragma unroll
  for (int g8 = 0; g8 < 4; ++g8) {
    const float4 s0 = *reinterpret_cast<const float4*>(esc + cc0 + g8 * 8);
    const float4 s1 = *reinterpret_cast<const float4*>(esc + cc0 + g8 * 8 + 4);
    const float4 b0 = *reinterpret_cast<const float4*>(ebi + cc0 + g8 * 8);
    const float4 b1 = *reinterpret_cast<const float4*>(ebi + cc0 + g8 * 8 + 4);
    const float sv[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
    const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    float y[8];
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      const float2 o = __ffma2_rn(make_float2(__uint_as_float(r[g8 * 8 + j]), __uint_as_float(r[g8 * 8 + j + 1])),
                                  make_float2(sv[j], sv[j + 1]), make_float2(bv[j], bv[j + 1]));
      y[j] = o.x; y[j + 1] = o.y;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) y[j] = fminf(fmaxf(y[j], lo), hi);
    const uint32_t ch = (uint32_t)((cin + g8 * 8) >> 3);
    sts128(wbuf_s + lane * 128 + ((ch ^ (lane & 7)) << 4), pack_bf16x2(y[0], y[1]), pack_bf16x2(y[2], y[3]),
           pack_bf16x2(y[4], y[5]), pack_bf16x2(y[6], y[7]));
  }
}
__device__ __forceinline__ void pin32(uint32_t (&r)[32]) {
#pragma unroll
  for (int i = 0; i < 32; ++i) asm volatile("" : "+r"(r[i]));
}
__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ CUtensorMap tmc, int bn, int reps, int use_tma, int variant, long long* out) {
  __shared__ __align__(1024) uint8_t stage[4 * 4096];
  __shared__ float esc[256], ebi[256];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, q = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 256; i += 128) { esc[i] = 1.0f + i * 1e-3f; ebi[i] = 0.01f * i; }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t taddr = tbase + ((uint32_t)(q * 32) << 16);
  const uint32_t wbuf_s = smem_u32(stage + q * 4096);
  const float lo = 0.0f, hi = INFINITY;
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    if (variant == 3) {
      uint32_t ra[32], rb[32];
      tmem_ld16_nw(taddr, ra); tmem_ld16_nw(taddr + 16, ra + 16);
      for (int c = 0; c < bn; c += 64) {
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        pin32(ra);
        const bool two = c + 32 < bn;
        if (two) { tmem_ld16_nw(taddr + c + 32, rb); tmem_ld16_nw(taddr + c + 48, rb + 16); }
        if (c > 0 && use_tma) {
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
        }
        epi_chunk32(ra, esc, ebi, c, 0, wbuf_s, lane, lo, hi);
        if (two) {
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          pin32(rb);
          if (c + 64 < bn) { tmem_ld16_nw(taddr + c + 64, ra); tmem_ld16_nw(taddr + c + 80, ra + 16); }
          epi_chunk32(rb, esc, ebi, c + 32, 32, wbuf_s, lane, lo, hi);
        }
        if (use_tma) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tmc), "r"(wbuf_s),
                         "r"(c), "r"((blockIdx.x * 128 + q * 32) % 4096) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      }
    } else if (variant == 4) {
      // variant 1 math, no TMEM pipelining, x32 load
      for (int c = 0; c < bn; c += 32) {
        uint32_t r[32];
        tmem_ld16_nw(taddr + c, r); tmem_ld16_nw(taddr + c + 16, r + 16);
        const int cin = c & 63;
        if (cin == 0 && c > 0 && use_tma) {
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        pin32(r);
        epi_chunk32(r, esc, ebi, c, cin, wbuf_s, lane, lo, hi);
        if ((cin == 32 || c + 32 >= bn) && use_tma) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tmc), "r"(wbuf_s),
                         "r"(c - cin), "r"((blockIdx.x * 128 + q * 32) % 4096) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      }
    } else if (variant == 2) {
      uint32_t ra[32], rb[32];
      tmem_ld16_nw(taddr, ra); tmem_ld16_nw(taddr + 16, ra + 16);
      for (int c = 0; c < bn; c += 64) {
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 32; ++i) asm volatile("" : "+r"(ra[i]));
        if (c + 32 < bn) { tmem_ld16_nw(taddr + c + 32, rb); tmem_ld16_nw(taddr + c + 48, rb + 16); }
        if (c > 0 && use_tma) {
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
        }
        for (int half = 0; half < 2; ++half) {
          if (half == 1) {
            if (c + 32 >= bn) break;
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < 32; ++i) asm volatile("" : "+r"(rb[i]));
            if (c + 64 < bn) { tmem_ld16_nw(taddr + c + 64, ra); tmem_ld16_nw(taddr + c + 80, ra + 16); }
          }
          const uint32_t* r = half ? rb : ra;
          const int cc0 = c + half * 32;
#pragma unroll
          for (int g8 = 0; g8 < 4; ++g8) {
            const float4 s0 = *reinterpret_cast<const float4*>(esc + cc0 + g8 * 8);
            const float4 s1 = *reinterpret_cast<const float4*>(esc + cc0 + g8 * 8 + 4);
            const float4 b0 = *reinterpret_cast<const float4*>(ebi + cc0 + g8 * 8);
            const float4 b1 = *reinterpret_cast<const float4*>(ebi + cc0 + g8 * 8 + 4);
            const float sv[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
            const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
            float y[8];
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
              const float2 o = __ffma2_rn(make_float2(__uint_as_float(r[g8 * 8 + j]), __uint_as_float(r[g8 * 8 + j + 1])),
                                          make_float2(sv[j], sv[j + 1]), make_float2(bv[j], bv[j + 1]));
              y[j] = o.x; y[j + 1] = o.y;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) y[j] = fminf(fmaxf(y[j], lo), hi);
            const uint32_t ch = (uint32_t)((half * 32 + g8 * 8) >> 3);
            sts128(wbuf_s + lane * 128 + ((ch ^ (lane & 7)) << 4), pack_bf16x2(y[0], y[1]), pack_bf16x2(y[2], y[3]),
                   pack_bf16x2(y[4], y[5]), pack_bf16x2(y[6], y[7]));
          }
        }
        if (use_tma) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tmc), "r"(wbuf_s),
                         "r"(c), "r"((blockIdx.x * 128 + q * 32) % 4096) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      }
    } else
    for (int c = 0; c < bn; c += 32) {
      uint32_t r[32];
      tmem_ld16_nw(taddr + c, r);
      tmem_ld16_nw(taddr + c + 16, r + 16);
      const float sc_l = esc[c + lane], bi_l = ebi[c + lane];
      const int cin = c & 63;
      if (cin == 0 && c > 0 && use_tma) {
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int g8 = 0; g8 < 4; ++g8) {
        float y[8];
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
          const int jj = g8 * 8 + j;
          float2 o;
          if (variant == 1) {
            o = __ffma2_rn(make_float2(__uint_as_float(r[jj]), __uint_as_float(r[jj + 1])),
                           *reinterpret_cast<const float2*>(esc + c + jj), *reinterpret_cast<const float2*>(ebi + c + jj));
          } else {
            o = __ffma2_rn(make_float2(__uint_as_float(r[jj]), __uint_as_float(r[jj + 1])),
                                      make_float2(__shfl_sync(0xffffffffu, sc_l, jj), __shfl_sync(0xffffffffu, sc_l, jj + 1)),
                                      make_float2(__shfl_sync(0xffffffffu, bi_l, jj), __shfl_sync(0xffffffffu, bi_l, jj + 1)));
          }
          y[j] = o.x; y[j + 1] = o.y;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) y[j] = fminf(fmaxf(y[j], lo), hi);
        const uint32_t ch = (uint32_t)((cin + g8 * 8) >> 3);
        sts128(wbuf_s + lane * 128 + ((ch ^ (lane & 7)) << 4), pack_bf16x2(y[0], y[1]), pack_bf16x2(y[2], y[3]),
               pack_bf16x2(y[4], y[5]), pack_bf16x2(y[6], y[7]));
      }
      if ((cin == 32 || c + 32 >= bn) && use_tma) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tmc), "r"(wbuf_s),
                       "r"(c - cin), "r"((blockIdx.x * 128 + q * 32) % 4096) : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (use_tma) {
      if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      __syncwarp();
    }
  }
  long long t1 = clock64();
  if (blockIdx.x == 0 && lane == 0) out[q] = (t1 - t0) / ((long long)reps * (bn / 32));
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}
int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc_t;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc_t, cudaEnableDefault, &qr);
  void* outbuf; cudaMalloc(&outbuf, 4096 * 256 * 2);
  CUtensorMap tm;
  cuuint64_t dims[2] = {256, 4096}; cuuint64_t st[1] = {256 * 2}; cuuint32_t box[2] = {64, 32}; cuuint32_t es[2] = {1, 1};
  enc_t(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, outbuf, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  long long* d; cudaMalloc(&d, 64);
  for (int variant : {0, 1, 3, 4}) for (int tma : {0, 1}) for (int bn : {64, 256}) for (int grid : {148}) {
    k<<<grid, 128>>>(tm, bn, 200, tma, variant, d);
    cudaDeviceSynchronize();
    long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("variant=%d tma_store=%d bn=%d grid=%d: clk per 32-col chunk %lld %lld %lld %lld (%s)\n", variant, tma, bn, grid, h[0], h[1], h[2], h[3],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
