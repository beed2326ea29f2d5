// executor.cu -- sm_100a device code of the GACER executor.
//
// * gacer_executor: the persistent multi-tenant kernel (one CTA per SM).
//   Each CTA loops: claim the next item of the open cluster from a tenant
//   queue (its preferred tenant first), wait on the item's producer-chunk
//   counters, run the tile function, release the chunk and cluster counters.
//   The cluster counters implement the paper's synchronisation pointers
//   (§4.3 l.767-771: "operators continue to be deployed only after
//   previously issued operators have completed") on the device instead of the
//   CPU-GPU sync whose cost T_SW the paper charges in Eq. 8 (l.780-799).
// * op_gemm_kernel / op_cc_kernel: the SAME tile functions launched one
//   kernel per fused op -- the sequential ("CuDNN-Seq") and
//   multi-stream ("Stream-Parallel") baselines.
//
// Tile functions
// * gemm_item: bf16 implicit-GEMM conv (A = im2col of NHWC input gathered
//   with cp.async into 128B-swizzled smem, B = K-major packed weights) or
//   swap-AB linear, on tcgen05.mma (kind::f16, M=128, N=bn<=128, K=16) with
//   the fp32 accumulator in TMEM; fused epilogue scale/bias(+skip)(+act)
//   read back with tcgen05.ld.  Split-K partials are reduced by the last
//   arriving CTA in fixed ks order (bit-identical in every mode).
// * cc_item: depthwise conv / max / avg / global-avg pool / elementwise on
//   CUDA cores, 8 channels per thread with 128-bit NHWC accesses.
// * simt_item: fp32 conv/linear with FFMA in fixed K order (fp32 tenants).
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "gacer_dev.h"

namespace gacer {

// =====================================================================
// PTX helpers
// =====================================================================
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(sz)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_128B canonical layout:
// 8-row x 128-byte atoms (row r, 16B chunk j stored at chunk j ^ (r & 7)),
// atoms stacked every 1024 bytes (SBO).  Bits: [0,14) start>>4, [16,30)
// LBO>>4 (=1, unused for swizzled K-major), [32,46) SBO>>4, [46,48)
// version=1 (sm_100), [61,64) layout = 2 (SWIZZLE_128B).
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
// Instruction descriptor kind::f16: D fp32 (bit 4), A bf16 (bits 7-9 = 1),
// B bf16 (bits 10-12 = 1), both K-major, N>>3 at bits 17-22, M>>4 at 24-28.
__device__ __forceinline__ uint32_t make_idesc(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(BM >> 4) << 24);
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// bf16 <-> float helpers
__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);  // RNE, .x = a (low half)
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float apply_act(float v, int act) {
  if (act == ACT_RELU) v = fmaxf(v, 0.0f);
  else if (act == ACT_RELU6) v = fminf(fmaxf(v, 0.0f), 6.0f);
  return v;
}

// =====================================================================
// shared memory layout
// =====================================================================
constexpr int A_STAGE_BYTES = BM * 128;
constexpr int B_STAGE_BYTES = BN_MAX * 128;
constexpr int SMEM_RING_BYTES = STAGES * (A_STAGE_BYTES + B_STAGE_BYTES);

struct SmemCtl {
  uint64_t mma_done[STAGES];
  uint64_t acc_bar;
  uint32_t tmem_base;
  int32_t flag;
  Item item;
  int32_t claimed;
  float red[NTHREADS * 8 / 8 + 8];
};
constexpr int SMEM_GEMM_BYTES = SMEM_RING_BYTES + 1024 /*align slack*/ + (int)sizeof(SmemCtl) + 64;
constexpr int GAP_RED_FLOATS = NTHREADS * 8;   // per-thread 8-channel partials

struct Ctx {               // per-CTA persistent state (uniform across threads)
  uint8_t* ring;           // 1024-aligned
  SmemCtl* ctl;
  float* gap_red;          // NTHREADS*8 floats (aliases the ring; used only by CC items)
  uint32_t tmem;
  uint32_t ring_pos;       // K-blocks issued so far (smem ring position)
  uint32_t acc_uses;       // accumulator commits so far
};

// =====================================================================
// GEMM tile (tcgen05)
// =====================================================================
struct ARowInfo {
  const __nv_bfloat16* img;  // image base for the row's sample (conv) or row pointer (rows mode)
  int hi0, wi0;
  bool ok;
};

__device__ __forceinline__ void load_rows_tile(uint32_t stage_base, const __nv_bfloat16* src, int ld, int row0,
                                               int nrows, int row_limit, int k, int k_limit, int chunk,
                                               int rsub) {
  const bool kok = k < k_limit;
  for (int r = rsub; r < nrows; r += 32) {
    const int row = row0 + r;
    const bool ok = kok && row < row_limit;
    const __nv_bfloat16* s = ok ? src + static_cast<size_t>(row) * ld + k : src;
    const uint32_t dst = stage_base + r * 128 + ((chunk ^ (r & 7)) << 4);
    cp_async16(dst, s, ok);
  }
}

__device__ void epilogue_store8(const OpDev& op, int m, int n, const float* v) {
  // m: GEMM row, n: first of 8 GEMM columns
  if (!op.swap) {
    if (m >= op.M) return;
    if (n + 8 <= op.Cout) {
      float y[8];
      const float4 s0 = *reinterpret_cast<const float4*>(op.scale + n);
      const float4 s1 = *reinterpret_cast<const float4*>(op.scale + n + 4);
      const float4 b0 = *reinterpret_cast<const float4*>(op.bias + n);
      const float4 b1 = *reinterpret_cast<const float4*>(op.bias + n + 4);
      const float sc[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
      const float bi[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) y[j] = fmaf(v[j], sc[j], bi[j]);
      if (op.has_skip) {
        const uint4 u = *reinterpret_cast<const uint4*>(
            static_cast<const __nv_bfloat16*>(op.skip) + static_cast<size_t>(m) * op.lds + n);
        float s[8];
        bf16x8_to_f32(u, s);
#pragma unroll
        for (int j = 0; j < 8; ++j) y[j] += s[j];
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) y[j] = apply_act(y[j], op.act);
      if (op.out_f32) {
        float* o = static_cast<float*>(op.out) + static_cast<size_t>(m) * op.ldo + n;
        *reinterpret_cast<float4*>(o) = make_float4(y[0], y[1], y[2], y[3]);
        *reinterpret_cast<float4*>(o + 4) = make_float4(y[4], y[5], y[6], y[7]);
      } else {
        uint4 u;
        u.x = pack_bf16x2(y[0], y[1]);
        u.y = pack_bf16x2(y[2], y[3]);
        u.z = pack_bf16x2(y[4], y[5]);
        u.w = pack_bf16x2(y[6], y[7]);
        *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(op.out) + static_cast<size_t>(m) * op.ldo + n) = u;
      }
    } else {
      for (int j = 0; j < 8; ++j) {
        const int nn = n + j;
        if (nn >= op.Cout) break;
        float y = fmaf(v[j], op.scale[nn], op.bias[nn]);
        if (op.has_skip)
          y += __bfloat162float(static_cast<const __nv_bfloat16*>(op.skip)[static_cast<size_t>(m) * op.lds + nn]);
        y = apply_act(y, op.act);
        if (op.out_f32) static_cast<float*>(op.out)[static_cast<size_t>(m) * op.ldo + nn] = y;
        else static_cast<__nv_bfloat16*>(op.out)[static_cast<size_t>(m) * op.ldo + nn] = __float2bfloat16_rn(y);
      }
    }
  } else {
    // swap-AB: GEMM row m = output feature, GEMM column n = sample
    if (m >= op.Cout) return;
    const float sc = op.scale[m], bi = op.bias[m];
    for (int j = 0; j < 8; ++j) {
      const int nn = n + j;
      if (nn >= op.B) break;
      const float y = apply_act(fmaf(v[j], sc, bi), op.act);
      if (op.out_f32) static_cast<float*>(op.out)[static_cast<size_t>(nn) * op.ldo + m] = y;
      else static_cast<__nv_bfloat16*>(op.out)[static_cast<size_t>(nn) * op.ldo + m] = __float2bfloat16_rn(y);
    }
  }
}

__device__ void gemm_item(const OpDev& op, const Item& it, Ctx& cx) {
  const int tid = threadIdx.x;
  const int bn = op.bn;
  const int kb0 = (it.ks * op.nkb) / op.split_k;
  const int kb1 = ((it.ks + 1) * op.nkb) / op.split_k;
  const int nk = kb1 - kb0;
  const int m0 = it.mt * BM, n0 = it.nt * bn;
  const int chunk = tid & 7, rsub = tid >> 3;
  const uint32_t ring_base = smem_u32(cx.ring);
  const uint32_t idesc = make_idesc(bn);

  // per-thread A-row info (conv im2col): rows rsub + 32*i
  ARowInfo ar[4];
  const __nv_bfloat16* in = static_cast<const __nv_bfloat16*>(op.in);
  if (!op.swap) {
    const int HoWo = op.Ho * op.Wo;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + rsub + 32 * i;
      ar[i].ok = m < op.M;
      const int mm = ar[i].ok ? m : 0;
      const int b = mm / HoWo;
      const int rem = mm - b * HoWo;
      const int ho = rem / op.Wo;
      const int wo = rem - ho * op.Wo;
      ar[i].img = in + static_cast<size_t>(b) * op.H * op.W * op.ldi;
      ar[i].hi0 = ho * op.stride - op.ph;
      ar[i].wi0 = wo * op.stride - op.pw;
    }
  }

  auto load_stage = [&](int kb, uint32_t stage) {
    const uint32_t a_base = ring_base + stage * A_STAGE_BYTES;
    const uint32_t b_base = ring_base + STAGES * A_STAGE_BYTES + stage * B_STAGE_BYTES;
    const int k = kb * BK + chunk * 8;
    if (!op.swap) {
      // A: im2col gather, one 16-byte chunk = 8 channels of one filter tap
      const bool kok = k < op.K;
      const int tap = k / op.C;
      const int c = k - tap * op.C;
      const int r = tap / op.kw;
      const int s = tap - r * op.kw;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int row = rsub + 32 * i;
        const int hi = ar[i].hi0 + r, wi = ar[i].wi0 + s;
        const bool ok = kok && ar[i].ok && hi >= 0 && hi < op.H && wi >= 0 && wi < op.W;
        const __nv_bfloat16* src = ok ? ar[i].img + (static_cast<size_t>(hi) * op.W + wi) * op.ldi + c : in;
        cp_async16(a_base + row * 128 + ((chunk ^ (row & 7)) << 4), src, ok);
      }
      // B: packed weights [Npad][Kpad], zero-padded
      load_rows_tile(b_base, static_cast<const __nv_bfloat16*>(op.wt), op.ldw, n0, bn, op.tiles_n * bn, k,
                     op.Kpad, chunk, rsub);
    } else {
      load_rows_tile(a_base, static_cast<const __nv_bfloat16*>(op.wt), op.ldw, m0, BM, op.tiles_m * BM, k,
                     op.Kpad, chunk, rsub);
      load_rows_tile(b_base, static_cast<const __nv_bfloat16*>(op.act_b), op.ldb, n0, bn, op.B, k, op.K, chunk,
                     rsub);
    }
  };
  auto wait_free = [&](uint32_t g) {
    if (g >= STAGES) mbar_wait(&cx.ctl->mma_done[g % STAGES], ((g / STAGES) + 1) & 1);
  };

  // ---- main loop: STAGES-1 K-blocks in flight
#pragma unroll 1
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) {
      wait_free(cx.ring_pos + s);
      load_stage(kb0 + s, (cx.ring_pos + s) % STAGES);
    }
    cp_async_commit();
  }
#pragma unroll 1
  for (int i = 0; i < nk; ++i) {
    const int il = i + STAGES - 1;
    if (il < nk) {
      wait_free(cx.ring_pos + il);
      load_stage(kb0 + il, (cx.ring_pos + il) % STAGES);
    }
    cp_async_commit();
    cp_async_wait<STAGES - 1>();
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t stage = (cx.ring_pos + i) % STAGES;
      const uint32_t a_base = ring_base + stage * A_STAGE_BYTES;
      const uint32_t b_base = ring_base + STAGES * A_STAGE_BYTES + stage * B_STAGE_BYTES;
#pragma unroll
      for (int kk = 0; kk < BK / 16; ++kk) {
        umma_bf16(cx.tmem, make_sdesc(a_base + kk * 32), make_sdesc(b_base + kk * 32), idesc,
                  (i > 0 || kk > 0) ? 1u : 0u);
      }
      umma_commit(&cx.ctl->mma_done[stage]);
      if (i == nk - 1) umma_commit(&cx.ctl->acc_bar);
    }
  }
  cx.ring_pos += nk;

  // ---- accumulator ready
  mbar_wait(&cx.ctl->acc_bar, cx.acc_uses & 1);
  cx.acc_uses++;
  tc_fence_after();

  const int warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, h = warp >> 2;
  const int row = q * 32 + lane;
  const int half = bn >> 1;
  const uint32_t tbase = cx.tmem + (static_cast<uint32_t>(q * 32) << 16);

  if (op.split_k == 1) {
    for (int c = 0; c < half; c += 8) {
      float v[8];
      tmem_ld8(tbase + h * half + c, v);
      epilogue_store8(op, m0 + row, n0 + h * half + c, v);
    }
    tc_fence_before();
  } else {
    // write fp32 partial, last arriver reduces in fixed ks order
    const int tile = it.mt * op.tiles_n + it.nt;
    float* part = op.partial + (static_cast<size_t>(tile) * op.split_k) * (BM * bn);
    float* mine = part + static_cast<size_t>(it.ks) * (BM * bn) + row * bn;
    for (int c = 0; c < half; c += 8) {
      float v[8];
      tmem_ld8(tbase + h * half + c, v);
      float* o = mine + h * half + c;
      __stcg(reinterpret_cast<float4*>(o), make_float4(v[0], v[1], v[2], v[3]));
      __stcg(reinterpret_cast<float4*>(o + 4), make_float4(v[4], v[5], v[6], v[7]));
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      const uint32_t old = atomicAdd(op.tile_cnt + tile, 1u);
      const int last = (old == static_cast<uint32_t>(op.split_k - 1));
      if (last) op.tile_cnt[tile] = 0;  // all arrivals done: re-arm for the next round
      cx.ctl->flag = last;
      __threadfence();
    }
    __syncthreads();
    if (cx.ctl->flag) {
      for (int c = 0; c < half; c += 8) {
        float acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.0f;
        for (int ks = 0; ks < op.split_k; ++ks) {
          const float* p = part + static_cast<size_t>(ks) * (BM * bn) + row * bn + h * half + c;
          const float4 a = __ldcg(reinterpret_cast<const float4*>(p));
          const float4 b = __ldcg(reinterpret_cast<const float4*>(p + 4));
          acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
          acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
        }
        epilogue_store8(op, m0 + row, n0 + h * half + c, acc);
      }
    }
  }
}

// =====================================================================
// fp32 SIMT GEMM (fp32 tenants): conv / linear-as-conv, fixed K order
// =====================================================================
__device__ void simt_item(const OpDev& op, const Item& it) {
  const float* in = static_cast<const float*>(op.in);
  const float* w = static_cast<const float*>(op.wt);
  const int m0 = it.mt * op.bm, n0 = it.nt * op.bn;
  const int HoWo = op.Ho * op.Wo;
  for (int e = threadIdx.x; e < op.bm * op.bn; e += NTHREADS) {
    const int m = m0 + e / op.bn, n = n0 + e % op.bn;
    if (m >= op.M || n >= op.Cout) continue;
    const int b = m / HoWo, rem = m - b * HoWo, ho = rem / op.Wo, wo = rem - ho * op.Wo;
    const float* img = in + static_cast<size_t>(b) * op.H * op.W * op.ldi;
    const float* wr = w + static_cast<size_t>(n) * op.K;
    float acc = 0.0f;
    for (int r = 0; r < op.kh; ++r) {
      const int hi = ho * op.stride - op.ph + r;
      for (int s = 0; s < op.kw; ++s) {
        const int wi = wo * op.stride - op.pw + s;
        const bool ok = hi >= 0 && hi < op.H && wi >= 0 && wi < op.W;
        const float* px = img + (static_cast<size_t>(hi) * op.W + wi) * op.ldi;
        const float* wk = wr + (r * op.kw + s) * op.C;
        for (int c = 0; c < op.C; ++c) acc = fmaf(ok ? px[c] : 0.0f, wk[c], acc);
      }
    }
    float y = fmaf(acc, op.scale[n], op.bias[n]);
    if (op.has_skip) y += static_cast<const float*>(op.skip)[static_cast<size_t>(m) * op.lds + n];
    y = apply_act(y, op.act);
    static_cast<float*>(op.out)[static_cast<size_t>(m) * op.ldo + n] = y;
  }
}

// =====================================================================
// CUDA-core ops: 8 channels per thread, 128-bit NHWC accesses
// =====================================================================
template <bool F32>
__device__ __forceinline__ void load8(const void* base, size_t idx, float* f) {
  if (F32) {
    const float4 a = *reinterpret_cast<const float4*>(static_cast<const float*>(base) + idx);
    const float4 b = *reinterpret_cast<const float4*>(static_cast<const float*>(base) + idx + 4);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  } else {
    const uint4 u = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(base) + idx);
    bf16x8_to_f32(u, f);
  }
}
template <bool F32>
__device__ __forceinline__ void store8(void* base, size_t idx, const float* y, bool out_f32) {
  if (F32 || out_f32) {
    float* o = static_cast<float*>(base) + idx;
    *reinterpret_cast<float4*>(o) = make_float4(y[0], y[1], y[2], y[3]);
    *reinterpret_cast<float4*>(o + 4) = make_float4(y[4], y[5], y[6], y[7]);
  } else {
    uint4 u;
    u.x = pack_bf16x2(y[0], y[1]);
    u.y = pack_bf16x2(y[2], y[3]);
    u.z = pack_bf16x2(y[4], y[5]);
    u.w = pack_bf16x2(y[6], y[7]);
    *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(base) + idx) = u;
  }
}

// tile: bm output pixels x bn channels; G = bn/8 channel groups, each thread
// handles pixel p = tid / G + j * (NTHREADS / G), group tid % G.
template <bool F32>
__device__ void cc_item(const OpDev& op, const Item& it, Ctx& cx) {
  const int tid = threadIdx.x;
  const int G = op.bn >> 3;
  const int g = tid % G;
  const int pstep = NTHREADS / G;
  const int c = it.nt * op.bn + g * 8;
  if (op.kind == DK_GAP) {
    // rows are samples; each (sample, 8 channels) is the mean over H*W pixels,
    // summed in a fixed order: lane l sums pixels l, l+L, ..., then the L lane
    // partials are added in lane order.
    const int L = pstep;
    const int lane = tid / G;
    const int HW = op.H * op.W;
    float* red = cx.gap_red;
    for (int b = it.mt * op.bm; b < min(op.B, (it.mt + 1) * op.bm); ++b) {
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (c < op.C) {
        for (int p = lane; p < HW; p += L) {
          float f[8];
          load8<F32>(op.in, (static_cast<size_t>(b) * HW + p) * op.ldi + c, f);
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] += f[j];
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) red[(lane * G + g) * 8 + j] = acc[j];
      __syncthreads();
      if (tid < G * 8) {
        const int gg = tid >> 3, jj = tid & 7;
        const int cc = it.nt * op.bn + gg * 8 + jj;
        float s = 0.0f;
        for (int l = 0; l < L; ++l) s += red[(l * G + gg) * 8 + jj];
        if (cc < op.C) {
          const float y = s / static_cast<float>(HW);
          if (F32 || op.out_f32) static_cast<float*>(op.out)[static_cast<size_t>(b) * op.ldo + cc] = y;
          else static_cast<__nv_bfloat16*>(op.out)[static_cast<size_t>(b) * op.ldo + cc] = __float2bfloat16_rn(y);
        }
      }
      __syncthreads();
    }
    return;
  }
  if (c >= op.Cout) return;
  const int HoWo = op.Ho * op.Wo;
  for (int j = 0; j < CC_TASKS_PER_THREAD; ++j) {
    const int m = it.mt * op.bm + tid / G + j * pstep;
    if (m >= op.M) break;
    const int b = m / HoWo, rem = m - b * HoWo, ho = rem / op.Wo, wo = rem - ho * op.Wo;
    const size_t img = static_cast<size_t>(b) * op.H * op.W;
    float y[8];
    if (op.kind == DK_ELTWISE) {
      load8<F32>(op.in, static_cast<size_t>(m) * op.ldi + c, y);
      if (op.has_skip) {
        float s[8];
        load8<F32>(op.skip, static_cast<size_t>(m) * op.lds + c, s);
#pragma unroll
        for (int q = 0; q < 8; ++q) y[q] += s[q];
      }
    } else if (op.kind == DK_MAXPOOL) {
#pragma unroll
      for (int q = 0; q < 8; ++q) y[q] = -INFINITY;
      for (int r = 0; r < op.kh; ++r) {
        const int hi = ho * op.stride - op.ph + r;
        if (hi < 0 || hi >= op.H) continue;
        for (int s = 0; s < op.kw; ++s) {
          const int wi = wo * op.stride - op.pw + s;
          if (wi < 0 || wi >= op.W) continue;
          float f[8];
          load8<F32>(op.in, (img + static_cast<size_t>(hi) * op.W + wi) * op.ldi + c, f);
#pragma unroll
          for (int q = 0; q < 8; ++q) y[q] = fmaxf(y[q], f[q]);
        }
      }
    } else if (op.kind == DK_AVGPOOL) {
#pragma unroll
      for (int q = 0; q < 8; ++q) y[q] = 0.0f;
      int cnt = 0;
      for (int r = 0; r < op.kh; ++r) {
        const int hi = ho * op.stride - op.ph + r;
        for (int s = 0; s < op.kw; ++s) {
          const int wi = wo * op.stride - op.pw + s;
          if (hi < -op.ph || hi >= op.H + op.ph || wi < -op.pw || wi >= op.W + op.pw) continue;
          const bool in_b = hi >= 0 && hi < op.H && wi >= 0 && wi < op.W;
          if (op.cip || in_b) ++cnt;
          if (!in_b) continue;
          float f[8];
          load8<F32>(op.in, (img + static_cast<size_t>(hi) * op.W + wi) * op.ldi + c, f);
#pragma unroll
          for (int q = 0; q < 8; ++q) y[q] += f[q];
        }
      }
      const float inv = static_cast<float>(cnt);
#pragma unroll
      for (int q = 0; q < 8; ++q) y[q] = y[q] / inv;
    } else {  // DK_DW: depthwise conv, weights [kh*kw][C] fp32, fused BN scale/bias + act
#pragma unroll
      for (int q = 0; q < 8; ++q) y[q] = 0.0f;
      const float* wt = static_cast<const float*>(op.wt);
      for (int r = 0; r < op.kh; ++r) {
        const int hi = ho * op.stride - op.ph + r;
        if (hi < 0 || hi >= op.H) continue;
        for (int s = 0; s < op.kw; ++s) {
          const int wi = wo * op.stride - op.pw + s;
          if (wi < 0 || wi >= op.W) continue;
          float f[8];
          load8<F32>(op.in, (img + static_cast<size_t>(hi) * op.W + wi) * op.ldi + c, f);
          const float4 w0 = *reinterpret_cast<const float4*>(wt + (r * op.kw + s) * op.C + c);
          const float4 w1 = *reinterpret_cast<const float4*>(wt + (r * op.kw + s) * op.C + c + 4);
          const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
          for (int q = 0; q < 8; ++q) y[q] = fmaf(f[q], wv[q], y[q]);
        }
      }
      const float4 s0 = *reinterpret_cast<const float4*>(op.scale + c);
      const float4 s1 = *reinterpret_cast<const float4*>(op.scale + c + 4);
      const float4 b0 = *reinterpret_cast<const float4*>(op.bias + c);
      const float4 b1 = *reinterpret_cast<const float4*>(op.bias + c + 4);
      const float sc[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
      const float bi[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int q = 0; q < 8; ++q) y[q] = fmaf(y[q], sc[q], bi[q]);
      if (op.has_skip) {
        float s[8];
        load8<F32>(op.skip, static_cast<size_t>(m) * op.lds + c, s);
#pragma unroll
        for (int q = 0; q < 8; ++q) y[q] += s[q];
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) y[q] = apply_act(y[q], op.act);
    store8<F32>(op.out, static_cast<size_t>(m) * op.ldo + c, y, op.out_f32);
  }
}

__device__ __forceinline__ void run_item(const OpDev& op, const Item& it, Ctx& cx) {
  switch (op.kind) {
    case DK_GEMM: gemm_item(op, it, cx); break;
    case DK_SIMT_GEMM: simt_item(op, it); break;
    default:
      if (op.f32) cc_item<true>(op, it, cx);
      else cc_item<false>(op, it, cx);
  }
}

// =====================================================================
// CTA setup shared by the executor and the standalone GEMM kernel
// =====================================================================
__device__ __forceinline__ void cta_setup(Ctx& cx, uint8_t* smem_raw, uint32_t tmem_cols, bool need_tmem) {
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  cx.ring = base;
  cx.ctl = reinterpret_cast<SmemCtl*>(base + SMEM_RING_BYTES);
  cx.gap_red = reinterpret_cast<float*>(base);
  cx.ring_pos = 0;
  cx.acc_uses = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&cx.ctl->mma_done[s], 1);
    mbar_init(&cx.ctl->acc_bar, 1);
    fence_mbar_init();
  }
  if (need_tmem && (threadIdx.x >> 5) == 0) tmem_alloc(&cx.ctl->tmem_base, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  cx.tmem = need_tmem ? cx.ctl->tmem_base : 0;
}

// =====================================================================
// The persistent multi-tenant executor
// =====================================================================
// Spin until *ctr >= target, with watchdog; returns false on abort.
__device__ bool spin_ge(const uint32_t* ctr, uint32_t target, const ExecParams& p) {
  if (ld_acquire(ctr) >= target) return true;
  const uint64_t t0 = globaltimer();
  uint32_t it = 0;
  while (ld_acquire(ctr) < target) {
    __nanosleep(64);
    if ((++it & 255) == 0) {
      if (*reinterpret_cast<volatile int32_t*>(p.error)) return false;
      if (static_cast<int64_t>(globaltimer() - t0) > p.watchdog_ns) {
        atomicExch(p.error, 1);
        return false;
      }
    }
  }
  return true;
}

extern "C" __global__ void __launch_bounds__(NTHREADS, 1) gacer_executor(ExecParams p) {
  extern __shared__ uint8_t smem_raw[];
  Ctx cx;
  cta_setup(cx, smem_raw, 256, true);
  SmemCtl* ctl = cx.ctl;
  const int tid = threadIdx.x;
  const int32_t* pref = p.cta_pref + static_cast<size_t>(blockIdx.x) * p.n_tenants;
  int k = 0;  // open cluster (thread 0's view)

  for (;;) {
    if (tid == 0) {
      int claimed = -2;  // -2 = round finished, -3 = abort
      while (k < p.n_clusters) {
        int got = -1;
        for (int j = 0; j < p.n_tenants && got < 0; ++j) {
          const int t = pref[j];
          if (t < 0) break;
          const int si = t * p.n_clusters + k;
          const Seg sg = p.segs[si];
          if (sg.size == 0) continue;
          if (ld_relaxed(p.heads + si) >= static_cast<uint32_t>(sg.size)) continue;
          const uint32_t idx = atomicAdd(p.heads + si, 1u);
          if (idx < static_cast<uint32_t>(sg.size)) got = p.queue[sg.begin + idx];
        }
        if (got >= 0) { claimed = got; break; }
        // nothing left to claim in cluster k: the synchronisation pointer --
        // wait until every item of cluster k (all tenants) is done.
        if (!spin_ge(p.cluster_done + k, p.epoch * p.cluster_total[k], p)) { claimed = -3; break; }
        ++k;
      }
      if (claimed >= 0) {
        const Item it = p.items[claimed];
        ctl->item = it;
        // producer -> consumer dependencies (chunk counters)
        for (int d = 0; d < it.dep_count; ++d) {
          const Dep dp = p.deps[it.dep_begin + d];
          if (!spin_ge(p.chunk_done + dp.counter, p.epoch * dp.target, p)) { claimed = -3; break; }
        }
        __threadfence();  // acquire side: invalidate stale L1 lines before the CTA reads inputs
      }
      ctl->claimed = claimed;
    }
    __syncthreads();
    const int claimed = ctl->claimed;
    if (claimed < 0) break;
    const Item it = ctl->item;
    const OpDev& op = p.ops[it.op];
    uint64_t t_start = 0;
    if (p.trace && tid == 0) t_start = globaltimer();
    run_item(op, it, cx);
    __syncthreads();
    if (tid == 0) {
      __threadfence();  // release: the item's global writes before the counters
      atomicAdd(p.chunk_done + it.chunk, 1u);
      atomicAdd(p.cluster_done + it.cluster, 1u);
      if (p.trace) {
        int64_t* rec = p.trace + static_cast<size_t>(claimed) * 8;
        rec[0] = op.tenant; rec[1] = it.op; rec[2] = smid(); rec[3] = claimed;
        rec[4] = it.cluster; rec[5] = it.chunk;
        rec[6] = static_cast<int64_t>(t_start); rec[7] = static_cast<int64_t>(globaltimer());
      }
    }
  }

  // teardown
  tc_fence_before();
  __syncthreads();
  if ((tid >> 5) == 0) tmem_dealloc(cx.tmem, 256);
  if (tid == 0) {
    __threadfence();
    const uint32_t old = atomicAdd(p.exit_count, 1u);
    if (old == gridDim.x - 1) {  // last CTA out re-arms the claim counters
      for (int i = 0; i < p.n_heads; ++i) p.heads[i] = 0;
      *p.exit_count = 0;
      __threadfence();
    }
  }
}

// =====================================================================
// Standalone per-op kernels (baselines): same tile functions
// =====================================================================
extern "C" __global__ void __launch_bounds__(NTHREADS, 1) op_gemm_kernel(const OpDev* ops, int op_idx) {
  extern __shared__ uint8_t smem_raw[];
  Ctx cx;
  cta_setup(cx, smem_raw, 128, true);
  const OpDev& op = ops[op_idx];
  Item it;
  int b = blockIdx.x;
  it.op = op_idx;
  it.ks = b % op.split_k;
  b /= op.split_k;
  it.nt = b % op.tiles_n;
  it.mt = b / op.tiles_n;
  gemm_item(op, it, cx);
  tc_fence_before();
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) tmem_dealloc(cx.tmem, 128);
}

extern "C" __global__ void __launch_bounds__(NTHREADS) op_cc_kernel(const OpDev* ops, int op_idx) {
  __shared__ __align__(16) float red[GAP_RED_FLOATS];
  Ctx cx;
  cx.gap_red = red;
  const OpDev& op = ops[op_idx];
  Item it;
  it.op = op_idx;
  it.ks = 0;
  it.nt = blockIdx.x % op.tiles_n;
  it.mt = blockIdx.x / op.tiles_n;
  if (op.kind == DK_SIMT_GEMM) simt_item(op, it);
  else if (op.f32) cc_item<true>(op, it, cx);
  else cc_item<false>(op, it, cx);
}

// =====================================================================
// host-side launchers (C++ linkage, used by host.cpp)
// =====================================================================
int executor_smem_bytes() { return SMEM_GEMM_BYTES; }

cudaError_t configure_kernels() {
  cudaError_t e = cudaFuncSetAttribute(gacer_executor, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_GEMM_BYTES);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(op_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_GEMM_BYTES);
}

cudaError_t launch_executor(const ExecParams& p, int grid, cudaStream_t s) {
  gacer_executor<<<grid, NTHREADS, SMEM_GEMM_BYTES, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_op(const OpDev* ops_dev, int op_idx, int kind, int n_blocks, cudaStream_t s) {
  if (kind == DK_GEMM) op_gemm_kernel<<<n_blocks, NTHREADS, SMEM_GEMM_BYTES, s>>>(ops_dev, op_idx);
  else op_cc_kernel<<<n_blocks, NTHREADS, 0, s>>>(ops_dev, op_idx);
  return cudaGetLastError();
}

}  // namespace gacer
