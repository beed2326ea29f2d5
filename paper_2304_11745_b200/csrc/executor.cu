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
#include "train_dev.cuh"

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

// tcgen05.ld of 16 columns without waiting (batch several, then tmem_wait)
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
// tcgen05.ld of 32 columns without waiting
__device__ __forceinline__ void tmem_ld32_nw(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_pin16(uint32_t (&r)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) asm volatile("" : "+r"(r[i]));
}
// keep the uses of r after the preceding tcgen05.wait::ld (the registers are
// written asynchronously; the empty asm orders every use after the wait)
__device__ __forceinline__ void tmem_pin32(uint32_t* r) {
#pragma unroll
  for (int i = 0; i < 32; ++i) asm volatile("" : "+r"(r[i]));
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
// MN-major SWIZZLE_128B canonical layout (CUTLASS cute UMMA Layout_MN_SW128):
// 64 MN-elements per 128-byte row, one row per K index, 8 K rows per
// 1024-byte swizzle atom (SBO = 1024 between atoms along K), the next 64
// MN-elements LBO = 8192 bytes further (one 64 x 64 TMA box).  A K step of 16
// advances the start address by 16 rows = 2048 bytes.
__device__ __forceinline__ uint64_t make_sdesc_mn(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>(8192 >> 4) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
// K-major SWIZZLE_NONE ("interleave") canonical layout: core matrices of 8
// rows x 16 bytes (8 K-elements), rows 16 B apart; SBO = bytes between 8-row
// groups, LBO = bytes between the two 8-element K chunks of a K=16 step.
__device__ __forceinline__ uint64_t make_sdesc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  return d;   // layout type 0 (SWIZZLE_NONE)
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
// Diagnostics probes (GACER_DEBUG_TIMING=1 at run time) are compiled in only
// with -DGACER_DIAG=1: they hold registers across the role loops.
#ifndef GACER_DIAG
#define GACER_DIAG 0
#endif
__shared__ uint32_t g_dbg_seen;   // per-CTA: milestones already recorded (no global load per probe)
__device__ __forceinline__ void dbg_mark(const ExecParams& p, int ev) {
#if GACER_DIAG
  if (p.dbg && !(g_dbg_seen & (1u << ev))) {   // first occurrence only
    atomicOr(&g_dbg_seen, 1u << ev);
    p.dbg[static_cast<size_t>(blockIdx.x) * DBG_EVENTS + ev] = static_cast<int64_t>(globaltimer());
  }
#endif
}

// per-k-block timeline of CTA 0 (GACER_DEBUG_TIMING): [0,256) MMA saw stage
// full, [256,512) producer issued the stage, [512,768) epilogue (tfull, done)
constexpr size_t KDBG_OFF = static_cast<size_t>(400) * 148 * DBG_EVENTS;
__device__ __forceinline__ void kdbg(const ExecParams& p, int slot, uint32_t i) {
#if GACER_DIAG
  if (p.dbg && blockIdx.x == 0 && i < 256) p.dbg[KDBG_OFF + slot * 256 + i] = static_cast<int64_t>(globaltimer());
#endif
}

// scheduler stamps of CTA 0's first 24 claims (GACER_DEBUG_TIMING): globaltimer
__device__ __forceinline__ void sdbg(const ExecParams& p, uint32_t n, int j, int64_t v) {
#if GACER_DIAG
  if (p.dbg && blockIdx.x == 0 && n < 24) p.dbg[KDBG_OFF + 1024 + n * 8 + j] = v;
#endif
}

// epilogue clock64 stamps of CTA 0's first 8 GEMM items (GACER_DEBUG_TIMING)
__device__ __forceinline__ void edbg(const ExecParams& p, int point, uint32_t acc) {
#if GACER_DIAG
  if (p.dbg && blockIdx.x == 0 && acc < 8) p.dbg[KDBG_OFF + 768 + acc * 16 + point] = static_cast<int64_t>(clock64());
#endif
}

// gpu-scope fences.  __threadfence() is fence.sc.gpu: MEMBAR.SC.GPU plus an
// L1 invalidation (CCTL.IVALL) of the whole SM.  A release needs only
// MEMBAR.ALL.GPU and an acquire only the invalidation, so each side uses its
// own fence: completions no longer flush the co-resident warps' L1 working
// set (spills, op fields, residual rows).
__device__ __forceinline__ void fence_release_gpu() { asm volatile("fence.release.gpu;\n" ::: "memory"); }
__device__ __forceinline__ void fence_acquire_gpu() { asm volatile("fence.acquire.gpu;\n" ::: "memory"); }

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
// ReLU / ReLU6 only: MobileNetV3's hardswish / hardsigmoid are separate
// eltwise ops (cc_item_ext, out of line) -- inlined here, their extra
// branches perturbed the register allocation of the hot epilogue and window
// loops (same-box A/B: +10 us per op on plain conv+ReLU layers)
__device__ __forceinline__ float apply_act(float v, int act) {
  if (act == ACT_RELU) v = fmaxf(v, 0.0f);
  else if (act == ACT_RELU6) v = fminf(fmaxf(v, 0.0f), 6.0f);
  return v;
}

// more PTX helpers: mbarrier arrive / tx, TMA, named barriers
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void* tmap, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
          dst),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// L2 evict-first policy: for operands read exactly once per round (the
// swap-AB linear weights -- VGG-16's FC1 alone streams 205 MB through L2,
// which would otherwise evict the other tenants' L2-resident activations)
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_2d_hint(uint32_t dst, const void* tmap, uint64_t* bar, int c0, int c1,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;\n" ::"r"(dst),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void l2_prefetch(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_im2col_4d(uint32_t dst, const void* tmap, uint64_t* bar, int c, int w,
                                                   int h, int n, uint16_t ow, uint16_t oh) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};\n" ::"r"(dst),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(ow), "h"(oh)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const void* tmap, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];\n" ::"l"(tmap),
               "r"(src), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// =====================================================================
// shared memory layout of the executor CTA
// =====================================================================
constexpr int A_STAGE_BYTES = BM * 128;
constexpr int B_STAGE_BYTES = BN_MAX * 128;
constexpr int SMEM_RING_BYTES = STAGES * (A_STAGE_BYTES + B_STAGE_BYTES);
constexpr int TMEM_COLS = 2 * BN_MAX;   // double-buffered accumulators
constexpr int A2_OFF = 16384;            // M-pair tiles: second A block inside the stage's B region
constexpr int RING_CONSUMERS = 1 + 1 + NEPI / 32;  // worker group, MMA thread, epilogue warps

struct EpiItem {             // the epilogue's copy of an Item: the fields it and the releaser use
  int32_t op, mt, nt, ks, idx, chunk, cluster, bud;
};

struct RingSlot {            // scheduler -> workers / MMA / epilogue
  Item it;
  int32_t idx;               // item index, -1 = STOP
  int32_t kind;              // op kind (DK_GEMM items go to MMA + epilogue)
  uint64_t t0;               // claim time (trace)
};

struct SmemCtl {
  uint64_t full[STAGES];     // TMA/gather -> MMA
  uint64_t empty[STAGES];    // MMA -> workers
  uint64_t tfull[2];         // MMA -> epilogue (accumulator ready)
  uint64_t tempty[2];        // epilogue -> MMA (accumulator drained)
  uint64_t rfull[ITEM_RING];
  uint64_t rempty[ITEM_RING];
  RingSlot ring[ITEM_RING];
  uint64_t lfull[ITEM_RING];   // epilogue -> releaser (completed GEMM items)
  uint64_t lempty[ITEM_RING];
  RingSlot rel[ITEM_RING];
  uint32_t tmem_base;
  int32_t epi_flag;
  int32_t n_segs_smem;
  int32_t pad;
  unsigned long long st_ns[STAT_TENANTS + 2];   // this CTA's occupancy counters (flushed at exit)
  __align__(16) float red[CC_THREADS * 8]; // GAP fixed-order reduction scratch / dw weights (float4 reads)
  float epi_scale[BN_MAX];   // epilogue: folded BN scale / bias of the tile's columns
  float epi_bias[BN_MAX];
  Seg segs[MAX_SMEM_SEGS];   // (tenant, cluster) queue segments, cached
  OpDev wop;                 // the worker group's current op (staged once per item)
};
constexpr int STAGE_WARP_BYTES = 32 * 128;           // epilogue staging: 32 rows x 128 B per warp (SW128)
// TMA-store staging only with 4 epilogue warps: 8 warps' staging rows do not
// fit beside the ring; they store their rows directly (16 B per thread)
constexpr bool EPI_STAGED = NEPI == 128;
#ifndef GACER_PROD_SPLIT
#define GACER_PROD_SPLIT 1
#endif
#ifndef GACER_WPREFETCH
#define GACER_WPREFETCH 0  // L2 prefetch of the next GEMM ops' weights on an op's first tile
                           // (measured: D2 1.814 -> 1.906 ms -- the bulk prefetches occupy the
                           //  SM's TMA unit ahead of its own operand loads; not adopted)
#endif
#ifndef GACER_L2_HINTS
#define GACER_L2_HINTS 1   // evict-first L2 policy on read-once weight streams (swap-AB linear)
#endif
#ifndef GACER_EPI_DB
#define GACER_EPI_DB 1
#endif
constexpr bool EPI_DB = GACER_EPI_DB != 0;
// lean staged epilogue variant: 0 = 32-column steps, scale/bias by warp
// shuffles; 1 = software-pipelined 16-column TMEM loads, scale/bias as
// 16-byte smem broadcasts
#ifndef GACER_EPI_V
#define GACER_EPI_V 0
#endif              // double-buffered staging (needs the smem of a ring stage)
constexpr int SMEM_STAGE_BYTES = EPI_STAGED ? (NEPI / 32) * STAGE_WARP_BYTES * (EPI_DB ? 2 : 1) : 0;
constexpr int SMEM_BYTES = SMEM_RING_BYTES + SMEM_STAGE_BYTES + 1024 /*align slack*/;
// The control block is a static __shared__ object (not carved from the
// dynamic buffer) so every access compiles to LDS/STS instead of generic
// loads/stores.
__shared__ __align__(128) SmemCtl g_ctl;

struct Ctx {
  uint8_t* ring;             // 1024-aligned stage buffers
  uint8_t* stage;            // 1024-aligned epilogue staging (SWIZZLE_128B rows)
  SmemCtl* ctl;
  uint32_t tmem;
};

// =====================================================================
// epilogue math (shared by every mode): y = act(acc*scale + bias [+ skip])
// =====================================================================
// The OpDev fields the epilogue uses, copied once per item into registers
// (reading them through a reference to global memory re-loads them after
// every store, since the compiler cannot prove the stores do not alias).
struct EpiOp {
  void* out;
  const float* scale;
  const float* bias;
  const void* tmap_c;
  int32_t M, Cout, B, ldo, act, out_f32, has_skip, swap, c_tma;
};
__device__ __forceinline__ EpiOp make_epi(const OpDev& op) {
  EpiOp e;
  e.out = op.out; e.scale = op.scale; e.bias = op.bias; e.tmap_c = op.tmap_c;
  e.M = op.M; e.Cout = op.Cout; e.B = op.B; e.ldo = op.ldo; e.act = op.act;
  e.out_f32 = op.out_f32; e.has_skip = op.has_skip; e.swap = op.swap; e.c_tma = op.c_tma;
  return e;
}

// y = act(v*scale + bias [+ skip]) for 8 columns (no store)
__device__ __forceinline__ void epi_math8(const EpiOp& op, const float* v, const float* sc, const float* bi,
                                          const uint4& skip8, float* y) {
#pragma unroll
  for (int j = 0; j < 8; j += 2) {   // packed FFMA2: two IEEE fmas, same results as fmaf
    const float2 r = __ffma2_rn(make_float2(v[j], v[j + 1]), make_float2(sc[j], sc[j + 1]),
                                make_float2(bi[j], bi[j + 1]));
    y[j] = r.x;
    y[j + 1] = r.y;
  }
  if (op.has_skip) {
    float s[8];
    bf16x8_to_f32(skip8, s);
#pragma unroll
    for (int j = 0; j < 8; ++j) y[j] += s[j];
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) y[j] = apply_act(y[j], op.act);
}

// y = act(v*scale + bias [+ skip]) for 8 columns whose scale/bias live in
// lanes j0..j0+7 of (sc_l, bi_l): broadcast by warp shuffles instead of
// shared-memory loads (the smem port is saturated by the TMA fills and the
// tensor-core operand reads of the next tile).  Same IEEE ops as epi_math8.
__device__ __forceinline__ void epi_math8_shfl(const EpiOp& op, const float* v, float sc_l, float bi_l, int j0,
                                               const uint4& skip8, float* y) {
#pragma unroll
  for (int j = 0; j < 8; j += 2) {
    const float s0 = __shfl_sync(0xffffffffu, sc_l, j0 + j), s1 = __shfl_sync(0xffffffffu, sc_l, j0 + j + 1);
    const float b0 = __shfl_sync(0xffffffffu, bi_l, j0 + j), b1 = __shfl_sync(0xffffffffu, bi_l, j0 + j + 1);
    const float2 r = __ffma2_rn(make_float2(v[j], v[j + 1]), make_float2(s0, s1), make_float2(b0, b1));
    y[j] = r.x;
    y[j + 1] = r.y;
  }
  if (op.has_skip) {
    float s[8];
    bf16x8_to_f32(skip8, s);
#pragma unroll
    for (int j = 0; j < 8; ++j) y[j] += s[j];
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) y[j] = apply_act(y[j], op.act);
}

// Write 8 results of `row` at column offset `col` (within the staged chunk)
// into the warp's 32x128B staging block with the 128-byte swizzle (16-byte
// chunk j of row r at j ^ (r & 7)), the layout the TMA store reads.
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void stage8(uint32_t wbuf, int row, int col, const float* y, bool f32) {
  const int sw = row & 7;
  const uint32_t rb = wbuf + row * 128;
  if (f32) {
    const int j0 = (col * 4) >> 4;
    sts128(rb + ((j0 ^ sw) << 4), __float_as_uint(y[0]), __float_as_uint(y[1]), __float_as_uint(y[2]),
           __float_as_uint(y[3]));
    sts128(rb + (((j0 + 1) ^ sw) << 4), __float_as_uint(y[4]), __float_as_uint(y[5]), __float_as_uint(y[6]),
           __float_as_uint(y[7]));
  } else {
    const int j = (col * 2) >> 4;
    sts128(rb + ((j ^ sw) << 4), pack_bf16x2(y[0], y[1]), pack_bf16x2(y[2], y[3]), pack_bf16x2(y[4], y[5]),
           pack_bf16x2(y[6], y[7]));
  }
}

// m: GEMM row; n: first of 8 GEMM columns; sc/bi: the 8 columns' scale/bias
// (non-swap); skip8: the 8 residual values (bf16) when op.has_skip.
__device__ __forceinline__ void epilogue_store8(const EpiOp& op, int m, int n, const float* v, const float* sc,
                                                const float* bi, const uint4& skip8) {
  if (m >= op.M) return;
  float y[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) y[j] = fmaf(v[j], sc[j], bi[j]);
  if (op.has_skip) {
    float s[8];
    bf16x8_to_f32(skip8, s);
#pragma unroll
    for (int j = 0; j < 8; ++j) y[j] += s[j];
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) y[j] = apply_act(y[j], op.act);
  if (n + 8 <= op.Cout) {
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
    for (int j = 0; j < 8 && n + j < op.Cout; ++j) {
      if (op.out_f32) static_cast<float*>(op.out)[static_cast<size_t>(m) * op.ldo + n + j] = y[j];
      else static_cast<__nv_bfloat16*>(op.out)[static_cast<size_t>(m) * op.ldo + n + j] = __float2bfloat16_rn(y[j]);
    }
  }
}

// swap-AB (linear): GEMM row m = output feature, GEMM column n = sample
__device__ __forceinline__ void epilogue_store8_swap(const EpiOp& op, int m, int n, const float* v, float sc,
                                                     float bi) {
  if (m >= op.Cout) return;
  for (int j = 0; j < 8; ++j) {
    const int nn = n + j;
    if (nn >= op.B) break;
    const float y = apply_act(fmaf(v[j], sc, bi), op.act);
    if (op.out_f32) static_cast<float*>(op.out)[static_cast<size_t>(nn) * op.ldo + m] = y;
    else static_cast<__nv_bfloat16*>(op.out)[static_cast<size_t>(nn) * op.ldo + m] = __float2bfloat16_rn(y);
  }
}

// =====================================================================
// worker side of a GEMM item: fill the smem ring for its K-blocks
// =====================================================================
__device__ __forceinline__ void kb_range(const OpDev& op, int ks, int& kb0, int& nk) {
  kb0 = (ks * op.nkb) / op.split_k;
  nk = ((ks + 1) * op.nkb) / op.split_k - kb0;
}

__device__ void produce_gemm(const OpDev& op, const Item& it, Ctx& cx, uint32_t& g, int wtid,
                             const ExecParams& p) {
  SmemCtl* ctl = &g_ctl;
  int kb0, nk;
  kb_range(op, it.ks, kb0, nk);
  const uint32_t ring_base = smem_u32(cx.ring);
  const uint32_t bbytes = static_cast<uint32_t>(op.bn) * 128u;
  const int mrep = op.mrep;
  const int m0 = it.mt * BM * mrep, n0 = it.nt * op.bn;
  if (op.a_mode != A_GATHER) {
    // NPROD producer threads (lane 0 of worker warps 0..NPROD-1), producer j
    // filling the stages gi = j (mod NPROD): one thread's TMA loads complete
    // at only ~27-35 B/clk (measured, scripts/micro/tma_rate.cu), far below
    // what the MMA consumes, so the issue is spread over several threads.
    // GACER_PROD_SPLIT: the A and the B loads of a stage are issued by two
    // threads (lane 0 of worker warps pj and pj + NPROD), doubling the TMA
    // issue parallelism of the plain im2col / rows paths
    const int pw = wtid >> 5;
    const int role = (GACER_PROD_SPLIT && pw >= NPROD) ? 1 : 0;   // 0: A loads + arrival, 1: B loads
    const int pj = pw - role * NPROD;
    const bool split_ab = GACER_PROD_SPLIT && (op.a_mode == A_IM2COL || op.a_mode == A_ROWS);
    if ((wtid & 31) == 0 && pj < NPROD && (role == 0 || split_ab)) {
      // every OpDev field the loop needs is loaded once into registers: the
      // SM's L1 is invalidated by the gpu-scope fences of the other roles,
      // so a global re-load per K-block would cost an L2 round trip each
      const int a_mode = op.a_mode, C = op.C, kw = op.kw;
      const void* tmap_a = op.tmap_a;
      const void* tmap_b = op.tmap_b;
      // swap-AB linear: A = the weights, each element read by one item only
      const bool stream_a = op.swap == 2 && a_mode == A_ROWS && GACER_L2_HINTS;
      const uint64_t pol_ef = stream_a ? l2_policy_evict_first() : 0ull;
      fence_proxy_async_global();   // acquired producer data -> this thread's TMA reads
      // im2col start (top-left input tap) of each 128-row half of the tile
      // (scalars, not arrays: a dynamically indexed array lives in local
      //  memory, and the other roles' gpu-scope fences invalidate L1, so each
      //  K-block's reload would be an L2 round trip)
      int w0a = 0, h0a = 0, img0a = 0, w0b = 0, h0b = 0, img0b = 0;
      if (a_mode == A_IM2COL || a_mode == A_IM2COL8) {
        const int HoWo = op.Ho * op.Wo, Wo = op.Wo;
        img0a = m0 / HoWo;
        int rem = m0 - img0a * HoWo;
        w0a = (rem % Wo) * op.stride - op.pw;
        h0a = (rem / Wo) * op.stride - op.ph;
        if (mrep > 1) {
          const int mm = m0 + BM;
          img0b = mm / HoWo;
          rem = mm - img0b * HoWo;
          w0b = (rem % Wo) * op.stride - op.pw;
          h0b = (rem / Wo) * op.stride - op.ph;
        }
      }
      // M-pair tiles: the second 128-row A block lands in the stage's B region
      // after the (<= 16 KB, bn <= 128) B block
      // A_MN: only the 64-column B boxes inside the GEMM's N (columns past it
      // are never stored, their smem is left as is)
      // A_MN8: one 1 KB box per tap (8 GEMM columns) inside the GEMM's N
      const int nbq = a_mode == A_MN ? min(op.bn, op.N - n0 + 63) / 64
                                     : (a_mode == A_MN8 ? min(op.bn, op.N - n0 + 7) / 8 : 0);
      const uint32_t tx = a_mode == A_MN ? A_STAGE_BYTES + static_cast<uint32_t>(nbq) * 8192u
                          : a_mode == A_MN8 ? A_STAGE_BYTES + static_cast<uint32_t>(nbq) * 1024u
                                            : A_STAGE_BYTES * mrep + bbytes;
      // first K-block of this item whose stage (g + i) % NPROD belongs to producer pj
      const int i0 = (pj - static_cast<int>(g % NPROD) + NPROD) % NPROD;
#pragma unroll 1
      for (int i = i0; i < nk; i += NPROD) {
        const uint32_t gi = g + i, stage = gi % STAGES;
        if (gi >= STAGES) mbar_wait(&ctl->empty[stage], ((gi / STAGES) + 1) & 1);
        uint64_t* bar = &ctl->full[stage];
        const uint32_t a_dst = ring_base + stage * A_STAGE_BYTES;
        const uint32_t b_dst = ring_base + STAGES * A_STAGE_BYTES + stage * B_STAGE_BYTES;
        const int k = (kb0 + i) * BK;
        if (role == 1) {   // (the stage's tx count is armed by its A producer; complete_tx may come first)
          tma_load_2d(b_dst, tmap_b, bar, k, n0);
          continue;
        }
        mbar_arrive_expect_tx(bar, tx);
#ifndef GACER_NO_I8_CODE
        if (a_mode == A_IM2COL8) {
          // 8 taps of 8 channels: one 128-pixel x 16-byte im2col box per tap
          // (taps past kh*kw: a channel start past the tensor -> zero fill),
          // then the pre-packed weight block with one bulk copy
          const int taps = op.kh * kw;
          const int kb = kb0 + i;
#pragma unroll 1
          for (int j = 0; j < 8; ++j) {
            const int tap = kb * 8 + j;
            const bool ok = tap < taps;
            const int r = ok ? tap / kw : 0, sx = ok ? tap - (tap / kw) * kw : 0;
            tma_load_im2col_4d(a_dst + j * 2048, tmap_a, bar, ok ? 0 : 8, w0a, h0a, img0a,
                               static_cast<uint16_t>(sx), static_cast<uint16_t>(r));
          }
          const size_t blk = (static_cast<size_t>(it.nt) * op.nkb + kb) * static_cast<size_t>(bbytes);
          vgs_load(cx.ring + (b_dst - ring_base), static_cast<const uint8_t*>(op.wt) + blk, bbytes, bar);
          kdbg(p, 1, gi);
          continue;
        }
#endif
        if (a_mode == A_MN || a_mode == A_MN8) {
          // K-block = output pixels [k, k + 64): A = dy rows (two 64-channel
          // boxes), B = one im2col box per 64 GEMM columns (tap, c0) -- or,
          // 8 channels (A_MN8), one 8-column box per tap
          tma_load_2d(a_dst, tmap_a, bar, m0, k);
          tma_load_2d(a_dst + 8192, tmap_a, bar, m0 + 64, k);
          const int HoWo = op.Ho * op.Wo;
          const int img = k / HoWo, rem = k - img * HoWo;
          const int ho = rem / op.Wo, wo = rem - ho * op.Wo;
          const int wi = wo * op.stride - op.pw, hi = ho * op.stride - op.ph;
          const int qw = a_mode == A_MN ? 64 : 8;
          const uint32_t qb = a_mode == A_MN ? 8192u : 1024u;
          for (int q = 0; q < nbq; ++q) {
            const int n = n0 + q * qw;
            const int tap = n / C, c0 = n - tap * C;
            tma_load_im2col_4d(b_dst + q * qb, tmap_b, bar, c0, wi, hi, img, static_cast<uint16_t>(tap % kw),
                               static_cast<uint16_t>(tap / kw));
          }
          kdbg(p, 1, gi);
          continue;
        }
        if (a_mode == A_IM2COL) {
          const int tap = k / C;
          const int c0 = k - tap * C;
          const int r = tap / kw, sx = tap - r * kw;
          tma_load_im2col_4d(a_dst, tmap_a, bar, c0, w0a, h0a, img0a, static_cast<uint16_t>(sx),
                             static_cast<uint16_t>(r));
          if (mrep > 1)
            tma_load_im2col_4d(b_dst + A2_OFF, tmap_a, bar, c0, w0b, h0b, img0b, static_cast<uint16_t>(sx),
                               static_cast<uint16_t>(r));
        } else if (stream_a) {
          tma_load_2d_hint(a_dst, tmap_a, bar, k, m0, pol_ef);
        } else {
          tma_load_2d(a_dst, tmap_a, bar, k, m0);
          if (mrep > 1) tma_load_2d(b_dst + A2_OFF, tmap_a, bar, k, m0 + BM);
        }
        if (!split_ab) tma_load_2d(b_dst, tmap_b, bar, k, n0);
        kdbg(p, 1, gi);
      }
      if (pj == 0) dbg_mark(p, 2);
    }
  } else {
    // im2col gather with cp.async (C not a multiple of 64): 16-byte chunks of
    // 8 channels of one tap; thread -> chunk j = wtid & 7, rows (wtid>>3) + 12i
    constexpr int RSTEP = NWORK / 8;                  // 12
    constexpr int ROWS = (2 * BM + RSTEP - 1) / RSTEP; // 22: covers M-pair tiles (256 rows)
    constexpr int LAG = STAGES - 1;                   // stages in flight per thread (< STAGES)
    const int rows_tile = BM * mrep;
    const int chunk = wtid & 7, rsub = wtid >> 3;
    const __nv_bfloat16* in = static_cast<const __nv_bfloat16*>(op.in);
    int img_off[ROWS], hi0[ROWS], wi0[ROWS];          // per gathered row: image offset, top-left tap
    const int HoWo = op.Ho * op.Wo;
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {
      const int row = rsub + RSTEP * i;
      const int m = m0 + row;
      const bool ok = m < op.M && row < rows_tile;
      const int mm = ok ? m : 0;
      const int b = mm / HoWo, rem = mm - b * HoWo, ho = rem / op.Wo, wo = rem - (rem / op.Wo) * op.Wo;
      img_off[i] = b * op.H * op.W * op.ldi;
      hi0[i] = ok ? ho * op.stride - op.ph : -100000;
      wi0[i] = wo * op.stride - op.pw;
    }
#pragma unroll 1
    for (int i = 0; i < nk; ++i) {
      const uint32_t gi = g + i, stage = gi % STAGES;
      if (gi >= STAGES) mbar_wait(&ctl->empty[stage], ((gi / STAGES) + 1) & 1);
      const uint32_t a_dst = ring_base + stage * A_STAGE_BYTES;
      const uint32_t b_dst = ring_base + STAGES * A_STAGE_BYTES + stage * B_STAGE_BYTES;
      const int k0 = (kb0 + i) * BK;
      if (wtid == 0) {
        mbar_expect_tx(&ctl->full[stage], bbytes);
        tma_load_2d(b_dst, op.tmap_b, &ctl->full[stage], k0, n0);
      }
      const int k = k0 + chunk * 8;
      const bool kok = k < op.K;
      const int tap = k / op.C;
      const int c = k - tap * op.C;
      const int r = tap / op.kw, s = tap - (tap / op.kw) * op.kw;
#pragma unroll
      for (int j = 0; j < ROWS; ++j) {
        const int row = rsub + RSTEP * j;
        if (row < rows_tile) {
          const int hi = hi0[j] + r, wi = wi0[j] + s;
          const bool ok = kok && hi >= 0 && hi < op.H && wi >= 0 && wi < op.W;
          const __nv_bfloat16* src = ok ? in + img_off[j] + (static_cast<size_t>(hi) * op.W + wi) * op.ldi + c : in;
          // rows of the second 128-row half land after the B block (M-pair tiles)
          const uint32_t dst = row < BM ? a_dst + row * 128 : b_dst + A2_OFF + (row - BM) * 128;
          cp_async16(dst + ((chunk ^ (row & 7)) << 4), src, ok);
        }
      }
      cp_async_commit();
      if (i >= LAG) {
        cp_async_wait<LAG>();
        fence_proxy_async_smem();
        named_bar_sync(1, NWORK);
        if (wtid == 0) mbar_arrive(&ctl->full[(g + i - LAG) % STAGES]);
      }
    }
    cp_async_wait<0>();
    fence_proxy_async_smem();
    named_bar_sync(1, NWORK);
    if (wtid == 0)
      for (int i = (nk > LAG ? nk - LAG : 0); i < nk; ++i) mbar_arrive(&ctl->full[(g + i) % STAGES]);
  }
  g += nk;
}

// =====================================================================
// fp32 SIMT GEMM (fp32 tenants): conv / linear-as-conv, fixed K order
// =====================================================================
__device__ void simt_item(const OpDev& op, const Item& it, int tid, int nthr) {
  // task = (output pixel m, 8 consecutive output channels): one input load
  // feeds 8 FMAs, the 8 weights of a K step are two float4 loads from the
  // K-outer weight layout [K][Cout rounded to 8].  Each output is still
  // accumulated with fmaf in the fixed (r, s, c) order from 0.
  const float* in = static_cast<const float*>(op.in);
  const float* w = static_cast<const float*>(op.wt);
  const int cpad = (op.Cout + 7) & ~7;
  const int m0 = it.mt * op.bm, n0 = it.nt * op.bn;
  const int HoWo = op.Ho * op.Wo;
  const int G = op.bn >> 3;
  for (int e = tid; e < op.bm * G; e += nthr) {
    const int m = m0 + e / G, n = n0 + (e % G) * 8;
    if (m >= op.M || n >= op.Cout) continue;
    const int b = m / HoWo, rem = m - b * HoWo, ho = rem / op.Wo, wo = rem - ho * op.Wo;
    const float* img = in + static_cast<size_t>(b) * op.H * op.W * op.ldi;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int r = 0; r < op.kh; ++r) {
      const int hi = ho * op.stride - op.ph + r;
      for (int s = 0; s < op.kw; ++s) {
        const int wi = wo * op.stride - op.pw + s;
        const bool ok = hi >= 0 && hi < op.H && wi >= 0 && wi < op.W;
        const float* px = img + (static_cast<size_t>(hi) * op.W + wi) * op.ldi;
        const float* wk = w + static_cast<size_t>((r * op.kw + s) * op.C) * cpad + n;
        for (int c = 0; c < op.C; ++c) {
          const float x = ok ? px[c] : 0.0f;
          const float4 w0 = *reinterpret_cast<const float4*>(wk + static_cast<size_t>(c) * cpad);
          const float4 w1 = *reinterpret_cast<const float4*>(wk + static_cast<size_t>(c) * cpad + 4);
          acc[0] = fmaf(x, w0.x, acc[0]); acc[1] = fmaf(x, w0.y, acc[1]);
          acc[2] = fmaf(x, w0.z, acc[2]); acc[3] = fmaf(x, w0.w, acc[3]);
          acc[4] = fmaf(x, w1.x, acc[4]); acc[5] = fmaf(x, w1.y, acc[5]);
          acc[6] = fmaf(x, w1.z, acc[6]); acc[7] = fmaf(x, w1.w, acc[7]);
        }
      }
    }
    for (int j = 0; j < 8 && n + j < op.Cout; ++j) {
      float y = fmaf(acc[j], op.scale[n + j], op.bias[n + j]);
      if (op.has_skip) y += static_cast<const float*>(op.skip)[static_cast<size_t>(m) * op.lds + n + j];
      y = apply_act(y, op.act);
      static_cast<float*>(op.out)[static_cast<size_t>(m) * op.ldo + n + j] = y;
    }
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

// One output pixel x 8 channels of a pool / depthwise / eltwise op.
template <bool F32>
__device__ __forceinline__ void cc_pixel(const OpDev& op, int m, int c, int HoWo) {
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

// Shared-memory window op (bf16 depthwise conv / max-pool / avg-pool, any
// kernel <= 3x3 taps... any kh*kw <= 9): the item is bm output pixels (whole
// output rows, chosen on the host) x bn channels.  Per image segment of the
// item, every input row the segment's windows touch is copied into shared
// memory with cp.async at once (coalesced 16-byte chunks, ~all of it in
// flight: the op is latency/bandwidth bound, not compute bound), then each
// thread computes (pixel, 8 channels) outputs from shared memory.  Per output
// the taps are reduced in the same fixed (r, s) order with IEEE fma as
// cc_pixel, so results are bit-identical to the other window paths.
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];\n" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ float4 lds128f(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32f(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;\n" ::"r"(a), "f"(v) : "memory");
}
// Outputs of one staged image segment: task (pixel, 8-channel group).  KH,
// KW, S > 0: compile-time window (taps unrolled, the tap loads of a pixel
// issued together); 0: runtime window.  Same fixed (r, s) reduction order.
template <int KH_, int KW_, int S_>
__device__ __forceinline__ void window_segment(const OpDev& op, int tid, int nthr, uint32_t sbuf, uint32_t wsm,
                                               int img, int m, int seg_end, int h_lo, int c0, int bnc) {
  const int KH = KH_ ? KH_ : op.kh, KW = KW_ ? KW_ : op.kw, S = S_ ? S_ : op.stride;
  constexpr int TMAX = KH_ ? KH_ * KW_ : 9;
  const int PH = op.ph, PW = op.pw, H = op.H, W = op.W, Wo = op.Wo;
  const int HoWo = op.Ho * Wo;
  const int kind = op.kind;
  const int G8 = bnc >> 3;
  const int tasks = (seg_end - m) * G8;
  // nthr % G8 == 0: a thread keeps its channel group (no division per task)
  const bool fixed_cg = (nthr % G8) == 0;
  for (int i = tid; i < tasks; i += nthr) {
    const int cg = fixed_cg ? (tid % G8) : (i % G8);
    const int px = m + i / G8;
    const int rem = px - img * HoWo, ho = rem / Wo, wo = rem - ho * Wo;
    const int hb = ho * S - PH, wb = wo * S - PW;
    uint4 raw[TMAX];
    uint32_t valid = 0;
    int cnt = 0;
#pragma unroll
    for (int t = 0; t < TMAX; ++t) {
      if (KH_ == 0 && t >= KH * KW) break;
      const int r = t / KW, s2 = t - (t / KW) * KW;
      const int hi = hb + r, wi = wb + s2;
      const bool ok = hi >= 0 && hi < H && wi >= 0 && wi < W;
      if (kind == DK_AVGPOOL) {
        const bool in_frame = hi >= -PH && hi < H + PH && wi >= -PW && wi < W + PW;
        cnt += (op.cip ? in_frame : ok) ? 1 : 0;
      }
      valid |= (ok ? 1u : 0u) << t;
      const int hc = ok ? hi - h_lo : 0, wc = ok ? wi : 0;
      raw[t] = lds128(sbuf + ((hc * W + wc) * bnc + cg * 8) * 2);
    }
    float y[8];
    const float init = kind == DK_MAXPOOL ? -INFINITY : 0.0f;
#pragma unroll
    for (int q = 0; q < 8; ++q) y[q] = init;
#pragma unroll
    for (int t = 0; t < TMAX; ++t) {
      if (KH_ == 0 && t >= KH * KW) break;
      if (!((valid >> t) & 1u)) continue;
      float f[8];
      bf16x8_to_f32(raw[t], f);
      if (kind == DK_MAXPOOL) {
#pragma unroll
        for (int q = 0; q < 8; ++q) y[q] = fmaxf(y[q], f[q]);
      } else if (kind == DK_AVGPOOL) {
#pragma unroll
        for (int q = 0; q < 8; ++q) y[q] += f[q];
      } else {
        const uint32_t wa = wsm + 4 * (t * bnc + cg * 8);
        const float4 w0 = lds128f(wa), w1 = lds128f(wa + 16);
        y[0] = fmaf(f[0], w0.x, y[0]); y[1] = fmaf(f[1], w0.y, y[1]);
        y[2] = fmaf(f[2], w0.z, y[2]); y[3] = fmaf(f[3], w0.w, y[3]);
        y[4] = fmaf(f[4], w1.x, y[4]); y[5] = fmaf(f[5], w1.y, y[5]);
        y[6] = fmaf(f[6], w1.z, y[6]); y[7] = fmaf(f[7], w1.w, y[7]);
      }
    }
    if (kind == DK_AVGPOOL) {
      const float inv = static_cast<float>(cnt);
#pragma unroll
      for (int q = 0; q < 8; ++q) y[q] = y[q] / inv;
    } else if (kind == DK_DW) {
      const uint32_t sa = wsm + 4 * (KH * KW * bnc + cg * 8), ba = sa + 4 * bnc;
      const float4 s0 = lds128f(sa), s1 = lds128f(sa + 16), b0 = lds128f(ba), b1 = lds128f(ba + 16);
      y[0] = fmaf(y[0], s0.x, b0.x); y[1] = fmaf(y[1], s0.y, b0.y);
      y[2] = fmaf(y[2], s0.z, b0.z); y[3] = fmaf(y[3], s0.w, b0.w);
      y[4] = fmaf(y[4], s1.x, b1.x); y[5] = fmaf(y[5], s1.y, b1.y);
      y[6] = fmaf(y[6], s1.z, b1.z); y[7] = fmaf(y[7], s1.w, b1.w);
      if (op.has_skip) {
        float sk[8];
        load8<false>(op.skip, static_cast<size_t>(px) * op.lds + c0 + cg * 8, sk);
#pragma unroll
        for (int q = 0; q < 8; ++q) y[q] += sk[q];
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) y[q] = apply_act(y[q], op.act);
    store8<false>(op.out, static_cast<size_t>(px) * op.ldo + c0 + cg * 8, y, op.out_f32);
  }
}

__device__ void window_smem(const OpDev& op, const Item& it, int tid, int nthr, uint32_t sbuf, int bar_id) {
  const int c0 = it.nt * op.bn;
  const int bnc = min(op.bn, op.Cout - c0);          // channels of this item (multiple of 8)
  const int G8 = bnc >> 3;
  const int HoWo = op.Ho * op.Wo;
  const int KH = op.kh, KW = op.kw, S = op.stride, PH = op.ph, H = op.H, W = op.W;
  const __nv_bfloat16* in = static_cast<const __nv_bfloat16*>(op.in);
  const uint32_t wsm = sbuf + WIN_IN_BYTES;           // dw weights [tap][bnc], scale[bnc], bias[bnc]
  if (op.kind == DK_DW) {
    const float* wt = static_cast<const float*>(op.wt);
    const int T = KH * KW;
    for (int i = tid; i < T * bnc; i += nthr) {
      const int t = i / bnc, cc = i - t * bnc;
      sts32f(wsm + 4 * i, wt[t * op.C + c0 + cc]);
    }
    for (int i = tid; i < bnc; i += nthr) {
      sts32f(wsm + 4 * (T * bnc + i), op.scale[c0 + i]);
      sts32f(wsm + 4 * (T * bnc + bnc + i), op.bias[c0 + i]);
    }
  }
  const int m_end = min(op.M, (it.mt + 1) * op.bm);
  for (int m = it.mt * op.bm; m < m_end;) {
    const int img = m / HoWo;
    const int seg_end = min(m_end, (img + 1) * HoWo);
    const int ho_a = (m - img * HoWo) / op.Wo, ho_b = (seg_end - 1 - img * HoWo) / op.Wo;
    const int h_lo = max(0, ho_a * S - PH), h_hi = min(H - 1, ho_b * S - PH + KH - 1);
    const int nrows = h_hi - h_lo + 1;
    // ---- stage input rows [h_lo, h_hi] x W x bnc channels (row-major, channel-minor)
    const int chunks = nrows * W * G8;
    const __nv_bfloat16* src0 = in + (static_cast<size_t>(img) * H + h_lo) * W * op.ldi + c0;
    for (int i = tid; i < chunks; i += nthr) {
      const int cg = i % G8, pw_ = i / G8;          // pw_ = row * W + w
      cp_async16(sbuf + (pw_ * bnc + cg * 8) * 2, src0 + static_cast<size_t>(pw_) * op.ldi + cg * 8, true);
    }
    cp_async_commit();
    cp_async_wait<0>();
    named_bar_sync(bar_id, nthr);
    if (KH == 3 && KW == 3 && S == 1)
      window_segment<3, 3, 1>(op, tid, nthr, sbuf, wsm, img, m, seg_end, h_lo, c0, bnc);
    else if (KH == 3 && KW == 3 && S == 2)
      window_segment<3, 3, 2>(op, tid, nthr, sbuf, wsm, img, m, seg_end, h_lo, c0, bnc);
    else if (KH == 2 && KW == 2 && S == 2)
      window_segment<2, 2, 2>(op, tid, nthr, sbuf, wsm, img, m, seg_end, h_lo, c0, bnc);
    else
      window_segment<0, 0, 0>(op, tid, nthr, sbuf, wsm, img, m, seg_end, h_lo, c0, bnc);
    named_bar_sync(bar_id, nthr);   // smem free for the next segment
    m = seg_end;
  }
}

// tile: bm output pixels x bn channels; G = bn/8 channel groups; thread tid
// (of CC_THREADS) handles pixels tid / G + j * (CC_THREADS / G), group tid % G.
// Runs on the worker warps (named barrier 1) or a standalone CTA.
template <bool F32>
__device__ void cc_item(const OpDev& op, const Item& it, int tid, float* red) {
  const int G = op.bn >> 3;
  const int g = tid % G;
  const int pstep = CC_THREADS / G;
  const int c = it.nt * op.bn + g * 8;
  if (op.kind == DK_GAP) {
    // rows are samples; (sample, 8 channels) = mean over H*W pixels, summed in
    // a fixed order: lane l sums pixels l, l+L, ..., then the L lane partials
    // are added in lane order.
    const int L = pstep;
    const int lane = tid / G;
    const int HW = op.H * op.W;
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
      named_bar_sync(1, CC_THREADS);
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
      named_bar_sync(1, CC_THREADS);
    }
    return;
  }
  const int HoWo = op.Ho * op.Wo;
  const int mb = it.mt * op.bm + tid / G;
  if (c >= op.Cout) return;
  // (bf16 window ops normally run as staged items, window_smem)
  const int m_end = min(op.M, (it.mt + 1) * op.bm);   // bm: a multiple of pstep (host)
  for (int m = mb; m < m_end; m += pstep) cc_pixel<F32>(op, m, c, HoWo);
}

// Eltwise ops of the NEXT-2 tenants, out of line (own register allocation):
// a standalone BatchNorm (folded scale / bias; DenseNet's pre-activation on
// a concat), the squeeze-and-excitation channel scale x * s[n][c], and the
// hardswish / hardsigmoid activations (PyTorch's definitions); y = act(
// (x * scale + bias) [+ skip | * s]), 8 channels per task as cc_item.
__device__ __noinline__ void cc_item_ext(const OpDev& op, const Item& it, int tid) {
  const int G = op.bn >> 3;
  const int c = it.nt * op.bn + (tid % G) * 8;
  if (c >= op.Cout) return;
  const int HoWo = op.Ho * op.Wo;
  const int pstep = CC_THREADS / G;
  const int mb = it.mt * op.bm + tid / G;
  float sc[8], bi[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) { sc[q] = op.affine ? op.scale[c + q] : 1.0f; bi[q] = op.affine ? op.bias[c + q] : 0.0f; }
  const int m_end = min(op.M, (it.mt + 1) * op.bm);   // bm: a multiple of pstep (host)
  for (int m = mb; m < m_end; m += pstep) {
    float y[8], s[8];
    if (op.f32) load8<true>(op.in, static_cast<size_t>(m) * op.ldi + c, y);
    else load8<false>(op.in, static_cast<size_t>(m) * op.ldi + c, y);
    if (op.affine) {
#pragma unroll
      for (int q = 0; q < 8; ++q) y[q] = fmaf(y[q], sc[q], bi[q]);
    }
    if (op.has_skip) {
      const size_t row = op.has_skip == 2 ? static_cast<size_t>(m / HoWo) : static_cast<size_t>(m);
      if (op.f32) load8<true>(op.skip, row * op.lds + c, s);
      else load8<false>(op.skip, row * op.lds + c, s);
#pragma unroll
      for (int q = 0; q < 8; ++q) y[q] = op.has_skip == 2 ? y[q] * s[q] : y[q] + s[q];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float v = y[q];
      if (op.act == ACT_RELU) v = fmaxf(v, 0.0f);
      else if (op.act == ACT_RELU6) v = fminf(fmaxf(v, 0.0f), 6.0f);
      else if (op.act == ACT_HSWISH) v = v * (fminf(fmaxf(v + 3.0f, 0.0f), 6.0f) * (1.0f / 6.0f));
      else if (op.act == ACT_HSIGMOID) v = fminf(fmaxf(v + 3.0f, 0.0f), 6.0f) * (1.0f / 6.0f);
      y[q] = v;
    }
    if (op.f32) store8<true>(op.out, static_cast<size_t>(m) * op.ldo + c, y, op.out_f32);
    else store8<false>(op.out, static_cast<size_t>(m) * op.ldo + c, y, op.out_f32);
  }
}

__device__ __forceinline__ void run_cc(const OpDev& op, const Item& it, int tid, float* red) {
  if (op.kind == DK_ELTWISE && (op.act > ACT_RELU6 || op.affine || op.has_skip == 2)) cc_item_ext(op, it, tid);
  else if (op.kind == DK_SIMT_GEMM) simt_item(op, it, tid, CC_THREADS);
  else if (op.f32) cc_item<true>(op, it, tid, red);
  else cc_item<false>(op, it, tid, red);
}

__device__ __forceinline__ Item decode_single(const OpDev& op, int op_idx, int b) {
  Item it;
  it.op = op_idx;
  const int split = op.kind == DK_GEMM ? op.split_k : 1;
  it.ks = b % split;
  b /= split;
  it.nt = b % op.tiles_n;
  it.mt = b / op.tiles_n;
  it.dep_begin = it.dep_count = 0;
  it.chunk = -1;
  it.bud = -1;
  it.cluster = 0;
  it.prio = 0;
  it.idx = -1;
  return it;
}

// =====================================================================
// scheduler: dependency-aware, rank-ordered claiming
// =====================================================================
// Spin until *ctr >= target, with watchdog; returns false on abort.
__device__ bool spin_ge(const uint32_t* ctr, uint32_t target, const ExecParams& p) {
  // relaxed polling (an acquire load invalidates the SM's L1 on every poll,
  // evicting the co-resident warps' working set); one fence on success
  if (ld_relaxed(ctr) >= target) { fence_acquire_gpu(); return true; }
  const uint64_t t0 = globaltimer();
  uint32_t it = 0, ns = 32;
  while (ld_relaxed(ctr) < target) {
    if (it >= 8) {                // a few back-to-back polls first (the release is often imminent),
      __nanosleep(ns);            // then exponential backoff: 148 CTAs poll a few hot lines
      ns = ns < 512 ? ns * 2 : 512;
    }
    if ((++it & 63) == 0) {
      if (*reinterpret_cast<volatile int32_t*>(p.error)) return false;
      if (static_cast<int64_t>(globaltimer() - t0) > p.watchdog_ns) {
        atomicExch(p.error, 1);
        return false;
      }
    }
  }
  fence_acquire_gpu();
  return true;
}

// Non-blocking readiness test of an item's producer-chunk dependencies
// (relaxed loads; the caller fences once after claiming).
__device__ __forceinline__ bool deps_ready(const ExecParams& p, const Item& it) {
  if (it.bud >= 0 && ld_relaxed(p.chunk_done + it.bud) < (p.epoch - 1u) * it.btot + it.boff) return false;
  if (it.dep_count <= INLINE_DEPS) {
    bool ok = true;
#pragma unroll
    for (int d = 0; d < INLINE_DEPS; ++d)
      if (d < it.dep_count) ok &= ld_relaxed(p.chunk_done + it.dc[d]) >= p.epoch * it.dt[d];
    return ok;
  }
  // overflow list (tile-level dependencies of wide windows): the Dep entries
  // and then their counters are loaded in groups of 8 independent loads --
  // two L2 round trips per group instead of two per dependency
  bool ok = true;
  for (int d0 = 0; d0 < it.dep_count && ok; d0 += 8) {
    Dep dp[8];
    uint32_t v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (d0 + j < it.dep_count) dp[j] = p.deps[it.dep_begin + d0 + j];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (d0 + j < it.dep_count) v[j] = ld_relaxed(p.chunk_done + dp[j].counter);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (d0 + j < it.dep_count) ok &= v[j] >= p.epoch * dp[j].target;
  }
  return ok;
}

__device__ __forceinline__ Seg get_seg(const ExecParams& p, const SmemCtl* ctl, int si) {
  return si < ctl->n_segs_smem ? ctl->segs[si] : p.segs[si];
}

// Find the best claimable item of the open cluster k without claiming it.
// Greedy, dependency-aware issue (§3, l.438-444: an operator that
// cannot be deployed now "is moved to the next cycle"): among the head items
// of the tenant queues this CTA may serve, pick the READY one (producers
// complete) with the highest upward rank (longest estimated remaining chain,
// computed by the plan compiler).  The critical tenant's chain advances while
// the others fill its residue (l.447-453).  Unready heads are never claimed,
// which keeps the wait-for graph acyclic.
// Returns 1 (candidate in si/h/cand), 0 (unclaimed work, none ready),
// 2 (every item of cluster k claimed), 3 (claim-ahead: no ready head, the
// best unready head in si/h/cand).
__device__ int scan_ready(const ExecParams& p, const SmemCtl* ctl, int k, int& best_si, uint32_t& best_h,
                          Item& cand) {
  const int32_t* pref = p.cta_pref + static_cast<size_t>(blockIdx.x) * p.n_tenants;
  bool unclaimed = false;
  best_si = -1;
  uint32_t best_prio = 0;
  int u_si = -1;
  uint32_t u_h = 0, u_prio = 0;
  for (int j = 0; j < p.n_tenants; ++j) {
    const int t = pref[j];
    if (t < 0) break;
    const int si = t * p.n_clusters + k;
    const Seg sg = get_seg(p, ctl, si);
    if (sg.size == 0) continue;
    const uint32_t h = ld_relaxed(p.heads + si);
    if (h >= static_cast<uint32_t>(sg.size)) continue;
    unclaimed = true;
    const Item* ip = p.items + sg.begin + h;
    const uint32_t prio = ip->prio;
    if (best_si >= 0 && prio <= best_prio) continue;
    const Item c = *ip;
    if (!deps_ready(p, c)) {
      if (p.claim_ahead && (u_si < 0 || prio > u_prio)) { u_si = si; u_h = h; u_prio = prio; }
      continue;
    }
    best_si = si;
    best_h = h;
    best_prio = prio;
    cand = c;
    if (j == 0 && p.own_first) return 1;  // the CTA's own tenant (SM partition) comes first
  }
  if (best_si >= 0) return 1;
  if (u_si >= 0) {
    best_si = u_si;
    best_h = u_h;
    cand = p.items[get_seg(p, ctl, u_si).begin + u_h];
    return 3;
  }
  return unclaimed ? 0 : 2;
}

__device__ __forceinline__ void release_item(const ExecParams& p, const Item& it, uint64_t t0, const OpDev& op) {
  // caller: all writes of the item are ordered before this thread (barrier);
  // the release fence makes them visible at gpu scope before the counters.
  // The trace's end stamp is taken BEFORE the counters publish the item, so a
  // dependent item's claim stamp is never earlier than it.
  const uint64_t t_end = (p.trace || p.stats) ? globaltimer() : 0;
  if (p.stats && op.tenant < STAT_TENANTS)
    atomicAdd(&g_ctl.st_ns[op.tenant], static_cast<unsigned long long>(t_end - t0));
  fence_release_gpu();
  dbg_mark(p, 8);
  atomicAdd(p.chunk_done + it.chunk, 1u);
  if (it.bud >= 0) atomicAdd(p.chunk_done + it.bud, 1u);
  atomicAdd(p.cluster_done + it.cluster, 1u);
  dbg_mark(p, 9);
  if (p.trace) {
    int64_t* rec = p.trace + static_cast<size_t>(it.idx) * TRACE_FIELDS;
    rec[0] = op.tenant; rec[1] = it.op; rec[2] = smid(); rec[3] = it.idx;
    rec[4] = it.cluster; rec[5] = it.chunk;
    rec[6] = static_cast<int64_t>(t0); rec[7] = static_cast<int64_t>(t_end);
  }
}

// Wait (blocking) until the item's dependencies are complete; false on abort.
__device__ bool wait_deps(const ExecParams& p, const Item& it) {
  if (deps_ready(p, it)) { fence_acquire_gpu(); return true; }   // usual case: one parallel check
  if (it.bud >= 0 && !spin_ge(p.chunk_done + it.bud, (p.epoch - 1u) * it.btot + it.boff, p)) return false;
  if (it.dep_count <= INLINE_DEPS) {
#pragma unroll
    for (int d = 0; d < INLINE_DEPS; ++d)   // (static indices: the Item stays in registers)
      if (d < it.dep_count && !spin_ge(p.chunk_done + it.dc[d], p.epoch * it.dt[d], p)) return false;
  } else {
    for (int d = 0; d < it.dep_count; ++d) {
      const Dep dp = p.deps[it.dep_begin + d];
      if (!spin_ge(p.chunk_done + dp.counter, p.epoch * dp.target, p)) return false;
    }
  }
  return true;
}

// The scheduler (warp 0, lane 0).  It finds the best ready candidate BEFORE
// waiting for room in the CTA's item ring (the scan latency overlaps the
// items in flight), then claims it.  In-flight depth: items continuing the
// same large op may be claimed up to LOOKAHEAD deep (hides claim latency);
// any other item only when the ring is drained to depth 1, so a
// latency-critical item of a small op never queues behind several long tiles
// of a big op (head-of-line blocking inside the CTA).
#ifndef GACER_BIGOP_DEPTH2
#define GACER_BIGOP_DEPTH2 1   // a large op's first item may join one item in flight (D2 -0.6 %, D3 -0.4 %, B=64 mix -0.5 %)
#endif
#ifndef GACER_TAIL_DEPTH
#define GACER_TAIL_DEPTH 1   // in-flight depth for the last #CTAs items of an op (A/B knob)
#endif
#ifndef GACER_TAIL_DEPTH_CC
#define GACER_TAIL_DEPTH_CC 0   // depth 2 for the tail of CUDA-core ops only (A/B knob)
#endif
#ifndef GACER_BIGOP_MULT
#define GACER_BIGOP_MULT 4   // "large": more than this many items per CTA left in the segment
#endif
#ifndef GACER_NEWOP_DEPTH
#define GACER_NEWOP_DEPTH 1   // in-flight depth allowed when the candidate starts a different op
#endif
__device__ void scheduler_role(const ExecParams& p, Ctx& cx) {
  SmemCtl* ctl = &g_ctl;
  uint32_t islot = 0, consumed = 0;
  int k = p.k_first;
  int sidx = blockIdx.x;
  int last_op = -1;
  const int big = 4 * static_cast<int>(gridDim.x);
  for (;;) {
    // one claimed item per pass, in scalars (an indexed Item array would
    // live in local memory: L2 round trips after every acquire fence)
    Item itm;
    int32_t iidx = -1;
    int n_claimed = 0;
    int claimed = -1;
    if (p.single_op >= 0) {
      while (islot - consumed >= 2) {
        mbar_wait(&ctl->rempty[consumed % ITEM_RING], (consumed / ITEM_RING) & 1);
        ++consumed;
      }
      const OpDev& op = p.ops[p.single_op];
      const int n = op.tiles_m * op.tiles_n * (op.kind == DK_GEMM ? op.split_k : 1);
      claimed = sidx < n ? sidx : -2;
      if (claimed >= 0) {
        itm = decode_single(op, p.single_op, sidx);
        itm.kind = op.kind;
        iidx = claimed;
        n_claimed = 1;
      }
      sidx += gridDim.x;
    } else {
      uint64_t t0 = 0;
      uint32_t spins = 0;
      while (claimed == -1) {
        if (k > p.k_last) { claimed = -2; break; }
        int si;
        uint32_t h;
        Item cand;
        sdbg(p, islot, 0, static_cast<int64_t>(globaltimer()));
        const int st = scan_ready(p, ctl, k, si, h, cand);
        sdbg(p, islot, 1, static_cast<int64_t>(globaltimer()));
        if (st == 2) {
          // every item of cluster k is claimed: the synchronisation pointer --
          // wait until every item of cluster k (all tenants) is done.
          const uint64_t tb = p.stats ? globaltimer() : 0;
          if (!spin_ge(p.cluster_done + k, p.epoch * p.cluster_total[k], p)) { claimed = -3; break; }
          if (p.stats && k < p.k_last) ctl->st_ns[STAT_TENANTS] += globaltimer() - tb;
          dbg_mark(p, 10);
          ++k;
          spins = 0;
          continue;
        }
        if (st == 0) {  // unclaimed work exists but none of it is ready: back off, rescan
          const uint64_t tw = p.stats ? globaltimer() : 0;
          __nanosleep(spins < 4 ? 64u : (spins < 8 ? 256u : 512u));
          if (p.stats) ctl->st_ns[STAT_TENANTS + 1] += globaltimer() - tw;
          if (spins++ == 0) t0 = globaltimer();
          if ((spins & 31) == 0) {
            if (*reinterpret_cast<volatile int32_t*>(p.error)) { claimed = -3; break; }
            if (static_cast<int64_t>(globaltimer() - t0) > p.watchdog_ns) {
              atomicExch(p.error, 1);
              claimed = -3;
              break;
            }
          }
          continue;
        }
        const int G1 = static_cast<int>(gridDim.x);
        // claim-ahead (st == 3): only once this CTA's ring is drained (the
        // CTA would otherwise idle); the dependency wait below then overlaps
        // the producers' tails instead of following them
        const uint32_t allowed =
            st == 3 ? 1u
                    : (cand.op != last_op) ? ((GACER_BIGOP_DEPTH2 && cand.op_left > GACER_BIGOP_MULT * G1) ? 2u
                                                                                      : static_cast<uint32_t>(GACER_NEWOP_DEPTH))
                                           : (cand.op_left > big ? static_cast<uint32_t>(LOOKAHEAD)
                                                                 : (cand.op_left > G1 ? 2u
                                                                    : ((GACER_TAIL_DEPTH_CC && cand.kind != DK_GEMM)
                                                                           ? 2u
                                                                           : static_cast<uint32_t>(GACER_TAIL_DEPTH))));
        sdbg(p, islot, 5, static_cast<int64_t>(allowed) * 1000 + (islot - consumed));
        while (islot - consumed >= allowed) {
          mbar_wait(&ctl->rempty[consumed % ITEM_RING], (consumed / ITEM_RING) & 1);
          ++consumed;
        }
        sdbg(p, islot, 2, static_cast<int64_t>(globaltimer()));
        const Seg sg = get_seg(p, ctl, si);
        const uint32_t idx = atomicAdd(p.heads + si, 1u);
        sdbg(p, islot, 3, static_cast<int64_t>(globaltimer()));
        if (idx >= static_cast<uint32_t>(sg.size)) continue;  // lost the race for the last item(s)
        if (idx == h && st != 3) {
          itm = cand;
        } else {
          // a later item than the one checked: its dependencies are items
          // claimed before it, so this wait terminates
          itm = p.items[sg.begin + idx];
          if (!wait_deps(p, itm)) { claimed = -3; break; }
        }
        iidx = sg.begin + static_cast<int>(idx);
        n_claimed = 1;
        claimed = iidx;
        last_op = itm.op;
      }
      if (claimed >= 0) fence_acquire_gpu();  // acquire side (pairs with the producers' release)
    }
    dbg_mark(p, 1);
    sdbg(p, islot, 4, static_cast<int64_t>(globaltimer()));
    sdbg(p, islot, 6, claimed >= 0 ? itm.op : -1);
    if (claimed < 0) n_claimed = 0;
    {
      const uint32_t slot = islot % ITEM_RING;  // free: islot - consumed < LOOKAHEAD < ITEM_RING
      RingSlot& rs = ctl->ring[slot];
      if (n_claimed > 0) rs.it = itm;
      rs.idx = n_claimed > 0 ? iidx : -1;
      rs.kind = n_claimed > 0 ? itm.kind : 0;
      rs.t0 = (p.trace || p.stats) ? globaltimer() : 0;
      mbar_arrive(&ctl->rfull[slot]);
      ++islot;
    }
    if (claimed < 0) break;
#if GACER_WPREFETCH
    // the op's first tile (exactly one per op in every plan): pull the next
    // GEMM ops' weights into L2 while this op runs (after the hand-off, so
    // the claimed item is not delayed)
    if (p.single_op < 0 && itm.mt == 0 && itm.nt == 0 && itm.ks == 0) {
      const OpDev& op = p.ops[itm.op];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const uint32_t bytes = op.pf_bytes[j];
        const char* src = static_cast<const char*>(op.pf_ptr[j]);
        for (uint32_t off = 0; off < bytes; off += 262144u)
          l2_prefetch(src + off, min(262144u, bytes - off));
      }
    }
#endif
  }
}

// A training-tenant operator's item: virtual blocks [mt * bm, ...) of its
// grid on the worker group.  Not inlined: the operators' register needs stay
// out of the worker loop's allocation (the GEMM producer path shares it).
__device__ __noinline__ void vgrid_item(const OpDev& op, int mt, int wtid, uint8_t* smem) {
  const int v0 = mt * op.bm, v1 = min(v0 + op.bm, op.vblocks);
  if (vg_streamable(op.vfn)) {   // HBM-streaming operators: staged through the ring with bulk copies
    vg_stream_item(op.vfn, op.va, v0, v1, op.vblocks, wtid, NWORK, smem, SMEM_RING_BYTES);
    return;
  }
  for (int vb = v0; vb < v1; ++vb) run_vgrid(op.vfn, op.va, vb, op.vblocks, wtid, NWORK, smem);
}

template <bool TRAIN>
__device__ void worker_role(const ExecParams& p, Ctx& cx) {
  SmemCtl* ctl = &g_ctl;
  const int wtid = threadIdx.x - WORK_WARP0 * 32;  // 0..NWORK-1
  uint32_t g = 0, islot = 0;
  int wop_cached = -1;   // op whose descriptor ctl->wop holds (uniform across the worker group)
  for (;;) {
    const uint32_t slot = islot % ITEM_RING;
    mbar_wait(&ctl->rfull[slot], (islot / ITEM_RING) & 1);
    const RingSlot rs = ctl->ring[slot];
    ++islot;
    if (rs.idx < 0) {
      named_bar_sync(1, NWORK);
      if (wtid == 0) mbar_arrive(&ctl->rempty[slot]);
      break;
    }
    if (rs.it.op != wop_cached) {  // stage the item's op descriptor in shared memory
       // (once per op run): the tile functions read its fields many times,
       // and global re-loads would each be an L2 round trip (L1 is
       // invalidated by the scheduler's acquire fences)
      constexpr int WORDS = static_cast<int>(sizeof(OpDev) / 4);
      static_assert(WORDS <= NWORK, "OpDev staging");
      if (wtid < WORDS)
        reinterpret_cast<uint32_t*>(&ctl->wop)[wtid] = reinterpret_cast<const uint32_t*>(p.ops + rs.it.op)[wtid];
      named_bar_sync(1, NWORK);
      wop_cached = rs.it.op;
    }
    const OpDev& op = ctl->wop;
    if (rs.kind == DK_GEMM) {
      produce_gemm(op, rs.it, cx, g, wtid, p);
      if (wtid == 0) dbg_mark(p, 3);
      named_bar_sync(1, NWORK);
    } else {
      if (wtid == 0 && p.trace && p.single_op < 0)
        p.trace[static_cast<size_t>(rs.it.idx) * TRACE_FIELDS + 8] = static_cast<int64_t>(globaltimer());
      if (op.win || op.kind == DK_VGRID) {
        // the staged window op / virtual-grid op borrows the GEMM smem ring:
        // wait until the MMA has consumed every stage produced so far (MMAs
        // complete in order)
        if (g > 0) mbar_wait(&ctl->empty[(g - 1) % STAGES], ((g - 1) / STAGES) & 1);
        if (wtid == 0 && p.trace && p.single_op < 0)   // ring drained (diagnostics)
          p.trace[static_cast<size_t>(rs.it.idx) * TRACE_FIELDS + 9] = static_cast<int64_t>(globaltimer());
        if (TRAIN && op.kind == DK_VGRID) {
          vgrid_item(op, rs.it.mt, wtid, cx.ring);
        } else {
          window_smem(op, rs.it, wtid, NWORK, smem_u32(cx.ring), 1);
        }
      } else {
        run_cc(op, rs.it, wtid, ctl->red);
      }
      named_bar_sync(1, NWORK);
      if (wtid == 0 && p.single_op < 0) release_item(p, rs.it, rs.t0, op);
    }
    if (wtid == 0) mbar_arrive(&ctl->rempty[slot]);
  }
}

__device__ void mma_role(const ExecParams& p, Ctx& cx) {
  SmemCtl* ctl = &g_ctl;
  uint32_t g = 0, islot = 0, acc = 0;
  const uint32_t ring_base = smem_u32(cx.ring);
  for (;;) {
    const uint32_t slot = islot % ITEM_RING;
    mbar_wait(&ctl->rfull[slot], (islot / ITEM_RING) & 1);
    const int idx = ctl->ring[slot].idx;
    const int kind = ctl->ring[slot].kind;
    const Item it = ctl->ring[slot].it;
    mbar_arrive(&ctl->rempty[slot]);
    ++islot;
    if (idx < 0) break;
    if (kind != DK_GEMM) continue;
    const OpDev& op = p.ops[it.op];
    int kb0, nk;
    kb_range(op, it.ks, kb0, nk);
    const uint32_t abuf = acc & 1;
    if (acc >= 2) mbar_wait(&ctl->tempty[abuf], ((acc / 2) + 1) & 1);
    tc_fence_after();
    const uint32_t d = cx.tmem + abuf * BN_MAX;
    const bool mn = op.a_mode == A_MN || op.a_mode == A_MN8;   // both operands MN-major (weight gradient)
    const bool mn8 = op.a_mode == A_MN8;
    const bool i8 = op.a_mode == A_IM2COL8;   // no-swizzle core-matrix layout (8-channel stems)
    const uint32_t idesc = make_idesc(op.bn) | (mn ? ((1u << 15) | (1u << 16)) : 0u);
    const int mrep = op.mrep;
    const uint32_t d2 = d + static_cast<uint32_t>(op.bn);   // second accumulator (M-pair tiles)
    bool stamped = false;
#pragma unroll 1
    for (int i = 0; i < nk; ++i) {
      const uint32_t stage = g % STAGES;
      mbar_wait(&ctl->full[stage], (g / STAGES) & 1);
      kdbg(p, 0, g);
      if (i == 0) dbg_mark(p, 4);
      if (p.trace && !stamped && p.single_op < 0) {
        p.trace[static_cast<size_t>(it.idx) * TRACE_FIELDS + 8] = static_cast<int64_t>(globaltimer());
        stamped = true;
      }
      tc_fence_after();
      const uint32_t a_base = ring_base + stage * A_STAGE_BYTES;
      const uint32_t b_base = ring_base + STAGES * A_STAGE_BYTES + stage * B_STAGE_BYTES;
      if (!(GACER_DIAG && p.dbg && (p.dbg_spin & 1))) {  // diagnostics: odd dbg_spin skips the MMAs
        if (mn8) {
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_bf16(d, make_sdesc_mn(a_base + kk * 2048), make_sdesc_none(b_base + kk * 256, 128, 1024), idesc,
                      (i > 0 || kk > 0) ? 1u : 0u);
        } else if (mn) {
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_bf16(d, make_sdesc_mn(a_base + kk * 2048), make_sdesc_mn(b_base + kk * 2048), idesc,
                      (i > 0 || kk > 0) ? 1u : 0u);
#ifndef GACER_NO_I8_CODE
        } else if (i8) {
          const uint32_t lbo_b = static_cast<uint32_t>(op.bn) * 16u;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_bf16(d, make_sdesc_none(a_base + kk * 4096, 2048, 128),
                      make_sdesc_none(b_base + kk * 2 * lbo_b, lbo_b, 128), idesc, (i > 0 || kk > 0) ? 1u : 0u);
#endif
        } else {
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk)
          umma_bf16(d, make_sdesc(a_base + kk * 32), make_sdesc(b_base + kk * 32), idesc,
                    (i > 0 || kk > 0) ? 1u : 0u);
        }
        if (mrep > 1) {
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_bf16(d2, make_sdesc(b_base + A2_OFF + kk * 32), make_sdesc(b_base + kk * 32), idesc,
                      (i > 0 || kk > 0) ? 1u : 0u);
        }
      }
      umma_commit(&ctl->empty[stage]);
      ++g;
    }
    umma_commit(&ctl->tfull[abuf]);
    dbg_mark(p, 5);
    ++acc;
  }
}

// One 16-column sub-chunk of the lean staged epilogue: y = clamp(acc *
// scale + bias [+ skip], lo, hi) -> bf16 RNE -> the warp's 128-byte-swizzled
// staging rows (columns cin..cin+15 of the 64-column chunk).  scale/bias: the
// tile's staged columns, read as warp-uniform 16-byte broadcasts.  Same IEEE
// operations in the same order as every other epilogue path.
__device__ __forceinline__ void epi_chunk16(const uint32_t (&r)[16], const float* esc, const float* ebi, bool skip,
                                            const uint4 (&sk)[2], float lo, float hi, int cin, uint32_t sbuf,
                                            int lane) {
#pragma unroll
  for (int g8 = 0; g8 < 2; ++g8) {
    const float4 s0 = *reinterpret_cast<const float4*>(esc + g8 * 8);
    const float4 s1 = *reinterpret_cast<const float4*>(esc + g8 * 8 + 4);
    const float4 b0 = *reinterpret_cast<const float4*>(ebi + g8 * 8);
    const float4 b1 = *reinterpret_cast<const float4*>(ebi + g8 * 8 + 4);
    const float sv[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
    const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    float y[8];
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      const float2 o = __ffma2_rn(make_float2(__uint_as_float(r[g8 * 8 + j]), __uint_as_float(r[g8 * 8 + j + 1])),
                                  make_float2(sv[j], sv[j + 1]), make_float2(bv[j], bv[j + 1]));
      y[j] = o.x;
      y[j + 1] = o.y;
    }
    if (skip) {
      float sv8[8];
      bf16x8_to_f32(sk[g8], sv8);
#pragma unroll
      for (int j = 0; j < 8; ++j) y[j] += sv8[j];
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) y[j] = fminf(fmaxf(y[j], lo), hi);
    const uint32_t ch = static_cast<uint32_t>((cin + g8 * 8) >> 3);   // 16-byte chunk of the 128-byte row
    sts128(sbuf + lane * 128 + ((ch ^ (lane & 7)) << 4), pack_bf16x2(y[0], y[1]), pack_bf16x2(y[2], y[3]),
           pack_bf16x2(y[4], y[5]), pack_bf16x2(y[6], y[7]));
  }
}
__device__ __forceinline__ void load_skip16(uint4 (&k)[2], const __nv_bfloat16* skrow, int c, int c_hi, int cout_left) {
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int cc = c + u * 8;
    k[u] = (cc < c_hi && cc < cout_left) ? *reinterpret_cast<const uint4*>(skrow + cc) : make_uint4(0, 0, 0, 0);
  }
}

// Epilogue: 8 warps; warp e reads TMEM lane quarter e % 4 (tile rows
// 32*(e%4)..) and the column half e / 4 (when bn is a multiple of 32, else
// the first four warps take every column).  Per 32 columns: two tcgen05.ld
// x16 behind one wait, fused scale/bias(/residual)/act with FFMA2, a
// 64-byte-swizzled 32x64B smem chunk, and a TMA tensor store of that chunk
// (coalesced; rows >= M and columns >= Cout clipped by the tensor map).
__device__ void epilogue_role(const ExecParams& p, Ctx& cx) {
  SmemCtl* ctl = &g_ctl;
  const int etid = threadIdx.x - EPI_WARP0 * 32;  // 0..NEPI-1
  const int ew = etid >> 5, lane = etid & 31;
  const int q = ew & 3, hcol = ew >> 2;
  uint8_t* wbuf = cx.stage + ew * STAGE_WARP_BYTES * (EPI_DB ? 2 : 1);
  const uint32_t wbuf_s = smem_u32(wbuf);
  uint32_t islot = 0, acc = 0, nrel = 0;
  for (;;) {
    const uint32_t slot = islot % ITEM_RING;
    mbar_wait(&ctl->rfull[slot], (islot / ITEM_RING) & 1);
    const int idx = ctl->ring[slot].idx;
    const int kind = ctl->ring[slot].kind;
    // only the Item fields the epilogue and the release need (a whole Item
    // held across the epilogue spilled to local memory)
    const RingSlot& rsl = ctl->ring[slot];
    const EpiItem it{rsl.it.op, rsl.it.mt, rsl.it.nt, rsl.it.ks, rsl.it.idx, rsl.it.chunk, rsl.it.cluster, rsl.it.bud};
    const uint64_t t0 = ctl->ring[slot].t0;
    __syncwarp();
    if (lane == 0) mbar_arrive(&ctl->rempty[slot]);
    if (etid == 0 && idx >= 0 && kind == DK_GEMM) edbg(p, 0, acc);
    ++islot;
    if (idx < 0) break;
    if (kind != DK_GEMM) continue;
    const OpDev& opg = p.ops[it.op];
    const EpiOp op = make_epi(opg);
    const int bn = opg.bn;
    const int split = opg.split_k;
    const bool swap = op.swap;
    const int row = q * 32 + lane;
    const int mrep = opg.mrep;
    const int m0t = it.mt * BM * mrep, n0 = it.nt * bn;
    int m0 = m0t;                 // first row of the current 128-row half
    int m = m0 + row;
    const int tile = it.mt * opg.tiles_n + it.nt;
    const int cout_left = op.Cout - n0;
    // this warp's tile columns: halves split at a multiple of 32, so a staged
    // 32-column box never reaches into the other warp's columns (boxes past
    // bn only cover columns >= Cout, which the tensor map clips)
    const int c_split = (NEPI / 128 > 1) ? 32 * ((bn + 63) / 64) : bn;
    const int c_lo = hcol ? (c_split < bn ? c_split : bn) : 0;
    const int c_hi = hcol ? bn : (c_split < bn ? c_split : bn);
    // ---- global reads issued before the accumulator is waited on
    float sc_row = 1.0f, bi_row = 0.0f;
    if (swap) {
      if (m < op.Cout) { sc_row = op.scale[m]; bi_row = op.bias[m]; }
    } else {
      for (int j = etid; j < bn; j += NEPI) {   // columns past Cout (a ragged last N-tile) are never stored
        const bool in = n0 + j < op.Cout;
        ctl->epi_scale[j] = in ? op.scale[n0 + j] : 0.0f;
        ctl->epi_bias[j] = in ? op.bias[n0 + j] : 0.0f;
      }
    }
    bool do_skip = op.has_skip && split == 1 && m < op.M && !swap;
    const __nv_bfloat16* skrow =
        do_skip ? static_cast<const __nv_bfloat16*>(opg.skip) + static_cast<size_t>(m) * opg.lds + n0 : nullptr;
    uint4 skA[4], skB[4];  // residual values of the current / next 32 columns
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int cc = c_lo + u * 8;
      skA[u] = (do_skip && cc < c_hi && cc < cout_left) ? *reinterpret_cast<const uint4*>(skrow + cc)
                                                       : make_uint4(0, 0, 0, 0);
    }
    named_bar_sync(2, NEPI);  // epi_scale / epi_bias visible
    if (etid == 0) { dbg_mark(p, 12); edbg(p, 1, acc); }
    const uint32_t abuf = acc & 1;
    mbar_wait(&ctl->tfull[abuf], (acc / 2) & 1);
    if (etid == 0) { dbg_mark(p, 6); kdbg(p, 2, 2 * acc); edbg(p, 2, acc); }
    if (etid == 0 && p.trace && p.single_op < 0)
      p.trace[static_cast<size_t>(it.idx) * TRACE_FIELDS + 9] = static_cast<int64_t>(globaltimer());
    tc_fence_after();
#if GACER_DIAG
    if (p.dbg && p.dbg_spin) {   // diagnostic: delay the TMEM read after tfull
      const long long ts = clock64();
      while (clock64() - ts < p.dbg_spin) {}
    }
#endif
    if (etid == 0) edbg(p, 11, acc);
    uint32_t taddr = cx.tmem + abuf * BN_MAX + (static_cast<uint32_t>(q * 32) << 16);
    float* part = opg.partial + static_cast<size_t>(tile) * split * (BM * bn);
    const bool staged = EPI_STAGED && op.c_tma && !swap;
    const int CW = op.out_f32 ? 32 : 64;          // columns per 128-byte staged row
    for (int hf = 0; hf < mrep; ++hf) {         // M-pair tiles: two 128-row accumulators
    if (hf > 0) {
      m0 = m0t + hf * BM;
      m = m0 + row;
      taddr += static_cast<uint32_t>(bn);         // the second accumulator follows the first's bn columns
      do_skip = op.has_skip && m < op.M;
      skrow = do_skip ? static_cast<const __nv_bfloat16*>(opg.skip) + static_cast<size_t>(m) * opg.lds + n0 : nullptr;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int cc = c_lo + u * 8;
        skA[u] = (do_skip && cc < c_hi && cc < cout_left) ? *reinterpret_cast<const uint4*>(skrow + cc)
                                                         : make_uint4(0, 0, 0, 0);
      }
    }
    if (split == 1 && !staged && !op.out_f32 && !swap) {
      // lean direct bf16 path: same math as the staged path below, each
      // thread storing its row's 8-column groups with 16-byte global stores
      // (no staging buffer, no TMA-store waits)
      const float lo = op.act == ACT_NONE ? -INFINITY : 0.0f;
      const float hi = op.act == ACT_RELU6 ? 6.0f : INFINITY;
      const bool skip = do_skip;
      __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(op.out) + static_cast<size_t>(m) * op.ldo + n0;
      const bool row_ok = m < op.M;
      for (int c = c_lo; c < c_hi; c += 32) {
        uint32_t r[32];
        tmem_ld16_nw(taddr + c, r);
        tmem_ld16_nw(taddr + c + 16, r + 16);
        const float sc_l = ctl->epi_scale[c + lane], bi_l = ctl->epi_bias[c + lane];
        if (skip) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int cc = c + 32 + u * 8;
            skB[u] = (cc < c_hi && cc < cout_left) ? *reinterpret_cast<const uint4*>(skrow + cc) : make_uint4(0, 0, 0, 0);
          }
        }
        tmem_wait();
#pragma unroll
        for (int g8 = 0; g8 < 4; ++g8) {
          float y[8];
#pragma unroll
          for (int j = 0; j < 8; j += 2) {
            const int jj = g8 * 8 + j;
            const float2 o = __ffma2_rn(make_float2(__uint_as_float(r[jj]), __uint_as_float(r[jj + 1])),
                                        make_float2(__shfl_sync(0xffffffffu, sc_l, jj), __shfl_sync(0xffffffffu, sc_l, jj + 1)),
                                        make_float2(__shfl_sync(0xffffffffu, bi_l, jj), __shfl_sync(0xffffffffu, bi_l, jj + 1)));
            y[j] = o.x;
            y[j + 1] = o.y;
          }
          if (skip) {
            float sv[8];
            bf16x8_to_f32(skA[g8], sv);
#pragma unroll
            for (int j = 0; j < 8; ++j) y[j] += sv[j];
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) y[j] = fminf(fmaxf(y[j], lo), hi);
          const int cc = c + g8 * 8;
          if (row_ok && cc < cout_left) {
            if (cc + 8 <= cout_left) {
              *reinterpret_cast<uint4*>(orow + cc) = make_uint4(pack_bf16x2(y[0], y[1]), pack_bf16x2(y[2], y[3]),
                                                                pack_bf16x2(y[4], y[5]), pack_bf16x2(y[6], y[7]));
            } else {
              for (int j = 0; j < 8 && cc + j < cout_left; ++j) orow[cc + j] = __float2bfloat16_rn(y[j]);
            }
          }
        }
        if (skip) {
#pragma unroll
          for (int u = 0; u < 4; ++u) skA[u] = skB[u];
        }
      }
      if (etid == 0 && p.trace && p.single_op < 0)   // column loop done (diagnostics)
        p.trace[static_cast<size_t>(it.idx) * TRACE_FIELDS + 11] = static_cast<int64_t>(globaltimer());
    } else if (split == 1 && staged && !op.out_f32) {
#if GACER_EPI_V == 0
      // lean staged bf16 path: branch-free activation clamp, 64-column
      // staging chunks (a compile-time constant), scale/bias by shuffle
      const float lo = op.act == ACT_NONE ? -INFINITY : 0.0f;
      const float hi = op.act == ACT_RELU6 ? 6.0f : INFINITY;
      const bool skip = do_skip;
      const int row0 = m0 + q * 32;
      for (int c = c_lo; c < c_hi; c += 32) {
        uint32_t r[32];
        tmem_ld16_nw(taddr + c, r);
        tmem_ld16_nw(taddr + c + 16, r + 16);   // c + 32 <= BN_MAX: columns past c_hi are never stored
        const float sc_l = ctl->epi_scale[c + lane], bi_l = ctl->epi_bias[c + lane];
        if (skip) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int cc = c + 32 + u * 8;
            skB[u] = (cc < c_hi && cc < cout_left) ? *reinterpret_cast<const uint4*>(skrow + cc) : make_uint4(0, 0, 0, 0);
          }
        }
        const int cin = (c - c_lo) & 63;
        // staging buffer of this 64-column chunk (EPI_DB: two per warp, the
        // store of one chunk overlaps the conversion of the next)
        const uint32_t sbuf = wbuf_s + (EPI_DB ? (((c - c_lo) >> 6) & 1) * STAGE_WARP_BYTES : 0);
        if (cin == 0 && c > c_lo) {            // a new chunk: its buffer's previous store must have been read
          if (lane == 0) {
            if (EPI_DB) bulk_wait_read1();
            else bulk_wait_read0();
          }
          __syncwarp();
        }
        tmem_wait();
#pragma unroll
        for (int g8 = 0; g8 < 4; ++g8) {
          float y[8];
#pragma unroll
          for (int j = 0; j < 8; j += 2) {
            const int jj = g8 * 8 + j;
            const float2 o = __ffma2_rn(make_float2(__uint_as_float(r[jj]), __uint_as_float(r[jj + 1])),
                                        make_float2(__shfl_sync(0xffffffffu, sc_l, jj), __shfl_sync(0xffffffffu, sc_l, jj + 1)),
                                        make_float2(__shfl_sync(0xffffffffu, bi_l, jj), __shfl_sync(0xffffffffu, bi_l, jj + 1)));
            y[j] = o.x;
            y[j + 1] = o.y;
          }
          if (skip) {
            float sv[8];
            bf16x8_to_f32(skA[g8], sv);
#pragma unroll
            for (int j = 0; j < 8; ++j) y[j] += sv[j];
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) y[j] = fminf(fmaxf(y[j], lo), hi);
          const uint32_t ch = static_cast<uint32_t>((cin + g8 * 8) >> 3);   // 16-byte chunk of the 128-byte row
          sts128(sbuf + lane * 128 + ((ch ^ (lane & 7)) << 4), pack_bf16x2(y[0], y[1]), pack_bf16x2(y[2], y[3]),
                 pack_bf16x2(y[4], y[5]), pack_bf16x2(y[6], y[7]));
        }
        if (cin == 32 || c + 32 >= c_hi) {     // 64-column chunk complete: TMA-store it
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(op.tmap_c, sbuf, n0 + c - cin, row0);
            bulk_commit();
          }
        }
        if (skip) {
#pragma unroll
          for (int u = 0; u < 4; ++u) skA[u] = skB[u];
        }
      }
      if (etid == 0 && p.trace && p.single_op < 0)   // column loop done (diagnostics)
        p.trace[static_cast<size_t>(it.idx) * TRACE_FIELDS + 11] = static_cast<int64_t>(globaltimer());
      if (lane == 0) bulk_wait0();        // stores complete before the item is released
      __syncwarp();
#else
      // lean staged bf16 path, software-pipelined over 64-column steps: the
      // TMEM load of the second 32 columns is in flight while the first are
      // converted (and the next step's first 32 while the second are);
      // scale/bias are read as warp-uniform 16-byte smem broadcasts; the
      // activation clamp is branch-free; each 64-column step is one
      // double-buffered staging chunk and one TMA store.
      const float lo = op.act == ACT_NONE ? -INFINITY : 0.0f;
      const float hi = op.act == ACT_RELU6 ? 6.0f : INFINITY;
      const bool skip = do_skip;
      const int row0 = m0 + q * 32;
      // 16-column sub-chunks ping-pong between two register sets: the TMEM
      // load of sub-chunk k+1 is in flight while sub-chunk k is converted
      uint32_t ra[16], rb[16];
      uint4 ka[2], kb[2];                    // residual values of the current / next sub-chunk
      ka[0] = skA[0]; ka[1] = skA[1];
      tmem_ld16_nw(taddr + c_lo, ra);
      for (int c = c_lo; c < c_hi; c += 64) {
        const uint32_t sbuf = wbuf_s + (EPI_DB ? (((c - c_lo) >> 6) & 1) * STAGE_WARP_BYTES : 0);
        if (c > c_lo) {                        // this buffer's previous store must have been read
          if (lane == 0) {
            if (EPI_DB) bulk_wait_read1();
            else bulk_wait_read0();
          }
          __syncwarp();
        }
#pragma unroll
        for (int sub = 0; sub < 4; sub += 2) {
          const int ca = c + sub * 16, cb = ca + 16;   // columns of ra / rb
          if (ca >= c_hi) break;
          tmem_wait();
          tmem_pin16(ra);
          if (cb < c_hi) tmem_ld16_nw(taddr + cb, rb);   // cb + 16 <= BN_MAX: never past the accumulator
          if (skip) load_skip16(kb, skrow, cb, c_hi, cout_left);
          epi_chunk16(ra, ctl->epi_scale + ca, ctl->epi_bias + ca, skip, ka, lo, hi, sub * 16, sbuf, lane);
          if (cb >= c_hi) break;
          tmem_wait();
          tmem_pin16(rb);
          if (cb + 16 < c_hi) tmem_ld16_nw(taddr + cb + 16, ra);
          if (skip) load_skip16(ka, skrow, cb + 16, c_hi, cout_left);
          epi_chunk16(rb, ctl->epi_scale + cb, ctl->epi_bias + cb, skip, kb, lo, hi, sub * 16 + 16, sbuf, lane);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(op.tmap_c, sbuf, n0 + c, row0);
          bulk_commit();
        }
      }
      if (etid == 0 && p.trace && p.single_op < 0)   // column loop done (diagnostics)
        p.trace[static_cast<size_t>(it.idx) * TRACE_FIELDS + 11] = static_cast<int64_t>(globaltimer());
      if (lane == 0) bulk_wait0();        // stores complete before the item is released
      __syncwarp();
#endif
    } else if (split == 1) {
      for (int c = c_lo; c < c_hi; c += 32) {
        uint32_t r[32];
        if (etid == 0 && c == c_lo) edbg(p, 12, acc);
        tmem_ld16_nw(taddr + c, r);
        if (c + 16 < c_hi) tmem_ld16_nw(taddr + c + 16, r + 16);
        tmem_wait();
        if (etid == 0) { dbg_mark(p, 16); edbg(p, 3, acc); }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int cc = c + 32 + u * 8;
          skB[u] = (do_skip && cc < c_hi && cc < cout_left) ? *reinterpret_cast<const uint4*>(skrow + cc)
                                                           : make_uint4(0, 0, 0, 0);
        }
        const float* v = reinterpret_cast<const float*>(r);
        if (swap) {
#pragma unroll
          for (int u = 0; u < 32; u += 8)
            if (c + u < c_hi) epilogue_store8_swap(op, m, n0 + c + u, v + u, sc_row, bi_row);
        } else if (staged) {
          const int cin = (c - c_lo) % CW;       // column offset inside the staged chunk
          if (cin == 0 && c > c_lo) {            // a new chunk: wait until the last store read the buffer
            if (lane == 0) bulk_wait_read0();
            __syncwarp();
          }
          const float sc_l = ctl->epi_scale[c + lane], bi_l = ctl->epi_bias[c + lane];  // one LDS per lane
#pragma unroll
          for (int sub = 0; sub < 32; sub += 16) {
            if (c + sub < c_hi) {
              float y[8];
              epi_math8_shfl(op, v + sub, sc_l, bi_l, sub, skA[sub / 8], y);
              stage8(wbuf_s, lane, cin + sub, y, op.out_f32);
              epi_math8_shfl(op, v + sub + 8, sc_l, bi_l, sub + 8, skA[sub / 8 + 1], y);
              stage8(wbuf_s, lane, cin + sub + 8, y, op.out_f32);
            }
          }
          if (cin + 32 == CW || c + 32 >= c_hi) {  // chunk complete: TMA-store it
            if (etid == 0) { dbg_mark(p, 17); edbg(p, 4, acc); }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(op.tmap_c, wbuf_s, n0 + c - cin, m0 + q * 32);
              bulk_commit();
            }
            if (etid == 0) { dbg_mark(p, 18); edbg(p, 5, acc); }
          }
        } else {
#pragma unroll
          for (int u = 0; u < 32; u += 8)
            if (c + u < c_hi) epilogue_store8(op, m, n0 + c + u, v + u, ctl->epi_scale + c + u, ctl->epi_bias + c + u, skA[u / 8]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) skA[u] = skB[u];
      }
      if (etid == 0 && p.trace && p.single_op < 0)   // column loop done (diagnostics)
        p.trace[static_cast<size_t>(it.idx) * TRACE_FIELDS + 11] = static_cast<int64_t>(globaltimer());
      if (staged) {
        if (etid == 0) { dbg_mark(p, 14); edbg(p, 6, acc); }
        if (lane == 0) bulk_wait0();        // stores complete before the item is released
        __syncwarp();
        if (etid == 0) edbg(p, 8, acc);
      }
    } else {
      // partial layout [tile][ks][bn/4][BM] float4: a warp's 32 rows of one
      // float4 column are 512 contiguous bytes (coalesced write and read)
      float4* mine = reinterpret_cast<float4*>(part + static_cast<size_t>(it.ks) * (BM * bn)) + row;
      for (int c = c_lo; c < c_hi; c += 32) {
        uint32_t r[32];
        tmem_ld16_nw(taddr + c, r);
        if (c + 16 < c_hi) tmem_ld16_nw(taddr + c + 16, r + 16);
        tmem_wait();
        const float* v = reinterpret_cast<const float*>(r);
#pragma unroll
        for (int u = 0; u < 32; u += 4)
          if (c + u < c_hi) __stcg(mine + ((c + u) >> 2) * BM, make_float4(v[u], v[u + 1], v[u + 2], v[u + 3]));
      }
    }
    }  // halves
    if (etid == 0) { dbg_mark(p, 13); edbg(p, 7, acc - 0); }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&ctl->tempty[abuf]);
    ++acc;
    if (split > 1 && !opg.partials_only) {   // last arrival reduces the splits in order
      named_bar_sync(2, NEPI);
      if (etid == 0) {
        __threadfence();
        const uint32_t old = atomicAdd(opg.tile_cnt + tile, 1u);
        const int last = (old == static_cast<uint32_t>(split - 1));
        if (last) opg.tile_cnt[tile] = 0;  // all arrivals done: re-arm for the next round
        ctl->epi_flag = last;
        __threadfence();
      }
      named_bar_sync(2, NEPI);
      if (ctl->epi_flag) {
        // fixed ks order (bit-identical in every mode); the partial loads of
        // an 8-column chunk are in flight together
        const __nv_bfloat16* skb = static_cast<const __nv_bfloat16*>(opg.skip);
        for (int c = c_lo; c < c_hi; c += 8) {
          if (staged && c > c_lo && ((c - c_lo) % CW) == 0) {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(op.tmap_c, wbuf_s, n0 + c - CW, m0 + q * 32);
              bulk_commit();
              bulk_wait_read0();
            }
            __syncwarp();
          }
          float4 ld[MAX_SPLIT][2];
#pragma unroll
          for (int ks = 0; ks < MAX_SPLIT; ++ks)
            if (ks < split) {
              const float4* qp = reinterpret_cast<const float4*>(part + static_cast<size_t>(ks) * (BM * bn)) + row;
              ld[ks][0] = __ldcg(qp + (c >> 2) * BM);
              ld[ks][1] = __ldcg(qp + ((c >> 2) + 1) * BM);
            }
          float s8[8] = {ld[0][0].x, ld[0][0].y, ld[0][0].z, ld[0][0].w, ld[0][1].x, ld[0][1].y, ld[0][1].z, ld[0][1].w};
#pragma unroll
          for (int ks = 1; ks < MAX_SPLIT; ++ks)
            if (ks < split) {
              s8[0] += ld[ks][0].x; s8[1] += ld[ks][0].y; s8[2] += ld[ks][0].z; s8[3] += ld[ks][0].w;
              s8[4] += ld[ks][1].x; s8[5] += ld[ks][1].y; s8[6] += ld[ks][1].z; s8[7] += ld[ks][1].w;
            }
          for (int ks = MAX_SPLIT; ks < split; ++ks) {   // long reductions (weight gradients), in split order
            const float4* qp = reinterpret_cast<const float4*>(part + static_cast<size_t>(ks) * (BM * bn)) + row;
            const float4 a = __ldcg(qp + (c >> 2) * BM), b = __ldcg(qp + ((c >> 2) + 1) * BM);
            s8[0] += a.x; s8[1] += a.y; s8[2] += a.z; s8[3] += a.w;
            s8[4] += b.x; s8[5] += b.y; s8[6] += b.z; s8[7] += b.w;
          }
          if (swap) {
            epilogue_store8_swap(op, m, n0 + c, s8, sc_row, bi_row);
          } else {
            uint4 k8 = make_uint4(0, 0, 0, 0);
            if (op.has_skip && m < op.M && c < cout_left)
              k8 = *reinterpret_cast<const uint4*>(skb + static_cast<size_t>(m) * opg.lds + n0 + c);
            if (staged) {
              float y[8];
              epi_math8(op, s8, ctl->epi_scale + c, ctl->epi_bias + c, k8, y);
              stage8(wbuf_s, lane, (c - c_lo) % CW, y, op.out_f32);
            } else {
              epilogue_store8(op, m, n0 + c, s8, ctl->epi_scale + c, ctl->epi_bias + c, k8);
            }
          }
        }
        if (staged && c_hi > c_lo) {
          const int last = c_lo + ((c_hi - c_lo - 1) / CW) * CW;
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(op.tmap_c, wbuf_s, n0 + last, m0 + q * 32);
            bulk_commit();
            bulk_wait0();
          }
          __syncwarp();
        }
      }
    }
    fence_proxy_async_global();  // generic stores -> later TMA reads by consumers
    if (etid == 0) { dbg_mark(p, 15); kdbg(p, 2, 2 * acc - 1); edbg(p, 9, acc - 1); }
    named_bar_sync(2, NEPI);     // also: epi_scale/bias free for the next item
    if (etid == 0) { dbg_mark(p, 7); edbg(p, 10, acc - 1); }
    if (etid == 0 && p.trace && p.single_op < 0)
      p.trace[static_cast<size_t>(it.idx) * TRACE_FIELDS + 10] = static_cast<int64_t>(globaltimer());
    if (etid == 0 && p.single_op < 0) {   // hand the release to the releaser lane
      const uint32_t ls = nrel % ITEM_RING;
      if (nrel >= ITEM_RING) mbar_wait(&ctl->lempty[ls], ((nrel / ITEM_RING) + 1) & 1);
      Item& ri = ctl->rel[ls].it;   // what release_item reads
      ri.op = it.op; ri.idx = it.idx; ri.chunk = it.chunk; ri.cluster = it.cluster; ri.bud = it.bud;
      ctl->rel[ls].t0 = t0;
      ctl->rel[ls].idx = idx;
      mbar_arrive(&ctl->lfull[ls]);
      ++nrel;
    }
  }
  if (etid == 0 && p.single_op < 0) {     // STOP for the releaser
    const uint32_t ls = nrel % ITEM_RING;
    if (nrel >= ITEM_RING) mbar_wait(&ctl->lempty[ls], ((nrel / ITEM_RING) + 1) & 1);
    ctl->rel[ls].idx = -1;
    mbar_arrive(&ctl->lfull[ls]);
  }
}

// Releaser (warp 1, lane 1): publishes completed GEMM items -- fence, then
// the chunk and cluster counters -- off the epilogue warps' critical path.
// Ordering: the epilogue's stores (TMA stores waited to completion, generic
// stores) precede its named barrier and mbarrier arrive (release.cta); this
// lane's wait is an acquire, and the (cumulative) fence.release.gpu orders the chain
// at GPU scope before the counter atomics.
__device__ void releaser_role(const ExecParams& p, Ctx& cx) {
  SmemCtl* ctl = &g_ctl;
  uint32_t n = 0;
  for (;;) {
    const uint32_t ls = n % ITEM_RING;
    mbar_wait(&ctl->lfull[ls], (n / ITEM_RING) & 1);
    const RingSlot r = ctl->rel[ls];
    mbar_arrive(&ctl->lempty[ls]);
    ++n;
    if (r.idx < 0) break;
    release_item(p, r.it, r.t0, p.ops[r.it.op]);
  }
}

template <bool TRAIN>
__device__ void executor_body(const ExecParams& p, uint8_t* smem_raw) {
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Ctx cx;
  cx.ring = base;
  cx.stage = base + SMEM_RING_BYTES;
  cx.ctl = &g_ctl;
  SmemCtl* ctl = &g_ctl;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    g_dbg_seen = 0;
    for (int s = 0; s < STAGES; ++s) { mbar_init(&ctl->full[s], 1); mbar_init(&ctl->empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&ctl->tfull[a], 1); mbar_init(&ctl->tempty[a], NEPI / 32); }
    for (int r = 0; r < ITEM_RING; ++r) { mbar_init(&ctl->rfull[r], 1); mbar_init(&ctl->rempty[r], RING_CONSUMERS); }
    for (int r = 0; r < ITEM_RING; ++r) { mbar_init(&ctl->lfull[r], 1); mbar_init(&ctl->lempty[r], 1); }
    fence_mbar_init();
  }
  for (int i = tid; i < STAT_TENANTS + 2; i += NTHREADS) ctl->st_ns[i] = 0;
  if (p.single_op < 0) {  // cache the queue segments
    const int ns = p.n_tenants * p.n_clusters;
    const int nc = ns < MAX_SMEM_SEGS ? ns : MAX_SMEM_SEGS;
    for (int i = tid; i < nc; i += NTHREADS) ctl->segs[i] = p.segs[i];
    if (tid == 0) ctl->n_segs_smem = nc;
  } else if (tid == 0) {
    ctl->n_segs_smem = 0;
  }
  if (p.self_gates && blockIdx.x == 0 && tid == 0) {   // device-resident inputs: open the input gates
    for (int i = 0; i < p.n_gates; ++i) atomicMax(p.chunk_done + p.gate0 + i, p.epoch);
    fence_release_gpu();
  }
  if (warp == MMA_WARP) tmem_alloc(&ctl->tmem_base, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  cx.tmem = ctl->tmem_base;
  if (tid == 0) dbg_mark(p, 0);

  if (warp == SCHED_WARP) {
    if (tid == 0) scheduler_role(p, cx);
  } else if (warp == MMA_WARP) {
    if ((tid & 31) == 0) mma_role(p, cx);
    else if ((tid & 31) == 1 && p.single_op < 0) releaser_role(p, cx);
  } else if (warp < EPI_WARP0) {
    worker_role<TRAIN>(p, cx);
  } else {
    epilogue_role(p, cx);
  }

  tc_fence_before();
  __syncthreads();
  if (tid == 0) dbg_mark(p, 11);
  if (warp == MMA_WARP) tmem_dealloc(cx.tmem, TMEM_COLS);
  if (p.stats && p.single_op < 0 && tid < STAT_TENANTS + 2 && ctl->st_ns[tid])
    atomicAdd(p.stats + tid, ctl->st_ns[tid]);
  if (tid == 0 && p.single_op < 0) {
    __threadfence();
    const uint32_t old = atomicAdd(p.exit_count, 1u);
    if (old == gridDim.x - 1) {  // last CTA out re-arms the claim counters
      for (int i = 0; i < p.n_heads; ++i) p.heads[i] = 0;
      // an aborted round (watchdog): saturate every completion counter so
      // that stream-side waits on them (gacer_stream_wait_grads) release
      // instead of blocking their stream forever; the host resets the
      // counters before the next round (sticky GACER_E_DEADLOCK path)
      if (*reinterpret_cast<volatile int32_t*>(p.error))
        for (int i = 0; i < p.n_counters; ++i) p.chunk_done[i] = 0xFFFFFFFFu;
      *p.exit_count = 0;
      __threadfence();
    }
  }
}

extern "C" __global__ void __launch_bounds__(NTHREADS, 1) gacer_executor(ExecParams p) {
  extern __shared__ uint8_t smem_raw[];
  executor_body<false>(p, smem_raw);
}

// The same executor with the training tenant's virtual-grid items (DK_VGRID)
// compiled in; launched only for rounds with a training tenant.  A separate
// instantiation keeps the operators' call out of the inference kernel's
// register allocation (it made the TMA producer loop spill).
extern "C" __global__ void __launch_bounds__(NTHREADS, 1) gacer_executor_train(ExecParams p) {
  extern __shared__ uint8_t smem_raw[];
  executor_body<true>(p, smem_raw);
}

// Standalone CUDA-core op kernel (baselines): one item per CTA, same tile function.
extern "C" __global__ void __launch_bounds__(CC_THREADS) op_cc_kernel(const OpDev* ops, int op_idx) {
  __shared__ __align__(16) float red[CC_THREADS * 8];
  extern __shared__ __align__(1024) uint8_t win_buf[];
  const OpDev& op = ops[op_idx];
  const Item it = decode_single(op, op_idx, blockIdx.x);
  if (op.kind == DK_VGRID) {
    const int v0 = it.mt * op.bm, v1 = min(v0 + op.bm, op.vblocks);
    if (vg_streamable(op.vfn)) {
      vg_stream_item(op.vfn, op.va, v0, v1, op.vblocks, threadIdx.x, CC_THREADS, win_buf, WIN_SMEM_BYTES);
      return;
    }
    for (int vb = v0; vb < v1; ++vb) run_vgrid(op.vfn, op.va, vb, op.vblocks, threadIdx.x, CC_THREADS, win_buf);
  } else if (op.win) {
    window_smem(op, it, threadIdx.x, CC_THREADS, smem_u32(win_buf), 1);
  } else {
    run_cc(op, it, threadIdx.x, red);
  }
}

// =====================================================================
// host-side launchers (C++ linkage, used by host.cpp)
// =====================================================================
int executor_smem_bytes() { return SMEM_BYTES; }

cudaError_t configure_kernels() {
  static_assert(WIN_SMEM_BYTES <= SMEM_RING_BYTES, "window staging must fit in the GEMM ring");
  cudaError_t e = cudaFuncSetAttribute(gacer_executor, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(gacer_executor_train, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(op_cc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, WIN_SMEM_BYTES);
}

cudaError_t launch_executor(const ExecParams& p, int grid, cudaStream_t s, bool train) {
  if (train) gacer_executor_train<<<grid, NTHREADS, SMEM_BYTES, s>>>(p);
  else gacer_executor<<<grid, NTHREADS, SMEM_BYTES, s>>>(p);
  return cudaGetLastError();
}

// Standalone per-op launch (sequential / multi-stream baselines).  GEMM ops
// run the executor kernel in single-op mode: persistent over the op's tiles,
// the same warp-specialised pipeline and tile functions.
cudaError_t launch_op(const ExecParams& base, const OpDev* ops_dev, int op_idx, int kind, int n_items, int num_sms,
                      cudaStream_t s) {
  if (kind == DK_GEMM) {
    ExecParams p = base;
    p.ops = ops_dev;
    if (p.dbg) p.dbg += static_cast<size_t>(op_idx) * 148 * DBG_EVENTS;
    p.single_op = op_idx;
    p.trace = nullptr;
    const int grid = n_items < num_sms ? n_items : num_sms;
    gacer_executor<<<grid, NTHREADS, SMEM_BYTES, s>>>(p);
  } else {
    op_cc_kernel<<<n_items, CC_THREADS, WIN_SMEM_BYTES, s>>>(ops_dev, op_idx);
  }
  return cudaGetLastError();
}

}  // namespace gacer
