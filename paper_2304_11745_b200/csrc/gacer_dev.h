// gacer_dev.h -- structures shared by the host runtime (host.cpp) and the
// sm_100a kernels (executor.cu).  Plain old data, uploaded once per
// registration / plan.
#pragma once
#include <stdint.h>

namespace gacer {

// ---------------------------------------------------------------- op kinds
// Lowered ("fused") operator kinds executed by the device.
enum DevKind : int32_t {
  DK_GEMM = 1,     // bf16 implicit-GEMM conv (im2col A) or swap-AB linear, tcgen05 + TMEM
  DK_DW = 2,       // depthwise 3x3-style conv (groups == C), CUDA cores
  DK_MAXPOOL = 3,
  DK_AVGPOOL = 4,
  DK_GAP = 5,
  DK_SIMT_GEMM = 6,// fp32 conv / linear on CUDA cores (FFMA), fixed K order
  DK_ELTWISE = 7,  // y = act(a [+ b]) standalone elementwise
  DK_VGRID = 8,    // a training-tenant CUDA-core operator run as a virtual grid (train_dev.cuh)
};

// Virtual-grid operators of the training tenant (train_dev.cuh documents each
// one's argument mapping).
enum VFn : int32_t {
  VF_NONE = 0,
  VF_BN_PARTIAL, VF_BN_FINALIZE, VF_BN_APPLY, VF_RELU_BWD, VF_ADD,
  VF_MAXPOOL_FWD, VF_MAXPOOL_ARGMAX, VF_MAXPOOL_BWD, VF_GAP_FWD, VF_GAP_BWD,
  VF_LINEAR_FWD, VF_LINEAR_DX, VF_LINEAR_DW, VF_SOFTMAX_CE, VF_MEAN, VF_SGD,
  VF_FILTER, VF_DILATE, VF_TRANSPOSE_IM2COL, VF_WGRAD_PERMUTE, VF_WGRAD_REDUCE, VF_PHASE_SCATTER,
  VF_FILTER_ALL,
};

// One filter-packing job of the training tenant's step (VF_FILTER_ALL packs
// every conv's forward and data-gradient GEMM operand in one operator):
// the vg_filter arguments with resolved pointers; `start` = the job's first
// element in the concatenated output index space.
struct FilterJob {
  const float* w;
  void* out;
  int64_t start;
  int32_t i[14];        // vg_filter's i0..i13
  int32_t pad[2];
};

// Phase decomposition of a strided conv's data gradient (stride S): input
// pixel h with (h + p) mod S = a receives exactly the taps r = a + S i, from
// dy rows u - i with u = (h + p - a) / S -- a stride-1 conv of dy with the
// KI = ceil((K - a) / S)-tap sub-filter over the output rows u in [u0, u1).
struct DgPhase {
  int K;        // taps of the phase along this dimension (0: no tap reaches it)
  int u0, n;    // first output index u and the count of them (u in [u0, u0 + n))
  int pad;      // the phase conv's low padding: K - 1 - u0 (its first window starts at u0 - (K - 1))
};
__host__ __device__ inline DgPhase dg_phase(int a, int K, int S, int p, int H) {
  DgPhase d;
  d.K = a < K ? (K - a + S - 1) / S : 0;
  const int lo = p - a;                                   // h + p - a = S u  =>  u >= (p - a) / S for h >= 0
  d.u0 = lo <= 0 ? 0 : (lo + S - 1) / S;
  const int hi = H - 1 + p - a;                           // h <= H - 1
  d.n = hi < 0 ? 0 : hi / S + 1 - d.u0;
  if (d.n < 0) d.n = 0;
  d.pad = d.K - 1 - d.u0;
  return d;
}

// Virtual-grid geometry, shared by the host lowering and the standalone calls.
constexpr int VG_THREADS = 192;               // = NWORK: the executor's worker group
constexpr int VG_MAX_PARTIALS = 148 * 4;      // row blocks of a BN reduction
constexpr int VG_ROWS_PER_BLOCK_MIN = 32;
inline int vg_bn_partials(int64_t M) {        // BN partial-sum row blocks for M rows
  int64_t p = (M + VG_ROWS_PER_BLOCK_MIN - 1) / VG_ROWS_PER_BLOCK_MIN;
  return static_cast<int>(p < VG_MAX_PARTIALS ? (p < 1 ? 1 : p) : VG_MAX_PARTIALS);
}
inline int vg_grid_for(int64_t work) {        // grid-stride ops: blocks for `work` thread tasks
  int64_t b = (work + VG_THREADS - 1) / VG_THREADS;
  const int64_t cap = 148 * 8;
  return static_cast<int>(b < cap ? (b < 1 ? 1 : b) : cap);
}

// BN apply: a grid whose thread stride (blocks x VG_THREADS) is a multiple of
// C / 8 for every C / 8 dividing 768 (C <= 2048: a multiple of 4 blocks), so
// each thread keeps one channel group
inline int vg_apply_blocks(int64_t work) { return (vg_grid_for(work) + 3) / 4 * 4; }

// Weight-gradient operand transpose tiles: TC channels x (16384 / TC) pixels
// (narrow inputs, e.g. the 8-channel stem image, take long pixel runs)
#ifdef __CUDACC__
#define GACER_HD __host__ __device__
#else
#define GACER_HD
#endif
GACER_HD inline int vg_transpose_tc(int C) { int c = (C + 7) / 8 * 8; return c < 64 ? c : 64; }
constexpr int VG_TRANSPOSE_TILE = 16384;       // elements per transpose tile (32 KB of smem)
GACER_HD inline int vg_transpose_blocks(int C, int KH, int KW, int Kpad) {
  const int tc = vg_transpose_tc(C), tp = VG_TRANSPOSE_TILE / tc;
  return ((Kpad + tp - 1) / tp) * ((C + tc - 1) / tc) * KH * KW;
}
constexpr int VG_MAX_BN_C = 2048;             // BN channels (per-channel constants staged in smem)

// Arguments of a virtual-grid operator: pointers, 64-bit sizes, ints, floats.
struct VArgs {
  const void* p[8];
  int64_t n[2];
  int32_t i[14];
  float f[4];
};

enum Act : int32_t { ACT_NONE = 0, ACT_RELU = 1, ACT_RELU6 = 2, ACT_HSWISH = 3, ACT_HSIGMOID = 4 };

// GEMM tile geometry
constexpr int BM = 128;           // rows per tile (UMMA M)
constexpr int BK = 64;            // bf16 elements per K-block = one 128-byte swizzle row
constexpr int BN_MAX = 256;       // max UMMA N per tile
#ifndef GACER_STAGES
#define GACER_STAGES 3
#endif
// smem ring depth (A 16 KB + B 32 KB per stage).  3 stages leave room for the
// double-buffered epilogue staging (GACER_EPI_DB); same-box A/B vs 4 stages
// with a single staging buffer: ~1.5% shorter D2 rounds.
constexpr int STAGES = GACER_STAGES;
// TMA-issuing producer threads per CTA (lane 0 of worker warps 0..NPROD-1).
// Producer j owns the stages s = j (mod NPROD); NPROD == STAGES so that no two
// producers ever wait on the same stage barrier (a parity wait cannot tell
// phase u from phase u - 2).
constexpr int NPROD = STAGES;
constexpr int ITEM_RING = 4;      // scheduler -> MMA/epilogue item queue depth
// warp roles of the executor CTA (16 warps; 4 per SM sub-partition, <= 128 registers)
constexpr int SCHED_WARP = 0;     // warp 0: scheduler (lane 0) -- claims ready items into the item ring
constexpr int MMA_WARP = 1;       // warp 1: single-thread tcgen05.mma issue
constexpr int WORK_WARP0 = 2;     // warps 2-7: TMA / gather loads of GEMM items, CUDA-core items
constexpr int NWORK = 192;
constexpr int EPI_WARP0 = 8;      // warps 8-11: TMEM -> register epilogue; warp w reads TMEM lane
constexpr int NEPI = 128;         //   quarter w % 4 (8 warps splitting the columns measured no faster)
constexpr int NTHREADS = 384;
constexpr int CC_THREADS = NWORK; // threads that execute a CUDA-core item
constexpr int CC_RUN = 8;         // consecutive output pixels per thread in the row-run window kernel
constexpr int CC_TASKS_PER_THREAD = 4;
constexpr int MAX_SPLIT = 4;      // split-K factor cap of forward layers (fixed per layer shape)
constexpr int MAX_SPLIT_LONG = 64; // cap for the long pixel reductions of weight gradients
constexpr int LOOKAHEAD = 3;      // max claimed items not yet picked up by every role (per CTA)
#ifndef GACER_INLINE_DEPS
#define GACER_INLINE_DEPS 4
#endif
constexpr int INLINE_DEPS = GACER_INLINE_DEPS;    // dependencies stored inside the Item
constexpr int MAX_SMEM_SEGS = 256;
constexpr int WIN_IN_BYTES = 96 * 1024;   // window_smem: staged input rows of one image segment
constexpr int WIN_SMEM_BYTES = WIN_IN_BYTES + (9 + 2) * 64 * 4 + 1024;  // + dw weights/scale/bias (kh*kw <= 9)

// operand A load mode of a GEMM op
// A_MN: weight-gradient GEMM with both operands MN-major, read in place (no
// staged transposes): A = dy [pixels][Cout] (2-D TMA, 64 channels x 64
// pixels per box), B = im2col(x) (im2col TMA, 64 pixels x 64 channels of one
// tap per box); K runs over the output pixels.
// A_IM2COL8: an 8-channel input (the graph's RGB image padded to 8): each
// K-block holds 8 filter taps; A = 8 im2col TMA boxes of 128 pixels x 8
// channels (16 B) in the no-swizzle K-major core-matrix layout (8 rows x
// 16 B per core matrix, SBO 128 B, the next tap LBO 2 KB), B = the weights
// pre-packed in the same layout per (N-tile, K-block) and fetched with one
// bulk copy.  Replaces the cp.async gather for stems (7x7 s2, 11x11 s4, 3x3).
// A_MN8: A_MN for an 8-channel input (the stem's weight gradient): B = one
// im2col box of 64 pixels x 8 channels per tap, in the no-swizzle MN-major
// core-matrix layout (K rows 16 B apart, LBO 128 B, the next tap SBO 1 KB).
enum AMode : int32_t { A_GATHER = 0, A_IM2COL = 1, A_ROWS = 2, A_MN = 3, A_IM2COL8 = 4, A_MN8 = 5 };

struct OpDev {
  int32_t kind;            // DevKind
  int32_t tenant;
  int32_t act;             // Act
  int32_t out_f32;         // output dtype: 1 = float32, 0 = bf16 (or f32 for fp32 tenants: see elem)
  int32_t f32;             // 1 = fp32 tenant (inputs/weights fp32), 0 = bf16
  int32_t swap;            // GEMM: 1 = swap-AB linear (A = weights, B = activations); 2 = same, A loaded L2 evict-first
  int32_t cip;             // avgpool count_include_pad
  int32_t has_skip;        // 1: + skip (same shape); 2: * skip[n][c] (channel scale, DK_ELTWISE)

  // input activation tensor, NHWC: elem(n,h,w,c) = in[((n*H + h)*W + w)*ldi + c]
  const void* in;
  int32_t B, H, W, C, ldi; // C = channels read (multiple of 8 for bf16)
  // output tensor NHWC (Ho x Wo pixels, Cout channels), row stride ldo
  void* out;
  int32_t Ho, Wo, Cout, ldo;
  // residual operand (same shape/layout as out), row stride lds
  const void* skip;
  int32_t lds, mrep;       // mrep: 128-row accumulators per GEMM tile (2: M-pair tile of 256 rows)

  int32_t kh, kw, stride, ph, pw, win; // win: 1 = window op staged through shared memory (window_smem)

  // GEMM view
  int32_t M, N, K;         // conv: M = B*Ho*Wo, N = Cout, K = kh*kw*C;  swap: M = Cout, N = B, K = C_flat
  int32_t Kpad;            // multiple of BK (weights row length)
  int32_t tiles_m, tiles_n;
  int32_t bm, bn;          // tile sizes (GEMM: bm = 128; CC ops: pixel rows / channels per tile)
  int32_t split_k, nkb;    // nkb = Kpad / BK
  const void* wt;          // packed weights: bf16 [Npad or Mpad][Kpad] K-major (fp32 [Cout][K] for SIMT);
                           // DW: [kh*kw][C] channel-minor
  int32_t ldw;
  int32_t affine;          // DK_ELTWISE: y = x * scale + bias first (a standalone BatchNorm)
  const void* act_b;       // swap-AB: activations as the B operand, row stride ldb (elements)
  int32_t ldb;
  int32_t partials_only;   // split-K: write the per-split partials only (reduced by a separate kernel)
  const float* scale;      // [Cout] folded BN scale (1 if no BN)
  const float* bias;       // [Cout] folded BN shift + conv bias
  float* partial;          // split-K workspace [tiles][split][BM*bn] fp32
  uint32_t* tile_cnt;      // split-K arrival counters [tiles]
  const void* tmap_a;      // CUtensorMap (64 B aligned, device memory): im2col or tiled A
  const void* tmap_b;      // CUtensorMap: tiled B (weights, or activations for swap-AB)
  int32_t a_mode;          // AMode
  int32_t c_tma;           // 1: epilogue stores through smem staging + TMA tensor store (tmap_c)
  const void* tmap_c;      // CUtensorMap of the output [M rows][Cout] (row stride ldo)
  // DK_VGRID: operator, virtual grid size; an item runs virtual blocks
  // [mt * bm, min((mt + 1) * bm, vblocks))
  int32_t vfn, vblocks;
  VArgs va;
  // L2 prefetch on this op's first item (tile 0, 0, 0): the packed weights of
  // the tenant's next GEMM ops (a chain op's first weight tiles otherwise
  // come from DRAM on its critical path).  bytes 0 = none.
  const void* pf_ptr[2];
  uint32_t pf_bytes[2];
};

// One work item: one output tile (mt, nt) of one op, K-slice ks.  Items are
// stored in queue order (grouped by (tenant, cluster) segment).
struct Item {
  int32_t op;
  int32_t mt, nt, ks;
  int32_t chunk;           // global chunk counter id (released on completion)
  int32_t cluster;
  uint32_t prio;           // upward rank: estimated remaining critical path (ns) of its tenant
  int32_t idx;             // position in the item array (trace / diagnostics)
  int32_t op_left;         // items of the same op after this one in its queue segment
  int32_t kind;            // DevKind of the op (saves the scheduler a global load per claim)
  int32_t dep_count;       // <= INLINE_DEPS: dc/dt hold them, else dep list at dep_begin
  int32_t dep_begin;
  int32_t dc[INLINE_DEPS]; // producer chunk counters
  uint32_t dt[INLINE_DEPS];// their per-round targets
  // SM budget of the item's chunk (gacer_chunking.sm_budget; the paper's
  // W(O^B) share): bud = the chunk's budget counter (-1:
  // none), incremented by every released item of the chunk; this item (the
  // j-th of its chunk in queue order, budget b) is ready only once
  // counter >= (epoch - 1) * btot + boff, boff = max(0, j - b + 1), so at most
  // b items of the chunk are claimed and not yet complete at any time.
  int32_t bud;
  uint32_t btot, boff;
};

struct Dep {
  int32_t counter;         // chunk counter id
  uint32_t target;         // items of that chunk per round
};

struct Seg {                // queue segment for (tenant, cluster)
  int32_t begin, size;
};

struct ExecParams {
  const OpDev* ops;
  const Item* items;        // queue order, grouped by segment
  const Dep* deps;          // overflow dependency lists (dep_count > INLINE_DEPS)
  const Seg* segs;          // [n_tenants * n_clusters]
  const int32_t* cta_pref;  // [num_ctas * n_tenants] tenant preference (-1 = none)
  uint32_t* heads;          // [n_tenants * n_clusters] claim counters (reset by last CTA)
  uint32_t* chunk_done;     // [n_chunks] epoch-accumulated completion counts
  uint32_t* cluster_done;   // [n_clusters] epoch-accumulated
  const uint32_t* cluster_total; // [n_clusters] items per round
  uint32_t* exit_count;
  int32_t* error;           // device error flag (deadlock watchdog)
  int64_t* trace;           // optional [n_items * 8]
  int32_t n_tenants, n_clusters;
  int32_t k_first, k_last;  // clusters served by this launch (host-synchronised pointers: one each)
  int32_t gate0, n_gates;   // per-tenant input-gate counters (chunk_done[gate0 .. gate0 + n_gates))
  int32_t self_gates;       // 1: inputs are device-resident, the kernel opens the gates itself
  uint32_t epoch;           // round number since plan install, >= 1
  int32_t n_heads;
  int64_t watchdog_ns;
  int32_t single_op;        // >= 0: standalone mode, run every tile of this op (strided over CTAs)
  int32_t own_first;        // 1: the CTA's own tenant (pref[0]) wins over higher-ranked items
  int64_t* dbg;             // optional [gridDim.x * DBG_EVENTS] %globaltimer milestones (diagnostics)
  int64_t dbg_spin;         // diagnostics: epilogue delay (clocks) between tfull and the TMEM read
  int32_t claim_ahead;      // 1: with no ready item, claim the best unready head and wait on its deps
  int32_t n_counters;       // chunk_done entries (saturated on a watchdog abort)
  unsigned long long* stats;// [STAT_TENANTS + 2] accumulating ns: per-tenant item time (claim -> release),
                            // then CTA time at cluster barriers, then CTA time with only unready work
};
constexpr int STAT_TENANTS = 16;
constexpr int DBG_EVENTS = 24;
// trace record per item: tenant, op, smid, idx, cluster, chunk, t_claim,
// t_release, t_start, t_acc_ready (GEMM), t_epilogue_done (GEMM), reserved
constexpr int TRACE_FIELDS = 12;

}  // namespace gacer
