// host.cpp -- C ABI of the GACER executor (include/gacer.h).
//
// Registration lowers a tenant DFG (§4.1 l.605-607) into fused
// device ops; gacer_set_regulation compiles the paper's regulation variables
// -- mask/list_B (§4.2 l.657-685, Eq. 5) and Matrix_P (§4.3 l.742-753,
// Eq. 6/7) -- into per-(tenant, cluster) work queues, per-item dependency
// lists and cluster totals that the persistent kernel enforces on-device.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "../../include/gacer.h"
#include "gacer_dev.h"

namespace gacer {
int executor_smem_bytes();
cudaError_t configure_kernels();
cudaError_t launch_executor(const ExecParams& p, int grid, cudaStream_t s, bool train);
cudaError_t launch_op(const ExecParams& base, const OpDev* ops_dev, int op_idx, int kind, int n_items, int num_sms,
                      cudaStream_t s);
cudaError_t launch_dgrad_filter(const float* w, int Cout, int Cin, int KH, int KW, int cread, int Kpad, int rows,
                                void* out, cudaStream_t s);
cudaError_t launch_fill(float* p, int n, float v, cudaStream_t s);
cudaError_t launch_dgrad_phase_filter(const float* w, int Cout, int Cin, int KI, int KJ, int cread, int Kpad, int rows,
                                      int S, int pa, int pb, int KH, int KW, void* out, cudaStream_t s);
cudaError_t launch_phase_scatter(const void* const* phase_out, int N, int H, int W, int C, int S, int ph, int pw,
                                 int KH, int KW, void* dx, cudaStream_t s);
cudaError_t launch_dilate(const void* dy, int N, int Hd, int Wd, int C, int S, int Hdd, int Wdd, void* out,
                          cudaStream_t s);
cudaError_t launch_transpose_im2col(const void* x, int N, int H, int W, int C, int Ho, int Wo, int KH, int KW, int S,
                                    int ph, int pw, int64_t M, int Kpad, void* out, cudaStream_t s);
cudaError_t launch_wgrad_permute(const float* g, int Cout, int Cin, int KH, int KW, float* dw, cudaStream_t s);
cudaError_t launch_fwd_filter(const float* w, int Cout, int Cin, int KH, int KW, int cread, int Kpad, int rows,
                              void* out, cudaStream_t s, int block_bn = 0);
cudaError_t launch_wgrad_reduce(const float* part, int Cout, int Cin, int KH, int KW, int bn, int tiles_n, int split,
                                float* dw, cudaStream_t s);
}  // namespace gacer

using namespace gacer;

namespace {

thread_local std::string g_err;
int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

}  // namespace

namespace gacer {
// error reporting for the other translation units (train_ops.cu)
int set_error(int code, const char* msg) { return set_err(code, "%s", msg); }
}  // namespace gacer

namespace {

// diagnostic switches: set and non-empty
static bool env_flag(const char* name);
// claim-ahead scheduling (executor.cu scan_ready): GACER_CLAIM_AHEAD=0/1 overrides the default
static bool claim_ahead_enabled() {
  const char* e = getenv("GACER_CLAIM_AHEAD");
  return e ? e[0] == '1' : true;
}
static bool env_flag(const char* name) {
  const char* v = getenv(name);
  return v && v[0] && v[0] != '0';
}
constexpr int kSplitSms = 148;  // split-K is a function of the layer shape only (bit-identity, H4)

int roundup(int a, int b) { return (a + b - 1) / b * b; }
int cdiv(int a, int b) { return (a + b - 1) / b; }
int pow2ceil(int a) { int p = 1; while (p < a) p <<= 1; return p; }

uint16_t f32_to_bf16_rne(float f);
float f32_to_bf16_round_trip(float f) {
  const uint32_t u = static_cast<uint32_t>(f32_to_bf16_rne(f)) << 16;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}
uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return static_cast<uint16_t>(u >> 16);  // inf/nan
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

// ---------------------------------------------------------------- tenants
struct Tensor {
  int C = 0, H = 0, W = 0;
  int buf = -1;          // storage buffer id; -1 = graph input, -2 = user output
  int coff = 0, ldc = 0;
  int producer_orig = -1;  // original op producing it (-1 = input)
  std::vector<int> writers;  // fused ops writing (a slice of) it
  bool sliced = false;     // storage is a slice of a concat tensor
  // liveness-based buffer reuse: the tensors that occupied this tensor's
  // buffer before it, most recent first (the plan compiler adds
  // write-after-read dependencies on their readers, tile by tile)
  std::vector<int> war_prev;
};

struct FusedOp {
  int kind = 0;
  int head = -1, last = -1;  // original op indices (0-based)
  std::vector<int> members;
  int in_t = -1, skip_t = -1, out_t = -1;
  int act = ACT_NONE;
  bool swap = false;
  bool affine = false;   // DK_ELTWISE: a standalone BatchNorm (scale / bias applied first)
  bool mul = false;      // DK_ELTWISE: channel scale by skip_t [B][C] (squeeze-and-excitation)
  // geometry
  int Cin = 0, H = 0, W = 0, Cout = 0, Ho = 0, Wo = 0;
  int kh = 1, kw = 1, stride = 1, ph = 0, pw = 0;
  int cread = 0;  // channels read per tap (K = kh*kw*cread)
  bool win = false;  // window op staged through shared memory
  int mrep = 1;      // GEMM: 128-row accumulators per tile (2 = M-pair tile, bm = 256)
  int M = 0, N = 0, K = 0, Kpad = 0, tiles_m = 1, tiles_n = 1, bm = 0, bn = 0, split_k = 1, nkb = 0;
  bool cip = true;
  // packed params (host)
  std::vector<uint16_t> w_bf16;
  std::vector<float> w_f32;
  std::vector<float> scale, bias;
  // device
  void* d_w = nullptr;
  size_t w_bytes = 0;    // bytes of the packed device weights
  float* d_scale = nullptr;
  float* d_bias = nullptr;
  float* d_partial = nullptr;
  uint32_t* d_tile_cnt = nullptr;
  double flops = 0, bytes = 0;
  bool rows_are_pixels = true;  // output pixel rows are the GEMM/tile M axis
  int a_mode = A_GATHER;        // GEMM operand-A load path
};

// ---------------------------------------------------------------- training tenant (A11)
// A training tenant's round is its whole SGD step (SURVEY §8 "Rounds"):
// forward, softmax-CE, backward in reverse topological order, the update --
// lowered at registration into a list of executor ops (tcgen05 GEMMs and
// virtual-grid CUDA-core operators, train_dev.cuh) over library-owned
// buffers.  Buffers are referenced symbolically and resolved when the op
// table is built (the graph input / logits / labels are bound later).
constexpr int TBUF_IN = -2, TBUF_OUT = -3, TBUF_LABELS = -4;
struct TRef {
  int buf = -1;        // -1: null; >= 0 library buffer; TBUF_*: bound buffers
  size_t off = 0;      // byte offset
};
struct TrainOp {
  int kind = DK_VGRID;           // DK_VGRID or DK_GEMM
  int vfn = 0, vblocks = 0, per = 1;   // virtual-grid op: function, grid, virtual blocks per item
  VArgs va{};
  TRef vp[8];                    // VArgs pointer slots
  OpDev gd{};                    // GEMM: geometry (pointers resolved at build time)
  TRef g_in, g_out, g_wt, g_part, g_scale, g_bias;
  int gemm_kind = 0;             // 0 forward conv, 1 data gradient, 2 weight gradient
  int im2col_c = 0;              // real channels of the im2col tensor map
  bool has_upper = false;        // explicit im2col upper corner (dgrad phases)
  int im2col_upper[2] = {0, 0};
  int a_ld = 0, a_rows = 0, b_rows = 0;
  std::vector<int> deps;         // producer ops (indices into tops): RAW / WAR / WAW on buffers
  std::vector<std::pair<int64_t, int64_t>> grad_ranges;   // flat-gradient slices written (floats)
  bool reads_input = false;      // reads the bound images or labels (input gate)
  int step_pos = 1;              // 1-based position in the step's issue order (pointer clusters)
  int items = 1;
  double flops = 0, bytes = 0;
};

struct Tenant {
  int batch = 0, dtype = 0, n_orig = 0;
  // training tenant (gacer_graph.train != 0)
  bool train = false;
  int n_steps = 0;                   // 2 n_orig + 1 step positions (forward, backward, update)
  std::vector<TrainOp> tops;
  std::vector<size_t> tbuf_bytes;
  std::vector<void*> tbufs;
  std::vector<float> h_params;       // initial master parameters (uploaded once)
  int buf_params = -1, buf_grads = -1, buf_mom = -1, buf_loss = -1;
  bool grad_gate = false;            // A12: the SGD op waits for the gradient all-reduce gate
  // the step's filter packing as one operator (VF_FILTER_ALL): its jobs with
  // unresolved buffers, the op index and the device job table's buffer
  struct FJob { TRef w, out; int32_t i[14]; int64_t n; };
  std::vector<FJob> fjobs;
  int fall_op = -1, fall_table = -1;
  std::map<std::pair<int, int>, std::pair<int64_t, int64_t>> param_slice;  // (orig op, which) -> (offset, count)
  const void* labels_dev = nullptr;
  float lr = 0.1f, momentum = 0.9f;
  int in_c = 0, in_h = 0, in_w = 0, in_c_pad = 0;
  std::vector<int> orig_kind;
  std::vector<int> orig_out_c;    // c_out for chunk validation
  std::vector<int> orig_tensor;   // tensor id of each original op's output
  std::vector<int> orig_fused;    // fused op containing the original op (-1 for aliases)
  std::vector<Tensor> tensors;    // tensor 0 = graph input
  std::vector<FusedOp> fops;
  int out_t = -1;
  int out_features = 0;
  std::vector<void*> bufs;        // device activation buffers
  std::vector<size_t> buf_bytes;
  const void* in_dev = nullptr;
  void* out_dev = nullptr;
  double flops = 0;
  int op_base = 0;                // index of fops[0] in the global op table
};

// ---------------------------------------------------------------- plan
struct Chunking {
  int axis = GACER_AXIS_NONE;
  std::vector<int> sizes;
  std::vector<int> budget;   // per chunk: max items in flight (0 = unlimited); empty = none
};

struct Plan {
  int n_clusters = 1;
  std::vector<std::vector<int>> cuts;               // [tenant][pointer]
  std::map<std::pair<int, int>, Chunking> chunks;   // (tenant, orig op 0-based) -> chunking
  // compiled
  std::vector<Item> items;
  std::vector<Dep> deps;
  std::vector<int32_t> queue;
  std::vector<Seg> segs;
  std::vector<uint32_t> cluster_total;
  int n_chunk_counters = 0;
  int input_counter0 = 0;                           // first of the per-tenant input-gate counters
  int grad_gate0 = 0;                               // first of the per-tenant gradient gates (A12)
  std::vector<std::vector<int>> fop_cluster;        // [tenant][fused op]
  std::vector<double> auto_share;                   // per tenant: SM need (work / chain latency)
};

struct State {
  bool inited = false;
  bool host_only = true;
  int device = -1;
  int num_sms = 148;
  gacer_options opts{};
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;   // host-buffer rounds: H2D copies + input gates
  // A12 (gradient all-reduce of data-parallel training tenants): baseline-mode
  // gates (round-numbered words the SGD launch waits on) and backward-done events
  uint32_t* d_bgate = nullptr;
  uint32_t round_no = 0;
  std::vector<cudaEvent_t> bwd_event;
  std::vector<cudaStream_t> tstreams;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t ev_fork = nullptr;           // multi-stream baseline: fork / join (no timing)
  std::vector<cudaEvent_t> tjoin;
  cudaGraphExec_t base_graph = nullptr;    // captured baseline round (gacer_capture_baseline)
  int base_graph_mode = -1;
  int base_graph_launches = 0;
  std::vector<Tenant> tenants;
  std::vector<double> user_share;   // gacer_set_sm_shares (empty = automatic)
  Plan plan;
  int mode = GACER_MODE_EXECUTOR;
  bool sticky_cuda = false;
  // device op table + TMA descriptors (2 per op)
  OpDev* d_ops = nullptr;
  std::vector<OpDev> h_ops;
  CUtensorMap* d_tmaps = nullptr;
  size_t n_tmaps = 0;
  // device plan
  Item* d_items = nullptr;
  Dep* d_deps = nullptr;
  int32_t* d_queue = nullptr;
  Seg* d_segs = nullptr;
  int32_t* d_pref = nullptr;
  uint32_t* d_heads = nullptr;
  uint32_t* d_chunk_done = nullptr;
  uint32_t* d_cluster_done = nullptr;
  uint32_t* d_cluster_total = nullptr;
  uint32_t* d_exit = nullptr;
  int32_t* d_error = nullptr;
  unsigned long long* d_stats = nullptr;   // executor occupancy counters (accumulating)
  std::vector<unsigned long long> stats_prev;
  int stat_rounds = 0;                     // executor rounds since the last gacer_get_stats
  float* d_ones = nullptr;    // unit BN scale / zero bias of the standalone GEMM calls (A11)
  float* d_zeros = nullptr;
  int n_unit = 0;
  int64_t* d_trace = nullptr;
  int64_t* d_dbg = nullptr;     // GACER_DEBUG_TIMING=1: per-CTA milestones
  size_t n_dbg = 0;
  uint32_t epoch = 0;
  int grid = 0;
  double last_ms = 0;
  int last_launches = 0;
};
State S;

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) {                                                             \
      S.sticky_cuda = true;                                                              \
      return set_err(GACER_E_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));     \
    }                                                                                    \
  } while (0)

template <class T>
int dev_upload(T** dptr, const T* src, size_t n) {
  if (*dptr) { cudaFree(*dptr); *dptr = nullptr; }
  if (n == 0) return 0;
  CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(dptr), n * sizeof(T)));
  if (src) CUDA_TRY(cudaMemcpy(*dptr, src, n * sizeof(T), cudaMemcpyHostToDevice));
  else CUDA_TRY(cudaMemset(*dptr, 0, n * sizeof(T)));
  return 0;
}

bool is_alias(int k) { return k == GACER_OP_FLATTEN || k == GACER_OP_DROPOUT || k == GACER_OP_CONCAT; }

int lower_train(const gacer_graph* g, int batch, Tenant& T, const std::map<int, int>& pos);   // defined below
bool has_train_tenant();
int build_train_opdev(const Tenant& T, int tenant_id, const TrainOp& op, OpDev& d, CUtensorMap* maps, bool encode);
int upload_train_tenant(Tenant& T);

// ------------------------------------------------------------------------
// registration: validation + shape inference + fusion + packing
// activation op kind -> fused activation (ACT_NONE: not an activation)
int act_of(int kind) {
  switch (kind) {
    case GACER_OP_RELU: return ACT_RELU;
    case GACER_OP_RELU6: return ACT_RELU6;
    case GACER_OP_HARDSWISH: return ACT_HSWISH;
    case GACER_OP_HARDSIGMOID: return ACT_HSIGMOID;
    default: return ACT_NONE;
  }
}

// ------------------------------------------------------------------------
// Liveness-based reuse of activation buffers (a round wrote
// every activation to its own buffer, 685 MB of DRAM write-back per D2
// round).  In issue order, a tensor whose buffer holds only itself (no
// concat slices; one writer; not the graph input or output) takes over the
// buffer of an earlier tensor whose last reader is at least GACER_REUSE_DIST
// (default 2) fused ops before its writer: best fit among the free buffers
// large enough, else the largest free one, grown.  The tenant's footprint
// then stays near its live set, which L2 can hold.  Correctness does not
// rest on the issue order: the plan compiler gives every tile of the new
// writer write-after-read dependencies on the reader tiles of the previous
// occupants that touch its bytes (compile_plan, war_deps).
void reuse_buffers(Tenant& T) {
  const int nt = static_cast<int>(T.tensors.size());
  const int nb = static_cast<int>(T.bufs.size());
  int dist = 2;
  if (const char* e = getenv("GACER_REUSE_DIST")) dist = std::max(1, atoi(e));
  // only tensors of at least min_bytes take part (the small tensors of the
  // late, latency-bound layers would gain no DRAM traffic and pay the
  // write-after-read dependency checks)
  size_t min_bytes = 0;
  if (const char* e = getenv("GACER_REUSE_MIN_KB")) min_bytes = static_cast<size_t>(std::max(0, atoi(e))) * 1024u;
  std::vector<int> holders(nb, 0);
  for (int t = 1; t < nt; ++t)
    if (T.tensors[t].buf >= 0) ++holders[T.tensors[t].buf];
  std::vector<int> last_read(nt, -1);
  for (size_t f = 0; f < T.fops.size(); ++f)
    for (int tin : {T.fops[f].in_t, T.fops[f].skip_t})
      if (tin > 0) last_read[tin] = std::max(last_read[tin], static_cast<int>(f));
  std::vector<std::pair<int, int>> cand;   // (writer, tensor)
  for (int t = 1; t < nt; ++t) {
    const Tensor& X = T.tensors[t];
    if (X.buf < 0 || X.sliced || holders[X.buf] != 1 || X.writers.size() != 1 || T.buf_bytes[X.buf] < std::max<size_t>(1, min_bytes))
      continue;
    cand.push_back({X.writers[0], t});
  }
  std::sort(cand.begin(), cand.end());
  struct Slot { int buf; size_t bytes; int last; std::vector<int> occ; };
  std::vector<Slot> slots;
  for (const auto& wt : cand) {
    const int w = wt.first, t = wt.second;
    Tensor& X = T.tensors[t];
    const size_t need = T.buf_bytes[X.buf];
    const int last = std::max(w, last_read[t]);
    int best = -1;
    for (int s = 0; s < static_cast<int>(slots.size()); ++s) {
      if (slots[s].last > w - dist) continue;
      if (best < 0) { best = s; continue; }
      const Slot& a = slots[s];
      const Slot& b = slots[best];
      const bool af = a.bytes >= need, bf = b.bytes >= need;
      if (af != bf ? af : (af ? a.bytes < b.bytes : a.bytes > b.bytes)) best = s;
    }
    if (best < 0) {
      slots.push_back({X.buf, need, last, {t}});
      continue;
    }
    Slot& sl = slots[best];
    T.buf_bytes[X.buf] = 0;   // its own buffer is never allocated
    X.buf = sl.buf;
    X.war_prev.assign(sl.occ.rbegin(), sl.occ.rend());
    sl.occ.push_back(t);
    sl.bytes = std::max(sl.bytes, need);
    sl.last = last;
  }
  for (const Slot& sl : slots) T.buf_bytes[sl.buf] = sl.bytes;
}

int lower_tenant(const gacer_graph* g, int batch, Tenant& T) {
  const int n = g->n_ops;
  if (n <= 0 || !g->ops) return set_err(GACER_E_INVALID_ARG, "graph has no ops");
  if (batch < 1) return set_err(GACER_E_INVALID_ARG, "batch must be >= 1");
  if (g->dtype != GACER_DTYPE_BF16 && g->dtype != GACER_DTYPE_FP32)
    return set_err(GACER_E_INVALID_ARG, "unknown dtype %d", g->dtype);
  if (g->in_c < 1 || g->in_h < 1 || g->in_w < 1) return set_err(GACER_E_SHAPE, "bad input shape");
  const bool f32 = g->dtype == GACER_DTYPE_FP32;
  T.batch = batch;
  T.dtype = g->dtype;
  T.n_orig = n;
  T.in_c = g->in_c; T.in_h = g->in_h; T.in_w = g->in_w;
  T.in_c_pad = roundup(g->in_c, 8);

  // ---- ids, predecessors, cycles, issue order (SPEC S:56 error set)
  std::map<int, int> pos;
  for (int i = 0; i < n; ++i) {
    const gacer_op_desc& o = g->ops[i];
    if (o.id < 1) return set_err(GACER_E_INVALID_ARG, "op %d: id must be >= 1", i + 1);
    if (pos.count(o.id)) return set_err(GACER_E_DUPLICATE_ID, "duplicate op id %d", o.id);
    pos[o.id] = i;
  }
  for (int i = 0; i < n; ++i) {
    const gacer_op_desc& o = g->ops[i];
    if (o.n_preds < 0 || (o.n_preds > 0 && !o.preds)) return set_err(GACER_E_INVALID_ARG, "op %d: bad preds", o.id);
    for (int j = 0; j < o.n_preds; ++j)
      if (o.preds[j] != 0 && !pos.count(o.preds[j]))
        return set_err(GACER_E_UNKNOWN_PREDECESSOR, "op %d: unknown predecessor %d", o.id, o.preds[j]);
  }
  {  // cycle detection (iterative DFS colouring)
    std::vector<int> color(n, 0);
    for (int s0 = 0; s0 < n; ++s0) {
      if (color[s0]) continue;
      std::vector<std::pair<int, int>> st{{s0, 0}};
      color[s0] = 1;
      while (!st.empty()) {
        auto& [v, j] = st.back();
        const gacer_op_desc& o = g->ops[v];
        if (j < o.n_preds) {
          const int pid = o.preds[j++];
          if (pid == 0) continue;
          const int u = pos[pid];
          if (color[u] == 1) return set_err(GACER_E_CYCLE, "dependency cycle through op %d", g->ops[u].id);
          if (color[u] == 0) { color[u] = 1; st.push_back({u, 0}); }
        } else {
          color[v] = 2;
          st.pop_back();
        }
      }
    }
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < g->ops[i].n_preds; ++j) {
      const int pid = g->ops[i].preds[j];
      if (pid != 0 && pos[pid] >= i)
        return set_err(GACER_E_INVALID_ARG, "op %d: predecessor %d is not earlier in issue order", g->ops[i].id, pid);
    }

  // ---- shape inference; tensors
  T.tensors.clear();
  Tensor tin;
  tin.C = g->in_c; tin.H = g->in_h; tin.W = g->in_w; tin.buf = -1; tin.ldc = T.in_c_pad;
  T.tensors.push_back(tin);
  T.orig_kind.assign(n, 0);
  T.orig_out_c.assign(n, 0);
  T.orig_tensor.assign(n, -1);
  std::vector<std::vector<int>> consumers(n + 1);  // by original op (index+1; 0 = input) -> consumer op idx
  auto tens_of = [&](int pid) { return pid == 0 ? 0 : T.orig_tensor[pos[pid]]; };
  for (int i = 0; i < n; ++i) {
    const gacer_op_desc& o = g->ops[i];
    T.orig_kind[i] = o.kind;
    auto need_preds = [&](int k) -> int {
      if (o.n_preds != k) return set_err(GACER_E_INVALID_ARG, "op %d: expected %d predecessors", o.id, k);
      return 0;
    };
    int rc = 0;
    switch (o.kind) {
      case GACER_OP_ADD: rc = need_preds(2); break;
      case GACER_OP_CONCAT: if (o.n_preds < 1) rc = set_err(GACER_E_INVALID_ARG, "concat needs preds"); break;
      case GACER_OP_CONV2D: case GACER_OP_LINEAR: case GACER_OP_MAXPOOL: case GACER_OP_AVGPOOL:
      case GACER_OP_GAP: case GACER_OP_BN: case GACER_OP_RELU: case GACER_OP_RELU6:
      case GACER_OP_HARDSWISH: case GACER_OP_HARDSIGMOID:
      case GACER_OP_FLATTEN: case GACER_OP_DROPOUT: rc = need_preds(1); break;
      case GACER_OP_MUL: rc = need_preds(2); break;
      default: rc = set_err(GACER_E_UNSUPPORTED_OP, "op %d: unknown kind %d", o.id, o.kind);
    }
    if (rc) return rc;
    for (int j = 0; j < o.n_preds; ++j) consumers[o.preds[j] == 0 ? 0 : pos[o.preds[j]] + 1].push_back(i);
    const Tensor& x = T.tensors[tens_of(o.preds[0])];
    Tensor y;
    y.producer_orig = i;
    switch (o.kind) {
      case GACER_OP_CONV2D: {
        if (o.c_in != x.C) return set_err(GACER_E_SHAPE, "op %d: c_in %d != input channels %d", o.id, o.c_in, x.C);
        if (o.kh < 1 || o.kw < 1 || o.stride < 1 || o.pad_h < 0 || o.pad_w < 0 || o.groups < 1 || o.c_out < 1)
          return set_err(GACER_E_INVALID_ARG, "op %d: bad conv params", o.id);
        if (o.c_in % o.groups || o.c_out % o.groups) return set_err(GACER_E_SHAPE, "op %d: groups", o.id);
        if (o.groups != 1 && !(o.groups == o.c_in && o.c_in == o.c_out))
          return set_err(GACER_E_UNSUPPORTED_OP, "op %d: grouped conv with 1 < groups < C", o.id);
        if (!o.weight) return set_err(GACER_E_INVALID_ARG, "op %d: missing weight", o.id);
        y.C = o.c_out;
        y.H = (x.H + 2 * o.pad_h - o.kh) / o.stride + 1;
        y.W = (x.W + 2 * o.pad_w - o.kw) / o.stride + 1;
        if (y.H < 1 || y.W < 1) return set_err(GACER_E_SHAPE, "op %d: empty output", o.id);
        T.orig_out_c[i] = o.c_out;
        break;
      }
      case GACER_OP_LINEAR:
        if (o.c_in != x.C * x.H * x.W)
          return set_err(GACER_E_SHAPE, "op %d: linear c_in %d != %d", o.id, o.c_in, x.C * x.H * x.W);
        if (!o.weight || o.c_out < 1) return set_err(GACER_E_INVALID_ARG, "op %d: linear params", o.id);
        y.C = o.c_out; y.H = 1; y.W = 1;
        T.orig_out_c[i] = o.c_out;
        break;
      case GACER_OP_MAXPOOL: case GACER_OP_AVGPOOL:
        if (o.kh < 1 || o.kw < 1 || o.stride < 1 || o.pad_h < 0 || o.pad_w < 0)
          return set_err(GACER_E_INVALID_ARG, "op %d: bad pool params", o.id);
        y.C = x.C;
        y.H = (x.H + 2 * o.pad_h - o.kh) / o.stride + 1;
        y.W = (x.W + 2 * o.pad_w - o.kw) / o.stride + 1;
        if (y.H < 1 || y.W < 1) return set_err(GACER_E_SHAPE, "op %d: empty output", o.id);
        T.orig_out_c[i] = x.C;
        break;
      case GACER_OP_GAP:
        y.C = x.C; y.H = 1; y.W = 1; T.orig_out_c[i] = x.C;
        break;
      case GACER_OP_BN:
        if (o.c_out != 0 && o.c_out != x.C) return set_err(GACER_E_SHAPE, "op %d: bn channels", o.id);
        if (!o.bn_gamma || !o.bn_beta || !o.bn_mean || !o.bn_var)
          return set_err(GACER_E_INVALID_ARG, "op %d: missing BN params", o.id);
        y.C = x.C; y.H = x.H; y.W = x.W; T.orig_out_c[i] = x.C;
        break;
      case GACER_OP_RELU: case GACER_OP_RELU6: case GACER_OP_DROPOUT:
      case GACER_OP_HARDSWISH: case GACER_OP_HARDSIGMOID:
        y.C = x.C; y.H = x.H; y.W = x.W; T.orig_out_c[i] = x.C;
        break;
      case GACER_OP_MUL: {   // x [C,H,W] * s [C,1,1] (squeeze-and-excitation channel scale)
        const Tensor& sc = T.tensors[tens_of(o.preds[1])];
        if (sc.C != x.C || sc.H != 1 || sc.W != 1) return set_err(GACER_E_SHAPE, "op %d: mul scale shape", o.id);
        y.C = x.C; y.H = x.H; y.W = x.W; T.orig_out_c[i] = x.C;
        break;
      }
      case GACER_OP_FLATTEN:
        y.C = x.C; y.H = x.H; y.W = x.W; T.orig_out_c[i] = x.C;   // data unchanged (NHWC storage)
        break;
      case GACER_OP_ADD: {
        const Tensor& b = T.tensors[tens_of(o.preds[1])];
        if (b.C != x.C || b.H != x.H || b.W != x.W) return set_err(GACER_E_SHAPE, "op %d: add shapes", o.id);
        y.C = x.C; y.H = x.H; y.W = x.W; T.orig_out_c[i] = x.C;
        break;
      }
      case GACER_OP_CONCAT: {
        int c = 0;
        for (int j = 0; j < o.n_preds; ++j) {
          const Tensor& b = T.tensors[tens_of(o.preds[j])];
          if (b.H != x.H || b.W != x.W) return set_err(GACER_E_SHAPE, "op %d: concat spatial sizes", o.id);
          c += b.C;
        }
        y.C = c; y.H = x.H; y.W = x.W; T.orig_out_c[i] = c;
        break;
      }
    }
    if (o.kind == GACER_OP_FLATTEN || o.kind == GACER_OP_DROPOUT) {
      T.orig_tensor[i] = tens_of(o.preds[0]);  // alias
    } else {
      T.orig_tensor[i] = static_cast<int>(T.tensors.size());
      T.tensors.push_back(y);
    }
  }

  if (g->train) {
    if (f32) return set_err(GACER_E_UNSUPPORTED_OP, "training tenants run in bf16 (SURVEY Q1)");
    return lower_train(g, batch, T, pos);
  }

  // effective consumers: look through flatten / dropout aliases
  std::function<void(int, std::vector<int>&)> eff;
  eff = [&](int node, std::vector<int>& out) {  // node: orig index + 1 (0 = input)
    for (int c : consumers[node]) {
      const int k = g->ops[c].kind;
      if (k == GACER_OP_FLATTEN || k == GACER_OP_DROPOUT) eff(c + 1, out);
      else out.push_back(c);
    }
  };
  auto single_consumer = [&](int orig) -> int {
    std::vector<int> cs;
    eff(orig + 1, cs);
    return cs.size() == 1 ? cs[0] : -1;
  };
  const int last_op = n - 1;
  // the graph output is the last op's tensor; it may not be fused further
  const int out_tensor = T.orig_tensor[last_op];

  // ---- fusion
  T.orig_fused.assign(n, -1);
  std::vector<char> taken(n, 0);
  T.fops.clear();
  for (int i = 0; i < n; ++i) {
    if (taken[i]) continue;
    const gacer_op_desc& o = g->ops[i];
    if (is_alias(o.kind)) continue;
    FusedOp F;
    F.head = i;
    F.members = {i};
    taken[i] = 1;
    F.in_t = tens_of(o.preds[0]);
    int tail = i;
    auto try_extend = [&](bool allow_bn, bool allow_add) {
      bool has_bn = false, has_add = false;
      for (;;) {
        if (T.orig_tensor[tail] == out_tensor) break;
        const int c = single_consumer(tail);
        if (c < 0 || taken[c]) break;
        const gacer_op_desc& co = g->ops[c];
        if (co.kind == GACER_OP_BN && allow_bn && !has_bn && !has_add) {
          has_bn = true;
        } else if (co.kind == GACER_OP_ADD && allow_add && !has_add) {
          const int a = tens_of(co.preds[0]), b = tens_of(co.preds[1]);
          const int mine = T.orig_tensor[tail];
          const int other = (a == mine) ? b : a;
          if (a == b || other == 0) break;  // x + x or a skip from the raw input: not fused
          F.skip_t = other;
          has_add = true;
        } else if (co.kind == GACER_OP_RELU || co.kind == GACER_OP_RELU6) {
          // (hardswish / hardsigmoid stay separate eltwise ops: executor.cu cc_item_ext)
          F.act = act_of(co.kind);
          F.members.push_back(c);
          taken[c] = 1;
          tail = c;
          break;
        } else {
          break;
        }
        F.members.push_back(c);
        taken[c] = 1;
        tail = c;
      }
    };
    switch (o.kind) {
      case GACER_OP_CONV2D: {
        const bool dw = o.groups > 1;
        F.kind = f32 ? (dw ? DK_DW : DK_SIMT_GEMM) : (dw ? DK_DW : DK_GEMM);
        try_extend(true, true);
        break;
      }
      case GACER_OP_LINEAR:
        F.kind = f32 ? DK_SIMT_GEMM : DK_GEMM;
        try_extend(false, false);
        break;
      case GACER_OP_MAXPOOL: F.kind = DK_MAXPOOL; break;
      case GACER_OP_AVGPOOL: F.kind = DK_AVGPOOL; F.cip = (o.flags & GACER_FLAG_COUNT_INCLUDE_PAD) != 0; break;
      case GACER_OP_GAP: F.kind = DK_GAP; break;
      case GACER_OP_ADD: {
        F.kind = DK_ELTWISE;
        F.skip_t = tens_of(o.preds[1]);
        try_extend(false, false);
        break;
      }
      case GACER_OP_MUL: {
        F.kind = DK_ELTWISE;
        F.skip_t = tens_of(o.preds[1]);
        F.mul = true;
        try_extend(false, false);
        break;
      }
      case GACER_OP_RELU: case GACER_OP_RELU6: case GACER_OP_HARDSWISH: case GACER_OP_HARDSIGMOID:
        F.kind = DK_ELTWISE;
        F.act = act_of(o.kind);
        break;
      case GACER_OP_BN:
        // a BatchNorm no conv produces (DenseNet's pre-activation on a concat):
        // a per-channel affine CUDA-core op, its activation fused
        F.kind = DK_ELTWISE;
        F.affine = true;
        try_extend(false, false);
        break;
      default:
        return set_err(GACER_E_UNSUPPORTED_OP, "op %d: kind %d not lowered", o.id, o.kind);
    }
    F.last = tail;
    F.out_t = T.orig_tensor[tail];
    const int fi = static_cast<int>(T.fops.size());
    for (int m : F.members) T.orig_fused[m] = fi;
    T.fops.push_back(std::move(F));
  }
  // order fused ops by their last member (topological: see DESIGN.md)
  {
    std::vector<int> idx(T.fops.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = static_cast<int>(i);
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return T.fops[a].last < T.fops[b].last; });
    std::vector<FusedOp> sorted;
    std::vector<int> remap(idx.size());
    for (size_t i = 0; i < idx.size(); ++i) { remap[idx[i]] = static_cast<int>(i); sorted.push_back(std::move(T.fops[idx[i]])); }
    T.fops = std::move(sorted);
    for (int& f : T.orig_fused) if (f >= 0) f = remap[f];
  }
  for (size_t fi = 0; fi < T.fops.size(); ++fi) T.tensors[T.fops[fi].out_t].writers.push_back(static_cast<int>(fi));

  // ---- storage: user output, concat slices, own buffers
  T.out_t = out_tensor;
  {
    Tensor& ot = T.tensors[out_tensor];
    if (ot.producer_orig >= 0 && g->ops[ot.producer_orig].kind == GACER_OP_CONCAT)
      return set_err(GACER_E_UNSUPPORTED_OP, "graph output may not be a concat");
    if (ot.writers.empty()) return set_err(GACER_E_UNSUPPORTED_OP, "graph output is the raw input");
    ot.buf = -2;
    ot.coff = 0;
    T.out_features = ot.C * ot.H * ot.W;   // float32 NHWC [B][H][W][C] ([B][C] when 1x1)
    ot.ldc = ot.C;
  }
  // concat slices: outermost first (reverse issue order)
  for (int i = n - 1; i >= 0; --i) {
    if (g->ops[i].kind != GACER_OP_CONCAT) continue;
    const int ct = T.orig_tensor[i];
    Tensor& C = T.tensors[ct];
    if (C.buf == -1 && !C.sliced) {
      C.buf = static_cast<int>(T.bufs.size());
      T.bufs.push_back(nullptr);
      C.ldc = C.C;
      C.coff = 0;
    }
    int off = 0;
    for (int j = 0; j < g->ops[i].n_preds; ++j) {
      const int pt = tens_of(g->ops[i].preds[j]);
      Tensor& P = T.tensors[pt];
      std::vector<int> cs;
      eff(P.producer_orig + 1, cs);
      // the producer writes straight into the concat buffer: it may feed one
      // concat only (other consumers just read the slice -- DenseNet's
      // nested feature concats, feat_l = concat(feat_{l-1}, y_l))
      int n_concat = 0;
      for (int c : cs) n_concat += g->ops[c].kind == GACER_OP_CONCAT;
      if (pt == 0 || n_concat != 1 || P.sliced || P.buf == -2)
        return set_err(GACER_E_UNSUPPORTED_OP, "concat op %d: input %d must be an op output feeding only this concat",
                       g->ops[i].id, g->ops[i].preds[j]);
      P.buf = C.buf;
      P.coff = C.coff + off;
      P.ldc = C.ldc;
      P.sliced = true;
      off += P.C;
    }
  }
  // concat tensor writers = writers of its slices (recursively)
  for (int i = 0; i < n; ++i) {
    if (g->ops[i].kind != GACER_OP_CONCAT) continue;
    Tensor& C = T.tensors[T.orig_tensor[i]];
    for (int j = 0; j < g->ops[i].n_preds; ++j) {
      const Tensor& P = T.tensors[tens_of(g->ops[i].preds[j])];
      C.writers.insert(C.writers.end(), P.writers.begin(), P.writers.end());
    }
  }
  for (size_t t = 1; t < T.tensors.size(); ++t) {
    Tensor& X = T.tensors[t];
    if (X.buf == -1 && !X.sliced && !X.writers.empty()) {
      X.buf = static_cast<int>(T.bufs.size());
      T.bufs.push_back(nullptr);
      X.ldc = X.C;
      X.coff = 0;
    }
  }
  T.buf_bytes.assign(T.bufs.size(), 0);
  const int elem = f32 ? 4 : 2;
  for (size_t t = 1; t < T.tensors.size(); ++t) {
    const Tensor& X = T.tensors[t];
    if (X.buf >= 0 && !X.sliced)
      T.buf_bytes[X.buf] = std::max(T.buf_bytes[X.buf], static_cast<size_t>(batch) * X.H * X.W * X.ldc * elem);
  }
  // (off by default: on D2 it cuts DRAM writes 657 -> 533 MB per round but
  //  the write-after-read dependencies cost 1.7-2 % of the makespan, same-box
  //  A/B; GACER_REUSE=1 enables it)
  if (env_flag("GACER_REUSE")) reuse_buffers(T);

  // ---- per fused op geometry + packing
  T.flops = 0;
  for (FusedOp& F : T.fops) {
    const gacer_op_desc& o = g->ops[F.head];
    const Tensor& X = T.tensors[F.in_t];
    const Tensor& Y = T.tensors[F.out_t];
    F.Cin = X.C; F.H = X.H; F.W = X.W;
    F.Cout = Y.C; F.Ho = Y.H; F.Wo = Y.W;
    if (F.in_t != 0 && X.C % 8 && F.kind != DK_SIMT_GEMM)
      return set_err(GACER_E_UNSUPPORTED_OP, "op %d: channel count %d not a multiple of 8", o.id, X.C);
    if ((Y.coff % 8) || (Y.ldc % 8 && Y.buf != -2)) return set_err(GACER_E_UNSUPPORTED_OP, "op %d: unaligned concat slice", o.id);
    if (F.skip_t >= 0 && !F.mul) {
      const Tensor& Sk = T.tensors[F.skip_t];
      if (Sk.C != Y.C || Sk.H != Y.H || Sk.W != Y.W) return set_err(GACER_E_SHAPE, "op %d: residual shape", o.id);
    }
    // folded scale / bias (fp64 -> fp32), SURVEY Q3
    auto fold = [&](int cout, const float* conv_bias) {
      F.scale.assign(cout, 1.0f);
      F.bias.assign(cout, 0.0f);
      const gacer_op_desc* bn = nullptr;
      for (int m : F.members) if (g->ops[m].kind == GACER_OP_BN) bn = &g->ops[m];
      for (int c = 0; c < cout; ++c) {
        const double cb = conv_bias ? conv_bias[c] : 0.0;
        if (bn) {
          const double s = static_cast<double>(bn->bn_gamma[c]) /
                           std::sqrt(static_cast<double>(bn->bn_var[c]) + static_cast<double>(bn->bn_eps));
          F.scale[c] = static_cast<float>(s);
          F.bias[c] = static_cast<float>(static_cast<double>(bn->bn_beta[c]) - static_cast<double>(bn->bn_mean[c]) * s + cb * s);
        } else {
          F.bias[c] = static_cast<float>(cb);
        }
      }
    };
    const float* cbias = (o.flags & GACER_FLAG_BIAS) ? o.bias : nullptr;
    if ((o.flags & GACER_FLAG_BIAS) && !o.bias) return set_err(GACER_E_INVALID_ARG, "op %d: missing bias", o.id);
    const int B = batch;
    if (F.kind == DK_GEMM || F.kind == DK_SIMT_GEMM) {
      const bool lin = o.kind == GACER_OP_LINEAR;
      if (lin) { F.kh = X.H; F.kw = X.W; F.stride = 1; F.ph = F.pw = 0; }
      else { F.kh = o.kh; F.kw = o.kw; F.stride = o.stride; F.ph = o.pad_h; F.pw = o.pad_w; }
      F.flops = 2.0 * B * F.Ho * F.Wo * F.Cout * static_cast<double>(F.Cin) * F.kh * F.kw;
      fold(F.Cout, cbias);
      // weights in (tap, channel) K order; linear weights are NCHW-flatten ordered (c, h, w)
      auto wval = [&](int co, int c, int r, int s) -> float {
        if (lin) return o.weight[static_cast<size_t>(co) * o.c_in + (static_cast<size_t>(c) * X.H + r) * X.W + s];
        return o.weight[((static_cast<size_t>(co) * o.c_in + c) * o.kh + r) * o.kw + s];
      };
      if (F.kind == DK_SIMT_GEMM) {
        F.cread = F.Cin;
        F.K = F.kh * F.kw * F.cread;
        F.M = B * F.Ho * F.Wo; F.N = F.Cout;
        F.bm = 64; F.bn = 64;
        F.tiles_m = cdiv(F.M, F.bm); F.tiles_n = cdiv(F.Cout, F.bn);
        // K-outer [K][Cout rounded to 8]: a thread's 8 output channels of one
        // K step are two float4 loads (simt_item)
        const int cpad = roundup(F.Cout, 8);
        F.w_f32.assign(static_cast<size_t>(F.K) * cpad, 0.0f);
        for (int co = 0; co < F.Cout; ++co)
          for (int r = 0; r < F.kh; ++r)
            for (int s = 0; s < F.kw; ++s)
              for (int c = 0; c < F.Cin; ++c)
                F.w_f32[static_cast<size_t>((r * F.kw + s) * F.cread + c) * cpad + co] = wval(co, c, r, s);
      } else {
        F.swap = lin && X.ldc == X.C && F.skip_t < 0;
        // operand A: TMA im2col loads 64 channels of one tap per K-block and
        // zero-fills channels >= Cin, so the per-tap K stride is Cin rounded
        // up to 64; used when that padding wastes at most 1.5x (always for
        // 1x1), else the cp.async gather with a stride of Cin rounded to 8.
        {
          const int c8 = roundup(F.Cin, 8), c64 = roundup(F.Cin, 64);
          const bool tma = c64 == c8 || F.kh * F.kw == 1 || 2 * c64 <= 3 * c8;
          F.a_mode = F.swap ? A_ROWS : (tma ? A_IM2COL : A_GATHER);
          // an 8-channel input with a large filter (7x7, 11x11 stems): 8 taps
          // per K-block by TMA.  (3x3: the cp.async gather's M-pair tiles win
          // in a round -- same-box A/B on D2)
          if (F.a_mode == A_GATHER && c8 == 8 && X.ldc == 8 && F.kh * F.kw >= 25 && !env_flag("GACER_NO_IM2COL8"))
            F.a_mode = A_IM2COL8;
          F.cread = (F.a_mode == A_IM2COL) ? c64 : c8;
          // M-pair tiles (two 128-row accumulators sharing each B stage) for
          // narrow (Cout <= 128), very wide layers (>= 2 tiles per SM even
          // in pairs): half the items, so the per-item scheduling, epilogue
          // prologue and release costs are amortised over twice the work.
          const long long m_rows = static_cast<long long>(B) * F.Ho * F.Wo;
          const int bn_est = F.Cout >= 128 ? 128 : roundup(F.Cout, 16);
          F.mrep = 1;
          // (a gather layer only if the im2col K stays short: a 7x7 stem
          //  would grow from 7 to 49 K-blocks)
          // (the cp.async gather fills both 128-row halves too, so a small-Cin
          //  layer keeps its short 8-channel K stride)
          const int mpair_per_sm = [] {   // pair items per SM required (A/B knob)
            const char* e = getenv("GACER_MPAIR_PER_SM");
            return e ? std::max(1, atoi(e)) : 1;   // (was 2: D3 -3 %, D2 / Table-2 neutral)
          }();
          // (any Cin: the 256-row tile halves the items of deep layers too --
          //  D2 -0.9 %, Table-2 AlexNet mix -1.6 %, others neutral; the
          //  round-2 limit was Cin <= 64, GACER_MPAIR_CIN_MAX restores it)
          const int mpair_cin_max = [] {
            const char* e = getenv("GACER_MPAIR_CIN_MAX");
            return e ? atoi(e) : (1 << 30);
          }();
          if (!F.swap && F.a_mode != A_IM2COL8 && F.Cout <= 128 && F.Cin <= mpair_cin_max &&
              cdiv(static_cast<int>(m_rows), 2 * BM) * cdiv(F.Cout, bn_est) >= mpair_per_sm * kSplitSms &&
              !env_flag("GACER_NO_MPAIR"))
            F.mrep = 2;
          // 1x1 stride-1 conv over a dense NHWC tensor is a plain GEMM: tiled TMA rows
          if (!F.swap && F.kh * F.kw == 1 && F.stride == 1 && o.pad_h == 0 && o.pad_w == 0 && c64 == c8 &&
              !env_flag("GACER_IM2COL_1X1")) {
            F.a_mode = A_ROWS;
            F.cread = c64;
          }
        }
        if (F.in_t == 0 && F.a_mode == A_GATHER && F.cread > X.ldc)
          return set_err(GACER_E_UNSUPPORTED_OP, "input padding");
        F.K = F.kh * F.kw * F.cread;
        F.Kpad = roundup(F.K, BK);
        F.nkb = F.Kpad / BK;
        size_t rows;
        if (F.swap) {
          F.rows_are_pixels = false;
          F.M = F.Cout; F.N = B;
          F.tiles_m = cdiv(F.Cout, BM);
          F.bn = std::min(BN_MAX, roundup(B, 16));
          F.tiles_n = cdiv(B, F.bn);
          rows = static_cast<size_t>(F.tiles_m) * BM;
        } else {
          F.M = B * F.Ho * F.Wo; F.N = F.Cout;
          F.tiles_m = cdiv(F.M, BM * F.mrep);
          // 128x256 tiles (less L2 operand traffic per FLOP) when they still
          // give every SM a tile; else N <= 128.  A function of the layer
          // shape only, identical in every mode.
          // Also for every throughput-dominant layer (>= 2 GFLOP): a 128x256
          // tile moves (128+256)/(128*256) smem/L2 bytes per MAC against
          // (128+128)/(128*128) for 128x128 -- the mainloop is bound by the
          // shared-memory port (TMA fill + tensor-core operand reads,
          // scripts/micro/tma_rate2.cu), so the wide tile needs ~30% less
          // SM time per FLOP; in a multi-tenant round the other tenants'
          // items fill the SMs a layer no longer covers by itself.
          const double wide_gflop = [] {   // (A/B knob: FLOP threshold of the 128x256 tile)
            const char* e = getenv("GACER_WIDE_GFLOP");
            return e ? atof(e) : 2.0;
          }();
          if (F.Cout >= 256 && (F.tiles_m * cdiv(F.Cout, 256) >= kSplitSms || F.flops >= wide_gflop * 1e9)) F.bn = 256;
          else F.bn = F.Cout >= 128 ? 128 : roundup(F.Cout, 16);
          F.tiles_n = cdiv(F.Cout, F.bn);
          rows = static_cast<size_t>(F.tiles_n) * F.bn;
        }
        F.bm = BM * F.mrep;
        // split-K: a function of the layer shape only (same in every mode/plan)
        const int tiles = F.tiles_m * F.tiles_n;
        int sk = 1;
        // (each split keeps >= 8 K-blocks: below that the fixed-order
        //  reduction of the partials costs more than the MMA it parallelises)
        // Convolutions run without split-K by default: the last arrival's
        // fixed-order reduction is a serial tail of dependent L2 round trips
        // (bn = 256: 32 steps, ~27 us on VGG-16's conv5_x against 14 us of
        // MMA work per split), and the executor fills the SMs a narrow conv
        // leaves idle with other items.  Same-box A/B: D2 1.71 -> 1.57 ms,
        // D3 4.20 -> 3.47 ms, the Table-2 mixes -8 to -10 %, the sequential
        // baseline faster too.  The swap-AB linears keep theirs (VGG-16's
        // FC1: 392 K-blocks on 32 tiles).  GACER_SPLITK_MAX=2/4 re-enables it.
        const int split_max_conv = [] {
          const char* e = getenv("GACER_SPLITK_MAX");
          return e ? std::max(1, std::min(MAX_SPLIT, atoi(e))) : 1;
        }();
        const int split_max_swap = [] {
          const char* e = getenv("GACER_SPLITK_SWAP_MAX");
          return e ? std::max(1, std::min(MAX_SPLIT, atoi(e))) : MAX_SPLIT;
        }();
        const int split_max = F.swap ? split_max_swap : split_max_conv;
        while (sk < split_max && tiles * sk * 2 <= kSplitSms && F.nkb / (sk * 2) >= 8) sk *= 2;
        if (F.mrep > 1) sk = 1;
        F.split_k = sk;
        F.w_bf16.assign(rows * F.Kpad, 0);
        for (int co = 0; co < F.Cout; ++co)
          for (int r = 0; r < F.kh; ++r)
            for (int s = 0; s < F.kw; ++s)
              for (int c = 0; c < F.Cin; ++c) {
                const int k = (r * F.kw + s) * F.cread + c;
                size_t at = static_cast<size_t>(co) * F.Kpad + k;
                if (F.a_mode == A_IM2COL8) {
                  // per (N-tile, K-block) a contiguous bn x 64 block in the
                  // no-swizzle K-major core-matrix layout the MMA reads:
                  // (n % 8) * 16 B + (n / 8) * 128 B + (k % 8) * 2 B + (k % 64 / 8) * bn * 16 B
                  const int nt = co / F.bn, n = co % F.bn, kb = k / BK, kk = k % BK;
                  at = (static_cast<size_t>(nt) * F.nkb + kb) * F.bn * BK +
                       ((n % 8) * 8 + (n / 8) * 64 + (kk % 8) + (kk / 8) * F.bn * 8);
                }
                F.w_bf16[at] = f32_to_bf16_rne(wval(co, c, r, s));
              }
        F.scale.resize(roundup(F.Cout, 8) + 8, 0.0f);
        F.bias.resize(roundup(F.Cout, 8) + 8, 0.0f);
      }
    } else if (F.kind == DK_DW) {
      F.kh = o.kh; F.kw = o.kw; F.stride = o.stride; F.ph = o.pad_h; F.pw = o.pad_w;
      F.flops = 2.0 * B * F.Ho * F.Wo * F.Cout * F.kh * F.kw;
      fold(F.Cout, cbias);
      F.w_f32.assign(static_cast<size_t>(F.kh) * F.kw * F.Cout, 0.0f);
      for (int c = 0; c < F.Cout; ++c)
        for (int r = 0; r < F.kh; ++r)
          for (int s = 0; s < F.kw; ++s) {
            const float w = o.weight[(static_cast<size_t>(c) * o.kh + r) * o.kw + s];
            F.w_f32[(r * F.kw + s) * F.Cout + c] = f32 ? w : f32_to_bf16_round_trip(w);
          }
      F.M = B * F.Ho * F.Wo;
    } else if (F.kind == DK_MAXPOOL || F.kind == DK_AVGPOOL) {
      F.kh = o.kh; F.kw = o.kw; F.stride = o.stride; F.ph = o.pad_h; F.pw = o.pad_w;
      F.M = B * F.Ho * F.Wo;
    } else if (F.kind == DK_GAP) {
      F.M = B;
    } else if (F.kind == DK_ELTWISE) {
      F.M = B * F.Ho * F.Wo;
      fold(F.Cout, nullptr);
    }
    if (F.kind != DK_GEMM && F.kind != DK_SIMT_GEMM) {
      F.bn = std::min(64, pow2ceil(roundup(F.Cout, 8)));
      const int G = F.bn / 8;
      F.bm = (F.kind == DK_GAP) ? std::min(B, 64) : CC_TASKS_PER_THREAD * (CC_THREADS / G);
      if (F.kind != DK_GAP) {
        // per-pixel CUDA-core items (eltwise ops, 5x5 depthwise, fp32 window
        // ops): rows per item grown (in whole thread sweeps) until the op has
        // about cc_per_sm items per SM -- fewer, longer items amortise the
        // per-item scheduling, like the window items below
        const double cc_per_sm = [] {
          const char* e = getenv("GACER_CC_ITEMS_PER_SM");
          // 1 per SM: R101+D121+M3 3.24 -> 3.02 ms, D2 / D3 neutral, the
          // per-op baselines unchanged (0.5 gained a little more in the
          // executor but cost the baselines 5-7 %)
          return e ? std::max(0.05, atof(e)) : 1.0;
        }();
        const int pstep = CC_THREADS / G;
        const double items = static_cast<double>(cdiv(F.M, F.bm)) * cdiv(F.Cout, F.bn);
        if (items > cc_per_sm * kSplitSms) {
          const int sweeps = static_cast<int>(std::ceil(items / (cc_per_sm * kSplitSms)));
          F.bm *= std::max(1, sweeps);
          (void)pstep;
        }
      }
      F.tiles_n = cdiv(F.Cout, F.bn);
      // bf16 window ops (depthwise / max / avg pool, <= 9 taps): items of R
      // whole output rows whose input rows are staged in shared memory
      // (window_smem); R from the staging budget and ~0.75 items per SM (fewer,
      // longer items: each item drains the GEMM ring it borrows and pays the
      // per-item claim / release; D2 1.81 -> 1.71 ms vs 2 per SM, D3 -3.6 %)
      F.win = false;
      if (!f32 && (F.kind == DK_DW || F.kind == DK_MAXPOOL || F.kind == DK_AVGPOOL) && F.kh * F.kw <= 9) {
        const long long row_bytes = static_cast<long long>(F.W) * F.bn * 2;
        const long long rows_fit = WIN_IN_BYTES / row_bytes;   // input rows that fit
        if (rows_fit >= F.kh) {
          const int r_max = static_cast<int>((rows_fit - F.kh) / F.stride + 1);
          const long long out_rows = static_cast<long long>(B) * F.Ho;
          const double win_per_sm = [] {   // items per SM the row count aims at (A/B knob)
            const char* e = getenv("GACER_WIN_ITEMS_PER_SM");
            // (0.5 first: D2 1.81 -> 1.71 ms vs 2; re-tuned after the split-K /
            //  M-pair changes: 0.75 beats 0.5 by 1.7 % on D2, 1.2 % on D3)
            return e ? std::max(0.05, atof(e)) : 0.75;
          }();
          const int r_par = static_cast<int>(std::max<long long>(
              1, static_cast<long long>(static_cast<double>(out_rows * F.tiles_n) / (win_per_sm * kSplitSms))));
          const int R = std::max(1, std::min(r_max, r_par));
          F.bm = R * F.Wo;
          F.win = true;
        }
      }
      F.tiles_m = cdiv(F.M, F.bm);
      F.scale.resize(roundup(F.Cout, 8) + 8, 0.0f);
      F.bias.resize(roundup(F.Cout, 8) + 8, 0.0f);
    }
    const double e = elem;
    F.bytes = (static_cast<double>(B) * F.H * F.W * F.Cin + static_cast<double>(B) * F.Ho * F.Wo * F.Cout) * e +
              (F.w_bf16.size() * 2.0 + F.w_f32.size() * 4.0);
    T.flops += F.flops;
  }
  return 0;
}

}  // namespace

// ------------------------------------------------------------------------
// device residency of a tenant and the global op table
// ------------------------------------------------------------------------
namespace {

size_t elem_size(const Tenant& T) { return T.dtype == GACER_DTYPE_FP32 ? 4 : 2; }

char* tensor_addr(const Tenant& T, int t) {
  const Tensor& X = T.tensors[t];
  if (X.buf == -2) return static_cast<char*>(T.out_dev);  // float32 [B][features]
  char* base = X.buf == -1 ? const_cast<char*>(static_cast<const char*>(T.in_dev))
                           : static_cast<char*>(T.bufs[X.buf]);
  if (!base) return nullptr;
  return base + static_cast<size_t>(X.coff) * elem_size(T);
}

int upload_tenant(Tenant& T) {
  if (T.train) return upload_train_tenant(T);
  for (size_t b = 0; b < T.bufs.size(); ++b)
    if (T.buf_bytes[b]) CUDA_TRY(cudaMalloc(&T.bufs[b], T.buf_bytes[b]));
  for (FusedOp& F : T.fops) {
    if (!F.w_bf16.empty()) {
      F.w_bytes = F.w_bf16.size() * 2;
      CUDA_TRY(cudaMalloc(&F.d_w, F.w_bf16.size() * 2));
      CUDA_TRY(cudaMemcpy(F.d_w, F.w_bf16.data(), F.w_bf16.size() * 2, cudaMemcpyHostToDevice));
    } else if (!F.w_f32.empty()) {
      CUDA_TRY(cudaMalloc(&F.d_w, F.w_f32.size() * 4));
      CUDA_TRY(cudaMemcpy(F.d_w, F.w_f32.data(), F.w_f32.size() * 4, cudaMemcpyHostToDevice));
    }
    if (!F.scale.empty()) {
      if (int rc = dev_upload(&F.d_scale, F.scale.data(), F.scale.size())) return rc;
      if (int rc = dev_upload(&F.d_bias, F.bias.data(), F.bias.size())) return rc;
    }
    if (F.kind == DK_GEMM && F.split_k > 1) {
      const size_t tiles = static_cast<size_t>(F.tiles_m) * F.tiles_n;
      CUDA_TRY(cudaMalloc(&F.d_partial, tiles * F.split_k * BM * F.bn * sizeof(float)));
      if (int rc = dev_upload<uint32_t>(&F.d_tile_cnt, nullptr, tiles)) return rc;
    }
    // host copies of the packed weights are no longer needed
    std::vector<uint16_t>().swap(F.w_bf16);
    std::vector<float>().swap(F.w_f32);
  }
  return 0;
}

void free_tenant(Tenant& T) {
  for (void* p : T.bufs) if (p) cudaFree(p);
  for (void* p : T.tbufs) if (p) cudaFree(p);
  for (FusedOp& F : T.fops) {
    for (void* p : {static_cast<void*>(F.d_w), static_cast<void*>(F.d_scale), static_cast<void*>(F.d_bias),
                    static_cast<void*>(F.d_partial), static_cast<void*>(F.d_tile_cnt)})
      if (p) cudaFree(p);
  }
}

OpDev make_opdev(const Tenant& T, int tenant_id, const FusedOp& F) {
  OpDev d;
  std::memset(&d, 0, sizeof d);
  const Tensor& X = T.tensors[F.in_t];
  const Tensor& Y = T.tensors[F.out_t];
  const bool f32 = T.dtype == GACER_DTYPE_FP32;
  d.kind = F.kind;
  d.tenant = tenant_id;
  d.act = F.act;
  d.out_f32 = (Y.buf == -2 || f32) ? 1 : 0;
  d.f32 = f32 ? 1 : 0;
  // 2: swap-AB whose A operand (the weights, read once per round) is loaded
  // with an L2 evict-first policy (GACER_NO_L2_HINT=1: plain loads)
  d.swap = F.swap ? (env_flag("GACER_NO_L2_HINT") ? 1 : 2) : 0;
  d.cip = F.cip ? 1 : 0;
  d.has_skip = F.skip_t >= 0 ? (F.mul ? 2 : 1) : 0;
  d.affine = F.affine ? 1 : 0;
  d.in = tensor_addr(T, F.in_t);
  d.B = T.batch; d.H = F.H; d.W = F.W;
  d.C = (F.kind == DK_GEMM) ? F.cread : F.Cin;
  d.ldi = X.ldc;
  d.out = tensor_addr(T, F.out_t);
  d.Ho = F.Ho; d.Wo = F.Wo; d.Cout = F.Cout; d.ldo = Y.ldc;
  if (F.skip_t >= 0) { d.skip = tensor_addr(T, F.skip_t); d.lds = T.tensors[F.skip_t].ldc; }
  d.kh = F.kh; d.kw = F.kw; d.stride = F.stride; d.ph = F.ph; d.pw = F.pw;
  d.win = F.win ? 1 : 0;
  d.mrep = F.mrep;
  d.M = F.M; d.N = F.N; d.K = F.K; d.Kpad = F.Kpad;
  d.tiles_m = F.tiles_m; d.tiles_n = F.tiles_n; d.bm = F.bm; d.bn = F.bn;
  d.split_k = F.split_k; d.nkb = F.nkb;
  d.wt = F.d_w;
  d.ldw = (F.kind == DK_GEMM) ? F.Kpad : F.K;
  if (F.swap) { d.act_b = d.in; d.ldb = F.H * F.W * X.ldc; }
  d.scale = F.d_scale; d.bias = F.d_bias;
  d.partial = F.d_partial; d.tile_cnt = F.d_tile_cnt;
  return d;
}

// ---- TMA descriptors (driver entry points resolved through the runtime)
PFN_cuTensorMapEncodeTiled_v12000 g_encode_tiled = nullptr;
PFN_cuTensorMapEncodeIm2col_v12000 g_encode_im2col = nullptr;

PFN_cuStreamWriteValue32_v11070 g_write_value32 = nullptr;
PFN_cuStreamWaitValue32_v11070 g_wait_value32 = nullptr;

int load_tma_encoders() {
  if (!g_write_value32) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    CUDA_TRY(cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q));
    g_write_value32 = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(f);
    if (!g_write_value32) return set_err(GACER_E_CUDA, "cuStreamWriteValue32 not available");
    CUDA_TRY(cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q));
    g_wait_value32 = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(f);
    if (!g_wait_value32) return set_err(GACER_E_CUDA, "cuStreamWaitValue32 not available");
  }
  if (g_encode_tiled && g_encode_im2col) return 0;
  cudaDriverEntryPointQueryResult q;
  void* f = nullptr;
  CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
  g_encode_tiled = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f, cudaEnableDefault, &q));
  g_encode_im2col = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(f);
  if (!g_encode_tiled || !g_encode_im2col) return set_err(GACER_E_CUDA, "cuTensorMapEncode* not available");
  return 0;
}

// K-major bf16 matrix [rows][ld] (row stride ld elements), box {64, box_rows},
// 128-byte swizzle = the UMMA SWIZZLE_128B K-major canonical layout.
int encode_rows(CUtensorMap* m, const void* base, int cols, int rows, int ld, int box_rows) {
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(GACER_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return 0;
}

// NHWC bf16 activation as an im2col view: 128 output pixels x 64 channels of
// one filter tap per load (pixelsPerColumn = BM, channelsPerPixel = BK).
// Bounding box per CUTLASS fprop convention: lower = -pad, upper = pad - (k-1).
int encode_im2col(CUtensorMap* m, const OpDev& d, int real_c, int pix_box = BM, int ch_box = BK,
                  CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B, const int* upper_hw = nullptr) {
  // globalDim[0] is the tensor's real channel count: channels [Cin, cread)
  // of a 64-channel box are out of bounds and zero-filled by the TMA
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(real_c), static_cast<cuuint64_t>(d.W),
                              static_cast<cuuint64_t>(d.H), static_cast<cuuint64_t>(d.B)};
  const cuuint64_t st[3] = {static_cast<cuuint64_t>(d.ldi) * 2, static_cast<cuuint64_t>(d.ldi) * 2 * d.W,
                            static_cast<cuuint64_t>(d.ldi) * 2 * d.W * d.H};
  const int lower[2] = {-d.pw, -d.ph};
  // (upper_hw: an explicit upper corner -- the output count per row is
  //  W + upper - lower, e.g. the phases of a strided conv's data gradient)
  const int upper[2] = {upper_hw ? upper_hw[1] : d.pw - (d.kw - 1), upper_hw ? upper_hw[0] : d.ph - (d.kh - 1)};
  const cuuint32_t es[4] = {1, static_cast<cuuint32_t>(d.stride), static_cast<cuuint32_t>(d.stride), 1};
  CUresult r = g_encode_im2col(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(d.in), dims, st, lower, upper,
                               static_cast<cuuint32_t>(ch_box), static_cast<cuuint32_t>(pix_box), es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(GACER_E_CUDA, "cuTensorMapEncodeIm2col failed (%d)", static_cast<int>(r));
  return 0;
}

int rebuild_op_table() {
  if (S.base_graph) {   // the captured baseline bakes op-table pointers
    cudaGraphExecDestroy(S.base_graph);
    S.base_graph = nullptr;
    S.base_graph_mode = -1;
  }
  S.h_ops.clear();
  std::vector<const FusedOp*> fops;
  std::vector<std::pair<int, const TrainOp*>> tops;   // training ops: (tenant, op)
  for (size_t t = 0; t < S.tenants.size(); ++t) {
    Tenant& T = S.tenants[t];
    T.op_base = static_cast<int>(S.h_ops.size());
    for (const FusedOp& F : T.fops) {
      S.h_ops.push_back(make_opdev(T, static_cast<int>(t), F));
      fops.push_back(&F);
      tops.push_back({-1, nullptr});
    }
    // weight prefetch targets: the next two tcgen05 GEMM ops of the tenant in
    // issue order whose packed weights are small enough to sit in L2 ahead of
    // use (<= 8 MB; not the swap-AB linears, which stream their weights)
    if (!env_flag("GACER_NO_WPREFETCH")) {
      const int nf = static_cast<int>(T.fops.size());
      for (int f = 0; f < nf; ++f) {
        OpDev& d = S.h_ops[T.op_base + f];
        int k = 0;
        for (int g2 = f + 1; g2 < nf && k < 2; ++g2) {
          const FusedOp& G2 = T.fops[g2];
          if (G2.kind != DK_GEMM || G2.swap || !G2.d_w) continue;
          const size_t bytes = G2.w_bytes;
          if (bytes == 0 || bytes > (8u << 20)) continue;
          d.pf_ptr[k] = G2.d_w;
          d.pf_bytes[k] = static_cast<uint32_t>(bytes & ~static_cast<size_t>(15));
          ++k;
        }
      }
    }
    for (const TrainOp& op : T.tops) {
      OpDev d;
      if (int rc = build_train_opdev(T, static_cast<int>(t), op, d, nullptr, false)) return rc;
      S.h_ops.push_back(d);
      fops.push_back(nullptr);
      tops.push_back({static_cast<int>(t), &op});
    }
  }
  if (S.host_only) return 0;
  if (int rc = load_tma_encoders()) return rc;
  const size_t n = S.h_ops.size();
  if (S.n_tmaps < 3 * n) {
    if (S.d_tmaps) cudaFree(S.d_tmaps);
    S.d_tmaps = nullptr;
    CUDA_TRY(cudaMalloc(&S.d_tmaps, 3 * n * sizeof(CUtensorMap)));  // cudaMalloc: 256-byte aligned
    S.n_tmaps = 3 * n;
  }
  std::vector<CUtensorMap> maps(3 * n);
  std::memset(maps.data(), 0, maps.size() * sizeof(CUtensorMap));
  for (size_t i = 0; i < n; ++i) {
    OpDev& d = S.h_ops[i];
    if (d.kind != DK_GEMM) continue;
    if (tops[i].second) {   // training-tenant GEMM: its own operand layouts
      const Tenant& T = S.tenants[tops[i].first];
      if (int rc = build_train_opdev(T, tops[i].first, *tops[i].second, d, &maps[3 * i], true)) return rc;
      d.tmap_a = S.d_tmaps + 3 * i;
      d.tmap_b = S.d_tmaps + 3 * i + 1;
      d.tmap_c = S.d_tmaps + 3 * i + 2;
      continue;
    }
    const FusedOp& F = *fops[i];
    d.a_mode = F.a_mode;
    d.tmap_a = S.d_tmaps + 3 * i;
    d.tmap_b = S.d_tmaps + 3 * i + 1;
    d.tmap_c = S.d_tmaps + 3 * i + 2;
    d.c_tma = 0;
    if (!d.in || !d.out) continue;  // I/O not bound yet: re-encoded by gacer_bind_io
    int rc = 0;
    if (d.swap) {
      rc = encode_rows(&maps[3 * i], d.wt, d.Kpad, d.tiles_m * BM, d.Kpad, BM);
      if (!rc) rc = encode_rows(&maps[3 * i + 1], d.act_b, d.K, d.B, d.ldb, d.bn);
    } else {
      if (d.a_mode == A_IM2COL) rc = encode_im2col(&maps[3 * i], d, F.Cin);
      else if (d.a_mode == A_IM2COL8) rc = encode_im2col(&maps[3 * i], d, F.Cin, BM, 8, CU_TENSOR_MAP_SWIZZLE_NONE);
      else if (d.a_mode == A_ROWS) rc = encode_rows(&maps[3 * i], d.in, d.K, d.M, d.ldi, BM);
      if (!rc && d.a_mode != A_IM2COL8)   // (IM2COL8: B is a bulk copy of pre-packed blocks)
        rc = encode_rows(&maps[3 * i + 1], d.wt, d.Kpad, d.tiles_n * d.bn, d.Kpad, d.bn);
      // output [M][Cout] (row stride ldo) for the TMA-store epilogue
      const int esz = d.out_f32 ? 4 : 2;
      const bool ok = (static_cast<long long>(d.ldo) * esz) % 16 == 0 &&
                      (reinterpret_cast<uintptr_t>(d.out) & 15) == 0;
      // (GACER_DIRECT_SMALL=n, diagnostics: ops of <= n items store directly)
      const long long items = static_cast<long long>(d.tiles_m) * d.tiles_n * d.split_k;
      const char* ds = getenv("GACER_DIRECT_SMALL");
      const bool small_direct = ds && items <= atoll(ds);
      if (!rc && ok && !env_flag("GACER_NO_TMA_STORE") && !small_direct) {
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(d.Cout), static_cast<cuuint64_t>(d.M)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(d.ldo) * esz};
        const cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / esz), 32u};  // 32 rows x 128 B
        const cuuint32_t es[2] = {1, 1};
        CUresult r = g_encode_tiled(&maps[3 * i + 2],
                                    d.out_f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                    d.out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_err(GACER_E_CUDA, "cuTensorMapEncodeTiled (output) failed (%d)", static_cast<int>(r));
        d.c_tma = 1;
      }
    }
    if (rc) return rc;
  }
  CUDA_TRY(cudaMemcpy(S.d_tmaps, maps.data(), 3 * n * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  return dev_upload(&S.d_ops, S.h_ops.data(), S.h_ops.size());
}

// ------------------------------------------------------------------------
// plan compilation (Eq. 5 chunks -> tile ranges; Eq. 6/7 -> clusters)
// ------------------------------------------------------------------------
struct ChunkRange {
  int m0, m1, n0, n1;  // tile ranges
  int counter;
  uint32_t n_items;
  int budget = 0;      // gacer_chunking.sm_budget of this chunk (0 = unlimited)
  int bud = -1;        // its budget counter (items released), -1 = none
  // Completion counters at M-tile granularity (ops whose M axis is output
  // pixels or samples): mc[mt - m0] counts the items of M-tile mt in this
  // chunk (target mc_items).  A consumer waits only for the producer tiles
  // its input window reads, so consecutive ops of a chain overlap (a
  // wavefront) instead of meeting at whole-op barriers.  Chunk semantics
  // (Eq. 5) are unchanged: this only refines the dependency bookkeeping.
  std::vector<int> mc;
  uint32_t mc_items = 0;
};

int cluster_of_orig(const Plan& P, int t, int orig0) {  // orig0: 0-based op index
  if (P.cuts.empty()) return 0;
  int k = 0;
  for (int c : P.cuts[t]) if (c < orig0 + 1) ++k;  // cut p = boundary after op p
  return k;
}

// Input rows a tile of fused op F reads from tensor tin, as a flattened row
// range [lo, hi]: pixels (b*H + h)*W + w, or samples for [B][C] tensors.
void tile_read_rows(const Tenant& T, const FusedOp& F, int mt, int ntile, int tin, long long& lo, long long& hi) {
  long long s_lo, s_hi;   // samples
  long long px_lo = -1, px_hi = -1;  // input pixels of in_t (-1: whole samples)
  if (F.rows_are_pixels) {
    const long long R = (F.kind == DK_GAP) ? 1 : static_cast<long long>(F.Ho) * F.Wo;
    const long long r0 = static_cast<long long>(mt) * F.bm;
    const long long r1 = std::min<long long>(F.M, r0 + F.bm);
    s_lo = r0 / R;
    s_hi = (r1 - 1) / R;
    if (F.kind != DK_GAP) {
      const long long HW = static_cast<long long>(F.H) * F.W;
      const long long ho0 = (r0 % R) / F.Wo, ho1 = ((r1 - 1) % R) / F.Wo;
      const long long h_lo = std::max<long long>(0, ho0 * F.stride - F.ph);
      const long long h_hi = std::min<long long>(F.H - 1, ho1 * F.stride - F.ph + F.kh - 1);
      px_lo = s_lo * HW + h_lo * F.W;
      px_hi = s_hi * HW + h_hi * F.W + F.W - 1;
    }
  } else {
    s_lo = static_cast<long long>(ntile) * F.bn;
    s_hi = std::min<long long>(T.batch, static_cast<long long>(ntile + 1) * F.bn) - 1;
  }
  const Tensor& X = T.tensors[tin];
  const long long XHW = static_cast<long long>(X.H) * X.W;
  lo = s_lo * XHW;
  hi = (s_hi + 1) * XHW - 1;
  if (tin == F.skip_t && F.mul) {
    // channel scale [B][C]: the samples of the tile's rows (lo, hi as set)
  } else if (tin == F.skip_t && F.rows_are_pixels && F.kind != DK_GAP) {
    lo = static_cast<long long>(mt) * F.bm;   // residual: same pixels as the output
    hi = std::min<long long>(F.M, lo + F.bm) - 1;
  } else if (px_lo >= 0 && tin == F.in_t) {
    lo = px_lo;
    hi = px_hi;
  }
}

// Output rows [lo, hi] (flattened, as above) a tile of fused op F writes.
void tile_write_rows(const Tenant& T, const FusedOp& F, int mt, int ntile, long long& lo, long long& hi) {
  if (F.rows_are_pixels) {
    lo = static_cast<long long>(mt) * F.bm;
    hi = std::min<long long>(F.M, lo + F.bm) - 1;
  } else {
    lo = static_cast<long long>(ntile) * F.bn;
    hi = std::min<long long>(T.batch, lo + F.bn) - 1;
  }
}

int compile_plan(Plan& P) {
  const int nt = static_cast<int>(S.tenants.size());
  P.n_clusters = (P.cuts.empty() ? 0 : static_cast<int>(P.cuts[0].size())) + 1;
  P.items.clear(); P.deps.clear(); P.queue.clear(); P.segs.clear();
  P.cluster_total.assign(P.n_clusters, 0);
  P.fop_cluster.assign(nt, {});
  std::vector<std::vector<std::vector<ChunkRange>>> cr(nt);
  int counter = 0;
  for (int t = 0; t < nt; ++t) {
    const Tenant& T = S.tenants[t];
    if (T.train) {   // training tenant: whole-op counters, clusters by step position
      cr[t].resize(T.tops.size());
      P.fop_cluster[t].resize(T.tops.size());
      for (size_t f = 0; f < T.tops.size(); ++f) {
        const TrainOp& op = T.tops[f];
        P.fop_cluster[t][f] = cluster_of_orig(P, t, op.step_pos - 1);
        ChunkRange r{0, op.kind == DK_GEMM ? op.gd.tiles_m : op.items, 0, op.kind == DK_GEMM ? op.gd.tiles_n : 1, 0, 0};
        r.n_items = static_cast<uint32_t>(op.items);
        r.counter = counter++;
        cr[t][f].push_back(r);
      }
      continue;
    }
    cr[t].resize(T.fops.size());
    P.fop_cluster[t].resize(T.fops.size());
    for (size_t f = 0; f < T.fops.size(); ++f) {
      const FusedOp& F = T.fops[f];
      P.fop_cluster[t][f] = cluster_of_orig(P, t, F.last);
      const Chunking* ch = nullptr;
      for (int m : F.members) {
        auto it = P.chunks.find({t, m});
        if (it == P.chunks.end()) continue;
        if (ch && (ch->axis != it->second.axis || ch->sizes != it->second.sizes || ch->budget != it->second.budget))
          return set_err(GACER_E_INVALID_ARG, "tenant %d: fused ops %d and %d carry different chunkings", t,
                         F.head + 1, m + 1);
        ch = &it->second;
      }
      const int split = (F.kind == DK_GEMM) ? F.split_k : 1;
      std::vector<ChunkRange>& ranges = cr[t][f];
      if (!ch) {
        ranges.push_back({0, F.tiles_m, 0, F.tiles_n, 0, 0});
      } else {
        // which tile axis carries the split, and units per tile along it
        bool on_m;
        long long unit;  // rows (or channels) per chunk unit
        int tsz;
        if (ch->axis == GACER_AXIS_BATCH) {
          if (F.rows_are_pixels) { on_m = true; unit = (F.kind == DK_GAP) ? 1 : static_cast<long long>(F.Ho) * F.Wo; tsz = F.bm; }
          else { on_m = false; unit = 1; tsz = F.bn; }
        } else {
          if (F.rows_are_pixels) { on_m = false; unit = 1; tsz = F.bn; }
          else { on_m = true; unit = 1; tsz = BM; }
        }
        const int ntiles = on_m ? F.tiles_m : F.tiles_n;
        long long u = 0;
        for (size_t j = 0; j < ch->sizes.size(); ++j) {
          const int s = ch->sizes[j];
          const long long a = u * unit, b = (u + s) * unit;
          int t0 = static_cast<int>((a + tsz - 1) / tsz), t1 = static_cast<int>((b + tsz - 1) / tsz);
          t0 = std::min(t0, ntiles); t1 = std::min(t1, ntiles);
          if (on_m) ranges.push_back({t0, t1, 0, F.tiles_n, 0, 0});
          else ranges.push_back({0, F.tiles_m, t0, t1, 0, 0});
          if (!ch->budget.empty()) ranges.back().budget = ch->budget[j];
          u += s;
        }
      }
      for (ChunkRange& r : ranges) {
        r.n_items = static_cast<uint32_t>(std::max(0, r.m1 - r.m0) * std::max(0, r.n1 - r.n0) * split);
        r.counter = -1;
        if (!r.n_items) continue;
        if (F.rows_are_pixels && !S.opts.coarse_deps) {
          r.mc_items = static_cast<uint32_t>((r.n1 - r.n0) * split);
          for (int mt = r.m0; mt < r.m1; ++mt) r.mc.push_back(counter++);
        } else {
          r.counter = counter++;
        }
        // SM budget W(O^B) (l.597-601): a semaphore counter of the chunk's
        // released items; only when it binds (fewer than the chunk's items)
        if (r.budget > 0 && static_cast<uint32_t>(r.budget) < r.n_items) r.bud = counter++;
      }
    }
  }
  // one input-gate counter per tenant (after the chunk counters): the items
  // that read the graph input wait for it, so a round whose H2D copies run on
  // a copy stream starts each tenant as soon as its own input has landed
  P.input_counter0 = counter;
  counter += nt;
  // A12: per-tenant gradient gates (opened by the communication stream after
  // the data-parallel all-reduce; the SGD op of a gated tenant waits for it)
  P.grad_gate0 = counter;
  counter += nt;
  P.n_chunk_counters = counter;

  // upward rank of every fused op (HEFT-style list scheduling): estimated
  // latency of the op + the longest rank among its consumers.  The device
  // scheduler claims the ready head item with the highest rank first.
  std::vector<std::vector<uint32_t>> rank(nt);
  P.auto_share.assign(nt, 1.0);
  for (int t = 0; t < nt; ++t) {
    const Tenant& T = S.tenants[t];
    if (T.train) {
      // per op: one item's latency (GEMM: its K-blocks at the executor's
      // measured per-SM rate; CUDA-core: its share of the op's bytes at
      // ~10 GB/s per SM) plus the per-op latency floor; rank = the longest
      // remaining dependency chain (HEFT upward rank over op.deps)
      const size_t nf = T.tops.size();
      std::vector<double> est(nf), rk(nf, 0.0), wk(nf, 0.0);
      for (size_t f = 0; f < nf; ++f) {
        const TrainOp& op = T.tops[f];
        double item_ns;
        if (op.kind == DK_GEMM) {
          const double kblocks = static_cast<double>(op.gd.nkb) / op.gd.split_k;
          item_ns = kblocks * BK * BM * op.gd.bn * 2.0 / 2700.0 + 1500.0;
        } else {
          item_ns = op.bytes / std::max(1, op.items) / 10.0 + 2000.0;
        }
        wk[f] = op.items * item_ns / kSplitSms;
        est[f] = 10000.0 + std::max(item_ns, wk[f]);
      }
      std::vector<double> best(nf, 0.0);
      for (size_t f = nf; f-- > 0;) {
        rk[f] = est[f] + best[f];
        for (int d : T.tops[f].deps) best[d] = std::max(best[d], rk[f]);
      }
      rank[t].resize(nf);
      double work_ns = 0.0, chain_ns = 0.0;
      for (size_t f = 0; f < nf; ++f) {
        rank[t][f] = static_cast<uint32_t>(std::min(rk[f], 4.0e9));
        work_ns += wk[f];
        chain_ns = std::max(chain_ns, rk[f]);
      }
      P.auto_share[t] = std::min(1.0, work_ns / std::max(1.0, chain_ns));
      continue;
    }
    const size_t nf = T.fops.size();
    std::vector<double> est(nf), rk(nf, 0.0), wk(nf, 0.0);
    for (size_t f = 0; f < nf; ++f) {
      const FusedOp& F = T.fops[f];
      const int split = (F.kind == DK_GEMM) ? F.split_k : 1;
      const double items = static_cast<double>(F.tiles_m) * F.tiles_n * split;
      const double waves = std::ceil(items / kSplitSms);
      // per-item time at the executor's measured rates (~2.7 TFLOP/s of
      // tensor work and ~10 GB/s of CUDA-core traffic per SM), and a per-op
      // latency floor (dependency notice + claim + first load + epilogue):
      // a chain of many small ops is long even when its work is tiny.
      double item_ns;
      if (F.kind == DK_GEMM) {
        const double kblocks = static_cast<double>(F.nkb) / split;
        item_ns = kblocks * BK * BM * F.bn * 2.0 / 2700.0 + 1500.0;
      } else {
        item_ns = F.bytes / std::max(1.0, items) / 10.0 + 2000.0;
      }
      // Rank = remaining chain LATENCY: per op a latency floor plus one item
      // (not the op's whole work).  Narrow ops of long chains (latency-bound)
      // then outrank the wide ops of a throughput-bound tenant, which absorb
      // the delay by filling whatever SMs the chains leave free.
      wk[f] = items * item_ns / kSplitSms;  // work, as full-GPU time
      (void)waves;
      // HEFT upward rank: the op's duration with the whole GPU (its work
      // spread over every SM, but never below one item) plus a per-op
      // latency floor.  A chain of few but wide ops (VGG-16) is then ranked
      // by its real length instead of its op count.
      est[f] = 10000.0 + std::max(item_ns, wk[f]);
    }
    for (size_t f = nf; f-- > 0;) {
      double best = 0.0;
      for (size_t g2 = f + 1; g2 < nf; ++g2) {
        const FusedOp& G2 = T.fops[g2];
        bool consumes = false;
        for (int tin : {G2.in_t, G2.skip_t})
          if (tin >= 0)
            for (int w : T.tensors[tin].writers) consumes |= (w == static_cast<int>(f));
        if (consumes) best = std::max(best, rk[g2]);
      }
      rk[f] = est[f] + best;
    }
    rank[t].resize(nf);
    for (size_t f = 0; f < nf; ++f) rank[t][f] = static_cast<uint32_t>(std::min(rk[f], 4.0e9));
    // SM need of the tenant (the paper's resource share W, §4.1 l.597-601):
    // the fraction of the GPU that sustains its work at its chain latency
    double work_ns = 0.0, chain_ns = 0.0;
    for (size_t f = 0; f < nf; ++f) {
      work_ns += wk[f];
      chain_ns = std::max(chain_ns, rk[f]);
    }
    P.auto_share[t] = std::min(1.0, work_ns / std::max(1.0, chain_ns));
  }

  // Write-after-read dependencies of reused activation buffers
  // (reuse_buffers): a tile writing bytes [a, b) of its output buffer waits
  // for every reader tile of the buffer's previous occupants that reads
  // those bytes (and, for bytes no reader touches, for the occupant's writer
  // tiles).  Older occupants matter only past the sizes of the more recent
  // ones: a more recent occupant's writer tiles waited for them already.
  std::vector<std::vector<int>> cdeps(P.n_chunk_counters);   // counter -> deps of its items
  struct WarEnt { long long lo, hi; Dep d; };
  struct WarSet { std::vector<WarEnt> rd, wr; long long span_rd = 0, span_wr = 0; };
  std::map<std::pair<int, int>, WarSet> war_cache;
  auto tile_dep = [&](int t, int f, const ChunkRange& q, int m) -> Dep {
    (void)t; (void)f;
    return q.mc.empty() ? Dep{q.counter, q.n_items} : Dep{q.mc[m - q.m0], q.mc_items};
  };
  auto war_set = [&](int t, int x) -> const WarSet& {
    auto it = war_cache.find({t, x});
    if (it != war_cache.end()) return it->second;
    WarSet& ws = war_cache[{t, x}];
    const Tenant& T = S.tenants[t];
    for (size_t f = 0; f < T.fops.size(); ++f) {
      const FusedOp& FR = T.fops[f];
      const bool reads = FR.in_t == x || FR.skip_t == x;
      const bool writes = FR.out_t == x;
      if (!reads && !writes) continue;
      for (const ChunkRange& q : cr[t][f]) {
        if (!q.n_items) continue;
        for (int m = q.m0; m < q.m1; ++m)
          for (int n = q.n0; n < q.n1; ++n) {
            const Dep d = tile_dep(t, static_cast<int>(f), q, m);
            for (int tin : {FR.in_t, FR.skip_t}) {
              if (tin != x) continue;
              long long lo, hi;
              tile_read_rows(T, FR, m, n, tin, lo, hi);
              ws.rd.push_back({lo, hi, d});
              ws.span_rd = std::max(ws.span_rd, hi - lo);
            }
            if (writes) {
              long long lo, hi;
              tile_write_rows(T, FR, m, n, lo, hi);
              ws.wr.push_back({lo, hi, d});
              ws.span_wr = std::max(ws.span_wr, hi - lo);
            }
          }
      }
    }
    auto by_lo = [](const WarEnt& u, const WarEnt& v) { return u.lo < v.lo; };
    std::stable_sort(ws.rd.begin(), ws.rd.end(), by_lo);
    std::stable_sort(ws.wr.begin(), ws.wr.end(), by_lo);
    return ws;
  };
  auto war_deps = [&](int t, const FusedOp& F, int mt, int ntile, const std::set<int>& dset, std::vector<Dep>& wl) {
    const Tenant& T = S.tenants[t];
    const Tensor& Y = T.tensors[F.out_t];
    if (Y.war_prev.empty()) return;
    const long long e = static_cast<long long>(elem_size(T));
    long long wlo, whi;
    tile_write_rows(T, F, mt, ntile, wlo, whi);
    const long long a = wlo * Y.ldc * e, b = (whi + 1) * Y.ldc * e;   // bytes [a, b)
    long long covered_to = 0;
    for (int x : Y.war_prev) {
      const Tensor& X = T.tensors[x];
      const long long xrow = static_cast<long long>(X.ldc) * e;
      const long long xb = static_cast<long long>(T.batch) * X.H * X.W * xrow;
      const long long lo_b = std::max(a, covered_to), hi_b = std::min(b, xb);
      if (lo_b < hi_b) {
        const long long r_lo = lo_b / xrow, r_hi = (hi_b - 1) / xrow;
        const WarSet& ws = war_set(t, x);
        auto add = [&](const Dep& d) { if (!dset.count(d.counter)) wl.push_back(d); };
        // reader tiles overlapping rows [r_lo, r_hi]; the rows they cover
        std::vector<std::pair<long long, long long>> cov;
        auto first = std::lower_bound(ws.rd.begin(), ws.rd.end(), WarEnt{r_lo - ws.span_rd, 0, {}},
                                      [](const WarEnt& u, const WarEnt& v) { return u.lo < v.lo; });
        for (auto itr = first; itr != ws.rd.end() && itr->lo <= r_hi; ++itr) {
          if (itr->hi < r_lo) continue;
          add(itr->d);
          cov.push_back({std::max(itr->lo, r_lo), std::min(itr->hi, r_hi)});
        }
        // rows no reader tile reads: the occupant's writer tiles there
        std::sort(cov.begin(), cov.end());
        std::vector<std::pair<long long, long long>> gaps;
        long long next = r_lo;
        for (const auto& c : cov) {
          if (c.first > next) gaps.push_back({next, c.first - 1});
          next = std::max(next, c.second + 1);
        }
        if (next <= r_hi) gaps.push_back({next, r_hi});
        for (const auto& gp : gaps) {
          auto fw = std::lower_bound(ws.wr.begin(), ws.wr.end(), WarEnt{gp.first - ws.span_wr, 0, {}},
                                     [](const WarEnt& u, const WarEnt& v) { return u.lo < v.lo; });
          for (auto itr = fw; itr != ws.wr.end() && itr->lo <= gp.second; ++itr)
            if (itr->hi >= gp.first) add(itr->d);
        }
      }
      covered_to = std::max(covered_to, xb);
      if (covered_to >= b) break;
    }
  };

  // items, grouped by (tenant, cluster) segment, in issue order
  std::vector<std::vector<std::vector<int32_t>>> seg_items(nt, std::vector<std::vector<int32_t>>(P.n_clusters));
  for (int t = 0; t < nt; ++t) {
    const Tenant& T = S.tenants[t];
    if (T.train) {
      for (size_t f = 0; f < T.tops.size(); ++f) {
        const TrainOp& op = T.tops[f];
        const ChunkRange& r = cr[t][f][0];
        const int k = P.fop_cluster[t][f];
        std::vector<Dep> dl;
        if (op.reads_input) dl.push_back({P.input_counter0 + t, 1u});   // input gate (images, labels)
        if (T.grad_gate && op.kind == DK_VGRID && op.vfn == VF_SGD)
          dl.push_back({P.grad_gate0 + t, 1u});                          // all-reduced gradients (A12)
        for (int d : op.deps) dl.push_back({cr[t][d][0].counter, cr[t][d][0].n_items});
        int dep_begin = 0;
        if (dl.size() > static_cast<size_t>(INLINE_DEPS)) {
          dep_begin = static_cast<int>(P.deps.size());
          P.deps.insert(P.deps.end(), dl.begin(), dl.end());
        }
        const int split = op.kind == DK_GEMM ? op.gd.split_k : 1;
        for (int mt = r.m0; mt < r.m1; ++mt)
          for (int ntile = r.n0; ntile < r.n1; ++ntile)
            for (int ks = 0; ks < split; ++ks) {
              Item it;
              std::memset(&it, 0, sizeof it);
              it.op = T.op_base + static_cast<int>(f);
              it.mt = mt; it.nt = ntile; it.ks = ks;
              it.dep_begin = dep_begin;
              it.dep_count = static_cast<int>(dl.size());
              if (dl.size() <= static_cast<size_t>(INLINE_DEPS))
                for (size_t d = 0; d < dl.size(); ++d) { it.dc[d] = dl[d].counter; it.dt[d] = dl[d].target; }
              it.chunk = r.counter;
              it.bud = -1;
              it.cluster = k;
              it.prio = rank[t][f];
              it.kind = op.kind;
              seg_items[t][k].push_back(static_cast<int32_t>(P.items.size()));
              P.items.push_back(it);
              P.cluster_total[k] += 1;
            }
      }
      continue;
    }
    for (size_t f = 0; f < T.fops.size(); ++f) {
      const FusedOp& F = T.fops[f];
      const int k = P.fop_cluster[t][f];
      const int split = (F.kind == DK_GEMM) ? F.split_k : 1;
      for (const ChunkRange& r : cr[t][f]) {
        if (!r.n_items) continue;
        uint32_t jchunk = 0;   // position of the next item within its chunk (queue order)
        for (int mt = r.m0; mt < r.m1; ++mt)
          for (int ntile = r.n0; ntile < r.n1; ++ntile) {
            std::set<int> dset;
            std::vector<Dep> dl;
            std::vector<int> full_extra;   // WAR deps pruned as implied (still implied by this item)
            if (F.in_t == 0) dl.push_back({P.input_counter0 + t, 1u});   // input gate (epoch-valued)
            for (int tin : {F.in_t, F.skip_t}) {
              if (tin < 0 || tin == 0) continue;
              const long long XHW = static_cast<long long>(T.tensors[tin].H) * T.tensors[tin].W;
              long long lo, hi;
              tile_read_rows(T, F, mt, ntile, tin, lo, hi);
              for (int w : T.tensors[tin].writers) {
                const FusedOp& Wf = T.fops[w];
                int wm0 = 0, wm1 = Wf.tiles_m, wn0 = 0, wn1 = Wf.tiles_n;
                if (Wf.rows_are_pixels) {
                  // producer rows are tin's pixels (or samples for GAP, XHW == 1)
                  wm0 = static_cast<int>(lo / Wf.bm);
                  wm1 = static_cast<int>(hi / Wf.bm) + 1;
                } else {
                  wn0 = static_cast<int>((lo / XHW) / Wf.bn);
                  wn1 = static_cast<int>((hi / XHW) / Wf.bn) + 1;
                }
                for (const ChunkRange& q : cr[t][w]) {
                  if (!q.n_items) continue;
                  if (q.m1 <= wm0 || q.m0 >= wm1 || q.n1 <= wn0 || q.n0 >= wn1) continue;
                  if (q.mc.empty()) {
                    if (dset.insert(q.counter).second) dl.push_back({q.counter, q.n_items});
                  } else {
                    for (int pm = std::max(q.m0, wm0); pm < std::min(q.m1, wm1); ++pm) {
                      const int c = q.mc[pm - q.m0];
                      if (dset.insert(c).second) dl.push_back({c, q.mc_items});
                    }
                  }
                }
              }
            }
            {
              std::vector<Dep> wl;
              war_deps(t, F, mt, ntile, dset, wl);
              if (!wl.empty()) {
                // drop write-after-read deps already implied by the RAW deps
                // (completion of a counter implies completion of every dep of
                // its items: closure over cdeps, a few levels deep)
                std::set<int> cl(dset.begin(), dset.end());
                std::vector<int> frontier(dset.begin(), dset.end());
                for (int depth = 0; depth < 2 && !frontier.empty() && cl.size() < 256; ++depth) {
                  std::vector<int> nxt;
                  for (int c : frontier)
                    if (c >= 0 && c < static_cast<int>(cdeps.size()))
                      for (int c2 : cdeps[c])
                        if (cl.insert(c2).second) nxt.push_back(c2);
                  frontier.swap(nxt);
                }
                for (const Dep& d : wl) {
                  full_extra.push_back(d.counter);
                  if (!cl.count(d.counter) && dset.insert(d.counter).second) dl.push_back(d);
                }
              }
            }
            int dep_begin = 0;
            if (dl.size() > static_cast<size_t>(INLINE_DEPS)) {
              dep_begin = static_cast<int>(P.deps.size());
              P.deps.insert(P.deps.end(), dl.begin(), dl.end());
            }
            for (int ks = 0; ks < split; ++ks) {
              Item it;
              std::memset(&it, 0, sizeof it);
              it.op = T.op_base + static_cast<int>(f);
              it.mt = mt; it.nt = ntile; it.ks = ks;
              it.dep_begin = dep_begin;
              it.dep_count = static_cast<int>(dl.size());
              if (dl.size() <= static_cast<size_t>(INLINE_DEPS))
                for (size_t d = 0; d < dl.size(); ++d) { it.dc[d] = dl[d].counter; it.dt[d] = dl[d].target; }
              it.chunk = r.mc.empty() ? r.counter : r.mc[mt - r.m0];
              if (ks == 0) {
                std::vector<int>& cd = cdeps[it.chunk];
                for (const Dep& d : dl) cd.push_back(d.counter);
                cd.insert(cd.end(), full_extra.begin(), full_extra.end());
                std::sort(cd.begin(), cd.end());
                cd.erase(std::unique(cd.begin(), cd.end()), cd.end());
              }
              it.bud = -1;
              if (r.bud >= 0) {   // every item of the chunk counts; item j >= budget waits
                it.bud = r.bud;
                it.btot = r.n_items;
                it.boff = jchunk >= static_cast<uint32_t>(r.budget) ? jchunk - static_cast<uint32_t>(r.budget) + 1u : 0u;
              }
              ++jchunk;
              it.cluster = k;
              it.prio = rank[t][f];
              it.kind = F.kind;
              seg_items[t][k].push_back(static_cast<int32_t>(P.items.size()));
              P.items.push_back(it);
              P.cluster_total[k] += 1;
            }
          }
      }
    }
  }
  // store the items in queue order: segment (tenant, cluster) after segment
  P.segs.assign(static_cast<size_t>(nt) * P.n_clusters, Seg{0, 0});
  std::vector<Item> ordered;
  ordered.reserve(P.items.size());
  for (int t = 0; t < nt; ++t)
    for (int k = 0; k < P.n_clusters; ++k) {
      Seg& sg = P.segs[static_cast<size_t>(t) * P.n_clusters + k];
      sg.begin = static_cast<int>(ordered.size());
      sg.size = static_cast<int>(seg_items[t][k].size());
      for (int32_t i : seg_items[t][k]) {
        ordered.push_back(P.items[i]);
        ordered.back().idx = static_cast<int32_t>(ordered.size() - 1);
      }
      int run = 0;  // op_left: items of the same op that follow in the segment
      for (int i = static_cast<int>(ordered.size()) - 1; i >= sg.begin; --i) {
        run = (i + 1 < static_cast<int>(ordered.size()) && i + 1 < sg.begin + sg.size &&
               ordered[i + 1].op == ordered[i].op) ? run + 1 : 0;
        ordered[i].op_left = run;
      }
    }
  P.items = std::move(ordered);
  if (env_flag("GACER_DEP_STATS")) {   // diagnostics: dependency-list lengths per tenant
    for (int t = 0; t < nt; ++t) {
      long long n = 0, tot = 0, over = 0;
      int mx = 0;
      for (const Item& it : P.items) {
        if (it.op < S.tenants[t].op_base || it.op >= S.tenants[t].op_base + static_cast<int>(S.tenants[t].fops.size()))
          continue;
        ++n; tot += it.dep_count; over += it.dep_count > INLINE_DEPS; mx = std::max(mx, it.dep_count);
      }
      fprintf(stderr, "[gacer] tenant %d: %lld items, mean deps %.2f, max %d, over inline %lld\n", t, n,
              n ? static_cast<double>(tot) / n : 0.0, mx, over);
    }
  }
  return 0;
}

// SM partition: CTA c prefers tenant own[c]; tenant shares are the plan's
// (gacer_set_sm_shares) or, by default, each tenant's SM need -- work divided
// by chain latency, the resource share W of §4.1 l.597-601 -- normalised;
// every tenant gets at least one CTA.
std::vector<int32_t> make_pref(int grid) {
  const int nt = static_cast<int>(S.tenants.size());
  std::vector<double> w(nt);
  double tot = 0;
  for (int t = 0; t < nt; ++t) {
    w[t] = (static_cast<int>(S.user_share.size()) == nt) ? S.user_share[t] : S.plan.auto_share[t];
    w[t] = std::max(w[t], 1e-6);
    tot += w[t];
  }
  std::vector<int> own(grid);
  std::vector<double> got(nt, 0.0);
  for (int c = 0; c < grid; ++c) {  // largest deficit first (weighted round robin)
    int best = 0;
    double bd = -1e300;
    for (int t = 0; t < nt; ++t) {
      const double deficit = w[t] / tot * (c + 1) - got[t];
      if (deficit > bd) { bd = deficit; best = t; }
    }
    own[c] = best;
    got[best] += 1.0;
  }
  for (int t = 0; t < nt && nt <= grid; ++t)  // at least one CTA per tenant
    if (got[t] < 1.0) {
      int donor = 0;
      for (int u = 1; u < nt; ++u) if (got[u] > got[donor]) donor = u;
      for (int c = grid - 1; c >= 0; --c)
        if (own[c] == donor) { own[c] = t; got[t] += 1; got[donor] -= 1; break; }
    }
  int bulk = 0;
  for (int t = 1; t < nt; ++t) if (w[t] > w[bulk]) bulk = t;
  std::vector<int32_t> pref(static_cast<size_t>(grid) * nt, -1);
  for (int c = 0; c < grid; ++c) {
    pref[static_cast<size_t>(c) * nt] = own[c];
    if (S.opts.partition == GACER_PARTITION_STRICT) continue;
    int j = 1;
    for (int d = 1; d < nt; ++d) {
      const int t = (own[c] + d) % nt;
      if (S.opts.partition == GACER_PARTITION_HYBRID && own[c] != bulk && t == bulk) continue;
      pref[static_cast<size_t>(c) * nt + j++] = t;
    }
  }
  return pref;
}

int upload_plan() {
  if (S.host_only) return 0;
  Plan& P = S.plan;
  S.grid = S.opts.num_ctas > 0 ? S.opts.num_ctas : S.num_sms;
  std::vector<int32_t> pref = make_pref(S.grid);
  const size_t nheads = static_cast<size_t>(S.tenants.size()) * P.n_clusters;
  int rc;
  if ((rc = dev_upload(&S.d_items, P.items.data(), P.items.size()))) return rc;
  if ((rc = dev_upload(&S.d_deps, P.deps.data(), std::max<size_t>(1, P.deps.size())))) return rc;
  if ((rc = dev_upload(&S.d_segs, P.segs.data(), P.segs.size()))) return rc;
  if ((rc = dev_upload(&S.d_pref, pref.data(), pref.size()))) return rc;
  if ((rc = dev_upload<uint32_t>(&S.d_heads, nullptr, nheads))) return rc;
  if ((rc = dev_upload<uint32_t>(&S.d_chunk_done, nullptr, std::max(1, P.n_chunk_counters)))) return rc;
  if ((rc = dev_upload<uint32_t>(&S.d_cluster_done, nullptr, P.n_clusters))) return rc;
  if ((rc = dev_upload(&S.d_cluster_total, P.cluster_total.data(), P.cluster_total.size()))) return rc;
  if (!S.d_exit && (rc = dev_upload<uint32_t>(&S.d_exit, nullptr, 1))) return rc;
  if (!S.d_error && (rc = dev_upload<int32_t>(&S.d_error, nullptr, 1))) return rc;
  if (!S.d_stats && (rc = dev_upload<unsigned long long>(&S.d_stats, nullptr, STAT_TENANTS + 2))) return rc;
  S.stats_prev.assign(STAT_TENANTS + 2, 0);
  CUDA_TRY(cudaMemset(S.d_stats, 0, (STAT_TENANTS + 2) * sizeof(unsigned long long)));
  S.stat_rounds = 0;
  if (S.d_trace) { cudaFree(S.d_trace); S.d_trace = nullptr; }
  if (S.opts.trace) {
    CUDA_TRY(cudaMalloc(&S.d_trace, P.items.size() * TRACE_FIELDS * sizeof(int64_t)));
    CUDA_TRY(cudaMemset(S.d_trace, 0, P.items.size() * TRACE_FIELDS * sizeof(int64_t)));
  }
  S.epoch = 0;
  return 0;
}

int reset_device_counters() {
  const Plan& P = S.plan;
  // rounds may still be in flight on any stream (gacer_run_round_async takes
  // the caller's non-blocking stream): drain the device before zeroing the
  // counters they are using (rare: once per ~2^31 / items rounds, and after a
  // watchdog abort)
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemset(S.d_heads, 0, S.tenants.size() * P.n_clusters * sizeof(uint32_t)));
  CUDA_TRY(cudaMemset(S.d_chunk_done, 0, std::max(1, P.n_chunk_counters) * sizeof(uint32_t)));
  CUDA_TRY(cudaMemset(S.d_cluster_done, 0, P.n_clusters * sizeof(uint32_t)));
  CUDA_TRY(cudaMemset(S.d_exit, 0, sizeof(uint32_t)));
  CUDA_TRY(cudaMemset(S.d_error, 0, sizeof(int32_t)));
  for (Tenant& T : S.tenants)
    for (FusedOp& F : T.fops)
      if (F.d_tile_cnt) CUDA_TRY(cudaMemset(F.d_tile_cnt, 0, sizeof(uint32_t) * F.tiles_m * F.tiles_n));
  S.epoch = 0;
  return 0;
}

int check_ready() {
  if (!S.inited) return set_err(GACER_E_STATE, "gacer_init not called");
  if (S.sticky_cuda) return set_err(GACER_E_CUDA, "sticky CUDA error: %s", g_err.c_str());
  if (S.host_only) return set_err(GACER_E_STATE, "host-only instance cannot run rounds");
  if (S.tenants.empty()) return set_err(GACER_E_STATE, "no tenants registered");
  for (size_t t = 0; t < S.tenants.size(); ++t)
    if (!S.tenants[t].in_dev || !S.tenants[t].out_dev || (S.tenants[t].train && !S.tenants[t].labels_dev))
      return set_err(GACER_E_STATE, "tenant %zu has unbound I/O%s", t, S.tenants[t].train ? " or labels" : "");
  return 0;
}

// keep epoch*target far from 32-bit wrap (called before a round's epoch is used)
int maybe_reset_epoch() {
  if (S.epoch >= 0x7FFFFF00u / std::max<uint32_t>(1, 1 + static_cast<uint32_t>(S.plan.items.size())))
    return reset_device_counters();
  return 0;
}

int enqueue_round(cudaStream_t st, bool record_events = true, bool gates_written = false) {
  if (int rc = check_ready()) return rc;
  if (!st) st = S.stream;
  if (record_events) CUDA_TRY(cudaEventRecord(S.ev0, st));
  int launches = 0;
  ++S.round_no;
  if (S.mode == GACER_MODE_EXECUTOR) {
    if (!gates_written) {
      if (int rc = maybe_reset_epoch()) return rc;
    }
    ExecParams p;
    std::memset(&p, 0, sizeof p);
    p.ops = S.d_ops; p.items = S.d_items; p.deps = S.d_deps; p.segs = S.d_segs;
    p.cta_pref = S.d_pref; p.heads = S.d_heads; p.chunk_done = S.d_chunk_done;
    p.cluster_done = S.d_cluster_done; p.cluster_total = S.d_cluster_total; p.exit_count = S.d_exit;
    p.error = S.d_error; p.trace = S.d_trace; p.stats = env_flag("GACER_NO_STATS") ? nullptr : S.d_stats;
    p.n_tenants = static_cast<int>(S.tenants.size());
    p.n_clusters = S.plan.n_clusters;
    p.epoch = ++S.epoch;
    ++S.stat_rounds;
    p.n_heads = p.n_tenants * p.n_clusters;
    p.watchdog_ns = static_cast<int64_t>(S.opts.watchdog_ms > 0 ? S.opts.watchdog_ms : 2000) * 1000000LL;
    p.single_op = -1;
    p.own_first = S.opts.partition == GACER_PARTITION_PRIORITY ? 0 : 1;
    p.claim_ahead = claim_ahead_enabled();
    p.n_counters = std::max(1, S.plan.n_chunk_counters);
    p.dbg = S.d_dbg;
    if (const char* e = getenv("GACER_DBG_SPIN")) p.dbg_spin = atoll(e);
    p.k_first = 0;
    p.k_last = p.n_clusters - 1;
    p.gate0 = S.plan.input_counter0;
    p.n_gates = static_cast<int32_t>(S.tenants.size());
    p.self_gates = gates_written ? 0 : 1;   // device-resident inputs: the kernel opens its gates
    CUDA_TRY(launch_executor(p, S.grid, st, has_train_tenant()));
    launches = 1;
  } else if (S.mode == GACER_MODE_EXECUTOR_HOSTSYNC) {
    // the paper's pointer mechanics (Fig. 6, Eq. 8): each cluster is issued
    // separately and the CPU waits for the GPU at every pointer before it
    // issues the next cluster -- the GPU idles for T_SW per pointer
    if (!gates_written) {
      if (int rc = maybe_reset_epoch()) return rc;
    }
    ExecParams p;
    std::memset(&p, 0, sizeof p);
    p.ops = S.d_ops; p.items = S.d_items; p.deps = S.d_deps; p.segs = S.d_segs;
    p.cta_pref = S.d_pref; p.heads = S.d_heads; p.chunk_done = S.d_chunk_done;
    p.cluster_done = S.d_cluster_done; p.cluster_total = S.d_cluster_total; p.exit_count = S.d_exit;
    p.error = S.d_error; p.trace = S.d_trace; p.stats = env_flag("GACER_NO_STATS") ? nullptr : S.d_stats;
    p.n_tenants = static_cast<int>(S.tenants.size());
    p.n_clusters = S.plan.n_clusters;
    p.epoch = ++S.epoch;
    ++S.stat_rounds;
    p.n_heads = p.n_tenants * p.n_clusters;
    p.watchdog_ns = static_cast<int64_t>(S.opts.watchdog_ms > 0 ? S.opts.watchdog_ms : 2000) * 1000000LL;
    p.single_op = -1;
    p.own_first = S.opts.partition == GACER_PARTITION_PRIORITY ? 0 : 1;
    p.claim_ahead = claim_ahead_enabled();
    p.n_counters = std::max(1, S.plan.n_chunk_counters);
    p.gate0 = S.plan.input_counter0;
    p.n_gates = static_cast<int32_t>(S.tenants.size());
    bool first = true;
    for (int k = 0; k < p.n_clusters; ++k) {
      if (S.plan.cluster_total[k] == 0) continue;   // empty segment: nothing to issue
      p.self_gates = (!gates_written && first) ? 1 : 0;   // the first launch opens the input gates
      first = false;
      p.k_first = p.k_last = k;
      CUDA_TRY(launch_executor(p, S.grid, st, has_train_tenant()));
      ++launches;
      if (k + 1 < p.n_clusters) CUDA_TRY(cudaStreamSynchronize(st));   // the CPU-side pointer
    }
  } else {
    const bool ms = S.mode == GACER_MODE_MULTISTREAM;
    if (ms) {
      while (S.tstreams.size() < S.tenants.size()) {
        cudaStream_t s;
        cudaEvent_t e;
        CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        S.tstreams.push_back(s);
        S.tjoin.push_back(e);
      }
      if (!S.ev_fork) CUDA_TRY(cudaEventCreateWithFlags(&S.ev_fork, cudaEventDisableTiming));
      CUDA_TRY(cudaEventRecord(S.ev_fork, st));   // fork: also joins the streams into a graph capture
    }
    for (size_t t = 0; t < S.tenants.size(); ++t) {
      cudaStream_t ts = st;
      if (ms) {
        ts = S.tstreams[t];
        CUDA_TRY(cudaStreamWaitEvent(ts, S.ev_fork, 0));
      }
      const Tenant& T = S.tenants[t];
      const size_t n_ops = T.train ? T.tops.size() : T.fops.size();
      for (size_t f = 0; f < n_ops; ++f) {
        int kind, nb;
        if (T.train && T.grad_gate && T.tops[f].kind == DK_VGRID && T.tops[f].vfn == VF_SGD) {
          // A12 in a baseline round: the gradients are complete here; the
          // update waits until the communication stream has reduced them
          CUDA_TRY(cudaEventRecord(S.bwd_event[t], ts));
          if (g_wait_value32(reinterpret_cast<CUstream>(ts), reinterpret_cast<CUdeviceptr>(S.d_bgate + t),
                             S.round_no, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
            return set_err(GACER_E_CUDA, "cuStreamWaitValue32 failed");
        }
        if (T.train) {
          kind = T.tops[f].kind;
          nb = T.tops[f].items;
        } else {
          const FusedOp& F = T.fops[f];
          kind = F.kind;
          nb = F.tiles_m * F.tiles_n * (F.kind == DK_GEMM ? F.split_k : 1);
        }
        ExecParams base;
        std::memset(&base, 0, sizeof base);
        base.error = S.d_error;
        base.watchdog_ns = 2000000000LL;
        base.dbg = S.d_dbg;
        if (const char* e = getenv("GACER_DBG_SPIN")) base.dbg_spin = atoll(e);
        CUDA_TRY(launch_op(base, S.d_ops, T.op_base + static_cast<int>(f), kind, nb, S.num_sms, ts));
        ++launches;
      }
    }
    if (ms) {
      for (size_t t = 0; t < S.tenants.size(); ++t) {
        CUDA_TRY(cudaEventRecord(S.tjoin[t], S.tstreams[t]));
        CUDA_TRY(cudaStreamWaitEvent(st, S.tjoin[t], 0));
      }
    }
  }
  if (record_events) CUDA_TRY(cudaEventRecord(S.ev1, st));
  S.last_launches = launches;
  return 0;
}

int finish_round() {
  CUDA_TRY(cudaEventSynchronize(S.ev1));
  float ms = 0;
  CUDA_TRY(cudaEventElapsedTime(&ms, S.ev0, S.ev1));
  S.last_ms = ms;
  if (S.mode == GACER_MODE_EXECUTOR) {
    int32_t err = 0;
    CUDA_TRY(cudaMemcpy(&err, S.d_error, sizeof err, cudaMemcpyDeviceToHost));
    if (err) {
      reset_device_counters();
      return set_err(GACER_E_DEADLOCK, "device watchdog fired (spin budget exceeded)");
    }
  }
  return 0;
}

void free_plan_device() {
  for (void* p : {static_cast<void*>(S.d_items), static_cast<void*>(S.d_deps), static_cast<void*>(S.d_queue),
                  static_cast<void*>(S.d_segs), static_cast<void*>(S.d_pref), static_cast<void*>(S.d_heads),
                  static_cast<void*>(S.d_chunk_done), static_cast<void*>(S.d_cluster_done),
                  static_cast<void*>(S.d_cluster_total), static_cast<void*>(S.d_exit),
                  static_cast<void*>(S.d_error), static_cast<void*>(S.d_trace), static_cast<void*>(S.d_stats)})
    if (p) cudaFree(p);
  S.d_stats = nullptr;
  S.d_items = nullptr; S.d_deps = nullptr; S.d_queue = nullptr; S.d_segs = nullptr; S.d_pref = nullptr;
  S.d_heads = nullptr; S.d_chunk_done = nullptr; S.d_cluster_done = nullptr; S.d_cluster_total = nullptr;
  S.d_exit = nullptr; S.d_error = nullptr; S.d_trace = nullptr;
}

}  // namespace

// ========================================================================
// C ABI
// ========================================================================
extern "C" {

int gacer_init(int cuda_device, const gacer_options* opts) {
  if (S.inited) gacer_shutdown();
  S = State();
  if (opts) S.opts = *opts;
  if (S.opts.partition < GACER_PARTITION_PRIORITY || S.opts.partition > GACER_PARTITION_HYBRID) {
    const int bad = S.opts.partition;
    S = State();
    return set_err(GACER_E_INVALID_ARG, "unknown partition mode %d", bad);
  }
  S.host_only = cuda_device < 0;
  S.device = cuda_device;
  S.inited = true;
  if (!S.host_only) {
    CUDA_TRY(cudaSetDevice(cuda_device));
    CUDA_TRY(cudaDeviceGetAttribute(&S.num_sms, cudaDevAttrMultiProcessorCount, cuda_device));
    int major = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, cuda_device));
    if (major != 10) {
      S.inited = false;
      return set_err(GACER_E_CUDA, "device %d is sm_%d0, this library is built for sm_100a", cuda_device, major);
    }
    CUDA_TRY(configure_kernels());
    if (const char* e = getenv("GACER_DEBUG_TIMING"); e && e[0] == '1') {
      S.n_dbg = static_cast<size_t>(512) * 148 * DBG_EVENTS;   // up to 512 ops x 148 CTAs
      CUDA_TRY(cudaMalloc(&S.d_dbg, S.n_dbg * sizeof(int64_t)));
      CUDA_TRY(cudaMemset(S.d_dbg, 0, S.n_dbg * sizeof(int64_t)));
    }
    CUDA_TRY(cudaStreamCreateWithFlags(&S.stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreate(&S.ev0));
    CUDA_TRY(cudaEventCreate(&S.ev1));
  }
  return GACER_OK;
}

int gacer_shutdown(void) {
  if (!S.inited) return GACER_OK;
  if (!S.host_only) {
    cudaDeviceSynchronize();
    for (Tenant& T : S.tenants) free_tenant(T);
    free_plan_device();
    if (S.d_ops) cudaFree(S.d_ops);
    if (S.d_tmaps) cudaFree(S.d_tmaps);
    for (cudaStream_t s : S.tstreams) cudaStreamDestroy(s);
    for (cudaEvent_t e : S.tjoin) cudaEventDestroy(e);
    if (S.ev_fork) cudaEventDestroy(S.ev_fork);
    if (S.base_graph) cudaGraphExecDestroy(S.base_graph);
    if (S.stream) cudaStreamDestroy(S.stream);
    if (S.copy_stream) cudaStreamDestroy(S.copy_stream);
    S.copy_stream = nullptr;
    if (S.ev0) cudaEventDestroy(S.ev0);
    if (S.ev1) cudaEventDestroy(S.ev1);
    if (S.d_ones) cudaFree(S.d_ones);
    if (S.d_zeros) cudaFree(S.d_zeros);
  }
  S = State();
  return GACER_OK;
}

int gacer_register_tenant(const gacer_graph* graph, int32_t batch) {
  if (!S.inited) return set_err(GACER_E_STATE, "gacer_init not called");
  if (S.sticky_cuda) return set_err(GACER_E_CUDA, "sticky CUDA error");
  if (!graph) return set_err(GACER_E_INVALID_ARG, "graph is NULL");
  Tenant T;
  if (int rc = lower_tenant(graph, batch, T)) return rc;
  if (!S.host_only) {
    if (int rc = upload_tenant(T)) { free_tenant(T); return rc; }
  }
  S.tenants.push_back(std::move(T));
  const int id = static_cast<int>(S.tenants.size()) - 1;
  if (int rc = rebuild_op_table()) return rc;
  // registration resets the plan to the identity plan
  S.plan = Plan();
  S.user_share.clear();
  if (int rc = compile_plan(S.plan)) return rc;
  if (int rc = upload_plan()) return rc;
  return id;
}

int gacer_get_tenant_info(int tenant, gacer_tenant_info* out) {
  if (!S.inited) return set_err(GACER_E_STATE, "gacer_init not called");
  if (tenant < 0 || tenant >= static_cast<int>(S.tenants.size()) || !out)
    return set_err(GACER_E_INVALID_ARG, "bad tenant id %d", tenant);
  const Tenant& T = S.tenants[tenant];
  out->n_orig_ops = T.n_orig;
  out->n_fused_ops = static_cast<int32_t>(T.train ? T.tops.size() : T.fops.size());
  out->batch = T.batch;
  out->in_c_pad = T.in_c_pad;
  out->in_h = T.in_h;
  out->in_w = T.in_w;
  out->out_features = T.out_features;
  out->in_bytes = static_cast<int64_t>(T.batch) * T.in_h * T.in_w * T.in_c_pad * elem_size(T);
  out->out_bytes = static_cast<int64_t>(T.batch) * T.out_features * 4;
  out->flops = T.flops;
  out->gemm_ops = out->mpair_ops = out->split_k_ops = out->swap_ops = out->wide_ops = out->cc_ops = 0;
  out->train = T.train ? 1 : 0;
  out->n_steps = T.n_steps;
  out->n_params = T.train ? static_cast<int64_t>(T.tbuf_bytes[T.buf_params] / 4) : 0;
  out->op_base = T.op_base;
  out->reused_tensors = 0;
  out->act_bytes = out->act_bytes_private = 0;
  for (size_t b = 0; b < T.buf_bytes.size(); ++b) out->act_bytes += static_cast<int64_t>(T.buf_bytes[b]);
  for (size_t t = 1; t < T.tensors.size(); ++t) {
    const Tensor& X = T.tensors[t];
    out->reused_tensors += X.war_prev.empty() ? 0 : 1;
    if (X.buf >= 0 && !X.sliced)
      out->act_bytes_private += static_cast<int64_t>(T.batch) * X.H * X.W * X.ldc * static_cast<int64_t>(elem_size(T));
  }
  for (const TrainOp& op : T.tops) {
    if (op.kind != DK_GEMM) { ++out->cc_ops; continue; }
    ++out->gemm_ops;
    out->split_k_ops += op.gd.split_k > 1;
    out->wide_ops += op.gd.bn > 128;
  }
  for (const FusedOp& F : T.fops) {
    if (F.kind != DK_GEMM) { ++out->cc_ops; continue; }
    ++out->gemm_ops;
    out->mpair_ops += F.mrep > 1;
    out->split_k_ops += F.split_k > 1;
    out->swap_ops += F.swap;
    out->wide_ops += F.bn > 128;
  }
  return GACER_OK;
}

int gacer_bind_io(int tenant, const void* input_dev, void* output_dev) {
  if (!S.inited) return set_err(GACER_E_STATE, "gacer_init not called");
  if (tenant < 0 || tenant >= static_cast<int>(S.tenants.size()))
    return set_err(GACER_E_INVALID_ARG, "bad tenant id %d", tenant);
  if (!input_dev || !output_dev) return set_err(GACER_E_INVALID_ARG, "NULL buffer");
  if ((reinterpret_cast<uintptr_t>(input_dev) | reinterpret_cast<uintptr_t>(output_dev)) & 15)
    return set_err(GACER_E_INVALID_ARG, "buffers must be 16-byte aligned");
  S.tenants[tenant].in_dev = input_dev;
  S.tenants[tenant].out_dev = output_dev;
  return rebuild_op_table();
}

int gacer_bind_labels(int tenant, const void* labels_dev) {
  if (!S.inited) return set_err(GACER_E_STATE, "gacer_init not called");
  if (tenant < 0 || tenant >= static_cast<int>(S.tenants.size()))
    return set_err(GACER_E_INVALID_ARG, "bad tenant id %d", tenant);
  if (!S.tenants[tenant].train) return set_err(GACER_E_INVALID_ARG, "tenant %d is not a training tenant", tenant);
  if (!labels_dev || (reinterpret_cast<uintptr_t>(labels_dev) & 3)) return set_err(GACER_E_INVALID_ARG, "bad labels buffer");
  S.tenants[tenant].labels_dev = labels_dev;
  return rebuild_op_table();
}

int gacer_get_train_state(int tenant, gacer_train_state* out) {
  if (!S.inited) return set_err(GACER_E_STATE, "gacer_init not called");
  if (tenant < 0 || tenant >= static_cast<int>(S.tenants.size()) || !out)
    return set_err(GACER_E_INVALID_ARG, "bad tenant id %d", tenant);
  const Tenant& T = S.tenants[tenant];
  if (!T.train) return set_err(GACER_E_INVALID_ARG, "tenant %d is not a training tenant", tenant);
  std::memset(out, 0, sizeof *out);
  out->n_params = static_cast<int64_t>(T.tbuf_bytes[T.buf_params] / 4);
  out->n_ops = static_cast<int32_t>(T.tops.size());
  if (S.host_only) return GACER_OK;
  out->loss = static_cast<const float*>(T.tbufs[T.buf_loss]);
  out->params = static_cast<float*>(T.tbufs[T.buf_params]);
  out->grads = static_cast<const float*>(T.tbufs[T.buf_grads]);
  out->momentum = static_cast<float*>(T.tbufs[T.buf_mom]);
  return GACER_OK;
}

int gacer_train_param(int tenant, int32_t op_index, int32_t which, int64_t* offset, int64_t* count) {
  if (!S.inited) return set_err(GACER_E_STATE, "gacer_init not called");
  if (tenant < 0 || tenant >= static_cast<int>(S.tenants.size()) || !offset || !count)
    return set_err(GACER_E_INVALID_ARG, "bad arguments");
  const Tenant& T = S.tenants[tenant];
  auto it = T.param_slice.find({op_index - 1, which});
  if (!T.train || op_index < 1 || it == T.param_slice.end())
    return set_err(GACER_E_INVALID_ARG, "op %d of tenant %d has no parameter %d", op_index, tenant, which);
  *offset = it->second.first;
  *count = it->second.second;
  return GACER_OK;
}

// ---- A12: the data-parallel gradient exchange of a training tenant
int gacer_train_set_allreduce(int tenant, int32_t enable) {
  if (!S.inited) return set_err(GACER_E_STATE, "gacer_init not called");
  if (tenant < 0 || tenant >= static_cast<int>(S.tenants.size()) || !S.tenants[tenant].train)
    return set_err(GACER_E_INVALID_ARG, "tenant %d is not a training tenant", tenant);
  Tenant& T = S.tenants[tenant];
  if (T.grad_gate == (enable != 0)) return GACER_OK;
  if (!S.host_only) {
    CUDA_TRY(cudaDeviceSynchronize());
    if (!S.d_bgate) {
      CUDA_TRY(cudaMalloc(&S.d_bgate, 64 * sizeof(uint32_t)));
      CUDA_TRY(cudaMemset(S.d_bgate, 0, 64 * sizeof(uint32_t)));
    }
    while (S.bwd_event.size() < S.tenants.size()) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      S.bwd_event.push_back(e);
    }
  }
  if (tenant >= 64) return set_err(GACER_E_INVALID_ARG, "at most 64 tenants with a gradient gate");
  T.grad_gate = enable != 0;
  Plan P;                      // recompile the current plan with / without the gate
  P.cuts = S.plan.cuts;
  P.chunks = S.plan.chunks;
  if (int rc = compile_plan(P)) return rc;
  S.plan = std::move(P);
  return upload_plan();
}

int gacer_train_buckets(int tenant, int64_t bucket_bytes, int64_t* out, int32_t cap) {
  if (!S.inited) return set_err(GACER_E_STATE, "gacer_init not called");
  if (tenant < 0 || tenant >= static_cast<int>(S.tenants.size()) || !S.tenants[tenant].train || bucket_bytes < 4)
    return set_err(GACER_E_INVALID_ARG, "bad arguments");
  const Tenant& T = S.tenants[tenant];
  // parameter slices from the END of the flat buffer (the last layers'
  // gradients are produced first in backward), grouped while <= bucket_bytes
  std::vector<std::pair<int64_t, int64_t>> sl;
  for (const auto& kv : T.param_slice)
    if (kv.first.first >= 0) sl.push_back(kv.second);
  std::sort(sl.begin(), sl.end());
  const int64_t cap_f = std::max<int64_t>(1, bucket_bytes / 4);
  std::vector<std::pair<int64_t, int64_t>> bk;   // (offset, count)
  int64_t hi = -1, lo = -1;
  for (auto it = sl.rbegin(); it != sl.rend(); ++it) {
    const int64_t a = it->first, e = it->first + it->second;
    if (hi < 0) { lo = a; hi = e; continue; }
    if (hi - a > cap_f) { bk.push_back({lo, hi - lo}); hi = e; }
    lo = a;
  }
  if (hi >= 0) bk.push_back({lo, hi - lo});
  if (out)
    for (int b = 0; b < static_cast<int>(bk.size()) && b < cap; ++b) { out[2 * b] = bk[b].first; out[2 * b + 1] = bk[b].second; }
  return static_cast<int>(bk.size());
}

int gacer_stream_wait_grads(void* stream, int tenant, int64_t offset, int64_t count) {
  if (int rc = check_ready()) return rc;
  if (tenant < 0 || tenant >= static_cast<int>(S.tenants.size()) || !S.tenants[tenant].grad_gate)
    return set_err(GACER_E_INVALID_ARG, "tenant %d has no gradient gate (gacer_train_set_allreduce)", tenant);
  const Tenant& T = S.tenants[tenant];
  auto st = reinterpret_cast<CUstream>(stream);
  if (S.mode != GACER_MODE_EXECUTOR) {   // baselines: the backward-done event of the enqueued round
    CUDA_TRY(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), S.bwd_event[tenant], 0));
    return GACER_OK;
  }
  // executor: the completion counters of every op writing into the range
  // (a training op's items share one whole-op counter; its first item carries it)
  std::vector<int> ctr(T.tops.size(), -1);
  for (const Item& it : S.plan.items) {
    const int f = it.op - T.op_base;
    if (f >= 0 && f < static_cast<int>(ctr.size()) && ctr[f] < 0) ctr[f] = it.chunk;
  }
  for (size_t f = 0; f < T.tops.size(); ++f) {
    const TrainOp& op = T.tops[f];
    bool hit = false;
    for (const auto& r : op.grad_ranges) hit |= r.first < offset + count && r.first + r.second > offset;
    if (!hit) continue;
    if (ctr[f] < 0) return set_err(GACER_E_STATE, "gradient op %zu has no items", f);
    const uint32_t target = S.epoch * static_cast<uint32_t>(op.items);
    if (g_wait_value32(st, reinterpret_cast<CUdeviceptr>(S.d_chunk_done + ctr[f]), target,
                       CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      return set_err(GACER_E_CUDA, "cuStreamWaitValue32 failed");
  }
  return GACER_OK;
}

int gacer_stream_open_grad_gate(void* stream, int tenant) {
  if (int rc = check_ready()) return rc;
  if (tenant < 0 || tenant >= static_cast<int>(S.tenants.size()) || !S.tenants[tenant].grad_gate)
    return set_err(GACER_E_INVALID_ARG, "tenant %d has no gradient gate", tenant);
  auto st = reinterpret_cast<CUstream>(stream);
  if (g_write_value32(st, reinterpret_cast<CUdeviceptr>(S.d_chunk_done + S.plan.grad_gate0 + tenant), S.epoch, 0) !=
          CUDA_SUCCESS ||
      g_write_value32(st, reinterpret_cast<CUdeviceptr>(S.d_bgate + tenant), S.round_no, 0) != CUDA_SUCCESS)
    return set_err(GACER_E_CUDA, "cuStreamWriteValue32 failed");
  return GACER_OK;
}

int gacer_set_regulation(const gacer_decomposition* dec, const gacer_sync_pointers* sp) {
  if (!S.inited) return set_err(GACER_E_STATE, "gacer_init not called");
  if (S.sticky_cuda) return set_err(GACER_E_CUDA, "sticky CUDA error");
  const int nt = static_cast<int>(S.tenants.size());
  if (nt == 0) return set_err(GACER_E_STATE, "no tenants registered");
  Plan P;
  if (sp) {
    if (sp->n_tenants != nt) return set_err(GACER_E_INVALID_ARG, "sync_pointers for %d tenants, %d registered", sp->n_tenants, nt);
    if (sp->n_pointers < 0) return set_err(GACER_E_POINTER_COUNT_MISMATCH, "negative pointer count");
    if (sp->n_pointers > 0 && !sp->cuts) return set_err(GACER_E_INVALID_ARG, "cuts is NULL");
    P.cuts.assign(nt, {});
    for (int t = 0; t < nt; ++t) {
      int prev = 0;
      for (int j = 0; j < sp->n_pointers; ++j) {
        const int c = sp->cuts[static_cast<size_t>(t) * sp->n_pointers + j];
        // a training tenant's operator list is its step: forward 1..n,
        // backward n+1..2n (reverse order), the update 2n+1
        const int lim = S.tenants[t].train ? S.tenants[t].n_steps : S.tenants[t].n_orig;
        if (c < 0 || c > lim)
          return set_err(GACER_E_CUT_OUT_OF_RANGE, "tenant %d pointer %d = %d outside [0, %d]", t, j, c, lim);
        if (c < prev) return set_err(GACER_E_UNSORTED_CUTS, "tenant %d pointers decrease at %d", t, j);
        prev = c;
        P.cuts[t].push_back(c);
      }
    }
  }
  if (dec) {
    if (dec->n < 0 || (dec->n > 0 && !dec->items)) return set_err(GACER_E_INVALID_ARG, "bad decomposition");
    for (int i = 0; i < dec->n; ++i) {
      const gacer_chunking& c = dec->items[i];
      if (c.tenant < 0 || c.tenant >= nt) return set_err(GACER_E_INVALID_ARG, "chunking %d: bad tenant", i);
      const Tenant& T = S.tenants[c.tenant];
      if (c.op_index < 1 || c.op_index > T.n_orig) return set_err(GACER_E_INVALID_ARG, "chunking %d: bad op_index", i);
      if (c.axis == GACER_AXIS_NONE) continue;  // mask(O) = 0
      if (T.train)   // BN statistics span the whole per-replica batch
        return set_err(GACER_E_INVALID_ARG, "chunking %d: a training tenant's operators are not decomposed", i);
      if (c.axis != GACER_AXIS_BATCH && c.axis != GACER_AXIS_CHANNEL)
        return set_err(GACER_E_INVALID_ARG, "chunking %d: bad axis", i);
      if (c.n_chunks < 1 || !c.sizes)
        return set_err(GACER_E_MASKED_OP_MISSING_CHUNKS, "chunking %d: decomposed op without list", i);
      const int o = c.op_index - 1;
      if (T.orig_fused[o] < 0) return set_err(GACER_E_INVALID_ARG, "chunking %d: op %d is an alias (flatten/dropout/concat)", i, c.op_index);
      long long sum = 0;
      for (int j = 0; j < c.n_chunks; ++j) {
        if (c.sizes[j] < 1) return set_err(GACER_E_CHUNK_SUM_MISMATCH, "chunking %d: chunk size < 1", i);
        sum += c.sizes[j];
      }
      const int want = c.axis == GACER_AXIS_BATCH ? T.batch : T.orig_out_c[o];
      if (sum != want)
        return set_err(GACER_E_CHUNK_SUM_MISMATCH, "chunking %d: sizes sum to %lld, expected %d (Eq. 5)", i, sum, want);
      Chunking ch;
      ch.axis = c.axis;
      ch.sizes.assign(c.sizes, c.sizes + c.n_chunks);
      if (c.sm_budget) {
        for (int j = 0; j < c.n_chunks; ++j)
          if (c.sm_budget[j] < 0) return set_err(GACER_E_INVALID_ARG, "chunking %d: negative sm_budget", i);
        ch.budget.assign(c.sm_budget, c.sm_budget + c.n_chunks);
      }
      if (!P.chunks.emplace(std::make_pair(c.tenant, o), ch).second)
        return set_err(GACER_E_INVALID_ARG, "chunking %d: op %d decomposed twice", i, c.op_index);
    }
  }
  if (int rc = compile_plan(P)) return rc;  // previous plan untouched on error
  S.plan = std::move(P);
  return upload_plan();
}

int gacer_query_op_clusters(int tenant, int32_t* out, int32_t n) {
  if (!S.inited) return set_err(GACER_E_STATE, "gacer_init not called");
  if (tenant < 0 || tenant >= static_cast<int>(S.tenants.size()) || !out)
    return set_err(GACER_E_INVALID_ARG, "bad tenant id %d", tenant);
  const Tenant& T = S.tenants[tenant];
  const int m = std::min(n, T.train ? T.n_steps : T.n_orig);   // training tenants: per step position
  for (int i = 0; i < m; ++i) out[i] = cluster_of_orig(S.plan, tenant, i);
  return m;
}

int gacer_query_op_fused(int tenant, int32_t* out, int32_t n) {
  if (!S.inited) return set_err(GACER_E_STATE, "gacer_init not called");
  if (tenant < 0 || tenant >= static_cast<int>(S.tenants.size()) || !out)
    return set_err(GACER_E_INVALID_ARG, "bad tenant id %d", tenant);
  const Tenant& T = S.tenants[tenant];
  if (T.train) return set_err(GACER_E_INVALID_ARG, "tenant %d is a training tenant", tenant);
  const int m = std::min(n, T.n_orig);
  for (int i = 0; i < m; ++i) out[i] = T.orig_fused[i];
  return m;
}

int gacer_set_sm_shares(const float* shares, int32_t n) {
  if (!S.inited) return set_err(GACER_E_STATE, "gacer_init not called");
  if (n == 0 || !shares) {
    S.user_share.clear();
  } else {
    if (n != static_cast<int32_t>(S.tenants.size()))
      return set_err(GACER_E_INVALID_ARG, "%d shares for %zu tenants", n, S.tenants.size());
    std::vector<double> v(n);
    for (int i = 0; i < n; ++i) {
      if (!(shares[i] > 0.0f)) return set_err(GACER_E_INVALID_ARG, "share %d must be > 0", i);
      v[i] = shares[i];
    }
    S.user_share = v;
  }
  return upload_plan();
}

int gacer_set_partition(int32_t partition) {
  if (!S.inited) return set_err(GACER_E_STATE, "gacer_init not called");
  if (partition < GACER_PARTITION_PRIORITY || partition > GACER_PARTITION_HYBRID)
    return set_err(GACER_E_INVALID_ARG, "unknown partition mode %d", partition);
  S.opts.partition = partition;
  return upload_plan();
}

int gacer_set_mode(int mode) {
  if (mode != GACER_MODE_EXECUTOR && mode != GACER_MODE_SEQUENTIAL && mode != GACER_MODE_MULTISTREAM &&
      mode != GACER_MODE_EXECUTOR_HOSTSYNC)
    return set_err(GACER_E_INVALID_ARG, "bad mode %d", mode);
  S.mode = mode;
  return GACER_OK;
}

int gacer_run_round_async(void* stream) { return enqueue_round(static_cast<cudaStream_t>(stream)); }

// The sequential / multi-stream baselines as a CUDA graph: one round of the
// mode's per-op launches (same tile functions, same order, same streams
// topology) captured once and replayed, so the comparison with the
// one-launch executor is not a comparison with host launch overhead
// ("Each is reported plain and with CUDA Graphs").
int gacer_capture_baseline(int mode) {
  if (int rc = check_ready()) return rc;
  if (mode != GACER_MODE_SEQUENTIAL && mode != GACER_MODE_MULTISTREAM)
    return set_err(GACER_E_INVALID_ARG, "only the sequential / multi-stream baselines are captured (mode %d)", mode);
  if (S.base_graph) { cudaGraphExecDestroy(S.base_graph); S.base_graph = nullptr; S.base_graph_mode = -1; }
  for (const Tenant& T : S.tenants)
    if (T.grad_gate)   // the round-numbered gradient gate cannot be baked into a graph
      return set_err(GACER_E_STATE, "baseline graphs are not captured with a data-parallel training tenant");
  const int saved = S.mode;
  S.mode = mode;
  CUDA_TRY(cudaStreamSynchronize(S.stream));
  CUDA_TRY(cudaStreamBeginCapture(S.stream, cudaStreamCaptureModeThreadLocal));
  const int rc = enqueue_round(S.stream, /*record_events=*/false);
  cudaGraph_t g = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(S.stream, &g);
  S.mode = saved;
  if (rc) { if (g) cudaGraphDestroy(g); return rc; }
  if (ec != cudaSuccess) return set_err(GACER_E_CUDA, "baseline capture failed: %s", cudaGetErrorString(ec));
  const cudaError_t ei = cudaGraphInstantiate(&S.base_graph, g, 0);
  cudaGraphDestroy(g);
  if (ei != cudaSuccess) return set_err(GACER_E_CUDA, "graph instantiate failed: %s", cudaGetErrorString(ei));
  S.base_graph_mode = mode;
  S.base_graph_launches = S.last_launches;
  return GACER_OK;
}

int gacer_run_baseline_graph(void* stream) {
  if (int rc = check_ready()) return rc;
  if (!S.base_graph) return set_err(GACER_E_STATE, "no captured baseline (gacer_capture_baseline)");
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : S.stream;
  CUDA_TRY(cudaEventRecord(S.ev0, st));
  CUDA_TRY(cudaGraphLaunch(S.base_graph, st));
  CUDA_TRY(cudaEventRecord(S.ev1, st));
  S.last_launches = S.base_graph_launches;
  return GACER_OK;
}

int gacer_run_round(void) {
  if (int rc = enqueue_round(S.stream)) return rc;
  return finish_round();
}

int gacer_run_round_host(const void* const* host_inputs, void* const* host_outputs) {
  if (int rc = check_ready()) return rc;
  if (!host_inputs || !host_outputs) return set_err(GACER_E_INVALID_ARG, "NULL host arrays");
  CUDA_TRY(cudaEventRecord(S.ev0, S.stream));  // the e2e time includes both copies
  const bool exec = S.mode == GACER_MODE_EXECUTOR || S.mode == GACER_MODE_EXECUTOR_HOSTSYNC;
  if (exec) {
    // executor: the input copies run on a copy stream, each followed by its
    // tenant's input gate, while the round already runs -- a tenant's first
    // items wait on the device for their own input only (copy/compute overlap)
    if (!S.copy_stream) CUDA_TRY(cudaStreamCreateWithFlags(&S.copy_stream, cudaStreamNonBlocking));
    if (int rc = maybe_reset_epoch()) return rc;
    const uint32_t ep = S.epoch + 1;
    CUDA_TRY(cudaStreamWaitEvent(S.copy_stream, S.ev0, 0));
    for (size_t t = 0; t < S.tenants.size(); ++t) {
      const Tenant& T = S.tenants[t];
      const size_t bytes = static_cast<size_t>(T.batch) * T.in_h * T.in_w * T.in_c_pad * elem_size(T);
      CUDA_TRY(cudaMemcpyAsync(const_cast<void*>(T.in_dev), host_inputs[t], bytes, cudaMemcpyHostToDevice,
                               S.copy_stream));
      const CUdeviceptr a = reinterpret_cast<CUdeviceptr>(S.d_chunk_done + S.plan.input_counter0 + t);
      if (g_write_value32(reinterpret_cast<CUstream>(S.copy_stream), a, ep, 0) != CUDA_SUCCESS)
        return set_err(GACER_E_CUDA, "cuStreamWriteValue32 failed");
    }
    if (int rc = enqueue_round(S.stream, false, true)) return rc;
    cudaEvent_t copied;   // the next round's copies must not overtake this one's reads
    CUDA_TRY(cudaEventCreateWithFlags(&copied, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(copied, S.copy_stream));
    CUDA_TRY(cudaStreamWaitEvent(S.stream, copied, 0));
    cudaEventDestroy(copied);
  } else {
    for (size_t t = 0; t < S.tenants.size(); ++t) {
      const Tenant& T = S.tenants[t];
      const size_t bytes = static_cast<size_t>(T.batch) * T.in_h * T.in_w * T.in_c_pad * elem_size(T);
      CUDA_TRY(cudaMemcpyAsync(const_cast<void*>(T.in_dev), host_inputs[t], bytes, cudaMemcpyHostToDevice, S.stream));
    }
    if (int rc = enqueue_round(S.stream, false)) return rc;
  }
  for (size_t t = 0; t < S.tenants.size(); ++t) {
    const Tenant& T = S.tenants[t];
    CUDA_TRY(cudaMemcpyAsync(host_outputs[t], T.out_dev, static_cast<size_t>(T.batch) * T.out_features * 4,
                             cudaMemcpyDeviceToHost, S.stream));
  }
  CUDA_TRY(cudaEventRecord(S.ev1, S.stream));
  return finish_round();
}

int gacer_get_stats(gacer_round_stats* out) {
  if (!S.inited) return set_err(GACER_E_STATE, "gacer_init not called");
  if (!out) return set_err(GACER_E_INVALID_ARG, "NULL");
  std::memset(out, 0, sizeof *out);
  out->last_round_ms = S.last_ms;
  out->n_items = static_cast<int64_t>(S.plan.items.size());
  out->n_clusters = S.plan.n_clusters;
  out->kernel_launches = S.last_launches;
  out->n_tenants = static_cast<int32_t>(S.tenants.size());
  for (const Tenant& T : S.tenants) {
    out->n_fused_ops += static_cast<int32_t>(T.fops.size() + T.tops.size());
    for (const TrainOp& op : T.tops) {
      if (op.kind == DK_GEMM) out->tensor_flops += op.flops;
      else out->cc_bytes += op.bytes;
    }
    for (const FusedOp& F : T.fops) {
      if (F.kind == DK_GEMM || F.kind == DK_SIMT_GEMM) out->tensor_flops += F.flops;
      else out->cc_bytes += F.bytes;
    }
  }
  if (!S.host_only && S.d_stats && S.stat_rounds > 0) {
    std::vector<unsigned long long> cur(STAT_TENANTS + 2, 0);
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpy(cur.data(), S.d_stats, cur.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    const double r = static_cast<double>(S.stat_rounds);
    out->stat_rounds = S.stat_rounds;
    for (int t = 0; t < STAT_TENANTS; ++t) out->tenant_sm_ns[t] = static_cast<double>(cur[t] - S.stats_prev[t]) / r;
    out->barrier_wait_ns = static_cast<double>(cur[STAT_TENANTS] - S.stats_prev[STAT_TENANTS]) / r;
    out->ready_wait_ns = static_cast<double>(cur[STAT_TENANTS + 1] - S.stats_prev[STAT_TENANTS + 1]) / r;
    S.stats_prev = cur;
    S.stat_rounds = 0;
  }
  return GACER_OK;
}

int gacer_get_trace(int64_t* records, int32_t cap) {
  if (!S.inited || S.host_only || !S.d_trace) return set_err(GACER_E_STATE, "tracing not enabled");
  if (!records || cap < 0) return set_err(GACER_E_INVALID_ARG, "bad buffer");
  const size_t n = std::min<size_t>(cap, S.plan.items.size());
  CUDA_TRY(cudaMemcpy(records, S.d_trace, n * TRACE_FIELDS * sizeof(int64_t), cudaMemcpyDeviceToHost));
  return static_cast<int>(n);
}

const char* gacer_last_error(void) { return g_err.c_str(); }

// Diagnostics: the lowered op `op` of the global op table (the trace's op
// field): out[0] = device kind (DK_*), [1] = virtual-grid function (VF_*),
// [2] = items per round, [3] = tenant, [4] = GEMM tile N, [5] = K-blocks.
int gacer_describe_op(int32_t op, int32_t* out) {
  if (!S.inited || !out || op < 0 || op >= static_cast<int>(S.h_ops.size()))
    return set_err(GACER_E_INVALID_ARG, "bad op index %d", op);
  const OpDev& d = S.h_ops[op];
  out[0] = d.kind;
  out[1] = d.vfn;
  out[2] = d.tiles_m * d.tiles_n * (d.kind == DK_GEMM ? d.split_k : 1);
  out[3] = d.tenant;
  out[4] = d.bn;
  out[5] = d.nkb;
  // algorithmic bytes (inputs + outputs + weights) and MFLOP of the fused op
  // (the planner's lookup table: HBM share W_bw, NEXT-3); training ops: 0
  double bytes = 0.0, flops = 0.0;
  for (const Tenant& T : S.tenants)
    if (!T.train && op >= T.op_base && op < T.op_base + static_cast<int>(T.fops.size())) {
      bytes = T.fops[op - T.op_base].bytes;
      flops = T.fops[op - T.op_base].flops;
    }
  out[6] = static_cast<int32_t>(std::min(bytes, 2147483647.0));
  out[7] = static_cast<int32_t>(std::min(flops / 1e6, 2147483647.0));
  return GACER_OK;
}

// Diagnostics (not part of the method): GACER_DEBUG_TIMING=1 milestones.
int gacer_debug_timing(int64_t* out, int64_t cap, int reset) {
  if (!S.inited || !S.d_dbg) return set_err(GACER_E_STATE, "GACER_DEBUG_TIMING not enabled");
  const size_t n = std::min<size_t>(static_cast<size_t>(cap), S.n_dbg);
  CUDA_TRY(cudaDeviceSynchronize());
  if (out) CUDA_TRY(cudaMemcpy(out, S.d_dbg, n * sizeof(int64_t), cudaMemcpyDeviceToHost));
  if (reset) CUDA_TRY(cudaMemset(S.d_dbg, 0, S.n_dbg * sizeof(int64_t)));
  return static_cast<int>(n);
}

}  // extern "C"

// Library-owned unit scale / zero bias vectors for the standalone GEMM calls
// (no folded BN): written once, grown on demand (cudaFree synchronises the
// device, so launches still reading the old vectors have finished).
namespace {
int unit_vectors(int n, const float** ones, const float** zeros) {
  if (n > S.n_unit) {
    const int m = std::max(n, 4096);
    if (S.d_ones) cudaFree(S.d_ones);
    if (S.d_zeros) cudaFree(S.d_zeros);
    S.d_ones = S.d_zeros = nullptr;
    S.n_unit = 0;
    CUDA_TRY(cudaMalloc(&S.d_ones, m * sizeof(float)));
    CUDA_TRY(cudaMalloc(&S.d_zeros, m * sizeof(float)));
    std::vector<float> h(m, 1.0f);
    CUDA_TRY(cudaMemcpy(S.d_ones, h.data(), m * sizeof(float), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemset(S.d_zeros, 0, m * sizeof(float)));
    S.n_unit = m;
  }
  *ones = S.d_ones;
  *zeros = S.d_zeros;
  return 0;
}
}  // namespace

// ------------------------------------------------------------------------
// A11: convolution data gradient on the tcgen05 implicit-GEMM path
// ------------------------------------------------------------------------
namespace {
struct DgPhaseGemm {        // one phase (a, b) of a strided conv's data gradient
  int a, b;
  DgPhase vh, vw;
  int K, Kpad, nkb, bn, tiles_m, tiles_n, rows, M, a_mode;
  int upper[2];              // explicit im2col upper corner (h, w)
  size_t off_op, off_maps, off_w, off_out;
};
struct DgradGeom {
  int cread, K, Kpad, nkb, bn, tiles_m, tiles_n, rows, M, a_mode, ph, pw, Hd, Wd, Hdd, Wdd;
  size_t off_op, off_maps, off_w, off_dil, bytes;
  // stride > 1: phase-decomposed (no zero-dilated dy): one stride-1 GEMM per
  // phase with taps, then a scatter into dx (GACER_DGRAD_DILATE=1: the
  // zero-dilated form)
  bool phased = false;
  std::vector<DgPhaseGemm> phases;
};

int dgrad_tile_bn(int Cin, int M) {
  return (Cin >= 256 && cdiv(M, BM) >= kSplitSms) ? 256 : (Cin >= 128 ? 128 : roundup(Cin, 16));
}

int dgrad_geom(int N, int H, int W, int Cin, int Cout, int KH, int KW, int stride, int pad_h, int pad_w,
               DgradGeom& g) {
  if (N < 1 || H < 1 || W < 1 || Cin < 8 || Cin % 8 || Cout < 64 || Cout % 64 || KH < 1 || KW < 1 || stride < 1 ||
      pad_h < 0 || pad_w < 0 || pad_h > KH - 1 || pad_w > KW - 1)
    return set_err(GACER_E_SHAPE, "conv_dgrad: need Cin %% 8 == 0, Cout %% 64 == 0, stride >= 1, 0 <= pad <= k-1");
  g.Hd = (H + 2 * pad_h - KH) / stride + 1;           // dy spatial size (the forward output)
  g.Wd = (W + 2 * pad_w - KW) / stride + 1;
  if (H + 2 * pad_h < KH || W + 2 * pad_w < KW) return set_err(GACER_E_SHAPE, "conv_dgrad: empty forward output");
  // stride > 1: dy zero-dilated by the stride, plus the rows/columns of x no
  // window reached ((H + 2p - K) mod S), so the stride-1 dgrad conv of the
  // dilated tensor has exactly H x W outputs
  g.Hdd = stride == 1 ? g.Hd : (g.Hd - 1) * stride + 1 + (H + 2 * pad_h - KH) % stride;
  g.Wdd = stride == 1 ? g.Wd : (g.Wd - 1) * stride + 1 + (W + 2 * pad_w - KW) % stride;
  g.ph = KH - 1 - pad_h;                              // the dgrad conv's padding
  g.pw = KW - 1 - pad_w;
  g.cread = Cout;                                     // dy channels, a multiple of 64
  g.a_mode = (KH * KW == 1 && g.ph == 0 && g.pw == 0) ? A_ROWS : A_IM2COL;
  g.K = KH * KW * g.cread;
  g.Kpad = roundup(g.K, BK);
  g.nkb = g.Kpad / BK;
  g.M = N * H * W;
  // 128x256 tiles for wide outputs (half the A-operand smem traffic per FLOP,
  // the mainloop being smem-port bound: DESIGN §4.1) when the M tiles still
  // cover the SMs
  g.bn = (Cin >= 256 && cdiv(g.M, BM) >= kSplitSms) ? 256 : (Cin >= 128 ? 128 : roundup(Cin, 16));
  g.tiles_m = cdiv(g.M, BM);
  g.tiles_n = cdiv(Cin, g.bn);
  g.rows = g.tiles_n * g.bn;
  size_t o = 0;
  auto take = [&](size_t n, size_t al) { o = (o + al - 1) / al * al; const size_t r = o; o += n; return r; };
  g.off_op = take(sizeof(OpDev), 256);
  g.off_maps = take(3 * sizeof(CUtensorMap), 128);
  g.off_w = take(static_cast<size_t>(g.rows) * g.Kpad * 2, 256);
  g.off_dil = stride == 1 ? 0 : take(static_cast<size_t>(N) * g.Hdd * g.Wdd * Cout * 2, 256);
  g.phased = false;
  g.phases.clear();
  // phases when the filter is no larger than the stride (1x1 / 2x2 at s2:
  // the dilated form would spend 3/4 of its MMA work on zeros and the phases
  // are few, dense GEMMs); larger filters keep the dilated form by default --
  // measured standalone at R50 B=64: 1x1 s2 phases 0.18 vs dilated 0.33 ms,
  // 3x3 s2 phases 0.17-0.22 vs dilated 0.12-0.18 ms (four small launches)
  // GACER_DGRAD_PHASES=1 / GACER_DGRAD_DILATE=1 force either form.
  const bool want_phases = env_flag("GACER_DGRAD_PHASES") || (KH <= stride && KW <= stride);
  if (stride > 1 && want_phases && !env_flag("GACER_DGRAD_DILATE")) {
    bool ok = true;
    for (int a = 0; a < stride && ok; ++a)
      for (int b = 0; b < stride && ok; ++b) {
        DgPhaseGemm q;
        q.a = a; q.b = b;
        q.vh = dg_phase(a, KH, stride, pad_h, H);
        q.vw = dg_phase(b, KW, stride, pad_w, W);
        if (q.vh.K == 0 || q.vw.K == 0 || q.vh.n == 0 || q.vw.n == 0) { q.K = 0; g.phases.push_back(q); continue; }
        if (q.vh.pad < 0 || q.vw.pad < 0) { ok = false; break; }
        q.K = q.vh.K * q.vw.K * Cout;
        q.Kpad = roundup(q.K, BK);
        q.nkb = q.Kpad / BK;
        q.M = N * q.vh.n * q.vw.n;
        q.a_mode = (q.vh.K * q.vw.K == 1 && q.vh.pad == 0 && q.vw.pad == 0 && q.vh.n == g.Hd && q.vw.n == g.Wd)
                       ? A_ROWS : A_IM2COL;
        q.bn = dgrad_tile_bn(Cin, q.M);
        q.tiles_m = cdiv(q.M, BM);
        q.tiles_n = cdiv(Cin, q.bn);
        q.rows = q.tiles_n * q.bn;
        q.upper[0] = q.vh.n - g.Hd - q.vh.pad;   // output rows per image = Hd + upper - lower
        q.upper[1] = q.vw.n - g.Wd - q.vw.pad;
        g.phases.push_back(q);
      }
    if (ok) {
      g.phased = true;
      for (DgPhaseGemm& q : g.phases) {
        if (q.K == 0) continue;
        q.off_op = take(sizeof(OpDev), 256);
        q.off_maps = take(3 * sizeof(CUtensorMap), 128);
        q.off_w = take(static_cast<size_t>(q.rows) * q.Kpad * 2, 256);
        q.off_out = take(static_cast<size_t>(q.M) * Cin * 2, 256);
      }
    } else {
      g.phases.clear();
    }
  }
  g.bytes = o;
  return 0;
}

// The OpDev of one phase GEMM (a stride-1 forward conv of dy with the
// phase's flipped sub-filter; dense output [N][n_a][n_b][Cin]).
void dgrad_phase_opdev(OpDev& d, const DgPhaseGemm& q, int N, int Hd, int Wd, int Cin, int Cout) {
  std::memset(&d, 0, sizeof d);
  d.kind = DK_GEMM; d.act = ACT_NONE;
  d.B = N; d.H = Hd; d.W = Wd; d.C = Cout; d.ldi = Cout;
  d.Ho = q.vh.n; d.Wo = q.vw.n; d.Cout = Cin; d.ldo = Cin;
  d.kh = q.vh.K; d.kw = q.vw.K; d.stride = 1; d.ph = q.vh.pad; d.pw = q.vw.pad; d.mrep = 1;
  d.M = q.M; d.N = Cin; d.K = q.K; d.Kpad = q.Kpad;
  d.tiles_m = q.tiles_m; d.tiles_n = q.tiles_n; d.bm = BM; d.bn = q.bn; d.split_k = 1; d.nkb = q.nkb;
  d.ldw = q.Kpad; d.a_mode = q.a_mode;
}
}  // namespace

extern "C" {

int64_t gacer_conv_dgrad_workspace(int32_t N, int32_t H, int32_t W, int32_t Cin, int32_t Cout, int32_t KH, int32_t KW,
                                   int32_t stride, int32_t pad_h, int32_t pad_w) {
  DgradGeom g;
  if (int rc = dgrad_geom(N, H, W, Cin, Cout, KH, KW, stride, pad_h, pad_w, g)) return rc;
  return static_cast<int64_t>(g.bytes);
}

int32_t gacer_conv_dgrad(const void* dy_dev, const float* w_dev, int32_t N, int32_t H, int32_t W, int32_t Cin,
                         int32_t Cout, int32_t KH, int32_t KW, int32_t stride, int32_t pad_h, int32_t pad_w,
                         void* dx_dev, void* ws_dev, int64_t ws_bytes, void* stream) {
  if (!S.inited || S.host_only) return set_err(GACER_E_STATE, "conv_dgrad: gacer_init on a device first");
  DgradGeom g;
  if (int rc = dgrad_geom(N, H, W, Cin, Cout, KH, KW, stride, pad_h, pad_w, g)) return rc;
  if (!dy_dev || !w_dev || !dx_dev || !ws_dev || ws_bytes < static_cast<int64_t>(g.bytes) ||
      (reinterpret_cast<uintptr_t>(ws_dev) & 255) || (reinterpret_cast<uintptr_t>(dy_dev) & 15) ||
      (reinterpret_cast<uintptr_t>(dx_dev) & 15))
    return set_err(GACER_E_INVALID_ARG, "conv_dgrad: null/misaligned pointer or workspace too small");
  if (int rc = load_tma_encoders()) return rc;
  if (!S.d_error) { if (int rc = dev_upload<int32_t>(&S.d_error, nullptr, 1)) return rc; }
  auto st = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(ws_dev);
  void* wt = ws + g.off_w;
  const float *scale = nullptr, *bias = nullptr;
  const int nsb = g.rows + 8;
  if (g.phased) {
    // phase decomposition: per phase with taps a stride-1 GEMM of dy with the
    // flipped sub-filter (dense output), then one scatter into dx
    const void* outs[4] = {nullptr, nullptr, nullptr, nullptr};
    for (const DgPhaseGemm& q : g.phases) {
      if (q.K == 0) continue;
      void* qw = ws + q.off_w;
      void* qo = ws + q.off_out;
      outs[q.a * stride + q.b] = qo;
      CUDA_TRY(launch_dgrad_phase_filter(w_dev, Cout, Cin, q.vh.K, q.vw.K, Cout, q.Kpad, q.rows, stride, q.a, q.b, KH,
                                         KW, qw, st));
      if (int rc0 = unit_vectors(q.rows + 8, &scale, &bias)) return rc0;
      OpDev d;
      dgrad_phase_opdev(d, q, N, g.Hd, g.Wd, Cin, Cout);
      d.in = dy_dev; d.out = qo; d.wt = qw; d.scale = scale; d.bias = bias;
      CUtensorMap maps[3];
      std::memset(maps, 0, sizeof maps);
      const CUtensorMap* dmaps = reinterpret_cast<const CUtensorMap*>(ws + q.off_maps);
      d.tmap_a = dmaps; d.tmap_b = dmaps + 1; d.tmap_c = dmaps + 2;
      int rc = q.a_mode == A_IM2COL ? encode_im2col(&maps[0], d, Cout, BM, BK, CU_TENSOR_MAP_SWIZZLE_128B, q.upper)
                                    : encode_rows(&maps[0], dy_dev, q.K, q.M, Cout, BM);
      if (!rc) rc = encode_rows(&maps[1], qw, q.Kpad, q.rows, q.Kpad, q.bn);
      if (rc) return rc;
      {
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(Cin), static_cast<cuuint64_t>(q.M)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(Cin) * 2};
        const cuuint32_t box[2] = {64u, 32u};
        const cuuint32_t es[2] = {1, 1};
        CUresult r = g_encode_tiled(&maps[2], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, qo, dims, strides, box, es,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_err(GACER_E_CUDA, "conv_dgrad: phase output map (%d)", static_cast<int>(r));
        d.c_tma = 1;
      }
      CUDA_TRY(cudaMemcpyAsync(ws + q.off_maps, maps, sizeof maps, cudaMemcpyHostToDevice, st));
      CUDA_TRY(cudaMemcpyAsync(ws + q.off_op, &d, sizeof d, cudaMemcpyHostToDevice, st));
      ExecParams base;
      std::memset(&base, 0, sizeof base);
      base.error = S.d_error;
      base.watchdog_ns = 2000000000LL;
      CUDA_TRY(launch_op(base, reinterpret_cast<const OpDev*>(ws + q.off_op), 0, DK_GEMM, q.tiles_m * q.tiles_n,
                         S.num_sms, st));
    }
    CUDA_TRY(launch_phase_scatter(outs, N, H, W, Cin, stride, pad_h, pad_w, KH, KW, dx_dev, st));
    return GACER_OK;
  }
  CUDA_TRY(launch_dgrad_filter(w_dev, Cout, Cin, KH, KW, g.cread, g.Kpad, g.rows, wt, st));
  const void* src = dy_dev;
  if (stride > 1) {
    CUDA_TRY(launch_dilate(dy_dev, N, g.Hd, g.Wd, Cout, stride, g.Hdd, g.Wdd, ws + g.off_dil, st));
    src = ws + g.off_dil;
  }
  if (int rc0 = unit_vectors(nsb, &scale, &bias)) return rc0;
  OpDev d;
  std::memset(&d, 0, sizeof d);
  d.kind = DK_GEMM;
  d.act = ACT_NONE;
  d.in = src;
  d.B = N; d.H = g.Hdd; d.W = g.Wdd; d.C = g.cread; d.ldi = Cout;
  d.out = dx_dev;
  d.Ho = H; d.Wo = W; d.Cout = Cin; d.ldo = Cin;
  d.kh = KH; d.kw = KW; d.stride = 1; d.ph = g.ph; d.pw = g.pw;
  d.mrep = 1;
  d.M = g.M; d.N = Cin; d.K = g.K; d.Kpad = g.Kpad;
  d.tiles_m = g.tiles_m; d.tiles_n = g.tiles_n; d.bm = BM; d.bn = g.bn;
  d.split_k = 1; d.nkb = g.nkb;
  d.wt = wt; d.ldw = g.Kpad;
  d.scale = scale; d.bias = bias;
  d.a_mode = g.a_mode;
  CUtensorMap maps[3];
  std::memset(maps, 0, sizeof maps);
  const CUtensorMap* dmaps = reinterpret_cast<const CUtensorMap*>(ws + g.off_maps);
  d.tmap_a = dmaps; d.tmap_b = dmaps + 1; d.tmap_c = dmaps + 2;
  int rc = (g.a_mode == A_IM2COL) ? encode_im2col(&maps[0], d, Cout) : encode_rows(&maps[0], src, g.K, g.M, Cout, BM);
  if (!rc) rc = encode_rows(&maps[1], wt, g.Kpad, g.rows, g.Kpad, g.bn);
  if (rc) return rc;
  if ((static_cast<long long>(Cin) * 2) % 16 == 0) {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(Cin), static_cast<cuuint64_t>(g.M)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(Cin) * 2};
    const cuuint32_t box[2] = {64u, 32u};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = g_encode_tiled(&maps[2], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dx_dev, dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(GACER_E_CUDA, "conv_dgrad: output tensor map (%d)", static_cast<int>(r));
    d.c_tma = 1;
  }
  // descriptors: pageable host -> device copies are staged before returning
  CUDA_TRY(cudaMemcpyAsync(ws + g.off_maps, maps, sizeof maps, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(ws + g.off_op, &d, sizeof d, cudaMemcpyHostToDevice, st));
  ExecParams base;
  std::memset(&base, 0, sizeof base);
  base.error = S.d_error;
  base.watchdog_ns = 2000000000LL;
  CUDA_TRY(launch_op(base, reinterpret_cast<const OpDev*>(ws + g.off_op), 0, DK_GEMM, g.tiles_m * g.tiles_n,
                     S.num_sms, st));
  return GACER_OK;
}

}  // extern "C"

// ------------------------------------------------------------------------
// A11: convolution weight gradient on the tcgen05 GEMM path
// ------------------------------------------------------------------------
namespace {
struct WgradGeom {
  int Ho, Wo, Ngemm, Kpad, nkb, bn, tiles_m, tiles_n, rows_a, rows_b, split;
  int64_t M;
  size_t off_op, off_maps, off_a, off_b, off_part, off_cnt, off_g, bytes;
};

int wgrad_geom(int N, int H, int W, int Cin, int Cout, int KH, int KW, int stride, int pad_h, int pad_w, WgradGeom& g) {
  if (N < 1 || H < 1 || W < 1 || Cin < 1 || Cout < 1 || KH < 1 || KW < 1 || stride < 1 || pad_h < 0 || pad_w < 0 ||
      H + 2 * pad_h < KH || W + 2 * pad_w < KW)
    return set_err(GACER_E_SHAPE, "conv_wgrad: inconsistent shape");
  g.Ho = (H + 2 * pad_h - KH) / stride + 1;
  g.Wo = (W + 2 * pad_w - KW) / stride + 1;
  g.M = static_cast<int64_t>(N) * g.Ho * g.Wo;          // the reduction length (pixels)
  if (g.M > (int64_t(1) << 30)) return set_err(GACER_E_SHAPE, "conv_wgrad: too many pixels");
  g.Ngemm = KH * KW * Cin;
  g.Kpad = roundup(static_cast<int>(g.M), BK);
  g.nkb = g.Kpad / BK;
  g.bn = g.Ngemm >= 256 ? 256 : (g.Ngemm >= 128 ? 128 : roundup(g.Ngemm, 16));   // 128x256 tiles: half the dy^T smem traffic per FLOP
  g.tiles_m = cdiv(Cout, BM);
  g.tiles_n = cdiv(g.Ngemm, g.bn);
  g.rows_a = g.tiles_m * BM;
  g.rows_b = g.tiles_n * g.bn;
  // split-K over the long pixel reduction, fixed by the shape (deterministic)
  // (about two waves of items over the SMs, each split >= 8 K-blocks)
  g.split = 1;
  while (g.split < MAX_SPLIT_LONG && g.tiles_m * g.tiles_n * g.split * 2 <= 2 * kSplitSms &&
         g.nkb / (g.split * 2) >= 8)
    g.split *= 2;
  const int tiles = g.tiles_m * g.tiles_n;
  size_t o = 0;
  auto take = [&](size_t n, size_t al) { o = (o + al - 1) / al * al; const size_t r = o; o += n; return r; };
  g.off_op = take(sizeof(OpDev), 256);
  g.off_maps = take(3 * sizeof(CUtensorMap), 128);
  g.off_a = take(static_cast<size_t>(g.rows_a) * g.Kpad * 2, 256);
  g.off_b = take(static_cast<size_t>(g.rows_b) * g.Kpad * 2, 256);
  g.off_part = take(static_cast<size_t>(tiles) * g.split * BM * g.bn * sizeof(float), 256);
  g.off_cnt = take(static_cast<size_t>(tiles) * sizeof(uint32_t), 256);
  g.off_g = take(static_cast<size_t>(Cout) * g.Ngemm * sizeof(float), 256);
  g.bytes = o;
  return 0;
}

// Weight gradient with MN-major operands read in place (A_MN): needs whole
// 64-channel boxes per tap (Cin % 64 == 0) and 16-byte NHWC rows.  Fills the
// GEMM fields of d that differ from the staged (A_ROWS) form and encodes the
// two tensor maps: dy [Mpix][Cout] as 64 x 64 boxes, x as an im2col view with
// 64-pixel columns.
bool wgrad_mn_ok(int Cin, int Cout) { return (Cin % 64 == 0 || Cin == 8) && Cout % 8 == 0; }

int wgrad_mn_setup(OpDev& d, CUtensorMap* maps, const void* x, const void* dy, int N, int H, int W, int Cin, int Cout,
                   int KH, int KW, int stride, int pad_h, int pad_w, const WgradGeom& g, bool encode) {
  d.a_mode = Cin == 8 ? A_MN8 : A_MN;
  d.in = dy;
  d.wt = x;
  d.B = N; d.H = H; d.W = W; d.C = Cin; d.ldi = Cin;
  d.Ho = g.Ho; d.Wo = g.Wo;
  d.kh = KH; d.kw = KW; d.stride = stride; d.ph = pad_h; d.pw = pad_w;
  if (!encode || !x || !dy) return 0;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(Cout), static_cast<cuuint64_t>(g.M)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(Cout) * 2};
  const cuuint32_t box[2] = {64u, static_cast<cuuint32_t>(BK)};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode_tiled(&maps[0], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(dy), dims, strides, box,
                              es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(GACER_E_CUDA, "wgrad: dy tensor map (%d)", static_cast<int>(r));
  OpDev v = d;          // the im2col view of x (the forward conv's geometry, 64-pixel columns)
  v.in = x;
  if (Cin == 8) return encode_im2col(&maps[1], v, Cin, BK, 8, CU_TENSOR_MAP_SWIZZLE_NONE);
  return encode_im2col(&maps[1], v, Cin, BK);
}
}  // namespace

extern "C" {

int64_t gacer_conv_wgrad_workspace(int32_t N, int32_t H, int32_t W, int32_t Cin, int32_t Cout, int32_t KH, int32_t KW,
                                   int32_t stride, int32_t pad_h, int32_t pad_w) {
  WgradGeom g;
  if (int rc = wgrad_geom(N, H, W, Cin, Cout, KH, KW, stride, pad_h, pad_w, g)) return rc;
  return static_cast<int64_t>(g.bytes);
}

int32_t gacer_conv_wgrad(const void* x_dev, const void* dy_dev, int32_t N, int32_t H, int32_t W, int32_t Cin,
                         int32_t Cout, int32_t KH, int32_t KW, int32_t stride, int32_t pad_h, int32_t pad_w,
                         float* dw_dev, void* ws_dev, int64_t ws_bytes, void* stream) {
  if (!S.inited || S.host_only) return set_err(GACER_E_STATE, "conv_wgrad: gacer_init on a device first");
  WgradGeom g;
  if (int rc = wgrad_geom(N, H, W, Cin, Cout, KH, KW, stride, pad_h, pad_w, g)) return rc;
  if (!x_dev || !dy_dev || !dw_dev || !ws_dev || ws_bytes < static_cast<int64_t>(g.bytes) ||
      (reinterpret_cast<uintptr_t>(ws_dev) & 255))
    return set_err(GACER_E_INVALID_ARG, "conv_wgrad: null/misaligned pointer or workspace too small");
  if (int rc = load_tma_encoders()) return rc;
  if (!S.d_error) { if (int rc = dev_upload<int32_t>(&S.d_error, nullptr, 1)) return rc; }
  auto st = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(ws_dev);
  void* a = ws + g.off_a;          // dy^T  [rows_a][Kpad]
  void* b = ws + g.off_b;          // im2col(x)^T [rows_b][Kpad]
  float* gbuf = reinterpret_cast<float*>(ws + g.off_g);
  const int nsb = g.rows_b + 8;
  // the transposes write every column < Kpad of the real rows; only the
  // padding rows (Cout.. and KH*KW*Cin.. up to the tile multiple) need zeros
  const size_t rowb = static_cast<size_t>(g.Kpad) * 2;
  if (g.rows_a > Cout) CUDA_TRY(cudaMemsetAsync(static_cast<uint8_t*>(a) + Cout * rowb, 0, (g.rows_a - Cout) * rowb, st));
  if (g.rows_b > g.Ngemm)
    CUDA_TRY(cudaMemsetAsync(static_cast<uint8_t*>(b) + g.Ngemm * rowb, 0, (g.rows_b - g.Ngemm) * rowb, st));
  CUDA_TRY(cudaMemsetAsync(ws + g.off_cnt, 0, static_cast<size_t>(g.tiles_m) * g.tiles_n * 4, st));
  const bool mn = wgrad_mn_ok(Cin, Cout) && !env_flag("GACER_WGRAD_STAGED");
  if (!mn) {
    // dy [M][Cout] viewed as a 1x1 "im2col" of itself: the transpose
    CUDA_TRY(launch_transpose_im2col(dy_dev, static_cast<int>(g.M), 1, 1, Cout, 1, 1, 1, 1, 1, 0, 0, g.M, g.Kpad, a, st));
    CUDA_TRY(launch_transpose_im2col(x_dev, N, H, W, Cin, g.Ho, g.Wo, KH, KW, stride, pad_h, pad_w, g.M, g.Kpad, b, st));
  }
  const float *ones = nullptr, *zeros = nullptr;
  if (int rc0 = unit_vectors(nsb, &ones, &zeros)) return rc0;
  OpDev d;
  std::memset(&d, 0, sizeof d);
  d.kind = DK_GEMM;
  d.act = ACT_NONE;
  d.out_f32 = 1;
  d.in = a;
  d.B = 1; d.H = 1; d.W = 1; d.C = g.Kpad; d.ldi = g.Kpad;
  d.out = gbuf;
  d.Ho = 1; d.Wo = 1; d.Cout = g.Ngemm; d.ldo = g.Ngemm;
  d.kh = 1; d.kw = 1; d.stride = 1;
  d.mrep = 1;
  d.M = Cout; d.N = g.Ngemm; d.K = g.Kpad; d.Kpad = g.Kpad;
  d.tiles_m = g.tiles_m; d.tiles_n = g.tiles_n; d.bm = BM; d.bn = g.bn;
  d.split_k = g.split; d.nkb = g.nkb;
  d.wt = b; d.ldw = g.Kpad;
  d.scale = ones;
  d.bias = zeros;
  d.partial = reinterpret_cast<float*>(ws + g.off_part);
  d.partials_only = g.split > 1 ? 1 : 0;
  d.tile_cnt = reinterpret_cast<uint32_t*>(ws + g.off_cnt);
  d.a_mode = A_ROWS;
  CUtensorMap maps[3];
  std::memset(maps, 0, sizeof maps);
  const CUtensorMap* dmaps = reinterpret_cast<const CUtensorMap*>(ws + g.off_maps);
  d.tmap_a = dmaps; d.tmap_b = dmaps + 1; d.tmap_c = dmaps + 2;
  d.c_tma = 0;                                   // fp32 rows stored directly
  int rc = 0;
  if (mn) {
    rc = wgrad_mn_setup(d, maps, x_dev, dy_dev, N, H, W, Cin, Cout, KH, KW, stride, pad_h, pad_w, g, true);
  } else {
    rc = encode_rows(&maps[0], a, g.Kpad, g.rows_a, g.Kpad, BM);
    if (!rc) rc = encode_rows(&maps[1], b, g.Kpad, g.rows_b, g.Kpad, g.bn);
  }
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(ws + g.off_maps, maps, sizeof maps, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(ws + g.off_op, &d, sizeof d, cudaMemcpyHostToDevice, st));
  ExecParams base;
  std::memset(&base, 0, sizeof base);
  base.error = S.d_error;
  base.watchdog_ns = 2000000000LL;
  CUDA_TRY(launch_op(base, reinterpret_cast<const OpDev*>(ws + g.off_op), 0, DK_GEMM,
                     g.tiles_m * g.tiles_n * g.split, S.num_sms, st));
  if (g.split > 1)   // the splits are summed in order by a parallel kernel, straight into dW's layout
    CUDA_TRY(launch_wgrad_reduce(d.partial, Cout, Cin, KH, KW, g.bn, g.tiles_n, g.split, dw_dev, st));
  else
    CUDA_TRY(launch_wgrad_permute(gbuf, Cout, Cin, KH, KW, dw_dev, st));
  return GACER_OK;
}

}  // extern "C"

// ------------------------------------------------------------------------
// A11: training forward conv (raw output, BN applied by gacer_bn_train_fwd)
// with device-resident fp32 master weights, on the same tcgen05 path
// ------------------------------------------------------------------------
namespace {
struct FwdGeom {
  int Ho, Wo, cread, K, Kpad, nkb, bn, tiles_m, tiles_n, rows, M, a_mode;
  size_t off_op, off_maps, off_w, bytes;
};

int fwd_geom(int N, int H, int W, int Cin, int Cout, int KH, int KW, int stride, int ph, int pw, FwdGeom& g) {
  if (N < 1 || H < 1 || W < 1 || Cin < 8 || Cin % 8 || Cout < 8 || Cout % 8 || KH < 1 || KW < 1 || stride < 1 ||
      ph < 0 || pw < 0 || H + 2 * ph < KH || W + 2 * pw < KW)
    return set_err(GACER_E_SHAPE, "conv_fwd: need Cin %% 8 == 0, Cout %% 8 == 0 and a non-empty output");
  g.Ho = (H + 2 * ph - KH) / stride + 1;
  g.Wo = (W + 2 * pw - KW) / stride + 1;
  if (Cin % 64 == 0) {
    g.cread = Cin;
    g.a_mode = (KH * KW == 1 && stride == 1 && ph == 0 && pw == 0) ? A_ROWS : A_IM2COL;
  } else if (Cin == 8 && KH * KW >= 25 && !env_flag("GACER_NO_IM2COL8")) {
    g.cread = 8;                         // the image stem: 8 taps per K-block by TMA (A_IM2COL8)
    g.a_mode = A_IM2COL8;
  } else {
    g.cread = Cin;                       // cp.async gather, 8-channel granules
    g.a_mode = A_GATHER;
  }
  g.K = KH * KW * g.cread;
  g.Kpad = roundup(g.K, BK);
  g.nkb = g.Kpad / BK;
  g.M = N * g.Ho * g.Wo;
  g.bn = (Cout >= 256 && cdiv(g.M, BM) >= kSplitSms) ? 256 : (Cout >= 128 ? 128 : roundup(Cout, 16));
  g.tiles_m = cdiv(g.M, BM);
  g.tiles_n = cdiv(Cout, g.bn);
  g.rows = g.tiles_n * g.bn;
  size_t o = 0;
  auto take = [&](size_t n, size_t al) { o = (o + al - 1) / al * al; const size_t r = o; o += n; return r; };
  g.off_op = take(sizeof(OpDev), 256);
  g.off_maps = take(3 * sizeof(CUtensorMap), 128);
  g.off_w = take(static_cast<size_t>(g.rows) * g.Kpad * 2, 256);
  g.bytes = o;
  return 0;
}
}  // namespace

extern "C" {

int64_t gacer_conv_fwd_workspace(int32_t N, int32_t H, int32_t W, int32_t Cin, int32_t Cout, int32_t KH, int32_t KW,
                                 int32_t stride, int32_t pad_h, int32_t pad_w) {
  FwdGeom g;
  if (int rc = fwd_geom(N, H, W, Cin, Cout, KH, KW, stride, pad_h, pad_w, g)) return rc;
  return static_cast<int64_t>(g.bytes);
}

int32_t gacer_conv_fwd(const void* x_dev, const float* w_dev, int32_t N, int32_t H, int32_t W, int32_t Cin,
                       int32_t Cout, int32_t KH, int32_t KW, int32_t stride, int32_t pad_h, int32_t pad_w, void* y_dev,
                       void* ws_dev, int64_t ws_bytes, void* stream) {
  if (!S.inited || S.host_only) return set_err(GACER_E_STATE, "conv_fwd: gacer_init on a device first");
  FwdGeom g;
  if (int rc = fwd_geom(N, H, W, Cin, Cout, KH, KW, stride, pad_h, pad_w, g)) return rc;
  if (!x_dev || !w_dev || !y_dev || !ws_dev || ws_bytes < static_cast<int64_t>(g.bytes) ||
      (reinterpret_cast<uintptr_t>(ws_dev) & 255) || (reinterpret_cast<uintptr_t>(x_dev) & 15) ||
      (reinterpret_cast<uintptr_t>(y_dev) & 15))
    return set_err(GACER_E_INVALID_ARG, "conv_fwd: null/misaligned pointer or workspace too small");
  if (int rc = load_tma_encoders()) return rc;
  if (!S.d_error) { if (int rc = dev_upload<int32_t>(&S.d_error, nullptr, 1)) return rc; }
  auto st = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(ws_dev);
  void* wt = ws + g.off_w;
  const float *scale = nullptr, *bias = nullptr;
  const int nsb = g.rows + 8;
  CUDA_TRY(launch_fwd_filter(w_dev, Cout, Cin, KH, KW, g.cread, g.Kpad, g.rows, wt, st,
                             g.a_mode == A_IM2COL8 ? g.bn : 0));
  if (int rc0 = unit_vectors(nsb, &scale, &bias)) return rc0;
  OpDev d;
  std::memset(&d, 0, sizeof d);
  d.kind = DK_GEMM;
  d.act = ACT_NONE;
  d.in = x_dev;
  d.B = N; d.H = H; d.W = W; d.C = g.cread; d.ldi = Cin;
  d.out = y_dev;
  d.Ho = g.Ho; d.Wo = g.Wo; d.Cout = Cout; d.ldo = Cout;
  d.kh = KH; d.kw = KW; d.stride = stride; d.ph = pad_h; d.pw = pad_w;
  d.mrep = 1;
  d.M = g.M; d.N = Cout; d.K = g.K; d.Kpad = g.Kpad;
  d.tiles_m = g.tiles_m; d.tiles_n = g.tiles_n; d.bm = BM; d.bn = g.bn;
  d.split_k = 1; d.nkb = g.nkb;
  d.wt = wt; d.ldw = g.Kpad;
  d.scale = scale; d.bias = bias;
  d.a_mode = g.a_mode;
  CUtensorMap maps[3];
  std::memset(maps, 0, sizeof maps);
  const CUtensorMap* dmaps = reinterpret_cast<const CUtensorMap*>(ws + g.off_maps);
  d.tmap_a = dmaps; d.tmap_b = dmaps + 1; d.tmap_c = dmaps + 2;
  int rc = 0;
  if (g.a_mode == A_IM2COL) rc = encode_im2col(&maps[0], d, Cin);
  else if (g.a_mode == A_IM2COL8) rc = encode_im2col(&maps[0], d, Cin, BM, 8, CU_TENSOR_MAP_SWIZZLE_NONE);
  else if (g.a_mode == A_ROWS) rc = encode_rows(&maps[0], x_dev, g.K, g.M, Cin, BM);
  if (!rc && g.a_mode != A_IM2COL8) rc = encode_rows(&maps[1], wt, g.Kpad, g.rows, g.Kpad, g.bn);
  if (rc) return rc;
  {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(Cout), static_cast<cuuint64_t>(g.M)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(Cout) * 2};
    const cuuint32_t box[2] = {64u, 32u};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = g_encode_tiled(&maps[2], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, y_dev, dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(GACER_E_CUDA, "conv_fwd: output tensor map (%d)", static_cast<int>(r));
    d.c_tma = 1;
  }
  CUDA_TRY(cudaMemcpyAsync(ws + g.off_maps, maps, sizeof maps, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(ws + g.off_op, &d, sizeof d, cudaMemcpyHostToDevice, st));
  ExecParams base;
  std::memset(&base, 0, sizeof base);
  base.error = S.d_error;
  base.watchdog_ns = 2000000000LL;
  CUDA_TRY(launch_op(base, reinterpret_cast<const OpDev*>(ws + g.off_op), 0, DK_GEMM, g.tiles_m * g.tiles_n,
                     S.num_sms, st));
  return GACER_OK;
}

}  // extern "C"

// ========================================================================
// A11: the training tenant's step as executor ops (gacer_graph.train != 0)
// ========================================================================
// The step is the one train_driver.SequentialTrainer issues call by call
// (the same operators, geometries, thread counts and reduction orders, so the
// two give identical bits), lowered once into executor ops: forward (conv =
// filter pack + tcgen05 GEMM, BN-train = partial sums / fp64 finalize /
// apply(+ReLU), residual add(+ReLU), max-pool, GAP, FC), softmax-CE + mean,
// the backward in reverse topological order (FC, GAP, ReLU, residual-add
// gradient sharing, BN backward with the fused ReLU mask, max-pool argmax /
// gather, conv weight gradient = operand transposes + split-K GEMM + ordered
// reduction, conv data gradient = flipped filter pack (+ zero dilation) +
// GEMM), and ONE SGD-momentum op over the flat parameter buffer.  Every op
// depends on the last writer of each buffer it touches and on the readers of
// each buffer it overwrites (op-level counters on the device).
namespace {

struct TrainLowering {
  Tenant& T;
  int B;
  std::vector<int> last_writer;               // per library buffer
  std::vector<std::vector<int>> readers;
  std::map<int, int> sp_writer;               // special (bound) buffers
  std::map<int, std::vector<int>> sp_readers;
  std::vector<int> grad_writers;              // ops writing (disjoint) slices of the flat gradients
  int step = 1;

  // A filter-packing job: appended to the step's single VF_FILTER_ALL op
  // (created at the first job, issued before every GEMM that reads a packed
  // operand); `out` becomes written by that op.
  void filter_job(TRef w, int out, const int32_t (&iv)[14]) {
    if (T.fall_op < 0) {
      TrainOp fa = vg(VF_FILTER_ALL, 1);
      T.fall_op = add(std::move(fa), {T.buf_params}, {});
    }
    Tenant::FJob j;
    j.w = w;
    j.out.buf = out;
    std::memcpy(j.i, iv, sizeof iv);
    j.n = static_cast<int64_t>(iv[6]) * iv[5];
    T.fjobs.push_back(j);
    writer_of(out) = T.fall_op;
    readers_of(out).clear();
  }
  // size the filter op's grid and job table once every job is known
  void finish_filters() {
    if (T.fall_op < 0) return;
    int64_t total = 0;
    for (const Tenant::FJob& j : T.fjobs) total += j.n;
    T.fall_table = buf(T.fjobs.size() * sizeof(FilterJob));
    TrainOp& fa = T.tops[T.fall_op];
    fa.vblocks = vg_grid_for(total);
    fa.va.n[0] = total;
    fa.va.i[0] = static_cast<int32_t>(T.fjobs.size());
    fa.vp[0].buf = T.fall_table;
    fa.bytes = static_cast<double>(total) * 6.0;
    const int grid = S.opts.num_ctas > 0 ? S.opts.num_ctas : (S.num_sms > 0 ? S.num_sms : kSplitSms);
    fa.per = std::max(1, cdiv(fa.vblocks, grid));
    fa.items = cdiv(fa.vblocks, fa.per);
  }

  explicit TrainLowering(Tenant& t, int b) : T(t), B(b) {}

  int buf(size_t bytes) {
    T.tbuf_bytes.push_back(std::max<size_t>(bytes, 16));
    T.tbufs.push_back(nullptr);
    last_writer.push_back(-1);
    readers.emplace_back();
    return static_cast<int>(T.tbuf_bytes.size()) - 1;
  }
  int& writer_of(int b) { return b >= 0 ? last_writer[b] : sp_writer.emplace(b, -1).first->second; }
  std::vector<int>& readers_of(int b) { return b >= 0 ? readers[b] : sp_readers[b]; }
  // bytes an op moves through buffer b (the flat parameter / gradient /
  // momentum buffers are touched per slice: not counted, see the SGD op)
  double bytes_of(int b) const {
    if (b < 0 || b == T.buf_params || b == T.buf_grads || b == T.buf_mom) return 0.0;
    return static_cast<double>(T.tbuf_bytes[b]);
  }

  // append op with its buffer accesses; returns its index
  int add(TrainOp&& op, std::initializer_list<int> rd, std::initializer_list<int> wr) {
    const int me = static_cast<int>(T.tops.size());
    std::set<int> dep;
    for (int b : rd) {
      if (b == -1) continue;
      if (b == TBUF_IN || b == TBUF_LABELS) op.reads_input = true;
      if (b == T.buf_grads) {   // the update reads every gradient slice
        dep.insert(grad_writers.begin(), grad_writers.end());
        continue;
      }
      if (writer_of(b) >= 0) dep.insert(writer_of(b));
      op.bytes += bytes_of(b);
    }
    for (int b : wr) {
      if (b == -1) continue;
      if (b == T.buf_grads) continue;   // disjoint per-parameter slices: no WAW between writers
      if (writer_of(b) >= 0) dep.insert(writer_of(b));
      for (int r : readers_of(b)) dep.insert(r);
      op.bytes += bytes_of(b);
    }
    dep.erase(me);
    op.deps.assign(dep.begin(), dep.end());
    for (int b : rd) if (b != -1 && b != T.buf_grads) readers_of(b).push_back(me);
    for (int b : wr) {
      if (b == -1) continue;
      if (b == T.buf_grads) {
        grad_writers.push_back(me);
        // the slices it writes (its VArgs pointer slots into the buffer)
        for (const TRef& r : op.vp)
          if (r.buf == T.buf_grads) {
            const int64_t off = static_cast<int64_t>(r.off / 4);
            for (const auto& kv : T.param_slice)
              if (kv.second.first == off) op.grad_ranges.push_back({off, kv.second.second});
          }
        continue;
      }
      writer_of(b) = me;
      readers_of(b).clear();
    }
    op.step_pos = step;
    if (op.kind == DK_VGRID) {
      // items: one wave of the executor's CTAs' worth of virtual-block ranges
      // (streaming operators: per-item claim/release overhead amortised).
      // The grid of this instance, not the SM count: with SMs reserved for a
      // collective, 148 items on 136 CTAs would take two waves.  Results do
      // not depend on it (the virtual-block decomposition is fixed).
      const int grid = S.opts.num_ctas > 0 ? S.opts.num_ctas : (S.num_sms > 0 ? S.num_sms : kSplitSms);
      op.per = std::max(1, cdiv(op.vblocks, grid));
      op.items = cdiv(op.vblocks, op.per);
    } else {
      op.items = op.gd.tiles_m * op.gd.tiles_n * op.gd.split_k;
    }
    T.tops.push_back(std::move(op));
    return me;
  }

  static TrainOp vg(int fn, int nvb) {
    TrainOp o;
    o.kind = DK_VGRID;
    o.vfn = fn;
    o.vblocks = std::max(1, nvb);
    std::memset(&o.va, 0, sizeof o.va);
    return o;
  }
};

}  // namespace

namespace {

int lower_train(const gacer_graph* g, int batch, Tenant& T, const std::map<int, int>& pos) {
  const int n = g->n_ops;
  const int B = batch;
  T.train = true;
  T.n_steps = 2 * n + 1;
  T.lr = g->lr;
  T.momentum = g->momentum;
  TrainLowering L(T, B);
  auto idx_of = [&](int id) { return id == 0 ? -1 : pos.at(id); };
  // ---- plan: shapes (NHWC, the input padded to 8 channels) and the fusable ReLUs
  struct Shp { int h, w, c; };
  std::vector<Shp> shp(n);
  const Shp in_shape{T.in_h, T.in_w, T.in_c_pad};
  auto shape_of = [&](int id) { return id == 0 ? in_shape : shp[pos.at(id)]; };
  std::vector<std::vector<int>> consumers(n + 1);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < g->ops[i].n_preds; ++j) consumers[idx_of(g->ops[i].preds[j]) + 1].push_back(i);
  std::vector<int> fused_relu(n, -1);   // producer (bn / add) -> its ReLU
  for (int i = 0; i < n; ++i) {
    const gacer_op_desc& o = g->ops[i];
    const Shp x = shape_of(o.preds[0]);
    switch (o.kind) {
      case GACER_OP_CONV2D:
        if (o.groups != 1 || (o.flags & GACER_FLAG_BIAS))
          return set_err(GACER_E_UNSUPPORTED_OP, "op %d: training supports ungrouped convs without bias", o.id);
        shp[i] = {(x.h + 2 * o.pad_h - o.kh) / o.stride + 1, (x.w + 2 * o.pad_w - o.kw) / o.stride + 1, o.c_out};
        if (o.c_out % 8) return set_err(GACER_E_UNSUPPORTED_OP, "op %d: training needs c_out %% 8 == 0", o.id);
        break;
      case GACER_OP_MAXPOOL:
        shp[i] = {(x.h + 2 * o.pad_h - o.kh) / o.stride + 1, (x.w + 2 * o.pad_w - o.kw) / o.stride + 1, x.c};
        break;
      case GACER_OP_GAP: shp[i] = {1, 1, x.c}; break;
      case GACER_OP_LINEAR:
        if (x.h != 1 || x.w != 1 || x.c != o.c_in)
          return set_err(GACER_E_UNSUPPORTED_OP, "op %d: training FC needs a [B][c_in] (1x1) input", o.id);
        shp[i] = {1, 1, o.c_out};
        break;
      case GACER_OP_BN:
        if (x.c > VG_MAX_BN_C) return set_err(GACER_E_UNSUPPORTED_OP, "op %d: training BN over > 2048 channels", o.id);
        shp[i] = x;
        break;
      case GACER_OP_FLATTEN: case GACER_OP_DROPOUT: case GACER_OP_RELU: case GACER_OP_ADD:
        shp[i] = x;
        break;
      default:
        return set_err(GACER_E_UNSUPPORTED_OP, "op %d: kind %d has no training lowering", o.id, o.kind);
    }
    if (o.kind == GACER_OP_RELU) {
      const int pr = idx_of(o.preds[0]);
      if (pr < 0 || (g->ops[pr].kind != GACER_OP_BN && g->ops[pr].kind != GACER_OP_ADD) || consumers[pr + 1].size() != 1)
        return set_err(GACER_E_UNSUPPORTED_OP, "op %d: a ReLU is trained fused into its BN or residual-add producer",
                       o.id);
      fused_relu[pr] = i;
    }
  }
  if (g->ops[n - 1].kind != GACER_OP_LINEAR)
    return set_err(GACER_E_UNSUPPORTED_OP, "training needs the last op to be the FC producing the logits");
  const int ncls = g->ops[n - 1].c_out;
  T.out_features = ncls;

  // ---- flat fp32 parameters (registration order: conv w (input channels
  //      padded), bn gamma, beta, linear w, b), gradients, momentum
  int64_t np = 0;
  for (int i = 0; i < n; ++i) {
    const gacer_op_desc& o = g->ops[i];
    auto slot = [&](int which, int64_t cnt) { T.param_slice[{i, which}] = {np, cnt}; np += cnt; };
    if (o.kind == GACER_OP_CONV2D) slot(0, static_cast<int64_t>(o.c_out) * shape_of(o.preds[0]).c * o.kh * o.kw);
    else if (o.kind == GACER_OP_BN) { slot(0, shape_of(o.preds[0]).c); slot(1, shape_of(o.preds[0]).c); }
    else if (o.kind == GACER_OP_LINEAR) { slot(0, static_cast<int64_t>(o.c_out) * o.c_in); if (o.flags & GACER_FLAG_BIAS) slot(1, o.c_out); }
  }
  T.h_params.assign(np, 0.0f);
  for (int i = 0; i < n; ++i) {
    const gacer_op_desc& o = g->ops[i];
    if (o.kind == GACER_OP_CONV2D) {
      if (!o.weight) return set_err(GACER_E_INVALID_ARG, "op %d: missing weight", o.id);
      const int cp = shape_of(o.preds[0]).c;
      float* w = T.h_params.data() + T.param_slice[{i, 0}].first;
      for (int co = 0; co < o.c_out; ++co)
        for (int ci = 0; ci < o.c_in; ++ci)
          for (int r = 0; r < o.kh * o.kw; ++r)
            w[(static_cast<size_t>(co) * cp + ci) * o.kh * o.kw + r] = o.weight[(static_cast<size_t>(co) * o.c_in + ci) * o.kh * o.kw + r];
    } else if (o.kind == GACER_OP_BN) {
      const int c = shape_of(o.preds[0]).c;
      std::memcpy(T.h_params.data() + T.param_slice[{i, 0}].first, o.bn_gamma, c * sizeof(float));
      std::memcpy(T.h_params.data() + T.param_slice[{i, 1}].first, o.bn_beta, c * sizeof(float));
    } else if (o.kind == GACER_OP_LINEAR) {
      std::memcpy(T.h_params.data() + T.param_slice[{i, 0}].first, o.weight,
                  static_cast<size_t>(o.c_out) * o.c_in * sizeof(float));
      if (o.flags & GACER_FLAG_BIAS) {
        if (!o.bias) return set_err(GACER_E_INVALID_ARG, "op %d: missing bias", o.id);
        std::memcpy(T.h_params.data() + T.param_slice[{i, 1}].first, o.bias, o.c_out * sizeof(float));
      }
    }
  }
  T.buf_params = L.buf(np * 4);
  T.buf_grads = L.buf(np * 4);
  T.buf_mom = L.buf(np * 4);
  T.buf_loss = L.buf(4);
  auto pref = [&](int i, int which) { TRef r; r.buf = T.buf_params; r.off = T.param_slice.at({i, which}).first * 4; return r; };
  auto gref = [&](int i, int which) { TRef r; r.buf = T.buf_grads; r.off = T.param_slice.at({i, which}).first * 4; return r; };
  auto bref = [](int b) { TRef r; r.buf = b; return r; };
  // unit scale / zero bias of the GEMM epilogues (no folded BN in training)
  int maxrows = 8;
  for (int i = 0; i < n; ++i) {
    const gacer_op_desc& o = g->ops[i];
    if (o.kind == GACER_OP_CONV2D) maxrows = std::max({maxrows, o.c_out, shape_of(o.preds[0]).c * o.kh * o.kw});
  }
  maxrows = roundup(maxrows, 256) + 8;
  const int buf_ones = L.buf(static_cast<size_t>(maxrows) * 4), buf_zeros = L.buf(static_cast<size_t>(maxrows) * 4);
  // (filled at upload: ones = 1.0f; zeros stay zero)
  T.param_slice[{-1, 0}] = {buf_ones, maxrows};

  // ---- forward
  std::vector<int> out(n, -1);   // output buffer of each op (after aliasing)
  std::map<int, int> pool_arg;   // max-pool op -> its argmax buffer (written by the forward pool)
  auto out_of = [&](int id) { return id == 0 ? TBUF_IN : out[pos.at(id)]; };
  std::vector<std::pair<int, int>> saved(n, {-1, -1});   // BN: (mean, var)
  int logits = -1;
  for (int i = 0; i < n; ++i) {
    const gacer_op_desc& o = g->ops[i];
    L.step = i + 1;
    const Shp x = shape_of(o.preds[0]), y = shp[i];
    const int xb = out_of(o.preds[0]);
    switch (o.kind) {
      case GACER_OP_CONV2D: {
        FwdGeom fg;
        if (int rc = fwd_geom(B, x.h, x.w, x.c, o.c_out, o.kh, o.kw, o.stride, o.pad_h, o.pad_w, fg)) return rc;
        const int wp = L.buf(static_cast<size_t>(fg.rows) * fg.Kpad * 2);
        {
          const int32_t iv[14] = {o.c_out, x.c, o.kh, o.kw, fg.cread, fg.Kpad, fg.rows, 1,
                                  fg.a_mode == A_IM2COL8 ? fg.bn : 0,   // block layout of the 8-channel TMA path
                                  0, 0, 0, 0, 0};
          L.filter_job(pref(i, 0), wp, iv);
        }
        const int yb = L.buf(static_cast<size_t>(B) * y.h * y.w * y.c * 2);
        TrainOp m;
        m.kind = DK_GEMM;
        m.gemm_kind = 0;
        OpDev& d = m.gd;
        std::memset(&d, 0, sizeof d);
        d.kind = DK_GEMM; d.act = ACT_NONE;
        d.B = B; d.H = x.h; d.W = x.w; d.C = fg.cread; d.ldi = x.c;
        d.Ho = fg.Ho; d.Wo = fg.Wo; d.Cout = o.c_out; d.ldo = o.c_out;
        d.kh = o.kh; d.kw = o.kw; d.stride = o.stride; d.ph = o.pad_h; d.pw = o.pad_w; d.mrep = 1;
        d.M = fg.M; d.N = o.c_out; d.K = fg.K; d.Kpad = fg.Kpad;
        d.tiles_m = fg.tiles_m; d.tiles_n = fg.tiles_n; d.bm = BM; d.bn = fg.bn; d.split_k = 1; d.nkb = fg.nkb;
        d.ldw = fg.Kpad; d.a_mode = fg.a_mode;
        m.g_in = bref(xb); m.g_out = bref(yb); m.g_wt = bref(wp);
        m.g_scale = bref(buf_ones); m.g_bias = bref(buf_zeros);
        m.im2col_c = x.c; m.a_ld = x.c; m.a_rows = fg.M; m.b_rows = fg.rows;
        m.flops = 2.0 * fg.M * o.c_out * static_cast<double>(x.c) * o.kh * o.kw;
        L.add(std::move(m), {xb, wp, buf_ones, buf_zeros}, {yb});
        out[i] = yb;
        break;
      }
      case GACER_OP_BN: {
        const int64_t M = static_cast<int64_t>(B) * x.h * x.w;
        const int C = x.c, P = vg_bn_partials(M);
        const int part = L.buf(static_cast<size_t>(P) * 2 * C * 4 + 4 * C * 4);
        const int mean = L.buf(C * 4), var = L.buf(C * 4);
        const int yb = L.buf(static_cast<size_t>(M) * C * 2);
        TRef coef = bref(part);
        coef.off = static_cast<size_t>(P) * 2 * C * 4;
        TrainOp a = TrainLowering::vg(VF_BN_PARTIAL, P);
        a.vp[0] = bref(xb); a.vp[5] = bref(part); a.va.n[0] = M; a.va.i[0] = 0; a.va.i[1] = C;
        L.add(std::move(a), {xb}, {part});
        TrainOp f = TrainLowering::vg(VF_BN_FINALIZE, cdiv(C, 32));
        f.vp[0] = bref(part); f.vp[1] = pref(i, 0); f.vp[2] = pref(i, 1); f.vp[3] = bref(xb); f.vp[5] = bref(mean);
        f.vp[6] = bref(var); f.vp[7] = coef;
        f.va.n[0] = M; f.va.i[0] = 0; f.va.i[1] = C; f.va.i[2] = P; f.va.f[0] = o.bn_eps;
        L.add(std::move(f), {part, T.buf_params, xb}, {mean, var, part});
        TrainOp e = TrainLowering::vg(VF_BN_APPLY, vg_apply_blocks(M * (C / 8)));
        e.vp[0] = bref(xb); e.vp[3] = coef; e.vp[4] = bref(yb);
        e.va.n[0] = M; e.va.i[0] = 0; e.va.i[1] = C; e.va.i[2] = fused_relu[i] >= 0 ? 1 : 0;
        L.add(std::move(e), {xb, part}, {yb});
        saved[i] = {mean, var};
        out[i] = yb;
        break;
      }
      case GACER_OP_RELU:
      case GACER_OP_FLATTEN:
      case GACER_OP_DROPOUT:
        out[i] = xb;        // fused into the producer / identity
        break;
      case GACER_OP_ADD: {
        const int bb = out_of(o.preds[1]);
        const int yb = L.buf(static_cast<size_t>(B) * x.h * x.w * x.c * 2);
        const int64_t n8 = static_cast<int64_t>(B) * x.h * x.w * x.c / 8;
        TrainOp a = TrainLowering::vg(VF_ADD, vg_grid_for(n8));
        a.vp[0] = bref(xb); a.vp[1] = bref(bb); a.vp[2] = bref(yb);
        a.va.n[0] = n8; a.va.i[0] = fused_relu[i] >= 0 ? 1 : 0;
        L.add(std::move(a), {xb, bb}, {yb});
        out[i] = yb;
        break;
      }
      case GACER_OP_MAXPOOL: {
        // the forward pool and the backward's argmax in one pass over x:
        // y (as VF_MAXPOOL_FWD computes it) and the per-channel window argmax
        // (as VF_MAXPOOL_ARGMAX) -- the backward then reads the stored argmax
        // instead of re-reading x at the end of the step
        const int yb = L.buf(static_cast<size_t>(B) * y.h * y.w * x.c * 2);
        const int arg = L.buf(static_cast<size_t>(B) * y.h * y.w * x.c);
        TrainOp a = TrainLowering::vg(VF_MAXPOOL_ARGMAX, vg_grid_for(static_cast<int64_t>(B) * y.h * y.w * (x.c / 8)));
        a.vp[0] = bref(xb); a.vp[1] = bref(arg); a.vp[2] = bref(yb);
        const int iv[11] = {B, x.h, x.w, x.c, o.kh, o.kw, o.stride, o.pad_h, o.pad_w, y.h, y.w};
        std::memcpy(a.va.i, iv, sizeof iv);
        L.add(std::move(a), {xb}, {yb, arg});
        out[i] = yb;
        pool_arg[i] = arg;
        break;
      }
      case GACER_OP_GAP: {
        const int yb = L.buf(static_cast<size_t>(B) * x.c * 2);
        TrainOp a = TrainLowering::vg(VF_GAP_FWD, vg_grid_for(static_cast<int64_t>(B) * (x.c / 8)));
        a.vp[0] = bref(xb); a.vp[1] = bref(yb);
        a.va.i[0] = B; a.va.i[1] = x.h * x.w; a.va.i[2] = x.c;
        L.add(std::move(a), {xb}, {yb});
        out[i] = yb;
        break;
      }
      case GACER_OP_LINEAR: {
        const bool last = i == n - 1;
        const int zb = last ? TBUF_OUT : L.buf(static_cast<size_t>(B) * o.c_out * 4);
        TrainOp a = TrainLowering::vg(VF_LINEAR_FWD, vg_grid_for(static_cast<int64_t>(B) * ((o.c_out + 3) / 4) * 32));
        a.vp[0] = bref(xb); a.vp[1] = pref(i, 0);
        if (o.flags & GACER_FLAG_BIAS) a.vp[2] = pref(i, 1);
        a.vp[3] = bref(zb);
        a.va.i[0] = B; a.va.i[1] = o.c_in; a.va.i[2] = o.c_out;
        L.add(std::move(a), {xb, T.buf_params}, {zb});
        out[i] = zb;
        if (last) logits = zb;
        break;
      }
    }
  }
  // ---- loss: mean softmax cross-entropy over the labels
  L.step = n;
  const int dz = L.buf(static_cast<size_t>(B) * ncls * 4), rowloss = L.buf(static_cast<size_t>(B) * 4);
  {
    TrainOp a = TrainLowering::vg(VF_SOFTMAX_CE, B);
    a.vp[0] = bref(logits); a.vp[1] = bref(TBUF_LABELS); a.vp[2] = bref(dz); a.vp[3] = bref(rowloss);
    a.va.i[0] = B; a.va.i[1] = ncls;
    L.add(std::move(a), {logits, TBUF_LABELS}, {dz, rowloss});
    TrainOp m = TrainLowering::vg(VF_MEAN, 1);
    m.vp[0] = bref(rowloss); m.vp[1] = bref(T.buf_loss); m.va.i[0] = B;
    L.add(std::move(m), {rowloss}, {T.buf_loss});
  }
  // ---- backward (reverse issue order)
  std::map<int, int> dval;            // orig op index (-1: input) -> gradient buffer of its output
  std::set<int> shared;               // gradient buffers held by two dval entries (a residual add): copy on write
  std::map<int, int> relu_mask;       // bn op -> the output of its fused ReLU
  dval[n - 1] = dz;
  auto acc = [&](int tid, int gb, size_t bytes) {
    if (tid < 0) return;
    auto it = dval.find(tid);
    if (it == dval.end()) { dval[tid] = gb; return; }
    const int cur = it->second;
    const int dst = shared.count(cur) ? L.buf(bytes) : cur;
    TrainOp a = TrainLowering::vg(VF_ADD, vg_grid_for(static_cast<int64_t>(bytes / 16)));
    a.vp[0] = bref(cur); a.vp[1] = bref(gb); a.vp[2] = bref(dst);
    a.va.n[0] = static_cast<int64_t>(bytes / 16); a.va.i[0] = 0;
    L.add(std::move(a), {cur, gb}, {dst});
    dval[tid] = dst;
  };
  for (int i = n - 1; i >= 0; --i) {
    const gacer_op_desc& o = g->ops[i];
    L.step = 2 * n - i;
    auto itd = dval.find(i);
    if (itd == dval.end()) continue;
    int dy = itd->second;
    dval.erase(itd);
    const int pred = idx_of(o.preds[0]);
    const Shp x = shape_of(o.preds[0]), y = shp[i];
    const int xb = out_of(o.preds[0]);
    const size_t xbytes = static_cast<size_t>(B) * x.h * x.w * x.c * 2;
    switch (o.kind) {
      case GACER_OP_LINEAR: {
        const int dx = L.buf(static_cast<size_t>(B) * x.c * 4);
        TrainOp a = TrainLowering::vg(VF_LINEAR_DX, vg_grid_for(static_cast<int64_t>((B + 3) / 4) * x.c));
        a.vp[0] = pref(i, 0); a.vp[1] = bref(dy); a.vp[2] = bref(dx);
        a.va.i[0] = B; a.va.i[1] = x.c; a.va.i[2] = o.c_out;
        L.add(std::move(a), {T.buf_params, dy}, {dx});
        TrainOp w = TrainLowering::vg(VF_LINEAR_DW, vg_grid_for(static_cast<int64_t>((o.c_out + 3) / 4) * x.c));
        w.vp[0] = bref(xb); w.vp[1] = bref(dy); w.vp[2] = gref(i, 0);
        if (o.flags & GACER_FLAG_BIAS) w.vp[3] = gref(i, 1);
        w.va.i[0] = B; w.va.i[1] = x.c; w.va.i[2] = o.c_out;
        L.add(std::move(w), {xb, dy}, {T.buf_grads});
        acc(pred, dx, static_cast<size_t>(B) * x.c * 4);
        break;
      }
      case GACER_OP_FLATTEN: case GACER_OP_DROPOUT:
        acc(pred, dy, 0);
        break;
      case GACER_OP_GAP: {
        const int dx = L.buf(xbytes);
        TrainOp a = TrainLowering::vg(VF_GAP_BWD, vg_grid_for(static_cast<int64_t>(B) * x.h * x.w * (x.c / 8)));
        a.vp[0] = bref(dy); a.vp[1] = bref(dx);
        a.va.i[0] = B; a.va.i[1] = x.h * x.w; a.va.i[2] = x.c;
        L.add(std::move(a), {dy}, {dx});
        acc(pred, dx, xbytes);
        break;
      }
      case GACER_OP_RELU: {
        if (g->ops[pred].kind == GACER_OP_BN) {
          relu_mask[pred] = out[i];           // applied inside the BN backward (fused)
        } else {
          const int dst = shared.count(dy) ? L.buf(xbytes) : dy;
          TrainOp a = TrainLowering::vg(VF_RELU_BWD, vg_grid_for(static_cast<int64_t>(xbytes / 16)));
          a.vp[0] = bref(out[i]); a.vp[1] = bref(dy); a.vp[2] = bref(dst);
          a.va.n[0] = static_cast<int64_t>(xbytes / 16); a.va.i[0] = 0;
          L.add(std::move(a), {out[i], dy}, {dst});
          dy = dst;
        }
        acc(pred, dy, xbytes);
        break;
      }
      case GACER_OP_ADD:
        shared.insert(dy);                    // both inputs receive dy itself (no copy)
        acc(idx_of(o.preds[0]), dy, xbytes);
        acc(idx_of(o.preds[1]), dy, xbytes);
        break;
      case GACER_OP_BN: {
        const int64_t M = static_cast<int64_t>(B) * x.h * x.w;
        const int C = x.c, P = vg_bn_partials(M);
        const int part = L.buf(static_cast<size_t>(P) * 2 * C * 4 + 4 * C * 4);
        const int dx = L.buf(xbytes);
        TRef coef = bref(part);
        coef.off = static_cast<size_t>(P) * 2 * C * 4;
        auto im = relu_mask.find(i);
        const int ym = im == relu_mask.end() ? -1 : im->second;
        if (im != relu_mask.end()) relu_mask.erase(im);
        TrainOp a = TrainLowering::vg(VF_BN_PARTIAL, P);
        a.vp[0] = bref(xb); a.vp[1] = bref(dy); if (ym >= 0) a.vp[2] = bref(ym);
        a.vp[3] = bref(saved[i].first); a.vp[4] = bref(saved[i].second); a.vp[5] = bref(part);
        a.va.n[0] = M; a.va.i[0] = 1; a.va.i[1] = C; a.va.f[0] = o.bn_eps;
        L.add(std::move(a), {xb, dy, ym, saved[i].first, saved[i].second}, {part});
        TrainOp f = TrainLowering::vg(VF_BN_FINALIZE, cdiv(C, 32));
        f.vp[0] = bref(part); f.vp[1] = pref(i, 0); f.vp[3] = bref(saved[i].first); f.vp[4] = bref(saved[i].second);
        f.vp[5] = gref(i, 0); f.vp[6] = gref(i, 1); f.vp[7] = coef;
        f.va.n[0] = M; f.va.i[0] = 1; f.va.i[1] = C; f.va.i[2] = P; f.va.f[0] = o.bn_eps;
        L.add(std::move(f), {part, T.buf_params, saved[i].first, saved[i].second}, {T.buf_grads, part});
        TrainOp e = TrainLowering::vg(VF_BN_APPLY, vg_apply_blocks(M * (C / 8)));
        e.vp[0] = bref(xb); e.vp[1] = bref(dy); if (ym >= 0) e.vp[2] = bref(ym); e.vp[3] = coef; e.vp[4] = bref(dx);
        e.va.n[0] = M; e.va.i[0] = 1; e.va.i[1] = C;
        L.add(std::move(e), {xb, dy, ym, part}, {dx});
        acc(pred, dx, xbytes);
        break;
      }
      case GACER_OP_MAXPOOL: {
        const int arg = pool_arg.at(i);   // written by the forward pool
        const int dx = L.buf(xbytes);
        const int iv[11] = {B, x.h, x.w, x.c, o.kh, o.kw, o.stride, o.pad_h, o.pad_w, y.h, y.w};
        TrainOp b2 = TrainLowering::vg(VF_MAXPOOL_BWD, vg_grid_for(static_cast<int64_t>(B) * x.h * x.w * (x.c / 8)));
        b2.vp[0] = bref(arg); b2.vp[1] = bref(dy); b2.vp[2] = bref(dx);
        std::memcpy(b2.va.i, iv, sizeof iv);
        L.add(std::move(b2), {arg, dy}, {dx});
        acc(pred, dx, xbytes);
        break;
      }
      case GACER_OP_CONV2D: {
        // weight gradient: dW = dy^T . im2col(x), both operands staged K-major
        // along the pixel index, split-K over the pixels, ordered reduction
        WgradGeom wg;
        if (int rc = wgrad_geom(B, x.h, x.w, x.c, o.c_out, o.kh, o.kw, o.stride, o.pad_h, o.pad_w, wg)) return rc;
        // MN-major operands read in place (no staged transposes) when every
        // 64-channel box lies inside one tap; the stem (3 channels) stages
        const bool mn = wgrad_mn_ok(x.c, o.c_out) && !env_flag("GACER_WGRAD_STAGED");
        const int ab = mn ? -1 : L.buf(static_cast<size_t>(wg.rows_a) * wg.Kpad * 2);
        const int bb = mn ? -1 : L.buf(static_cast<size_t>(wg.rows_b) * wg.Kpad * 2);
        const int tiles = wg.tiles_m * wg.tiles_n;
        const int part = L.buf(static_cast<size_t>(tiles) * wg.split * BM * wg.bn * 4);
        const int gbuf = wg.split > 1 ? -1 : L.buf(static_cast<size_t>(o.c_out) * wg.Ngemm * 4);
        if (!mn) {
          TrainOp t = TrainLowering::vg(VF_TRANSPOSE_IM2COL, vg_transpose_blocks(o.c_out, 1, 1, wg.Kpad));
          t.vp[0] = bref(dy); t.vp[1] = bref(ab);
          t.va.n[0] = wg.M;
          const int iv[12] = {static_cast<int>(wg.M), 1, 1, o.c_out, 1, 1, 1, 1, 0, 0, wg.Kpad, 1};
          std::memcpy(t.va.i, iv, sizeof iv);
          L.add(std::move(t), {dy}, {ab});
        }
        if (!mn) {
          TrainOp t = TrainLowering::vg(VF_TRANSPOSE_IM2COL, vg_transpose_blocks(x.c, o.kh, o.kw, wg.Kpad));
          t.vp[0] = bref(xb); t.vp[1] = bref(bb);
          t.va.n[0] = wg.M;
          const int iv[12] = {B, x.h, x.w, x.c, wg.Ho, wg.Wo, o.kw, o.stride, o.pad_h, o.pad_w, wg.Kpad, o.kh};
          std::memcpy(t.va.i, iv, sizeof iv);
          L.add(std::move(t), {xb}, {bb});
        }
        {
          TrainOp m;
          m.kind = DK_GEMM;
          m.gemm_kind = 2;
          OpDev& d = m.gd;
          std::memset(&d, 0, sizeof d);
          d.kind = DK_GEMM; d.act = ACT_NONE; d.out_f32 = 1;
          d.B = 1; d.H = 1; d.W = 1; d.C = wg.Kpad; d.ldi = wg.Kpad;
          d.Ho = 1; d.Wo = 1; d.Cout = wg.Ngemm; d.ldo = wg.Ngemm;
          d.kh = 1; d.kw = 1; d.stride = 1; d.mrep = 1;
          d.M = o.c_out; d.N = wg.Ngemm; d.K = wg.Kpad; d.Kpad = wg.Kpad;
          d.tiles_m = wg.tiles_m; d.tiles_n = wg.tiles_n; d.bm = BM; d.bn = wg.bn;
          d.split_k = wg.split; d.nkb = wg.nkb; d.ldw = wg.Kpad;
          d.partials_only = wg.split > 1 ? 1 : 0;
          d.a_mode = A_ROWS;
          m.g_part = bref(part); m.g_out = bref(gbuf);
          m.g_scale = bref(buf_ones); m.g_bias = bref(buf_zeros);
          m.flops = 2.0 * o.c_out * static_cast<double>(wg.Ngemm) * wg.M;
          if (mn) {
            wgrad_mn_setup(d, nullptr, nullptr, nullptr, B, x.h, x.w, x.c, o.c_out, o.kh, o.kw, o.stride, o.pad_h,
                           o.pad_w, wg, false);
            m.g_in = bref(dy); m.g_wt = bref(xb);
            L.add(std::move(m), {dy, xb, buf_ones, buf_zeros}, {part, gbuf});
          } else {
            m.g_in = bref(ab); m.g_wt = bref(bb);
            m.a_ld = wg.Kpad; m.a_rows = wg.rows_a; m.b_rows = wg.rows_b;
            L.add(std::move(m), {ab, bb, buf_ones, buf_zeros}, {part, gbuf});
          }
        }
        if (wg.split > 1) {
          TrainOp r = TrainLowering::vg(VF_WGRAD_REDUCE, vg_grid_for(static_cast<int64_t>((wg.Ngemm + 3) / 4) * o.c_out));
          r.vp[0] = bref(part); r.vp[1] = gref(i, 0);
          r.va.i[0] = o.c_out; r.va.i[1] = x.c; r.va.i[2] = o.kh; r.va.i[3] = o.kw; r.va.i[4] = wg.bn;
          r.va.i[5] = wg.tiles_n; r.va.i[6] = wg.split;
          L.add(std::move(r), {part}, {T.buf_grads});
        } else {
          TrainOp r = TrainLowering::vg(VF_WGRAD_PERMUTE, vg_grid_for(static_cast<int64_t>(o.c_out) * x.c * o.kh * o.kw));
          r.vp[0] = bref(gbuf); r.vp[1] = gref(i, 0);
          r.va.i[0] = o.c_out; r.va.i[1] = x.c; r.va.i[2] = o.kh; r.va.i[3] = o.kw;
          L.add(std::move(r), {gbuf}, {T.buf_grads});
        }
        if (pred >= 0) {
          // data gradient: a forward conv of (zero-dilated) dy with the
          // flipped, transposed filter
          DgradGeom dg;
          if (int rc = dgrad_geom(B, x.h, x.w, x.c, o.c_out, o.kh, o.kw, o.stride, o.pad_h, o.pad_w, dg)) return rc;
          if (dg.phased) {
            // phase decomposition (no zero-dilated dy, no S^2 zero work): per
            // phase with taps the flipped sub-filter and a stride-1 GEMM of dy,
            // then one scatter of the phases into dx
            int pbuf[4] = {-1, -1, -1, -1};
            for (const DgPhaseGemm& q : dg.phases) {
              if (q.K == 0) continue;
              const int qw = L.buf(static_cast<size_t>(q.rows) * q.Kpad * 2);
              const int32_t iv[14] = {o.c_out, x.c, q.vh.K, q.vw.K, o.c_out, q.Kpad, q.rows, 0, 0, o.stride, q.a,
                                      q.b, o.kh, o.kw};
              L.filter_job(pref(i, 0), qw, iv);
              const int qo = L.buf(static_cast<size_t>(q.M) * x.c * 2);
              pbuf[q.a * o.stride + q.b] = qo;
              TrainOp m;
              m.kind = DK_GEMM;
              m.gemm_kind = 1;
              dgrad_phase_opdev(m.gd, q, B, dg.Hd, dg.Wd, x.c, o.c_out);
              m.g_in = bref(dy); m.g_out = bref(qo); m.g_wt = bref(qw);
              m.g_scale = bref(buf_ones); m.g_bias = bref(buf_zeros);
              m.im2col_c = o.c_out; m.a_ld = o.c_out; m.a_rows = q.M; m.b_rows = q.rows;
              m.has_upper = q.a_mode == A_IM2COL;
              m.im2col_upper[0] = q.upper[0]; m.im2col_upper[1] = q.upper[1];
              m.flops = 2.0 * q.M * x.c * static_cast<double>(q.K);
              L.add(std::move(m), {dy, qw, buf_ones, buf_zeros}, {qo});
            }
            const int dx = L.buf(xbytes);
            TrainOp sc = TrainLowering::vg(VF_PHASE_SCATTER,
                                           vg_grid_for(static_cast<int64_t>(B) * x.h * x.w * (x.c / 8)));
            for (int k = 0; k < 4; ++k) sc.vp[k] = bref(pbuf[k]);
            sc.vp[4] = bref(dx);
            sc.va.n[0] = static_cast<int64_t>(B) * x.h * x.w * (x.c / 8);
            const int sv[9] = {B, x.h, x.w, x.c, o.stride, o.pad_h, o.pad_w, o.kh, o.kw};
            std::memcpy(sc.va.i, sv, sizeof sv);
            L.add(std::move(sc), {pbuf[0], pbuf[1], pbuf[2], pbuf[3]}, {dx});
            acc(pred, dx, xbytes);
            break;
          }
          const int wp = L.buf(static_cast<size_t>(dg.rows) * dg.Kpad * 2);
          {
            const int32_t iv[14] = {o.c_out, x.c, o.kh, o.kw, dg.cread, dg.Kpad, dg.rows, 0, 0, 0, 0, 0, 0, 0};
            L.filter_job(pref(i, 0), wp, iv);
          }
          int src = dy;
          if (o.stride > 1) {
            src = L.buf(static_cast<size_t>(B) * dg.Hdd * dg.Wdd * o.c_out * 2);
            TrainOp dl = TrainLowering::vg(VF_DILATE, vg_grid_for(static_cast<int64_t>(B) * dg.Hdd * dg.Wdd * (o.c_out / 8)));
            dl.vp[0] = bref(dy); dl.vp[1] = bref(src);
            const int iv[7] = {B, dg.Hd, dg.Wd, o.c_out, o.stride, dg.Hdd, dg.Wdd};
            std::memcpy(dl.va.i, iv, sizeof iv);
            L.add(std::move(dl), {dy}, {src});
          }
          const int dx = L.buf(xbytes);
          TrainOp m;
          m.kind = DK_GEMM;
          m.gemm_kind = 1;
          OpDev& d = m.gd;
          std::memset(&d, 0, sizeof d);
          d.kind = DK_GEMM; d.act = ACT_NONE;
          d.B = B; d.H = dg.Hdd; d.W = dg.Wdd; d.C = dg.cread; d.ldi = o.c_out;
          d.Ho = x.h; d.Wo = x.w; d.Cout = x.c; d.ldo = x.c;
          d.kh = o.kh; d.kw = o.kw; d.stride = 1; d.ph = dg.ph; d.pw = dg.pw; d.mrep = 1;
          d.M = dg.M; d.N = x.c; d.K = dg.K; d.Kpad = dg.Kpad;
          d.tiles_m = dg.tiles_m; d.tiles_n = dg.tiles_n; d.bm = BM; d.bn = dg.bn; d.split_k = 1; d.nkb = dg.nkb;
          d.ldw = dg.Kpad; d.a_mode = dg.a_mode;
          m.g_in = bref(src); m.g_out = bref(dx); m.g_wt = bref(wp);
          m.g_scale = bref(buf_ones); m.g_bias = bref(buf_zeros);
          m.im2col_c = o.c_out; m.a_ld = o.c_out; m.a_rows = dg.M; m.b_rows = dg.rows;
          m.flops = 2.0 * dg.M * x.c * static_cast<double>(o.c_out) * o.kh * o.kw;
          L.add(std::move(m), {src, wp, buf_ones, buf_zeros}, {dx});
          acc(pred, dx, xbytes);
        }
        break;
      }
    }
  }
  // ---- the update: SGD with momentum over the flat parameters
  L.step = 2 * n + 1;
  {
    TrainOp a = TrainLowering::vg(VF_SGD, vg_grid_for(np));
    a.vp[0] = bref(T.buf_params); a.vp[1] = bref(T.buf_grads); a.vp[2] = bref(T.buf_mom);
    a.va.n[0] = np; a.va.i[0] = 0; a.va.f[0] = T.lr; a.va.f[1] = T.momentum;
    a.bytes = 5.0 * 4.0 * static_cast<double>(np);   // read w, g, buf; write w, buf
    L.add(std::move(a), {T.buf_params, T.buf_grads, T.buf_mom}, {T.buf_params, T.buf_mom});
  }
  L.finish_filters();
  T.flops = 0;
  for (const TrainOp& o : T.tops) T.flops += o.flops;
  return 0;
}

}  // namespace

namespace {

bool has_train_tenant() {
  for (const Tenant& T : S.tenants) if (T.train) return true;
  return false;
}

// device address of a symbolic training-tenant buffer reference
void* tref_addr(const Tenant& T, const TRef& r) {
  char* base = nullptr;
  if (r.buf >= 0) base = static_cast<char*>(T.tbufs[r.buf]);
  else if (r.buf == TBUF_IN) base = const_cast<char*>(static_cast<const char*>(T.in_dev));
  else if (r.buf == TBUF_OUT) base = static_cast<char*>(T.out_dev);
  else if (r.buf == TBUF_LABELS) base = const_cast<char*>(static_cast<const char*>(T.labels_dev));
  return base ? base + r.off : nullptr;
}

// The OpDev of training op f with its buffers resolved; GEMM ops also get
// their tensor maps encoded into maps[0..2] (A, B, output) when every buffer
// exists (device mode, I/O bound).
int build_train_opdev(const Tenant& T, int tenant_id, const TrainOp& op, OpDev& d, CUtensorMap* maps, bool encode) {
  if (op.kind == DK_VGRID) {
    std::memset(&d, 0, sizeof d);
    d.kind = DK_VGRID;
    d.tenant = tenant_id;
    d.vfn = op.vfn;
    d.vblocks = op.vblocks;
    d.bm = op.per;
    d.tiles_m = op.items;
    d.tiles_n = 1;
    d.split_k = 1;
    d.va = op.va;
    for (int j = 0; j < 8; ++j) d.va.p[j] = tref_addr(T, op.vp[j]);
    return 0;
  }
  d = op.gd;
  d.tenant = tenant_id;
  d.in = tref_addr(T, op.g_in);
  d.out = tref_addr(T, op.g_out);
  d.wt = tref_addr(T, op.g_wt);
  d.partial = static_cast<float*>(tref_addr(T, op.g_part));
  d.scale = static_cast<const float*>(tref_addr(T, op.g_scale));
  d.bias = static_cast<const float*>(tref_addr(T, op.g_bias));
  d.c_tma = 0;
  if (!encode || !d.in || !d.wt) return 0;
  int rc = 0;
  if (d.a_mode == A_MN || d.a_mode == A_MN8) {
    WgradGeom wg;
    rc = wgrad_geom(d.B, d.H, d.W, d.C, d.M, d.kh, d.kw, d.stride, d.ph, d.pw, wg);
    if (!rc) rc = wgrad_mn_setup(d, maps, d.wt, d.in, d.B, d.H, d.W, d.C, d.M, d.kh, d.kw, d.stride, d.ph, d.pw, wg, true);
    if (rc) return rc;
  } else {
    if (d.a_mode == A_IM2COL)
      rc = encode_im2col(&maps[0], d, op.im2col_c, BM, BK, CU_TENSOR_MAP_SWIZZLE_128B,
                         op.has_upper ? op.im2col_upper : nullptr);
    else if (d.a_mode == A_IM2COL8) rc = encode_im2col(&maps[0], d, op.im2col_c, BM, 8, CU_TENSOR_MAP_SWIZZLE_NONE);
    else if (d.a_mode == A_ROWS) rc = encode_rows(&maps[0], d.in, op.gemm_kind == 2 ? d.Kpad : d.K, op.a_rows, op.a_ld, BM);
    if (!rc && d.a_mode != A_IM2COL8) rc = encode_rows(&maps[1], d.wt, d.Kpad, op.b_rows, d.Kpad, d.bn);
    if (rc) return rc;
  }
  if (op.gemm_kind != 2 && d.out && (static_cast<long long>(d.ldo) * 2) % 16 == 0) {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(d.Cout), static_cast<cuuint64_t>(d.M)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(d.ldo) * 2};
    const cuuint32_t box[2] = {64u, 32u};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = g_encode_tiled(&maps[2], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d.out, dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(GACER_E_CUDA, "training op: output tensor map (%d)", static_cast<int>(r));
    d.c_tma = 1;
  }
  return 0;
}

int upload_train_tenant(Tenant& T) {
  for (size_t b = 0; b < T.tbufs.size(); ++b) {
    CUDA_TRY(cudaMalloc(&T.tbufs[b], T.tbuf_bytes[b]));
    CUDA_TRY(cudaMemset(T.tbufs[b], 0, T.tbuf_bytes[b]));   // zero: padding rows, momentum, gradients
  }
  if (T.fall_table >= 0) {   // the filter op's job table with resolved pointers
    std::vector<FilterJob> jt(T.fjobs.size());
    int64_t start = 0;
    for (size_t k = 0; k < T.fjobs.size(); ++k) {
      std::memset(&jt[k], 0, sizeof jt[k]);
      jt[k].w = static_cast<const float*>(tref_addr(T, T.fjobs[k].w));
      jt[k].out = tref_addr(T, T.fjobs[k].out);
      jt[k].start = start;
      std::memcpy(jt[k].i, T.fjobs[k].i, sizeof jt[k].i);
      start += T.fjobs[k].n;
    }
    CUDA_TRY(cudaMemcpy(T.tbufs[T.fall_table], jt.data(), jt.size() * sizeof(FilterJob), cudaMemcpyHostToDevice));
  }
  CUDA_TRY(cudaMemcpy(T.tbufs[T.buf_params], T.h_params.data(), T.h_params.size() * 4, cudaMemcpyHostToDevice));
  const auto ones = T.param_slice.at({-1, 0});
  CUDA_TRY(launch_fill(static_cast<float*>(T.tbufs[ones.first]), static_cast<int>(ones.second), 1.0f, nullptr));
  CUDA_TRY(cudaDeviceSynchronize());
  std::vector<float>().swap(T.h_params);
  return 0;
}

}  // namespace
