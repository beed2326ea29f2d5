/*
 * gacer.h -- C ABI of the B200-native GACER multi-tenant executor.
 *
 * GACER (arXiv 2304.11745, "Granularity-Aware ConcurrEncy Regulation for
 * Multi-Tenant Deep Learning") regulates the concurrent execution of N tenant
 * DNNs M_1..M_n on one GPU (§4.1 l.603-607) with
 *   - spatial regulation: an operator O^B is decomposed into chunks
 *     O^{B^1},...,O^{B^j}, sum B^j = B (Eq. 5, l.657-668), selected by a mask
 *     list and list_B (l.683-684); plus channel split (north_star addition);
 *   - temporal regulation: per-model pointer lists P_n forming Matrix_P
 *     (Eq. 7, l.742-753) that cut every DFG into segments; same-index
 *     segments of all models form a cluster deployed together (Eq. 6,
 *     l.723-739); a pointer is a synchronisation point (l.767-771).
 *
 * This library executes one *round* (every registered tenant's forward once)
 * under such a plan with ONE persistent sm_100a kernel: operator chunks are
 * pulled from per-tenant device work queues, pointers are enforced by
 * device-side cluster counters (no host stream events), producer->consumer
 * order by device-side dependency counters.
 *
 * The training tenant's operators (conv forward / dgrad /
 * wgrad on the same tcgen05 path, BN-train, pooling / FC backward,
 * softmax-CE, SGD) are declared in gacer_train.h.
 *
 * Conventions (all calls):
 *   - return value >= 0 on success (an id where documented), else a negative
 *     gacer_status; gacer_last_error() then holds a message.
 *   - all pointer arguments are HOST pointers unless named *_dev.
 *   - the library is not thread-safe; one process drives one GPU.
 *   - a CUDA error is sticky: every later call returns GACER_E_CUDA.
 */
#ifndef GACER_H_
#define GACER_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- status */
typedef enum {
  GACER_OK = 0,
  GACER_E_INVALID_ARG = -1,
  GACER_E_DUPLICATE_ID = -2,            /* two ops share an id */
  GACER_E_UNKNOWN_PREDECESSOR = -3,     /* pred id not in the graph */
  GACER_E_CYCLE = -4,                   /* dependency cycle */
  GACER_E_UNSUPPORTED_OP = -5,          /* op kind / pattern not lowered               */
  GACER_E_CHUNK_SUM_MISMATCH = -6,      /* sum of list_B != B (Eq. 5, l.662)            */
  GACER_E_MASKED_OP_MISSING_CHUNKS = -7,/* axis set but no sizes */
  GACER_E_CUT_OUT_OF_RANGE = -8,        /* pointer outside [0, n_ops] */
  GACER_E_UNSORTED_CUTS = -9,           /* pointers decrease */
  GACER_E_POINTER_COUNT_MISMATCH = -10, /* "Each P has the same number of pointers" (l.753) */
  GACER_E_STATE = -11,                  /* call out of order (no init / no tenants / unbound I/O) */
  GACER_E_OOM = -12,
  GACER_E_CUDA = -13,                   /* sticky CUDA error */
  GACER_E_DEADLOCK = -14,               /* device watchdog fired (spin budget exceeded) */
  GACER_E_SHAPE = -15                   /* inconsistent tensor shapes in the graph */
} gacer_status;

/* ------------------------------------------------------------- operators */
/* PyTorch eval-mode semantics. */
typedef enum {
  GACER_OP_CONV2D = 1,  /* c_in c_out kh kw stride pad_h pad_w groups (1 or c_in==c_out); weight OIHW */
  GACER_OP_LINEAR = 2,  /* c_in c_out; weight [c_out][c_in]; input flattened in NCHW order */
  GACER_OP_MAXPOOL = 3, /* kh kw stride pad_h pad_w; floor mode, -inf padding */
  GACER_OP_AVGPOOL = 4, /* kh kw stride pad_h pad_w; flags & COUNT_INCLUDE_PAD */
  GACER_OP_GAP = 5,     /* adaptive average pool to 1x1 */
  GACER_OP_ADD = 6,     /* 2 preds, elementwise */
  GACER_OP_CONCAT = 7,  /* n preds, channel axis */
  GACER_OP_BN = 8,      /* inference BatchNorm2d: bn_gamma/beta/mean/var [c_out], bn_eps */
  GACER_OP_RELU = 9,
  GACER_OP_RELU6 = 10,
  GACER_OP_FLATTEN = 11, /* NCHW-order flatten (identity on the data; reorders LINEAR weights) */
  GACER_OP_DROPOUT = 12, /* identity (inference) */
  GACER_OP_HARDSWISH = 13,   /* x * relu6(x + 3) / 6 (MobileNetV3, "M3") */
  GACER_OP_HARDSIGMOID = 14, /* relu6(x + 3) / 6 (the squeeze-and-excitation gate) */
  GACER_OP_MUL = 15          /* 2 preds: x [C,H,W] * s [C,1,1] broadcast over H, W (SE channel scale) */
} gacer_op_kind;

typedef enum { GACER_DTYPE_BF16 = 1, GACER_DTYPE_FP32 = 2 } gacer_dtype;
typedef enum { GACER_AXIS_NONE = 0, GACER_AXIS_BATCH = 1, GACER_AXIS_CHANNEL = 2 } gacer_axis;
enum { GACER_FLAG_BIAS = 1, GACER_FLAG_COUNT_INCLUDE_PAD = 2 };

/* One operator O_{n,i} (SPEC OperatorSpec S:27).
 * Parameter arrays are HOST float32 arrays; they are copied (and, for BF16
 * graphs, rounded to bf16 RNE and repacked) during gacer_register_tenant, so
 * the caller may free them on return.  Unused fields are ignored. */
typedef struct {
  int32_t id;                 /* unique within the tenant, >= 1; id 0 = the graph input */
  int32_t kind;               /* gacer_op_kind */
  int32_t n_preds;
  const int32_t* preds;       /* predecessor ids, each < this op's position in issue order */
  int32_t c_in, c_out, kh, kw, stride, pad_h, pad_w, groups;
  int32_t flags;              /* GACER_FLAG_* */
  const float* weight;        /* CONV2D: [c_out][c_in/groups][kh][kw]; LINEAR: [c_out][c_in] */
  const float* bias;          /* [c_out] when flags & GACER_FLAG_BIAS */
  const float* bn_gamma;      /* BN: [c_out] each */
  const float* bn_beta;
  const float* bn_mean;
  const float* bn_var;
  float bn_eps;
} gacer_op_desc;

/* A tenant DFG M_n = [O_{n,1},...,O_{n,i}] in topological issue order
 * (l.605-607).  The last op is the tenant's output. */
typedef struct {
  int32_t n_ops;
  const gacer_op_desc* ops;
  int32_t in_c, in_h, in_w;   /* per-sample input shape (C, H, W) */
  int32_t dtype;              /* gacer_dtype of activations/weights on the GPU */
  int32_t train;              /* 1: a TRAINING tenant (the
                                 techniques "are applicable to both the training and inference
                                 phases").  Its round is one SGD step: BN in training mode
                                 (per-batch statistics), mean softmax cross-entropy over the
                                 labels (gacer_bind_labels), backward, SGD with momentum
                                 (lr, momentum; PyTorch semantics).  dtype must be BF16; the
                                 graph is a ResNet-style DFG (conv without bias, BN, ReLU fused
                                 into its BN / residual-add producer, add, max-pool, GAP,
                                 flatten, a final LINEAR producing the logits); other patterns
                                 return GACER_E_UNSUPPORTED_OP.  Pointers index its step
                                 (gacer_sync_pointers); it takes no decomposition. */
  float lr, momentum;
} gacer_graph;

/* Spatial regulation for one operator: the mask entry and list_B (l.667,
 * l.683-684).  op_index is the 1-based position of the op in the tenant's
 * ORIGINAL (pre-fusion) op list.  axis BATCH: sizes sum to the batch (Eq. 5);
 * axis CHANNEL: sizes sum to c_out.
 * sm_budget (nullable; [n_chunks], each >= 0, 0 = unlimited): the chunk's
 * resource share W(O^B) (l.597-601; "by controlling the number j, we can
 * control the spatial granularity", l.667-668): at most sm_budget[j] items of
 * chunk j are claimed-and-not-complete at any time, so the chunk occupies at
 * most that many SMs (one item runs on one SM; the others serve other
 * tenants).  Enforced on the device by a per-chunk semaphore counter; it
 * changes WHEN tiles run, never what they compute (results are bit-identical
 * with and without budgets).  A single chunk (n_chunks = 1, sizes = {B})
 * budgets an undecomposed operator.  Negative values: GACER_E_INVALID_ARG. */
typedef struct {
  int32_t tenant;
  int32_t op_index;
  int32_t axis;               /* gacer_axis */
  int32_t n_chunks;
  const int32_t* sizes;       /* [n_chunks], each >= 1 */
  const int32_t* sm_budget;   /* [n_chunks] max items in flight per chunk, 0 = unlimited; may be NULL */
} gacer_chunking;

typedef struct {
  int32_t n;
  const gacer_chunking* items; /* ops not listed: mask(O) = 0 (not decomposed) */
} gacer_decomposition;

/* Matrix_P (Eq. 7, l.742-753): cuts[t * n_pointers + j] is the j-th pointer
 * of tenant t (registration order).  A cut p is the segment boundary after
 * original op p; cuts are non-decreasing in [0, n_ops]; repeated / zero cuts
 * give empty segments (the paper's [None], Eq. 6 l.730).  Cluster k = the
 * k-th segment of every tenant; no op of cluster k+1 starts before every op
 * of cluster k has finished. */
typedef struct {
  int32_t n_tenants;          /* must equal the number of registered tenants */
  int32_t n_pointers;         /* |P_n|, the same for every tenant */
  const int32_t* cuts;        /* [n_tenants][n_pointers] */
} gacer_sync_pointers;

/* Execution mode of gacer_run_round*.  EXECUTOR is the method; the other two
 * are the paper's baselines run on the SAME tile functions. */
typedef enum {
  GACER_MODE_EXECUTOR = 0,    /* one persistent multi-tenant kernel per round */
  GACER_MODE_SEQUENTIAL = 1,  /* "CuDNN-Seq": one kernel per fused op, one stream, tenant after tenant */
  GACER_MODE_MULTISTREAM = 2, /* "Stream-Parallel": one kernel per fused op, one stream per tenant */
  GACER_MODE_EXECUTOR_HOSTSYNC = 3 /* the executor with the paper's CPU-side pointers: one launch per
                                      cluster (pointer segment), the host synchronising with the GPU
                                      between them (T_SW of Eq. 8); same results, measurement only */
} gacer_mode;

typedef enum {
  GACER_PARTITION_PRIORITY = 0,        /* default.  No tenant ownership: every CTA claims the ready item
                                          of highest upward rank over all tenants (global list
                                          scheduling, HEFT-style); the SM shares only order ties */
  GACER_PARTITION_WORK_CONSERVING = 1, /* each CTA prefers one tenant (SM share), steals from the others */
  GACER_PARTITION_STRICT = 2,          /* each CTA serves only its tenant (SM share per tenant) */
  GACER_PARTITION_HYBRID = 3           /* like WORK_CONSERVING, except that CTAs of the other tenants
                                          never take the bulk tenant's (largest share) items: its long
                                          tiles cannot delay the latency-bound chains */
} gacer_partition;

typedef struct {
  int32_t num_ctas;           /* executor grid; 0 = #SMs */
  int32_t partition;          /* gacer_partition */
  int32_t watchdog_ms;        /* device spin budget before GACER_E_DEADLOCK; 0 = 2000 */
  int32_t trace;              /* 1 = record per-item (tenant, op, sm, t0, t1) */
  int32_t coarse_deps;        /* 1 = an item waits for whole producer chunks (the paper's
                                 op-level dependency); 0 (default) = only for the producer
                                 M-tiles its input window reads (tile wavefront).  Results
                                 are bit-identical either way. */
} gacer_options;

#define GACER_MAX_STAT_TENANTS 16   /* tenants with per-tenant occupancy counters */

typedef struct {
  double last_round_ms;       /* device time of the last round (CUDA events) */
  int64_t n_items;            /* work items per round under the current plan */
  int32_t n_clusters;         /* |P| + 1 */
  int32_t n_fused_ops;        /* lowered ops over all tenants */
  int32_t kernel_launches;    /* kernels launched by the last round */
  int32_t n_tenants;
  double tensor_flops;        /* algorithmic conv+FC FLOPs per round (2*MAC) */
  double cc_bytes;            /* algorithmic bytes of the CUDA-core ops per round */
  /* Executor occupancy (the Fig. 8 analog, §5.3 l.979-981), from
   * device counters every executor round accumulates; averaged over the
   * executor rounds since the previous gacer_get_stats call (0 if none): */
  int32_t stat_rounds;        /* executor rounds the figures below average over */
  int32_t pad0;
  double tenant_sm_ns[GACER_MAX_STAT_TENANTS]; /* per tenant: sum over its items of (release - claim)
                                 time on its CTA (SM-ns; items pipelined inside one CTA overlap) */
  double barrier_wait_ns;     /* sum over CTAs of the time spent waiting at sync pointers
                                 (cluster barriers, A5) -- the device T_SW (CTA-ns) */
  double ready_wait_ns;       /* sum over CTAs of the time spent with unclaimed but unready work
                                 (dependency stalls; CTA-ns) */
} gacer_round_stats;

typedef struct {
  int32_t n_orig_ops;         /* ops given at registration */
  int32_t n_fused_ops;        /* ops after conv+BN+add+act fusion */
  int32_t batch;
  int32_t in_c_pad;           /* channel stride of the NHWC input buffer */
  int32_t in_h, in_w;
  int32_t out_features;       /* output row length (float32) */
  int64_t in_bytes;           /* bytes of the input buffer: batch*in_h*in_w*in_c_pad*elem */
  int64_t out_bytes;          /* batch*out_features*4 */
  double flops;               /* algorithmic FLOPs of one forward */
  int32_t gemm_ops;           /* fused ops on the tcgen05 GEMM tile path */
  int32_t mpair_ops;          /* ... of them with 256-row (M-pair) tiles */
  int32_t split_k_ops;        /* ... of them with a fixed split-K > 1 */
  int32_t swap_ops;           /* ... of them swap-AB linears (weights = the M operand) */
  int32_t wide_ops;           /* ... of them with 128x256 tiles */
  int32_t cc_ops;             /* fused ops on CUDA cores (depthwise, pools, GAP, eltwise, SIMT) */
  int32_t train;              /* 1: a training tenant (its round is one SGD step) */
  int32_t n_steps;            /* training: 2 n_orig_ops + 1 step positions (pointer range) */
  int64_t n_params;           /* training: floats in the flat parameter buffer */
  int32_t op_base;            /* global executor index of the tenant's first operator */
  int32_t reused_tensors;     /* activation tensors placed in an earlier tensor's buffer
                                 (liveness-based reuse: set GACER_REUSE=1
                                 before registration; off by default) */
  int64_t act_bytes;          /* device bytes of the tenant's activation buffers */
  int64_t act_bytes_private;  /* ... if every activation tensor had its own buffer */
} gacer_tenant_info;

/* Device buffers of a training tenant (library-owned; valid until
 * gacer_shutdown).  Flat fp32 parameter / gradient / momentum buffers in
 * registration order: CONV2D weight [c_out][c_in padded to 8][kh][kw], BN
 * gamma then beta, LINEAR weight [c_out][c_in] then bias (gacer_train_param
 * gives each slice). */
typedef struct {
  const float* loss;          /* 1 float: the step's mean softmax cross-entropy */
  float* params;              /* master weights, updated in place by each round's SGD step */
  const float* grads;         /* gradients of the last step */
  float* momentum;            /* SGD momentum buffers (zero before the first step) */
  int64_t n_params;
  int32_t n_ops;              /* executor ops of one step */
  int32_t pad;
} gacer_train_state;

/* ------------------------------------------------------------------ calls */

/* Bind the calling process to `cuda_device` (>= 0).  cuda_device = -1 opens
 * a HOST-ONLY instance: registration and plan compilation run (validation,
 * lowering, Eq. 6/7 segmentation) but nothing touches a GPU and run calls
 * return GACER_E_STATE.  opts may be NULL (defaults). */
int gacer_init(int cuda_device, const gacer_options* opts);
int gacer_shutdown(void);

/* Register tenant M_n with its batch B (>= 1).  Validates the DFG (ids,
 * predecessors, acyclicity, topological issue order, shapes), fuses
 * conv+BN(+add)(+ReLU/ReLU6), linear(+ReLU), elides dropout/flatten, turns
 * concat into channel-offset writes, and (device mode) packs the weights
 * into library-owned device memory.  Resets the regulation to the identity
 * plan (no chunks, no pointers).  Returns the tenant id (0, 1, ...). */
int gacer_register_tenant(const gacer_graph* graph, int32_t batch);

int gacer_get_tenant_info(int tenant, gacer_tenant_info* out);

/* Bind caller-owned DEVICE buffers.  input_dev: NHWC [B][in_h][in_w][in_c_pad]
 * of the graph dtype, padding channels zero.  output_dev: float32
 * [B][out_features] -- the last op's output in NHWC order [B][H][W][C]
 * (logits [B][classes] for a 1x1 output).  Both 16-byte aligned; both must
 * outlive every round that uses them. */
int gacer_bind_io(int tenant, const void* input_dev, void* output_dev);

/* Training tenants: bind the int32 [B] labels (device, 4-byte aligned; must
 * outlive the rounds using it); the graph input is bound with gacer_bind_io
 * (NHWC bf16 images) together with the float32 [B][classes] logits buffer. */
int gacer_bind_labels(int tenant, const void* labels_dev);
int gacer_get_train_state(int tenant, gacer_train_state* out);
/* Offset and length (floats) of parameter `which` (0: conv/linear weight or
 * BN gamma; 1: linear bias or BN beta) of ORIGINAL op op_index (1-based) in
 * the flat buffers. */
int gacer_train_param(int tenant, int32_t op_index, int32_t which, int64_t* offset, int64_t* count);

/* Install a regulation plan (mask/list_B/list_C and Matrix_P).  Either
 * argument may be NULL (no decomposition / no pointers).  Atomic: on error
 * the previous plan stays in force. */
int gacer_set_regulation(const gacer_decomposition* decomposition,
                         const gacer_sync_pointers* sync_pointers);

/* ---- A12: data-parallel gradient exchange of a training tenant (north_star:
 * "NCCL over NVLink is used only for the gradient all-reduce of data-parallel
 * training tenants").  The round's backward writes
 * the flat gradients; with the exchange enabled the SGD update additionally
 * waits for a per-tenant gradient gate.  The caller (one process per GPU,
 * torch.distributed / NCCL) enqueues on a communication stream, per bucket:
 * gacer_stream_wait_grads (device-side waits for the ops producing that
 * slice of the gradients, so the all-reduce of the last layers overlaps the
 * rest of the backward), its all-reduce + 1/G, and after the last bucket
 * gacer_stream_open_grad_gate.  Launch the executor with fewer CTAs than SMs
 * (gacer_options.num_ctas) so the collective's kernels find free SMs. */

/* Enable (1) / disable (0) the gradient gate of training tenant `tenant`
 * (recompiles the current plan; drains the device). */
int gacer_train_set_allreduce(int tenant, int32_t enable);

/* Buckets over the flat gradient buffer, last layers first: whole parameter
 * slices grouped up to bucket_bytes (a larger single slice is its own
 * bucket).  out[2b] = float offset, out[2b+1] = float count (out may be NULL
 * to count).  Returns the number of buckets. */
int gacer_train_buckets(int tenant, int64_t bucket_bytes, int64_t* out, int32_t cap);

/* Enqueue on `stream` a device-side wait until every op writing gradient
 * floats [offset, offset + count) of the most recently enqueued round has
 * completed (executor: cuStreamWaitValue32 on their completion counters;
 * baseline modes: the round's backward-done event). */
int gacer_stream_wait_grads(void* stream, int tenant, int64_t offset, int64_t count);

/* Enqueue on `stream` the opening of the tenant's gradient gate for the most
 * recently enqueued round (its SGD update may then run). */
int gacer_stream_open_grad_gate(void* stream, int tenant);

/* Cluster index of every ORIGINAL op of `tenant` under the current plan
 * (out[i] for op i+1), i.e. Eq. 6/7 as compiled.  n = capacity of out. */
int gacer_query_op_clusters(int tenant, int32_t* out, int32_t n);

/* Fused operator of every ORIGINAL op of `tenant` (out[i] for op i+1): the
 * tenant-local index of the executor operator that computes it (conv + BN +
 * add + activation lowered into one), -1 for aliases (flatten, dropout,
 * concat).  The executor's global op index (device trace, gacer_describe_op)
 * is gacer_tenant_info.op_base + out[i].  For the planner's lookup table
 * (W and T per operator).  Inference tenants only. */
int gacer_query_op_fused(int tenant, int32_t* out, int32_t n);

/* SM partition of the executor (the paper's resource share W, §4.1
 * l.597-601): shares[t] > 0 is tenant t's relative share of the executor's
 * CTAs; each CTA serves its tenant's ready items first and (in the
 * work-conserving partition) other tenants' items when its own has none
 * ready.  n = 0 / shares = NULL restores the automatic shares (each tenant's
 * SM need: estimated work / chain latency).  Part of the regulation state;
 * reset by gacer_register_tenant. */
int gacer_set_sm_shares(const float* shares, int32_t n);

/* Switch the SM-partition policy (gacer_partition) of the executor; the
 * initial value comes from gacer_options.partition.  Together with the
 * shares it forms the spatial part of the regulation: bench.py sweeps both.
 * GACER_E_INVALID_ARG for an unknown policy (the previous one stays). */
int gacer_set_partition(int32_t partition);

int gacer_set_mode(int mode);               /* gacer_mode */

/* One round: every tenant's forward once on its bound input.
 * gacer_run_round blocks until the outputs are visible;
 * gacer_run_round_async enqueues on `stream` (a cudaStream_t; NULL = the
 * library stream) and returns. */
int gacer_run_round(void);
int gacer_run_round_async(void* stream);

/* The baselines as CUDA graphs (sequential and multi-stream
 * "reported plain and with CUDA Graphs"; the paper's Stream-Parallel
 * comparator, §5.1 l.925).  gacer_capture_baseline(mode), mode =
 * GACER_MODE_SEQUENTIAL or GACER_MODE_MULTISTREAM, captures ONE round of that
 * mode's per-op launches (the same tile functions, order and stream topology
 * as gacer_run_round in that mode) into a library-owned CUDA graph, replacing
 * any previous capture; the current mode is left unchanged.  Needs bound I/O.
 * gacer_run_baseline_graph(stream) replays it on `stream` (NULL = the
 * library stream); gacer_get_stats().kernel_launches then reports the
 * captured round's kernel count.  Re-registration or re-binding I/O discards
 * the capture (GACER_E_STATE until captured again).  Outputs are
 * byte-identical to the executor's. */
int gacer_capture_baseline(int mode);
int gacer_run_baseline_graph(void* stream);

/* End-to-end round with HOST buffers: copies host_inputs[t] (layout as
 * gacer_bind_io, pinned memory recommended) to the bound device inputs, runs
 * the round, copies every output to host_outputs[t]; blocks.  Arrays are
 * indexed by tenant id.  gacer_get_stats().last_round_ms then covers the
 * copies and the round (CUDA events on the library stream). */
int gacer_run_round_host(const void* const* host_inputs, void* const* host_outputs);

int gacer_get_stats(gacer_round_stats* out);

/* Trace of the last executor round (options.trace = 1): up to `cap` records
 * of 10 int64 each, indexed by work item: tenant, global fused-op index, SM
 * id, item index, cluster, chunk counter, t_claim_ns, t_release_ns,
 * t_mma_start_ns, t_epilogue_start_ns (%globaltimer; the last two are 0 for
 * CUDA-core items).  Returns the number of records written. */
int gacer_get_trace(int64_t* records, int32_t cap);

const char* gacer_last_error(void);

/* Describe lowered op `op` of the global op table (the op field of
 * gacer_get_trace records): out[8] = {device kind, virtual-grid function,
 * items per round, tenant, GEMM tile N, K-blocks, algorithmic bytes (inputs +
 * outputs + weights, capped at 2^31 - 1), MFLOP}.  Diagnostics and the
 * planner's lookup table. */
int gacer_describe_op(int32_t op, int32_t* out);

/* Diagnostics only (not on the method's path): when the process runs with
 * GACER_DEBUG_TIMING=1, kernels record %globaltimer milestones per CTA
 * ([op slot][cta][16] int64; executor rounds use slot 0).  Copies up to cap
 * values to out (may be NULL), optionally zeroes the buffer.  Returns the
 * count copied. */
int gacer_debug_timing(int64_t* out, int64_t cap, int reset);

#ifdef __cplusplus
}
#endif
#endif /* GACER_H_ */
