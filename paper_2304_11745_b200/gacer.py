"""Thin ctypes binding of libgacer.so (include/gacer.h).

Argument marshalling only: every step of the path runs in the library and
its sm_100a kernels.  There is no Python or CPU fallback -- if the library is
missing this module raises at import of ``lib()``.

Function names mirror the C ABI (gacer_init, gacer_register_tenant,
gacer_set_regulation, gacer_run_round, ...).  ``graph_desc`` and
``regulation_desc`` marshal the plain-data graph / plan descriptions used by
the tests and bench into the C structs (keeping the backing arrays alive).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# GACER_LIB selects an alternative build of the same library (A/B timing of
# kernel variants on one box); default: the in-tree build.
LIB_PATH = os.environ.get("GACER_LIB") or os.path.join(_HERE, "libgacer.so")

# ---------------------------------------------------------------- constants
OK = 0
E = {
    -1: "GACER_E_INVALID_ARG", -2: "GACER_E_DUPLICATE_ID", -3: "GACER_E_UNKNOWN_PREDECESSOR",
    -4: "GACER_E_CYCLE", -5: "GACER_E_UNSUPPORTED_OP", -6: "GACER_E_CHUNK_SUM_MISMATCH",
    -7: "GACER_E_MASKED_OP_MISSING_CHUNKS", -8: "GACER_E_CUT_OUT_OF_RANGE", -9: "GACER_E_UNSORTED_CUTS",
    -10: "GACER_E_POINTER_COUNT_MISMATCH", -11: "GACER_E_STATE", -12: "GACER_E_OOM", -13: "GACER_E_CUDA",
    -14: "GACER_E_DEADLOCK", -15: "GACER_E_SHAPE",
}
STATUS = {v: k for k, v in E.items()}

OP = {"conv": 1, "linear": 2, "maxpool": 3, "avgpool": 4, "gap": 5, "add": 6, "concat": 7,
      "bn": 8, "relu": 9, "relu6": 10, "flatten": 11, "dropout": 12,
      "hardswish": 13, "hardsigmoid": 14, "mul": 15}
DTYPE = {"bf16": 1, "fp32": 2}
AXIS = {"none": 0, "batch": 1, "channel": 2}
MODE = {"executor": 0, "sequential": 1, "multistream": 2, "executor_hostsync": 3}
PARTITION = {"priority": 0, "work_conserving": 1, "strict": 2, "hybrid": 3}
FLAG_BIAS, FLAG_CIP = 1, 2

FP = C.POINTER(C.c_float)
IP = C.POINTER(C.c_int32)


class gacer_op_desc(C.Structure):
    _fields_ = [("id", C.c_int32), ("kind", C.c_int32), ("n_preds", C.c_int32), ("preds", IP),
                ("c_in", C.c_int32), ("c_out", C.c_int32), ("kh", C.c_int32), ("kw", C.c_int32),
                ("stride", C.c_int32), ("pad_h", C.c_int32), ("pad_w", C.c_int32), ("groups", C.c_int32),
                ("flags", C.c_int32), ("weight", FP), ("bias", FP), ("bn_gamma", FP), ("bn_beta", FP),
                ("bn_mean", FP), ("bn_var", FP), ("bn_eps", C.c_float)]


class gacer_graph(C.Structure):
    _fields_ = [("n_ops", C.c_int32), ("ops", C.POINTER(gacer_op_desc)), ("in_c", C.c_int32),
                ("in_h", C.c_int32), ("in_w", C.c_int32), ("dtype", C.c_int32), ("train", C.c_int32),
                ("lr", C.c_float), ("momentum", C.c_float)]


class gacer_chunking(C.Structure):
    _fields_ = [("tenant", C.c_int32), ("op_index", C.c_int32), ("axis", C.c_int32),
                ("n_chunks", C.c_int32), ("sizes", IP), ("sm_budget", IP)]


class gacer_decomposition(C.Structure):
    _fields_ = [("n", C.c_int32), ("items", C.POINTER(gacer_chunking))]


class gacer_sync_pointers(C.Structure):
    _fields_ = [("n_tenants", C.c_int32), ("n_pointers", C.c_int32), ("cuts", IP)]


class gacer_options(C.Structure):
    _fields_ = [("num_ctas", C.c_int32), ("partition", C.c_int32), ("watchdog_ms", C.c_int32),
                ("trace", C.c_int32), ("coarse_deps", C.c_int32)]


class gacer_round_stats(C.Structure):
    _fields_ = [("last_round_ms", C.c_double), ("n_items", C.c_int64), ("n_clusters", C.c_int32),
                ("n_fused_ops", C.c_int32), ("kernel_launches", C.c_int32), ("n_tenants", C.c_int32),
                ("tensor_flops", C.c_double), ("cc_bytes", C.c_double), ("stat_rounds", C.c_int32),
                ("pad0", C.c_int32), ("tenant_sm_ns", C.c_double * 16), ("barrier_wait_ns", C.c_double),
                ("ready_wait_ns", C.c_double)]


class gacer_tenant_info(C.Structure):
    _fields_ = [("n_orig_ops", C.c_int32), ("n_fused_ops", C.c_int32), ("batch", C.c_int32),
                ("in_c_pad", C.c_int32), ("in_h", C.c_int32), ("in_w", C.c_int32),
                ("out_features", C.c_int32), ("in_bytes", C.c_int64), ("out_bytes", C.c_int64),
                ("flops", C.c_double), ("gemm_ops", C.c_int32), ("mpair_ops", C.c_int32),
                ("split_k_ops", C.c_int32), ("swap_ops", C.c_int32), ("wide_ops", C.c_int32),
                ("cc_ops", C.c_int32), ("train", C.c_int32), ("n_steps", C.c_int32), ("n_params", C.c_int64),
                ("op_base", C.c_int32), ("reused_tensors", C.c_int32),
                ("act_bytes", C.c_int64), ("act_bytes_private", C.c_int64)]


class gacer_train_state(C.Structure):
    _fields_ = [("loss", C.c_void_p), ("params", C.c_void_p), ("grads", C.c_void_p), ("momentum", C.c_void_p),
                ("n_params", C.c_int64), ("n_ops", C.c_int32), ("pad", C.c_int32)]


EXPORTS = {
    "gacer_init": ([C.c_int, C.POINTER(gacer_options)], C.c_int),
    "gacer_shutdown": ([], C.c_int),
    "gacer_register_tenant": ([C.POINTER(gacer_graph), C.c_int32], C.c_int),
    "gacer_get_tenant_info": ([C.c_int, C.POINTER(gacer_tenant_info)], C.c_int),
    "gacer_capture_baseline": ([C.c_int], C.c_int),
    "gacer_run_baseline_graph": ([C.c_void_p], C.c_int),
    "gacer_bind_io": ([C.c_int, C.c_void_p, C.c_void_p], C.c_int),
    "gacer_bind_labels": ([C.c_int, C.c_void_p], C.c_int),
    "gacer_get_train_state": ([C.c_int, C.POINTER(gacer_train_state)], C.c_int),
    "gacer_train_param": ([C.c_int, C.c_int32, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], C.c_int),
    "gacer_set_regulation": ([C.POINTER(gacer_decomposition), C.POINTER(gacer_sync_pointers)], C.c_int),
    "gacer_query_op_clusters": ([C.c_int, IP, C.c_int32], C.c_int),
    "gacer_query_op_fused": ([C.c_int, IP, C.c_int32], C.c_int),
    "gacer_train_set_allreduce": ([C.c_int, C.c_int32], C.c_int),
    "gacer_train_buckets": ([C.c_int, C.c_int64, C.POINTER(C.c_int64), C.c_int32], C.c_int),
    "gacer_stream_wait_grads": ([C.c_void_p, C.c_int, C.c_int64, C.c_int64], C.c_int),
    "gacer_stream_open_grad_gate": ([C.c_void_p, C.c_int], C.c_int),
    "gacer_set_sm_shares": ([C.POINTER(C.c_float), C.c_int32], C.c_int),
    "gacer_set_partition": ([C.c_int32], C.c_int),
    "gacer_set_mode": ([C.c_int], C.c_int),
    "gacer_run_round": ([], C.c_int),
    "gacer_run_round_async": ([C.c_void_p], C.c_int),
    "gacer_run_round_host": ([C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)], C.c_int),
    "gacer_get_stats": ([C.POINTER(gacer_round_stats)], C.c_int),
    "gacer_get_trace": ([C.POINTER(C.c_int64), C.c_int32], C.c_int),
    "gacer_last_error": ([], C.c_char_p),
    "gacer_describe_op": ([C.c_int32, IP], C.c_int),
    "gacer_debug_timing": ([C.POINTER(C.c_int64), C.c_int64, C.c_int], C.c_int),
    # include/gacer_train.h: training-tenant CUDA-core steps (device pointers as ints, stream as int)
    "gacer_bn_partials": ([C.c_int64, C.c_int32], C.c_int32),
    "gacer_bn_train_fwd": ([C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p, C.c_float, C.c_int32,
                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int32),
    "gacer_bn_train_bwd": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p,
                            C.c_void_p, C.c_float, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p],
                           C.c_int32),
    "gacer_relu_bwd": ([C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p], C.c_int32),
    "gacer_maxpool_bwd": ([C.c_void_p, C.c_void_p] + [C.c_int32] * 11 + [C.c_void_p, C.c_void_p, C.c_void_p],
                          C.c_int32),
    "gacer_gap_bwd": ([C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p], C.c_int32),
    "gacer_linear_bwd": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                          C.c_void_p, C.c_void_p, C.c_void_p], C.c_int32),
    "gacer_conv_dgrad_workspace": ([C.c_int32] * 10, C.c_int64),
    "gacer_conv_dgrad": ([C.c_void_p, C.c_void_p] + [C.c_int32] * 10 + [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p],
                         C.c_int32),
    "gacer_conv_wgrad_workspace": ([C.c_int32] * 10, C.c_int64),
    "gacer_conv_wgrad": ([C.c_void_p, C.c_void_p] + [C.c_int32] * 10 + [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p],
                         C.c_int32),
    "gacer_conv_fwd_workspace": ([C.c_int32] * 10, C.c_int64),
    "gacer_conv_fwd": ([C.c_void_p, C.c_void_p] + [C.c_int32] * 10 + [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p],
                       C.c_int32),
    "gacer_maxpool_fwd": ([C.c_void_p] + [C.c_int32] * 11 + [C.c_void_p, C.c_void_p], C.c_int32),
    "gacer_add": ([C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p], C.c_int32),
    "gacer_gap_fwd": ([C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p], C.c_int32),
    "gacer_linear_fwd": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                          C.c_void_p], C.c_int32),
    "gacer_softmax_ce": ([C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                          C.c_void_p], C.c_int32),
    "gacer_sgd_momentum": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_float, C.c_float, C.c_int32,
                            C.c_void_p], C.c_int32),
}

_lib = None


def lib():
    """Load libgacer.so (built in-tree by __graft_entry__.build()).  Raises if
    absent: there is no fallback path."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built; run __graft_entry__.build()")
        _lib = C.CDLL(LIB_PATH)
        for name, (args, res) in EXPORTS.items():
            if os.environ.get("GACER_LIB") and not hasattr(_lib, name):
                continue          # an older A/B build may lack newer entry points
            f = getattr(_lib, name)
            f.argtypes = args
            f.restype = res
    return _lib


class GacerError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{E.get(code, code)}: {msg}")
        self.code = code
        self.name = E.get(code, str(code))


def _check(rc):
    if rc < 0:
        raise GacerError(rc, lib().gacer_last_error().decode())
    return rc


# ---------------------------------------------------------------- marshalling
def _fptr(a, keep):
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.float32)
    keep.append(a)
    return a.ctypes.data_as(FP)


def _iptr(a, keep):
    a = np.ascontiguousarray(a, dtype=np.int32)
    keep.append(a)
    return a.ctypes.data_as(IP)


def graph_desc(graph, params, dtype="bf16", train=False, lr=0.1, momentum=0.9):
    """Marshal a plain-data tenant graph (``graph.ops`` list of dicts,
    ``graph.in_c/in_h/in_w``) and its parameters into a gacer_graph.
    Returns (struct, keepalive)."""
    keep = []
    n = len(graph.ops)
    arr = (gacer_op_desc * n)()
    for i, op in enumerate(graph.ops):
        d = arr[i]
        d.id = op["id"]
        d.kind = OP[op["kind"]]
        d.n_preds = len(op["preds"])
        d.preds = _iptr(op["preds"], keep)
        p = params.get(op["id"], {})
        k = op["kind"]
        if k == "conv":
            d.c_in, d.c_out, d.kh, d.kw = op["c_in"], op["c_out"], op["kh"], op["kw"]
            d.stride, d.pad_h, d.pad_w, d.groups = op["stride"], op["ph"], op["pw"], op["groups"]
        elif k == "linear":
            d.c_in, d.c_out = op["c_in"], op["c_out"]
        elif k in ("maxpool", "avgpool"):
            d.kh, d.kw, d.stride, d.pad_h, d.pad_w = op["kh"], op["kw"], op["stride"], op["ph"], op["pw"]
            if k == "avgpool" and op.get("cip", True):
                d.flags |= FLAG_CIP
        elif k == "bn":
            d.c_out = op["c"]
            d.bn_eps = op["eps"]
            d.bn_gamma = _fptr(p["gamma"], keep)
            d.bn_beta = _fptr(p["beta"], keep)
            d.bn_mean = _fptr(p["mean"], keep)
            d.bn_var = _fptr(p["var"], keep)
        if "w" in p:
            d.weight = _fptr(p["w"], keep)
        if "b" in p:
            d.bias = _fptr(p["b"], keep)
            d.flags |= FLAG_BIAS
    keep.append(arr)
    g = gacer_graph(n_ops=n, ops=C.cast(arr, C.POINTER(gacer_op_desc)), in_c=graph.in_c,
                    in_h=graph.in_h, in_w=graph.in_w, dtype=DTYPE[dtype], train=int(bool(train)),
                    lr=float(lr), momentum=float(momentum))
    return g, keep


def regulation_desc(decomposition=None, pointers=None, n_tenants=None):
    """decomposition: list of (tenant, op_index (1-based), axis, sizes[, sm_budget]);
    pointers: list (per tenant) of cut lists.  Returns (dec*, ptr*, keep)."""
    keep = []
    dp = None
    if decomposition is not None:
        n = len(decomposition)
        arr = (gacer_chunking * max(n, 1))()
        for i, ent in enumerate(decomposition):
            t, oi, axis, sizes = ent[:4]
            budget = ent[4] if len(ent) > 4 else None   # per-chunk SM budgets (0 = unlimited)
            arr[i].tenant, arr[i].op_index = t, oi
            arr[i].axis = AXIS[axis] if isinstance(axis, str) else axis
            arr[i].n_chunks = len(sizes) if sizes is not None else 0
            arr[i].sizes = _iptr(sizes, keep) if sizes is not None else None
            arr[i].sm_budget = _iptr(budget, keep) if budget is not None else None
        keep.append(arr)
        dec = gacer_decomposition(n=n, items=C.cast(arr, C.POINTER(gacer_chunking)))
        keep.append(dec)
        dp = C.pointer(dec)
    pp = None
    if pointers is not None:
        nt = len(pointers) if n_tenants is None else n_tenants
        npt = len(pointers[0]) if pointers else 0
        flat = np.zeros(max(1, nt * npt), dtype=np.int32)
        for t, cuts in enumerate(pointers):
            flat[t * npt:(t + 1) * npt] = cuts
        sp = gacer_sync_pointers(n_tenants=nt, n_pointers=npt, cuts=_iptr(flat, keep))
        keep.append(sp)
        pp = C.pointer(sp)
    return dp, pp, keep


# ---------------------------------------------------------------- calls
def gacer_init(device=0, num_ctas=0, partition="priority", watchdog_ms=0, trace=False, coarse_deps=False):
    o = gacer_options(num_ctas=num_ctas, partition=PARTITION[partition], watchdog_ms=watchdog_ms,
                      trace=int(trace), coarse_deps=int(coarse_deps))
    return _check(lib().gacer_init(device, C.byref(o)))


def gacer_shutdown():
    return _check(lib().gacer_shutdown())


def gacer_register_tenant(graph, params, batch, dtype="bf16", train=False, lr=0.1, momentum=0.9):
    g, keep = graph_desc(graph, params, dtype, train, lr, momentum)
    rc = lib().gacer_register_tenant(C.byref(g), batch)
    del keep
    return _check(rc)


def gacer_get_tenant_info(tenant):
    info = gacer_tenant_info()
    _check(lib().gacer_get_tenant_info(tenant, C.byref(info)))
    return {f: getattr(info, f) for f, _ in gacer_tenant_info._fields_}


def gacer_bind_io(tenant, input_dev_ptr, output_dev_ptr):
    return _check(lib().gacer_bind_io(tenant, C.c_void_p(input_dev_ptr), C.c_void_p(output_dev_ptr)))


def gacer_bind_labels(tenant, labels_dev_ptr):
    return _check(lib().gacer_bind_labels(tenant, C.c_void_p(labels_dev_ptr)))


def gacer_get_train_state(tenant):
    st = gacer_train_state()
    _check(lib().gacer_get_train_state(tenant, C.byref(st)))
    return {f: (getattr(st, f) or 0) if f in ("loss", "params", "grads", "momentum") else getattr(st, f)
            for f, _ in gacer_train_state._fields_ if f != "pad"}


def gacer_train_param(tenant, op_index, which=0):
    off, cnt = C.c_int64(), C.c_int64()
    _check(lib().gacer_train_param(tenant, op_index, which, C.byref(off), C.byref(cnt)))
    return off.value, cnt.value


def gacer_set_regulation(decomposition=None, pointers=None, n_tenants=None):
    dp, pp, keep = regulation_desc(decomposition, pointers, n_tenants)
    rc = lib().gacer_set_regulation(dp, pp)
    del keep
    return _check(rc)


def gacer_query_op_clusters(tenant, n_ops):
    out = np.zeros(n_ops, dtype=np.int32)
    n = _check(lib().gacer_query_op_clusters(tenant, out.ctypes.data_as(IP), n_ops))
    return out[:n].tolist()


def gacer_query_op_fused(tenant, n_ops):
    out = np.zeros(n_ops, dtype=np.int32)
    n = _check(lib().gacer_query_op_fused(tenant, out.ctypes.data_as(IP), n_ops))
    return out[:n].tolist()


def gacer_train_set_allreduce(tenant, enable=True):
    return _check(lib().gacer_train_set_allreduce(tenant, int(bool(enable))))


def gacer_train_buckets(tenant, bucket_bytes):
    n = _check(lib().gacer_train_buckets(tenant, int(bucket_bytes), None, 0))
    out = np.zeros(2 * max(n, 1), dtype=np.int64)
    _check(lib().gacer_train_buckets(tenant, int(bucket_bytes), out.ctypes.data_as(C.POINTER(C.c_int64)), n))
    return [(int(out[2 * b]), int(out[2 * b + 1])) for b in range(n)]


def gacer_stream_wait_grads(stream, tenant, offset, count):
    return _check(lib().gacer_stream_wait_grads(C.c_void_p(stream), tenant, int(offset), int(count)))


def gacer_stream_open_grad_gate(stream, tenant):
    return _check(lib().gacer_stream_open_grad_gate(C.c_void_p(stream), tenant))


def gacer_set_partition(partition="priority"):
    return _check(lib().gacer_set_partition(PARTITION[partition] if isinstance(partition, str) else int(partition)))


def gacer_set_sm_shares(shares=None):
    if not shares:
        return _check(lib().gacer_set_sm_shares(None, 0))
    arr = np.ascontiguousarray(shares, dtype=np.float32)
    return _check(lib().gacer_set_sm_shares(arr.ctypes.data_as(FP), len(arr)))


def gacer_set_mode(mode):
    return _check(lib().gacer_set_mode(MODE[mode] if isinstance(mode, str) else mode))


def gacer_run_round():
    return _check(lib().gacer_run_round())


def gacer_run_round_async(stream_ptr=0):
    return _check(lib().gacer_run_round_async(C.c_void_p(stream_ptr)))


def gacer_capture_baseline(mode):
    return _check(lib().gacer_capture_baseline(MODE[mode] if isinstance(mode, str) else mode))


def gacer_run_baseline_graph(stream_ptr=0):
    return _check(lib().gacer_run_baseline_graph(C.c_void_p(stream_ptr)))


def gacer_run_round_host(host_in_ptrs, host_out_ptrs):
    n = len(host_in_ptrs)
    ins = (C.c_void_p * n)(*host_in_ptrs)
    outs = (C.c_void_p * n)(*host_out_ptrs)
    return _check(lib().gacer_run_round_host(ins, outs))


def gacer_get_stats():
    s = gacer_round_stats()
    _check(lib().gacer_get_stats(C.byref(s)))
    d = {f: getattr(s, f) for f, _ in gacer_round_stats._fields_ if f != "pad0"}
    d["tenant_sm_ns"] = list(s.tenant_sm_ns)[:max(0, min(16, s.n_tenants))]
    return d


def gacer_get_trace(cap):
    buf = np.zeros((cap, 12), dtype=np.int64)
    n = _check(lib().gacer_get_trace(buf.ctypes.data_as(C.POINTER(C.c_int64)), cap))
    return buf[:n]


def gacer_describe_op(op):
    out = np.zeros(8, dtype=np.int32)
    _check(lib().gacer_describe_op(op, out.ctypes.data_as(IP)))
    return dict(zip(("kind", "vfn", "items", "tenant", "bn", "nkb", "bytes", "mflop"), out.tolist()))


def gacer_last_error():
    return lib().gacer_last_error().decode()


def gacer_debug_timing(n_ops=1, reset=True, n_ctas=148, events=24):
    buf = np.zeros((n_ops, n_ctas, events), dtype=np.int64)
    _check(lib().gacer_debug_timing(buf.ctypes.data_as(C.POINTER(C.c_int64)), buf.size, int(reset)))
    return buf


# ------------------------------------------------- training-tenant steps (A11)
def _call(name, *args):
    return _check(getattr(lib(), name)(*args))


def bn_train_fwd(x, M, C_, gamma, beta, eps, relu, y, mean, var, scratch, stream=0):
    """gacer_bn_train_fwd on device pointers (ints)."""
    return _call("gacer_bn_train_fwd", x, M, C_, gamma, beta, eps, relu, y, mean, var, scratch, stream)


def bn_train_bwd(x, dy, M, C_, gamma, mean, var, eps, dx, dgamma, dbeta, scratch, stream=0, relu_y=None):
    return _call("gacer_bn_train_bwd", x, dy, relu_y, M, C_, gamma, mean, var, eps, dx, dgamma, dbeta, scratch, stream)


def relu_bwd(x, dy, n, six, dx, stream=0):
    return _call("gacer_relu_bwd", x, dy, n, six, dx, stream)


def maxpool_bwd(x, dy, N, H, W, C_, KH, KW, stride, ph, pw, Ho, Wo, dx, scratch, stream=0):
    return _call("gacer_maxpool_bwd", x, dy, N, H, W, C_, KH, KW, stride, ph, pw, Ho, Wo, dx, scratch, stream)


def gap_bwd(dy, N, HW, C_, dx, stream=0):
    return _call("gacer_gap_bwd", dy, N, HW, C_, dx, stream)


def linear_bwd(x, w, dy, N, K, O, dx, dw, db, stream=0):
    return _call("gacer_linear_bwd", x, w, dy, N, K, O, dx, dw, db, stream)


def conv_dgrad_workspace(N, H, W, Cin, Cout, KH, KW, stride, ph, pw):
    return _check(lib().gacer_conv_dgrad_workspace(N, H, W, Cin, Cout, KH, KW, stride, ph, pw))


def conv_dgrad(dy, w, N, H, W, Cin, Cout, KH, KW, stride, ph, pw, dx, ws, ws_bytes, stream=0):
    return _call("gacer_conv_dgrad", dy, w, N, H, W, Cin, Cout, KH, KW, stride, ph, pw, dx, ws, ws_bytes, stream)


def conv_wgrad_workspace(N, H, W, Cin, Cout, KH, KW, stride, ph, pw):
    return _check(lib().gacer_conv_wgrad_workspace(N, H, W, Cin, Cout, KH, KW, stride, ph, pw))


def conv_wgrad(x, dy, N, H, W, Cin, Cout, KH, KW, stride, ph, pw, dw, ws, ws_bytes, stream=0):
    return _call("gacer_conv_wgrad", x, dy, N, H, W, Cin, Cout, KH, KW, stride, ph, pw, dw, ws, ws_bytes, stream)


def conv_fwd_workspace(N, H, W, Cin, Cout, KH, KW, stride, ph, pw):
    return _check(lib().gacer_conv_fwd_workspace(N, H, W, Cin, Cout, KH, KW, stride, ph, pw))


def conv_fwd(x, w, N, H, W, Cin, Cout, KH, KW, stride, ph, pw, y, ws, ws_bytes, stream=0):
    return _call("gacer_conv_fwd", x, w, N, H, W, Cin, Cout, KH, KW, stride, ph, pw, y, ws, ws_bytes, stream)


def maxpool_fwd(x, N, H, W, C_, KH, KW, stride, ph, pw, Ho, Wo, y, stream=0):
    return _call("gacer_maxpool_fwd", x, N, H, W, C_, KH, KW, stride, ph, pw, Ho, Wo, y, stream)


def add(a, b, n, relu, y, stream=0):
    return _call("gacer_add", a, b, n, relu, y, stream)


def gap_fwd(x, N, HW, C_, y, stream=0):
    return _call("gacer_gap_fwd", x, N, HW, C_, y, stream)


def linear_fwd(x, w, b, N, K, O, z, stream=0):
    return _call("gacer_linear_fwd", x, w, b, N, K, O, z, stream)


def softmax_ce(z, labels, N, Cls, loss, dz, scratch, stream=0):
    return _call("gacer_softmax_ce", z, labels, N, Cls, loss, dz, scratch, stream)


def sgd_momentum(w, g, buf, n, lr, momentum, first, stream=0):
    return _call("gacer_sgd_momentum", w, g, buf, n, lr, momentum, first, stream)


def bn_partials(M, C_):
    return lib().gacer_bn_partials(M, C_)
