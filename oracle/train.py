"""Training-tenant step in fp64 -- TEST INFRASTRUCTURE ONLY.

SURVEY.md §8(a) A11 / §8(c) "Training": one step of a training tenant is a
forward pass with BatchNorm in TRAINING mode (statistics of the per-replica
batch), mean softmax cross-entropy over the labels, the backward pass, and an
SGD-with-momentum update (lr 0.1, momentum 0.9 proposed; the paper trains with
PyTorch defaults and states no hyper-parameters, §5.1 l.903-911).
A12: with G data-parallel replicas the update uses the MEAN of the replicas'
gradients (``allreduce_mean``), each replica's BN statistics its own.

Every backward operator is the plain derivative of the forward definition
(``gacer_oracle_train.c``); the graph backward walks the operator list in
reverse issue order, summing the gradients of tensors with several consumers
in consumer order.  BN running statistics follow PyTorch (momentum 0.1,
unbiased variance).  Pins: tests/test_oracle_train.py.
"""
from __future__ import annotations

import ctypes
from typing import Dict, List, Optional

import numpy as np

from . import ops

_bound = False


def _lib():
    global _bound
    L = ops.lib()
    if not _bound:
        D = ctypes.POINTER(ctypes.c_double)
        i, d, sz = ctypes.c_int, ctypes.c_double, ctypes.c_size_t
        L.oracle_conv2d_bwd_data.argtypes = [D, D] + [i] * 13 + [D]
        L.oracle_conv2d_bwd_weight.argtypes = [D, D] + [i] * 13 + [D, D]
        L.oracle_bn_train_fwd.argtypes = [D, i, i, i, D, D, d, D, D, D]
        L.oracle_bn_train_bwd.argtypes = [D, D, i, i, i, D, D, D, d, D, D, D]
        L.oracle_relu_bwd.argtypes = [D, D, sz, i, D]
        L.oracle_maxpool_bwd.argtypes = [D, D] + [i] * 11 + [D]
        L.oracle_gap_bwd.argtypes = [D, i, i, i, D]
        L.oracle_linear_bwd.argtypes = [D, D, D, i, i, i, D, D, D]
        L.oracle_softmax_ce.argtypes = [D, ctypes.POINTER(ctypes.c_int), i, i, D]
        L.oracle_softmax_ce.restype = ctypes.c_double
        L.oracle_sgd_momentum.argtypes = [D, D, D, sz, d, d, i]
        _bound = True
    return L


_p, _f = ops._p, ops._f64


# ------------------------------------------------------------------ operators
def conv2d_bwd(x, w, dy, stride=1, pad=(0, 0), groups=1, bias=False):
    """(dx, dw, db) of y = conv2d(x, w) (+ b)."""
    x, w, dy = _f(x), _f(w), _f(dy)
    N, Cin, H, W = x.shape
    Cout, _, KH, KW = w.shape
    ph, pw = pad
    Ho, Wo = dy.shape[2:]
    dx, dw = np.empty_like(x), np.empty_like(w)
    db = np.empty(Cout) if bias else None
    L = _lib()
    L.oracle_conv2d_bwd_data(_p(dy), _p(w), N, Cin, H, W, Cout, KH, KW, stride, ph, pw, groups, Ho, Wo, _p(dx))
    L.oracle_conv2d_bwd_weight(_p(x), _p(dy), N, Cin, H, W, Cout, KH, KW, stride, ph, pw, groups, Ho, Wo,
                               _p(dw), _p(db))
    return dx, dw, db


def bn_train_fwd(x, gamma, beta, eps):
    """(y, batch mean, biased batch var)."""
    x = _f(x)
    N, C = x.shape[:2]
    HW = int(np.prod(x.shape[2:])) if x.ndim > 2 else 1
    y, mean, var = np.empty_like(x), np.empty(C), np.empty(C)
    _lib().oracle_bn_train_fwd(_p(x), N, C, HW, _p(_f(gamma)), _p(_f(beta)), float(eps), _p(y), _p(mean), _p(var))
    return y, mean, var


def bn_train_bwd(x, dy, gamma, mean, var, eps):
    """(dx, dgamma, dbeta)."""
    x, dy = _f(x), _f(dy)
    N, C = x.shape[:2]
    HW = int(np.prod(x.shape[2:])) if x.ndim > 2 else 1
    dx, dg, db = np.empty_like(x), np.empty(C), np.empty(C)
    _lib().oracle_bn_train_bwd(_p(x), _p(dy), N, C, HW, _p(_f(gamma)), _p(_f(mean)), _p(_f(var)), float(eps),
                               _p(dx), _p(dg), _p(db))
    return dx, dg, db


def relu_bwd(x, dy, six=False):
    x, dy = _f(x), _f(dy)
    dx = np.empty_like(x)
    _lib().oracle_relu_bwd(_p(x), _p(dy), x.size, int(six), _p(dx))
    return dx


def maxpool_bwd(x, dy, k, stride, pad=(0, 0)):
    x, dy = _f(x), _f(dy)
    N, C, H, W = x.shape
    KH, KW = k
    Ho, Wo = dy.shape[2:]
    dx = np.empty_like(x)
    _lib().oracle_maxpool_bwd(_p(x), _p(dy), N, C, H, W, KH, KW, stride, pad[0], pad[1], Ho, Wo, _p(dx))
    return dx


def gap_bwd(dy, shape):
    N, C, H, W = shape
    dy = _f(dy).reshape(N, C)
    dx = np.empty(shape)
    _lib().oracle_gap_bwd(_p(dy), N, C, H * W, _p(dx))
    return dx


def linear_bwd(x, w, dy, bias=True):
    x, w, dy = _f(x), _f(w), _f(dy)
    N, K = x.shape
    O = w.shape[0]
    dx, dw = np.empty_like(x), np.empty_like(w)
    db = np.empty(O) if bias else None
    _lib().oracle_linear_bwd(_p(x), _p(w), _p(dy), N, K, O, _p(dx), _p(dw), _p(db))
    return dx, dw, db


def softmax_ce(z, labels):
    """(mean loss, dz)."""
    z = _f(z)
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    N, C = z.shape
    assert lab.shape == (N,) and lab.min() >= 0 and lab.max() < C
    dz = np.empty_like(z)
    loss = _lib().oracle_softmax_ce(_p(z), lab.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), N, C, _p(dz))
    return float(loss), dz


def sgd_momentum(w, g, buf, lr, momentum, first):
    """In-place SGD-momentum update of fp64 arrays ``w`` and ``buf``."""
    assert w.dtype == np.float64 and buf.dtype == np.float64 and w.flags.c_contiguous and buf.flags.c_contiguous
    _lib().oracle_sgd_momentum(_p(w), _p(_f(g)), _p(buf), w.size, float(lr), float(momentum), int(first))


def allreduce_mean(grads_per_replica: List[Dict]) -> Dict:
    """A12: the element-wise mean of the replicas' gradients, summed in replica
    order then divided by G (the result every replica applies)."""
    G = len(grads_per_replica)
    out = {}
    for oid, d in grads_per_replica[0].items():
        out[oid] = {}
        for name in d:
            acc = np.array(grads_per_replica[0][oid][name], dtype=np.float64)
            for r in range(1, G):
                acc = acc + grads_per_replica[r][oid][name]
            out[oid][name] = acc / G
    return out


# -------------------------------------------------------------- graph level
_TRAINABLE = {"conv": ("w", "b"), "linear": ("w", "b"), "bn": ("gamma", "beta")}


def forward_train(graph, params, x):
    """Forward with training-mode BN; returns (logits, tape) where the tape
    holds every op's input values and BN batch statistics."""
    vals = {0: _f(x)}
    tape = {}
    for op in graph.ops:
        k, oid = op["kind"], op["id"]
        ins = [vals[p] for p in op["preds"]]
        xi = ins[0]
        if k == "bn":
            p = params[oid]
            y, mean, var = bn_train_fwd(xi, p["gamma"], p["beta"], op["eps"])
            tape[oid] = (mean, var)
        elif k == "conv":
            p = params[oid]
            y = ops.conv2d(xi, p["w"], p.get("b"), op["stride"], (op["ph"], op["pw"]), op["groups"])
        elif k == "linear":
            p = params[oid]
            y = ops.linear(xi.reshape(xi.shape[0], -1), p["w"], p.get("b"))
        elif k in ("relu", "relu6"):
            y = ops.relu(xi, six=(k == "relu6"))
        elif k == "maxpool":
            y = ops.maxpool(xi, (op["kh"], op["kw"]), op["stride"], (op["ph"], op["pw"]))
        elif k == "gap":
            y = ops.gap(xi)
        elif k == "add":
            y = ops.add(ins[0], ins[1])
        elif k in ("flatten", "dropout"):
            y = xi.reshape(xi.shape[0], -1) if k == "flatten" else xi
        else:
            raise NotImplementedError(f"training backward of {k!r} is not defined in the oracle")
        vals[oid] = y
    out = vals[graph.ops[-1]["id"]]
    return out.reshape(out.shape[0], -1), (vals, tape)


def backward(graph, params, saved, dlogits):
    """Reverse-order backward; returns {op_id: {param: grad}}."""
    vals, tape = saved
    grads: Dict[int, Dict[str, np.ndarray]] = {}
    last = graph.ops[-1]["id"]
    dval: Dict[int, Optional[np.ndarray]] = {last: _f(dlogits).reshape(vals[last].shape)}

    def acc(tid, g):
        g = g.reshape(vals[tid].shape)
        dval[tid] = g if dval.get(tid) is None else dval[tid] + g

    for op in reversed(graph.ops):
        k, oid = op["kind"], op["id"]
        dy = dval.pop(oid, None)
        if dy is None:
            continue                              # output unused by the loss
        ins = [vals[p] for p in op["preds"]]
        xi = ins[0]
        if k == "conv":
            dx, dw, db = conv2d_bwd(xi, params[oid]["w"], dy, op["stride"], (op["ph"], op["pw"]), op["groups"],
                                    bias="b" in params[oid])
            grads[oid] = {"w": dw, **({"b": db} if db is not None else {})}
            acc(op["preds"][0], dx)
        elif k == "linear":
            x2 = xi.reshape(xi.shape[0], -1)
            dx, dw, db = linear_bwd(x2, params[oid]["w"], dy.reshape(dy.shape[0], -1), bias="b" in params[oid])
            grads[oid] = {"w": dw, **({"b": db} if db is not None else {})}
            acc(op["preds"][0], dx)
        elif k == "bn":
            mean, var = tape[oid]
            dx, dg, db = bn_train_bwd(xi, dy, params[oid]["gamma"], mean, var, op["eps"])
            grads[oid] = {"gamma": dg, "beta": db}
            acc(op["preds"][0], dx)
        elif k in ("relu", "relu6"):
            acc(op["preds"][0], relu_bwd(xi, dy, six=(k == "relu6")))
        elif k == "maxpool":
            acc(op["preds"][0], maxpool_bwd(xi, dy, (op["kh"], op["kw"]), op["stride"], (op["ph"], op["pw"])))
        elif k == "gap":
            acc(op["preds"][0], gap_bwd(dy, xi.shape))
        elif k == "add":
            acc(op["preds"][0], dy)
            acc(op["preds"][1], dy)
        elif k in ("flatten", "dropout"):
            acc(op["preds"][0], dy)
        else:
            raise NotImplementedError(k)
    return grads


def train_step(graph, params, x, labels, lr=0.1, momentum=0.9, state=None, grads_hook=None):
    """One SGD step of a training tenant.  ``state`` carries the momentum
    buffers and BN running statistics between steps ({} on the first step).
    ``grads_hook`` (A12) maps the local gradients to the applied ones, e.g.
    ``allreduce_mean`` over replicas.  Returns (loss, grads, new_params,
    new_state); inputs are not modified."""
    state = {"step": 0, "buf": {}, "running": {}} if state is None else state
    logits, saved = forward_train(graph, params, x)
    loss, dz = softmax_ce(logits, labels)
    grads = backward(graph, params, saved, dz)
    if grads_hook is not None:
        grads = grads_hook(grads)
    first = state["step"] == 0
    new_params, bufs = {}, {}
    for oid, p in params.items():
        new_params[oid] = {n: _f(v).copy() for n, v in p.items()}
        for n in _TRAINABLE.get(next(o["kind"] for o in graph.ops if o["id"] == oid), ()):
            if n in grads.get(oid, {}):
                buf = np.zeros(new_params[oid][n].shape) if first else state["buf"][(oid, n)].copy()
                sgd_momentum(new_params[oid][n], grads[oid][n], buf, lr, momentum, first)
                bufs[(oid, n)] = buf
    # BN running statistics (PyTorch: momentum 0.1, unbiased variance)
    _, tape = saved
    running = {}
    vals = saved[0]
    for op in graph.ops:
        if op["kind"] == "bn":
            oid = op["id"]
            mean, var = tape[oid]
            xi = vals[op["preds"][0]]
            M = xi.size // xi.shape[1]
            rm, rv = state["running"].get(oid, (_f(params[oid]["mean"]), _f(params[oid]["var"])))
            running[oid] = (0.9 * rm + 0.1 * mean, 0.9 * rv + 0.1 * var * M / (M - 1))
            new_params[oid]["mean"], new_params[oid]["var"] = running[oid]
    return loss, grads, new_params, {"step": state["step"] + 1, "buf": bufs, "running": running}
