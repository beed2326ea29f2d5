"""Tenant forward in fp64 -- TEST INFRASTRUCTURE ONLY.

``forward_graph`` computes y_n = M_n(x_n) for one tenant (§4.1
l.605-607: the model is the operator list O_{n,1..i}), operator by operator,
with the plain operators of ``oracle.ops``.  Activations are NCHW fp64.  BN
is applied unfolded, flatten is NCHW order (PyTorch),
dropout is the identity (inference).

``chunked_forward`` applies the paper's spatial regulation literally:
Eq. 5 (l.657-668) O^B -> O^{B^1},...,O^{B^j} with sum B^j = B, realised as
"torch.chunk() ... torch.cat()" (l.673): split the operator's inputs along
the batch axis per list_B, run the operator on every chunk, concatenate.
The channel split (a north_star addition absent from the
paper) splits along the output-channel axis the same way.  Because every
operator is per-sample (inference) or per-channel separable, the result is
exactly ``forward_graph`` (the paper: "without sacrificing model accuracy",
l.674) -- a property the tests check bit-for-bit.
"""
from __future__ import annotations

import numpy as np

from . import ops


def _apply(op, params, ins):
    """Apply one operator (definitions: SURVEY §8(c) C1) to fp64 inputs."""
    k = op["kind"]
    x = ins[0]
    if k == "conv":
        p = params[op["id"]]
        return ops.conv2d(x, p["w"], p.get("b"), op["stride"], (op["ph"], op["pw"]),
                          op["groups"])
    if k == "bn":
        p = params[op["id"]]
        return ops.batchnorm(x, p["gamma"], p["beta"], p["mean"], p["var"], op["eps"])
    if k == "relu":
        return ops.relu(x)
    if k == "relu6":
        return ops.relu(x, six=True)
    if k == "maxpool":
        return ops.maxpool(x, (op["kh"], op["kw"]), op["stride"], (op["ph"], op["pw"]))
    if k == "avgpool":
        return ops.avgpool(x, (op["kh"], op["kw"]), op["stride"], (op["ph"], op["pw"]),
                           op.get("cip", True))
    if k == "gap":
        return ops.gap(x)
    if k == "linear":
        p = params[op["id"]]
        return ops.linear(x.reshape(x.shape[0], -1), p["w"], p.get("b"))
    if k == "hardswish":
        return ops.hardswish(x)
    if k == "hardsigmoid":
        return ops.hardsigmoid(x)
    if k == "mul":          # squeeze-and-excitation scale: x * s broadcast over H, W
        return ops.scale_channels(x, ins[1])
    if k == "add":
        return ops.add(ins[0], ins[1])
    if k == "concat":
        return np.concatenate(ins, axis=1)
    if k == "flatten":
        return x.reshape(x.shape[0], -1)
    if k == "dropout":
        return x
    raise ValueError(f"unknown op kind {k}")


def forward_graph(graph, params, x, return_all=False):
    """fp64 forward of one tenant; ``x`` is NCHW.  Returns the output of the
    last operator (logits [B, classes] or GAP features [B, C])."""
    vals = {0: np.ascontiguousarray(x, dtype=np.float64)}
    for op in graph.ops:
        vals[op["id"]] = _apply(op, params, [vals[p] for p in op["preds"]])
    out = vals[graph.ops[-1]["id"]]
    out = out.reshape(out.shape[0], -1)
    return (out, vals) if return_all else out


def _slice_params(op, params, c0, c1):
    """Parameters of the output-channel slice [c0, c1) of ``op``."""
    p = params.get(op["id"])
    if p is None:
        return params
    q = {}
    for name, a in p.items():
        q[name] = a[c0:c1]
    out = dict(params)
    out[op["id"]] = q
    return out


def _channel_chunk(op, params, ins, c0, c1):
    """Run ``op`` restricted to output channels [c0, c1)."""
    k = op["kind"]
    sub = dict(op)
    if k == "conv":
        if op["groups"] == 1:
            return _apply(sub, _slice_params(op, params, c0, c1), ins)
        if op["groups"] == op["c_in"] == op["c_out"]:      # depthwise
            sub["groups"] = c1 - c0
            return _apply(sub, _slice_params(op, params, c0, c1), [ins[0][:, c0:c1]])
        raise ValueError("channel split of grouped conv with groups != C")
    if k == "linear":
        return _apply(sub, _slice_params(op, params, c0, c1), ins)
    if k in ("bn",):
        return _apply(sub, _slice_params(op, params, c0, c1), [ins[0][:, c0:c1]])
    if k in ("relu", "relu6", "hardswish", "hardsigmoid", "maxpool", "avgpool", "gap", "dropout"):
        return _apply(sub, params, [ins[0][:, c0:c1]])
    if k in ("add", "mul"):
        return _apply(sub, params, [a[:, c0:c1] for a in ins])
    raise ValueError(f"channel split not defined for {k}")


def chunked_forward(graph, params, x, decomposition):
    """Eq. 5 applied literally.  ``decomposition`` maps op id ->
    (axis, list) with axis in {"batch", "channel"} and sum(list) == B
    (batch, Eq. 5) or == C_out (channel).  Unlisted ops run undecomposed
    (mask(O) = 0, l.683-684)."""
    vals = {0: np.ascontiguousarray(x, dtype=np.float64)}
    for op in graph.ops:
        ins = [vals[p] for p in op["preds"]]
        d = decomposition.get(op["id"])
        if d is None:
            vals[op["id"]] = _apply(op, params, ins)
            continue
        axis, sizes = d
        assert all(s >= 1 for s in sizes)
        if axis == "batch":
            B = ins[0].shape[0]
            assert sum(sizes) == B, "Eq. 5: sum of B^j must equal B"
            outs, b0 = [], 0
            for sz in sizes:                      # torch.chunk -> op -> torch.cat
                outs.append(_apply(op, params, [a[b0:b0 + sz] for a in ins]))
                b0 += sz
            vals[op["id"]] = np.concatenate(outs, axis=0)
        elif axis == "channel":
            outs, c0 = [], 0
            for sz in sizes:
                outs.append(_channel_chunk(op, params, ins, c0, c0 + sz))
                c0 += sz
            vals[op["id"]] = np.concatenate(outs, axis=1)
        else:
            raise ValueError(axis)
    out = vals[graph.ops[-1]["id"]]
    return out.reshape(out.shape[0], -1)
