"""Sequential training step of one tenant from the device operators of
include/gacer_train.h (first version).

Host-side sequencing only: every arithmetic step is a call into libgacer.so
(tcgen05 conv forward / dgrad / wgrad through single-op executor launches,
the CUDA-core BN-train / pooling / FC / loss / SGD kernels); this module
walks the tenant's operator list forward and then in reverse, allocates the
saved activations and gradients in HBM, and issues the calls in order on one
stream.  It is the training analog of the inference path's sequential
baseline mode; running the step as executor work items (and in C) is the
next step.

Supported operator patterns (those of ResNet-18/34/50/101 and the test
CNNs): conv -> bn -> [relu], add -> [relu], maxpool, gap -> [flatten] ->
linear.  A ReLU is fused into its producer (BN apply or residual add); its
backward mask is taken from the ReLU output (y > 0 iff x > 0).  Layout:
NHWC bf16 activations, fp32 master weights / BN parameters / gradients /
momentum buffers; a 3-channel input is zero-padded to 8 channels (the conv
operand granule), with zero-padded filter channels that stay zero.
BN running statistics are not updated (they do not enter the step's loss
or gradients)."""
from __future__ import annotations

from typing import Dict, List

import numpy as np

from . import gacer as G


def _pad8(c: int) -> int:
    return (c + 7) // 8 * 8


def plan_graph(graph):
    """Host-side plan of a training graph: NHWC shape (H, W, C) of every
    tensor (the input's C padded to 8) and the ReLUs fused into their
    producer ({producer id: relu id}).  Raises NotImplementedError for
    operator patterns the device path does not train."""
    consumers: Dict[int, List[int]] = {}
    for op in graph.ops:
        for p in op["preds"]:
            consumers.setdefault(p, []).append(op["id"])
    ops = {op["id"]: op for op in graph.ops}
    shape = {0: (graph.in_h, graph.in_w, _pad8(graph.in_c))}
    fused: Dict[int, int] = {}
    for op in graph.ops:
        k, oid = op["kind"], op["id"]
        h, w, c = shape[op["preds"][0]]
        if k == "conv":
            if op["groups"] != 1 or op.get("bias"):
                raise NotImplementedError("grouped / biased conv training is not supported yet")
            st = op["stride"]
            shape[oid] = ((h + 2 * op["ph"] - op["kh"]) // st + 1, (w + 2 * op["pw"] - op["kw"]) // st + 1, op["c_out"])
        elif k == "maxpool":
            st = op["stride"]
            shape[oid] = ((h + 2 * op["ph"] - op["kh"]) // st + 1, (w + 2 * op["pw"] - op["kw"]) // st + 1, c)
        elif k == "gap":
            shape[oid] = (1, 1, c)
        elif k == "linear":
            # the trainer's FC reads a [B][C] activation (a GAP output): a
            # flatten -> linear head over a spatial tensor would need the
            # NCHW-flatten weight order, which it does not implement
            if (h, w) != (1, 1) or c != op["c_in"]:
                raise NotImplementedError("linear training needs a [B][c_in] (1x1 spatial) input")
            shape[oid] = (1, 1, op["c_out"])
        elif k in ("bn", "flatten", "dropout", "relu", "add"):
            shape[oid] = (h, w, c)
        else:
            raise NotImplementedError(f"training of {k!r}")
        if k == "relu":
            prod = op["preds"][0]
            if ops.get(prod, {}).get("kind") not in ("bn", "add") or len(consumers[prod]) != 1:
                raise NotImplementedError("a ReLU is trained fused into its BN or residual-add producer")
            fused[prod] = oid
    return shape, fused


class SequentialTrainer:
    def __init__(self, graph, params, batch: int, lr: float = 0.1, momentum: float = 0.9):
        import torch
        self.torch = torch
        self.g, self.B, self.lr, self.mom = graph, batch, lr, momentum
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
        self.shape, self.fused_relu = plan_graph(graph)
        self.kind = {op["id"]: op["kind"] for op in graph.ops}
        self.params: Dict[int, Dict[str, object]] = {}
        for op in graph.ops:
            k, oid = op["kind"], op["id"]
            if k == "conv":
                c = self.shape[op["preds"][0]][2]
                wt = np.zeros((op["c_out"], c, op["kh"], op["kw"]), np.float32)
                wt[:, :op["c_in"]] = params[oid]["w"]        # zero filter channels for the padded input
                self.params[oid] = {"w": dev(wt)}
            elif k == "bn":
                self.params[oid] = {"gamma": dev(params[oid]["gamma"]), "beta": dev(params[oid]["beta"])}
            elif k == "linear":
                self.params[oid] = {"w": dev(params[oid]["w"])}
                if "b" in params[oid]:
                    self.params[oid]["b"] = dev(params[oid]["b"])
        # one flat fp32 buffer each for the parameters, their gradients and
        # the momentum buffers: the SGD update is ONE launch over the whole
        # model, and the gradient all-reduce (A12) sees one contiguous buffer
        keys = [(pid, n) for pid in self.params for n in self.params[pid]]
        total = sum(self.params[pid][n].numel() for pid, n in keys)
        self.flat_p = torch.empty(total, device="cuda")
        self.flat_g = torch.zeros(total, device="cuda")
        self.flat_m = torch.zeros(total, device="cuda")
        self.gview: Dict[int, Dict[str, object]] = {}
        off = 0
        for pid, n in keys:
            t = self.params[pid][n]
            k = t.numel()
            self.flat_p[off:off + k].copy_(t.reshape(-1))
            self.params[pid][n] = self.flat_p[off:off + k].view(t.shape)
            self.gview.setdefault(pid, {})[n] = self.flat_g[off:off + k].view(t.shape)
            off += k
        self.first = True
        # one workspace for every conv call (the largest need)
        need = 1 << 20
        for op in graph.ops:
            if op["kind"] != "conv":
                continue
            h, w, c = self.shape[op["preds"][0]]
            a = (self.B, h, w, c, op["c_out"], op["kh"], op["kw"], op["stride"], op["ph"], op["pw"])
            need = max(need, G.conv_fwd_workspace(*a), G.conv_wgrad_workspace(*a))
            if op["preds"][0] != 0:
                need = max(need, G.conv_dgrad_workspace(*a))
        self.ws = torch.empty(need + 256, dtype=torch.uint8, device="cuda")
        self.WS, self.NB = (self.ws.data_ptr() + 255) // 256 * 256, need
        maxmc = max(self.B * s[0] * s[1] * s[2] for s in self.shape.values())
        maxc = max(s[2] for s in self.shape.values())
        self.bn_scratch = torch.empty(G.bn_partials(maxmc, 8) * 2 * maxc + 4 * maxc + 64, device="cuda")
        self.argmax = torch.empty(maxmc, dtype=torch.uint8, device="cuda")

    # ---------------------------------------------------------------- step
    def step(self, x_nhwc8, labels, grads_hook=None):
        """One SGD step: x_nhwc8 bf16 [B][H][W][pad8(C)] and labels int32 [B]
        on the device.  Returns the loss (a 1-element fp32 device tensor) and
        the parameter gradients {op_id: {name: tensor}}.

        grads_hook(flat_g), if given, runs after the backward pass and BEFORE
        the SGD update (e.g. the data-parallel gradient mean of A12,
        GradBuckets.reduce_mean); it must leave flat_g ready on the legacy
        default stream the libgacer calls use.  The library calls run on that
        stream; it is ordered after the caller's current stream on entry and
        the current stream after it on return."""
        torch, B, P = self.torch, self.B, (lambda t: t.data_ptr())
        cur, dflt = torch.cuda.current_stream(), torch.cuda.default_stream()
        if cur != dflt:
            dflt.wait_stream(cur)
        bf = lambda shape: torch.empty(shape, dtype=torch.bfloat16, device="cuda")
        f32 = lambda *shape: torch.empty(shape, device="cuda")
        out = {0: x_nhwc8}
        saved = {}
        logits = None
        for op in self.g.ops:
            k, oid = op["kind"], op["id"]
            pred = op["preds"][0]
            h, w, c = self.shape[pred]
            ho, wo, co = self.shape[oid]
            if k == "conv":
                y = bf((B, ho, wo, co))
                G.conv_fwd(P(out[pred]), P(self.params[oid]["w"]), B, h, w, c, co, op["kh"], op["kw"], op["stride"],
                           op["ph"], op["pw"], P(y), self.WS, self.NB)
                out[oid] = y
            elif k == "bn":
                y = bf((B, h, w, c))
                mean, var = f32(c), f32(c)
                relu = 1 if oid in self.fused_relu else 0
                G.bn_train_fwd(P(out[pred]), B * h * w, c, P(self.params[oid]["gamma"]), P(self.params[oid]["beta"]),
                               op["eps"], relu, P(y), P(mean), P(var), P(self.bn_scratch))
                saved[oid] = (mean, var)
                out[oid] = y
            elif k == "relu":
                out[oid] = out[pred]                  # fused into the producer
            elif k == "add":
                y = bf((B, h, w, c))
                G.add(P(out[op["preds"][0]]), P(out[op["preds"][1]]), y.numel(), 1 if oid in self.fused_relu else 0,
                      P(y))
                out[oid] = y
            elif k == "maxpool":
                y = bf((B, ho, wo, c))
                G.maxpool_fwd(P(out[pred]), B, h, w, c, op["kh"], op["kw"], op["stride"], op["ph"], op["pw"], ho, wo,
                              P(y))
                out[oid] = y
            elif k == "gap":
                y = bf((B, c))
                G.gap_fwd(P(out[pred]), B, h * w, c, P(y))
                out[oid] = y
            elif k in ("flatten", "dropout"):
                out[oid] = out[pred]
            elif k == "linear":
                z = f32(B, co)
                b = self.params[oid].get("b")
                G.linear_fwd(P(out[pred]), P(self.params[oid]["w"]), P(b) if b is not None else None, B, c, co, P(z))
                out[oid] = z
                logits = z
        ncls = logits.shape[1]
        loss, dz = f32(1), f32(B, ncls)
        G.softmax_ce(P(logits), P(labels), B, ncls, P(loss), P(dz), P(f32(B)))
        # ---------------------------------------------------------- backward
        grads: Dict[int, Dict[str, object]] = {}
        relu_mask: Dict[int, object] = {}
        dval = {self.g.ops[-1]["id"]: dz}

        shared = set()        # gradient tensors held by two dval entries (a residual add): copy on write

        def acc(tid, g):
            if tid == 0:
                return
            if tid in dval:
                cur = dval[tid]
                dst = cur if id(cur) not in shared else torch.empty_like(cur)
                G.add(P(cur), P(g), g.numel(), 0, P(dst))
                dval[tid] = dst
            else:
                dval[tid] = g

        for op in reversed(self.g.ops):
            k, oid = op["kind"], op["id"]
            dy = dval.pop(oid, None)
            if dy is None:
                continue
            pred = op["preds"][0]
            h, w, c = self.shape[pred]
            ho, wo, co = self.shape[oid]
            if k == "linear":
                dx = f32(B, c)
                gw = self.gview[oid]["w"]
                gb = self.gview[oid].get("b")
                G.linear_bwd(P(out[pred]), P(self.params[oid]["w"]), P(dy), B, c, co, P(dx), P(gw),
                             P(gb) if gb is not None else None)
                grads[oid] = {"w": gw, **({"b": gb} if gb is not None else {})}
                acc(pred, dx)
            elif k in ("flatten", "dropout"):
                acc(pred, dy)
            elif k == "gap":
                dx = bf((B, h, w, c))
                G.gap_bwd(P(dy), B, h * w, c, P(dx))
                acc(pred, dx)
            elif k == "relu":
                if self.kind[pred] == "bn":
                    relu_mask[pred] = out[oid]        # applied inside the BN backward (fused)
                else:
                    dst = dy if id(dy) not in shared else torch.empty_like(dy)
                    G.relu_bwd(P(out[oid]), P(dy), dy.numel(), 0, P(dst))
                    dy = dst
                acc(pred, dy)
            elif k == "add":
                shared.add(id(dy))                # both inputs receive dy itself (no copy)
                acc(op["preds"][0], dy)
                acc(op["preds"][1], dy)
            elif k == "bn":
                dx = bf((B, h, w, c))
                gg, gb = self.gview[oid]["gamma"], self.gview[oid]["beta"]
                mean, var = saved[oid]
                ym = relu_mask.pop(oid, None)
                G.bn_train_bwd(P(out[pred]), P(dy), B * h * w, c, P(self.params[oid]["gamma"]), P(mean), P(var),
                               op["eps"], P(dx), P(gg), P(gb), P(self.bn_scratch),
                               relu_y=P(ym) if ym is not None else None)
                grads[oid] = {"gamma": gg, "beta": gb}
                acc(pred, dx)
            elif k == "maxpool":
                dx = bf((B, h, w, c))
                G.maxpool_bwd(P(out[pred]), P(dy), B, h, w, c, op["kh"], op["kw"], op["stride"], op["ph"], op["pw"],
                              ho, wo, P(dx), P(self.argmax))
                acc(pred, dx)
            elif k == "conv":
                gw = self.gview[oid]["w"]
                a = (B, h, w, c, co, op["kh"], op["kw"], op["stride"], op["ph"], op["pw"])
                G.conv_wgrad(P(out[pred]), P(dy), *a, P(gw), self.WS, self.NB)
                grads[oid] = {"w": gw}
                if pred != 0:
                    dx = bf((B, h, w, c))
                    G.conv_dgrad(P(dy), P(self.params[oid]["w"]), *a, P(dx), self.WS, self.NB)
                    acc(pred, dx)
        # ---------------------------------------------------------- SGD
        # (every parameter has a gradient: a ResNet's whole parameter set is
        #  written by the backward pass above, so one launch updates it all)
        if grads_hook is not None:
            with torch.cuda.stream(dflt):
                grads_hook(self.flat_g)
        G.sgd_momentum(P(self.flat_p), P(self.flat_g), P(self.flat_m), self.flat_p.numel(), self.lr, self.mom,
                       int(self.first))
        self.first = False
        if cur != dflt:
            cur.wait_stream(dflt)
        return loss, grads
