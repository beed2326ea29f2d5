"""Tenant DFG descriptors (data only).

A tenant graph is the paper's model operator list M_n = [O_{n,1}, ..., O_{n,i}]
(§4.1, l.605-607): operators in topological issue order, each with a
unique id and its predecessor ids.  Predecessor id 0 denotes the graph input.
The last operator is the graph output.

Operator kinds and their parameters (PyTorch eval-mode meaning):

  conv     c_in c_out kh kw stride ph pw groups bias
  bn       c eps [res_last]          (inference BatchNorm2d)
  relu / relu6
  maxpool  kh kw stride ph pw        (floor mode, implicit -inf padding)
  avgpool  kh kw stride ph pw cip    (cip = count_include_pad)
  gap                                (adaptive avg-pool to 1x1)
  linear   c_in c_out bias
  add      (2 preds)   concat (n preds, channel axis)
  flatten  dropout                   (flatten is NCHW order, dropout = identity)

Model structures follow the torchvision definitions (§5.1 l.903 names
the models; BASELINE.json names the mixes).  Spatial input is 224x224.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List


@dataclass
class Graph:
    name: str
    in_c: int
    in_h: int
    in_w: int
    ops: List[dict] = field(default_factory=list)
    init_gain: float = 2.0      # He-normal gain for conv/linear weights (C4)
    n_classes: int = 0

    # ---- builder helpers -------------------------------------------------
    def _add(self, kind: str, preds: List[int], **p) -> int:
        oid = len(self.ops) + 1
        op = {"id": oid, "kind": kind, "preds": list(preds)}
        op.update(p)
        self.ops.append(op)
        return oid

    def conv(self, x, c_in, c_out, k, stride=1, pad=0, groups=1, bias=False):
        kh, kw = (k, k) if isinstance(k, int) else k
        ph, pw = (pad, pad) if isinstance(pad, int) else pad
        return self._add("conv", [x], c_in=c_in, c_out=c_out, kh=kh, kw=kw,
                         stride=stride, ph=ph, pw=pw, groups=groups, bias=bias)

    def bn(self, x, c, eps=1e-5, res_last=False):
        return self._add("bn", [x], c=c, eps=eps, res_last=res_last)

    def relu(self, x):
        return self._add("relu", [x])

    def relu6(self, x):
        return self._add("relu6", [x])

    def maxpool(self, x, k, stride, pad=0):
        return self._add("maxpool", [x], kh=k, kw=k, stride=stride, ph=pad, pw=pad)

    def avgpool(self, x, k, stride, pad=0, cip=True):
        return self._add("avgpool", [x], kh=k, kw=k, stride=stride, ph=pad, pw=pad, cip=cip)

    def gap(self, x):
        return self._add("gap", [x])

    def linear(self, x, c_in, c_out, bias=True):
        return self._add("linear", [x], c_in=c_in, c_out=c_out, bias=bias)

    def hardswish(self, x):
        return self._add("hardswish", [x])

    def hardsigmoid(self, x):
        return self._add("hardsigmoid", [x])

    def mul(self, x, s):
        """x [N, C, H, W] * s [N, C] broadcast over H, W (squeeze-and-excitation)"""
        return self._add("mul", [x, s])

    def add(self, a, b):
        return self._add("add", [a, b])

    def concat(self, xs):
        return self._add("concat", list(xs))

    def flatten(self, x):
        return self._add("flatten", [x])

    def dropout(self, x):
        return self._add("dropout", [x])

    # conv -> bn -> act
    def cba(self, x, c_in, c_out, k, stride=1, pad=0, groups=1, act="relu",
            eps=1e-5, res_last=False):
        y = self.conv(x, c_in, c_out, k, stride, pad, groups)
        y = self.bn(y, c_out, eps=eps, res_last=res_last)
        if act == "relu":
            y = self.relu(y)
        elif act == "relu6":
            y = self.relu6(y)
        elif act == "hardswish":
            y = self.hardswish(y)
        return y


# --------------------------------------------------------------------------
# tiny tenants (BASELINE config 1)
# --------------------------------------------------------------------------
def tiny_cnn() -> Graph:
    g = Graph("tiny_cnn", 3, 32, 32)
    x = g.conv(0, 3, 8, 3, 1, 1, bias=True); x = g.relu(x); x = g.maxpool(x, 2, 2)
    x = g.conv(x, 8, 16, 3, 1, 1, bias=True); x = g.relu(x); x = g.maxpool(x, 2, 2)
    x = g.conv(x, 16, 32, 3, 1, 1, bias=True); x = g.relu(x)
    x = g.gap(x)
    g.n_classes = 32
    return g


def tiny_mlp() -> Graph:
    # input [B, 784] is carried as a 784x1x1 "image" (flatten is the identity)
    g = Graph("tiny_mlp", 784, 1, 1)
    x = g.flatten(0)
    x = g.linear(x, 784, 256); x = g.relu(x)
    x = g.linear(x, 256, 10)
    g.n_classes = 10
    return g


# --------------------------------------------------------------------------
# ResNet-18/50/101 (torchvision v1.5: stride on the 3x3 of the bottleneck)
# --------------------------------------------------------------------------
def _resnet(name, block, layers) -> Graph:
    g = Graph(name, 3, 224, 224)
    x = g.cba(0, 3, 64, 7, 2, 3)
    x = g.maxpool(x, 3, 2, 1)
    c_in = 64
    for li, (planes, n) in enumerate(zip((64, 128, 256, 512), layers)):
        for bi in range(n):
            stride = 2 if (li > 0 and bi == 0) else 1
            if block == "basic":
                c_out = planes
                y = g.cba(x, c_in, planes, 3, stride, 1)
                y = g.cba(y, planes, planes, 3, 1, 1, act=None, res_last=True)
            else:
                c_out = planes * 4
                y = g.cba(x, c_in, planes, 1)
                y = g.cba(y, planes, planes, 3, stride, 1)
                y = g.cba(y, planes, c_out, 1, act=None, res_last=True)
            if stride != 1 or c_in != c_out:
                sc = g.cba(x, c_in, c_out, 1, stride, 0, act=None)
            else:
                sc = x
            x = g.relu(g.add(y, sc))
            c_in = c_out
    x = g.gap(x)
    x = g.flatten(x)
    x = g.linear(x, c_in, 1000)
    g.n_classes = 1000
    return g


def resnet18():
    return _resnet("resnet18", "basic", (2, 2, 2, 2))


def resnet34():
    return _resnet("resnet34", "basic", (3, 4, 6, 3))


def resnet50():
    return _resnet("resnet50", "bottleneck", (3, 4, 6, 3))


def resnet101():
    return _resnet("resnet101", "bottleneck", (3, 4, 23, 3))


# --------------------------------------------------------------------------
# VGG-16 (configuration D).  AdaptiveAvgPool2d((7,7)) is the identity at 224^2
# and is not emitted.
# --------------------------------------------------------------------------
def vgg16() -> Graph:
    g = Graph("vgg16", 3, 224, 224)
    cfg = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M",
           512, 512, 512, "M", 512, 512, 512, "M"]
    x, c = 0, 3
    for v in cfg:
        if v == "M":
            x = g.maxpool(x, 2, 2)
        else:
            x = g.relu(g.conv(x, c, v, 3, 1, 1, bias=True))
            c = v
    x = g.flatten(x)
    x = g.dropout(g.relu(g.linear(x, 512 * 7 * 7, 4096)))
    x = g.dropout(g.relu(g.linear(x, 4096, 4096)))
    x = g.linear(x, 4096, 1000)
    g.n_classes = 1000
    return g


# --------------------------------------------------------------------------
# AlexNet (torchvision).  AdaptiveAvgPool2d((6,6)) is the identity at 224^2.
# --------------------------------------------------------------------------
def alexnet() -> Graph:
    g = Graph("alexnet", 3, 224, 224)
    x = g.relu(g.conv(0, 3, 64, 11, 4, 2, bias=True)); x = g.maxpool(x, 3, 2)
    x = g.relu(g.conv(x, 64, 192, 5, 1, 2, bias=True)); x = g.maxpool(x, 3, 2)
    x = g.relu(g.conv(x, 192, 384, 3, 1, 1, bias=True))
    x = g.relu(g.conv(x, 384, 256, 3, 1, 1, bias=True))
    x = g.relu(g.conv(x, 256, 256, 3, 1, 1, bias=True)); x = g.maxpool(x, 3, 2)
    x = g.flatten(x)
    x = g.relu(g.linear(g.dropout(x), 256 * 6 * 6, 4096))
    x = g.relu(g.linear(g.dropout(x), 4096, 4096))
    x = g.linear(x, 4096, 1000)
    g.n_classes = 1000
    return g


# --------------------------------------------------------------------------
# MobileNetV2 (torchvision, width 1.0).  Gain-1 init.
# --------------------------------------------------------------------------
def mobilenet_v2() -> Graph:
    g = Graph("mobilenet_v2", 3, 224, 224, init_gain=1.0)
    x = g.cba(0, 3, 32, 3, 2, 1, act="relu6")
    c_in = 32
    for t, c, n, s in ((1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2),
                       (6, 96, 3, 1), (6, 160, 3, 2), (6, 320, 1, 1)):
        for i in range(n):
            stride = s if i == 0 else 1
            hidden = c_in * t
            use_res = stride == 1 and c_in == c
            y = x
            if t != 1:
                y = g.cba(y, c_in, hidden, 1, act="relu6")
            y = g.cba(y, hidden, hidden, 3, stride, 1, groups=hidden, act="relu6")
            y = g.cba(y, hidden, c, 1, act=None, res_last=use_res)
            x = g.add(y, x) if use_res else y
            c_in = c
    x = g.cba(x, c_in, 1280, 1, act="relu6")
    x = g.gap(x)
    x = g.flatten(x)
    x = g.dropout(x)
    x = g.linear(x, 1280, 1000)
    g.n_classes = 1000
    return g


# --------------------------------------------------------------------------
# Inception-v3 (torchvision, no aux logits, transform_input=False), 224^2 input
# (SURVEY Q11).  BasicConv2d = conv(no bias) + BN(eps=1e-3) + ReLU.
# --------------------------------------------------------------------------
def inception_v3() -> Graph:
    g = Graph("inception_v3", 3, 224, 224)

    def bc(x, ci, co, k, stride=1, pad=0):
        return g.cba(x, ci, co, k, stride, pad, eps=1e-3)

    def inc_a(x, ci, pf):
        b1 = bc(x, ci, 64, 1)
        b5 = bc(bc(x, ci, 48, 1), 48, 64, 5, pad=2)
        b3 = bc(bc(bc(x, ci, 64, 1), 64, 96, 3, pad=1), 96, 96, 3, pad=1)
        bp = bc(g.avgpool(x, 3, 1, 1), ci, pf, 1)
        return g.concat([b1, b5, b3, bp]), 64 + 64 + 96 + pf

    def inc_b(x, ci):
        b3 = bc(x, ci, 384, 3, stride=2)
        bd = bc(bc(bc(x, ci, 64, 1), 64, 96, 3, pad=1), 96, 96, 3, stride=2)
        bp = g.maxpool(x, 3, 2)
        return g.concat([b3, bd, bp]), 384 + 96 + ci

    def inc_c(x, ci, c7):
        b1 = bc(x, ci, 192, 1)
        b7 = bc(x, ci, c7, 1)
        b7 = bc(b7, c7, c7, (1, 7), pad=(0, 3))
        b7 = bc(b7, c7, 192, (7, 1), pad=(3, 0))
        bd = bc(x, ci, c7, 1)
        bd = bc(bd, c7, c7, (7, 1), pad=(3, 0))
        bd = bc(bd, c7, c7, (1, 7), pad=(0, 3))
        bd = bc(bd, c7, c7, (7, 1), pad=(3, 0))
        bd = bc(bd, c7, 192, (1, 7), pad=(0, 3))
        bp = bc(g.avgpool(x, 3, 1, 1), ci, 192, 1)
        return g.concat([b1, b7, bd, bp]), 768

    def inc_d(x, ci):
        b3 = bc(bc(x, ci, 192, 1), 192, 320, 3, stride=2)
        b7 = bc(x, ci, 192, 1)
        b7 = bc(b7, 192, 192, (1, 7), pad=(0, 3))
        b7 = bc(b7, 192, 192, (7, 1), pad=(3, 0))
        b7 = bc(b7, 192, 192, 3, stride=2)
        bp = g.maxpool(x, 3, 2)
        return g.concat([b3, b7, bp]), 320 + 192 + ci

    def inc_e(x, ci):
        b1 = bc(x, ci, 320, 1)
        b3 = bc(x, ci, 384, 1)
        b3 = g.concat([bc(b3, 384, 384, (1, 3), pad=(0, 1)),
                       bc(b3, 384, 384, (3, 1), pad=(1, 0))])
        bd = bc(bc(x, ci, 448, 1), 448, 384, 3, pad=1)
        bd = g.concat([bc(bd, 384, 384, (1, 3), pad=(0, 1)),
                       bc(bd, 384, 384, (3, 1), pad=(1, 0))])
        bp = bc(g.avgpool(x, 3, 1, 1), ci, 192, 1)
        return g.concat([b1, b3, bd, bp]), 2048

    x = bc(0, 3, 32, 3, stride=2)
    x = bc(x, 32, 32, 3)
    x = bc(x, 32, 64, 3, pad=1)
    x = g.maxpool(x, 3, 2)
    x = bc(x, 64, 80, 1)
    x = bc(x, 80, 192, 3)
    x = g.maxpool(x, 3, 2)
    c = 192
    x, c = inc_a(x, c, 32)
    x, c = inc_a(x, c, 64)
    x, c = inc_a(x, c, 64)
    x, c = inc_b(x, c)
    for c7 in (128, 160, 160, 192):
        x, c = inc_c(x, c, c7)
    x, c = inc_d(x, c)
    x, c = inc_e(x, c)
    x, c = inc_e(x, c)
    x = g.gap(x)
    x = g.dropout(x)
    x = g.flatten(x)
    x = g.linear(x, 2048, 1000)
    g.n_classes = 1000
    return g


# --------------------------------------------------------------------------
# MobileNetV3-large (torchvision mobilenet_v3_large; the paper's "M3", PAPER.md
# l.903).  BN eps 1e-3; squeeze-and-excitation = GAP -> FC(+ReLU) -> FC ->
# hardsigmoid -> channel scale (torchvision's 1x1 convs on the pooled map,
# written as linears); gain-1 init as for MobileNetV2.
# --------------------------------------------------------------------------
def _make_divisible(v, d=8):
    nv = max(d, int(v + d / 2) // d * d)
    if nv < 0.9 * v:
        nv += d
    return nv


def mobilenet_v3_large() -> Graph:
    g = Graph("mobilenet_v3_large", 3, 224, 224, init_gain=1.0)
    eps = 1e-3
    x = g.cba(0, 3, 16, 3, 2, 1, act="hardswish", eps=eps)
    c_in = 16
    cfg = [(3, 16, 16, False, "relu", 1), (3, 64, 24, False, "relu", 2), (3, 72, 24, False, "relu", 1),
           (5, 72, 40, True, "relu", 2), (5, 120, 40, True, "relu", 1), (5, 120, 40, True, "relu", 1),
           (3, 240, 80, False, "hardswish", 2), (3, 200, 80, False, "hardswish", 1),
           (3, 184, 80, False, "hardswish", 1), (3, 184, 80, False, "hardswish", 1),
           (3, 480, 112, True, "hardswish", 1), (3, 672, 112, True, "hardswish", 1),
           (5, 672, 160, True, "hardswish", 2), (5, 960, 160, True, "hardswish", 1),
           (5, 960, 160, True, "hardswish", 1)]
    for k, exp, out, se, act, stride in cfg:
        use_res = stride == 1 and c_in == out
        y = x
        if exp != c_in:
            y = g.cba(y, c_in, exp, 1, act=act, eps=eps)
        y = g.cba(y, exp, exp, k, stride, (k - 1) // 2, groups=exp, act=act, eps=eps)
        if se:
            sq = _make_divisible(exp // 4, 8)
            s = g.gap(y)
            s = g.relu(g.linear(s, exp, sq))
            s = g.hardsigmoid(g.linear(s, sq, exp))
            y = g.mul(y, s)
        y = g.cba(y, exp, out, 1, act=None, eps=eps, res_last=use_res)
        x = g.add(y, x) if use_res else y
        c_in = out
    x = g.cba(x, c_in, 960, 1, act="hardswish", eps=eps)
    x = g.gap(x)
    x = g.flatten(x)
    x = g.hardswish(g.linear(x, 960, 1280))
    x = g.dropout(x)
    x = g.linear(x, 1280, 1000)
    g.n_classes = 1000
    return g


# --------------------------------------------------------------------------
# DenseNet-121 (torchvision densenet121; the paper's "D121").
# Dense layer = BN -> ReLU -> conv1x1 (4 x 32) -> BN -> ReLU -> conv3x3 (32),
# its input the concatenation of every earlier feature map of the block
# (written as nested concats: feat_l = concat(feat_{l-1}, y_l), one channel
# prefix of the block's buffer each); transition = BN -> ReLU -> conv1x1
# (C/2) -> avgpool 2x2; head = BN -> ReLU -> GAP -> FC.
# --------------------------------------------------------------------------
def densenet121() -> Graph:
    g = Graph("densenet121", 3, 224, 224)
    x = g.conv(0, 3, 64, 7, 2, 3)
    x = g.relu(g.bn(x, 64))
    x = g.maxpool(x, 3, 2, 1)
    c = 64
    for bi, n_layers in enumerate((6, 12, 24, 16)):
        feat = x
        for _ in range(n_layers):
            h = g.relu(g.bn(feat, c))
            h = g.conv(h, c, 128, 1)
            h = g.relu(g.bn(h, 128))
            y = g.conv(h, 128, 32, 3, 1, 1)
            feat = g.concat([feat, y])
            c += 32
        x = feat
        if bi < 3:
            x = g.relu(g.bn(x, c))
            x = g.conv(x, c, c // 2, 1)
            x = g.avgpool(x, 2, 2)
            c //= 2
    x = g.relu(g.bn(x, c))
    x = g.gap(x)
    x = g.flatten(x)
    x = g.linear(x, c, 1000)
    g.n_classes = 1000
    return g


MODELS = {
    "tiny_cnn": tiny_cnn,
    "tiny_mlp": tiny_mlp,
    "resnet18": resnet18,
    "resnet34": resnet34,
    "resnet50": resnet50,
    "resnet101": resnet101,
    "vgg16": vgg16,
    "alexnet": alexnet,
    "mobilenet_v2": mobilenet_v2,
    "inception_v3": inception_v3,
    "mobilenet_v3_large": mobilenet_v3_large,
    "densenet121": densenet121,
}


def build_model(name: str, in_hw: int | None = None) -> Graph:
    """Return the tenant graph; ``in_hw`` overrides the spatial input size
    (used only for small parity cases; the models are defined for 224^2)."""
    g = MODELS[name]()
    if in_hw is not None and g.in_h > 1:
        g.in_h = g.in_w = in_hw
    return g


# BASELINE.json configs: name -> list of (model, batch, dtype)
CONFIGS: Dict[str, list] = {
    "d1_tiny": [("tiny_cnn", 2, "fp32"), ("tiny_mlp", 2, "fp32")],
    "d2_r50_v16_mv2": [("resnet50", 8, "bf16"), ("vgg16", 8, "bf16"),
                       ("mobilenet_v2", 8, "bf16")],
    "d3_five": [("alexnet", 16, "bf16"), ("resnet18", 16, "bf16"),
                ("resnet101", 16, "bf16"), ("inception_v3", 16, "bf16"),
                ("mobilenet_v2", 16, "bf16")],
    # the paper's Table 2 vision mixes at batch 8
    # (the paper's batches are unstated there): not BASELINE configs, used by
    # the plan sweeps and NEXT-2
    "t2_alex_v16_r18": [("alexnet", 8, "bf16"), ("vgg16", 8, "bf16"), ("resnet18", 8, "bf16")],
    "t2_r50_v16_m3": [("resnet50", 8, "bf16"), ("vgg16", 8, "bf16"), ("mobilenet_v3_large", 8, "bf16")],
    "t2_r101_d121_m3": [("resnet101", 8, "bf16"), ("densenet121", 8, "bf16"),
                        ("mobilenet_v3_large", 8, "bf16")],
}
CONFIG_INDEX = {"d1_tiny": 1, "d2_r50_v16_mv2": 2, "d3_five": 3, "d4_mixed": 4,
                "t2_alex_v16_r18": 6, "t2_r50_v16_m3": 7, "t2_r101_d121_m3": 8}
# BASELINE.json configs[3] (D4): ResNet-50 TRAINING (batch 64; one SGD step per
# round) co-located with MobileNetV2 + VGG-16 inference (batch 8, SURVEY §8(d)
# D4: the inference batch is unstated in BASELINE, 8 as in D2).  Entries:
# (model, batch, dtype, train)
TRAIN_CONFIGS: Dict[str, list] = {
    "d4_mixed": [("resnet50", 64, "bf16", True), ("vgg16", 8, "bf16", False),
                 ("mobilenet_v2", 8, "bf16", False)],
}


def config_tenants(cfg: str):
    return CONFIGS[cfg]
