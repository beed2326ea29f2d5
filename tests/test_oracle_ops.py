"""Pins for the oracle's operators -- none of these re-type
the oracle's own formula: they use a hand-computed example, closed forms for
constant inputs, brute force via numpy matmul, and torch-CPU fp64 library
routines."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import ops
from gacer_testutil import read_golden

RNG = np.random.default_rng(1234)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


# ---------------------------------------------------------------- hand value
def test_conv_hand_example():
    want = np.array([[float(v) for v in ln.split()] for ln in read_golden("conv_hand.txt")])
    x = np.arange(1, 10, dtype=np.float64).reshape(1, 1, 3, 3)
    w = np.ones((1, 1, 3, 3))
    y = ops.conv2d(x, w, None, 1, (1, 1))
    assert np.array_equal(y[0, 0], want)


# ---------------------------------------------------------------- closed forms
@pytest.mark.parametrize("groups", [1, 4])
def test_conv_constant_closed_form(groups):
    c, v, b = 0.75, -1.25, 0.5
    Cin, Cout, H = 8, 4, 6
    x = np.full((2, Cin, H, H), c)
    w = np.full((Cout, Cin // groups, 3, 3), v)
    y = ops.conv2d(x, w, np.full(Cout, b), 1, (1, 1), groups)
    cig = Cin // groups
    assert np.allclose(y[:, :, 1:-1, 1:-1], c * v * cig * 9 + b, rtol=0, atol=1e-12)
    assert np.allclose(y[:, :, 0, 0], c * v * cig * 4 + b, rtol=0, atol=1e-12)   # corner: 4 taps
    assert np.allclose(y[:, :, 0, 2], c * v * cig * 6 + b, rtol=0, atol=1e-12)   # edge: 6 taps
    assert np.allclose(y[:, :, -1, -1], c * v * cig * 4 + b, rtol=0, atol=1e-12)


def test_conv_stride2_taps_closed_form():
    # 7x7 stride 2 pad 3 on 9x9 ones: count in-bounds taps per output by enumeration
    x = np.ones((1, 1, 9, 9))
    y = ops.conv2d(x, np.ones((1, 1, 7, 7)), None, 2, (3, 3))
    for ho in range(y.shape[2]):
        for wo in range(y.shape[3]):
            rows = sum(0 <= ho * 2 - 3 + r < 9 for r in range(7))
            cols = sum(0 <= wo * 2 - 3 + s < 9 for s in range(7))
            assert y[0, 0, ho, wo] == rows * cols


def test_pool_relu_gap_constants():
    c = 1.5
    x = np.full((2, 3, 7, 7), c)
    assert np.all(ops.maxpool(x, 3, 2, (1, 1)) == c)
    assert np.all(ops.gap(x) == c)
    assert np.all(ops.relu(x) == c)
    assert np.all(ops.relu(np.full((4,), 7.0), six=True) == 6.0)
    assert np.all(ops.relu(np.full((4,), -7.0)) == 0.0)
    # avg-pool count_include_pad: border value c * (#valid taps) / k^2
    y = ops.avgpool(x, 3, 1, (1, 1), count_include_pad=True)
    assert np.isclose(y[0, 0, 0, 0], c * 4 / 9) and np.isclose(y[0, 0, 0, 3], c * 6 / 9)
    assert np.isclose(y[0, 0, 3, 3], c)
    y2 = ops.avgpool(x, 3, 1, (1, 1), count_include_pad=False)
    assert np.allclose(y2, c)


def test_linear_bn_closed_form():
    c, v, b = 0.5, 2.0, -0.25
    y = ops.linear(np.full((3, 10), c), np.full((4, 10), v), np.full(4, b))
    assert np.allclose(y, c * v * 10 + b)
    g, be, m, var, eps = 1.1, 0.2, -0.05, 0.9, 1e-5
    y = ops.batchnorm(np.full((2, 3, 2, 2), c), *(np.full(3, t) for t in (g, be, m, var)), eps)
    assert np.allclose(y, g * (c - m) / np.sqrt(var + eps) + be, rtol=1e-15)


# ---------------------------------------------------------------- brute force
def test_conv1x1_is_matmul():
    x = RNG.standard_normal((2, 16, 5, 5))
    w = RNG.standard_normal((8, 16, 1, 1))
    y = ops.conv2d(x, w)
    ref = np.einsum("nchw,oc->nohw", x, w[:, :, 0, 0])
    assert rel(y, ref) < 1e-13


# ---------------------------------------------------------------- library routines
@pytest.mark.parametrize("cfg", [
    dict(N=2, Cin=3, Cout=8, H=13, W=11, k=(3, 3), s=1, p=(1, 1), g=1, bias=True),
    dict(N=1, Cin=8, Cout=16, H=16, W=16, k=(7, 7), s=2, p=(3, 3), g=1, bias=False),
    dict(N=2, Cin=12, Cout=12, H=9, W=9, k=(3, 3), s=2, p=(1, 1), g=12, bias=False),
    dict(N=1, Cin=6, Cout=10, H=10, W=10, k=(1, 7), s=1, p=(0, 3), g=1, bias=False),
    dict(N=1, Cin=6, Cout=10, H=10, W=10, k=(7, 1), s=1, p=(3, 0), g=1, bias=True),
    dict(N=1, Cin=3, Cout=4, H=31, W=31, k=(11, 11), s=4, p=(2, 2), g=1, bias=True),
])
def test_conv_vs_torch(cfg):
    x = RNG.standard_normal((cfg["N"], cfg["Cin"], cfg["H"], cfg["W"]))
    w = RNG.standard_normal((cfg["Cout"], cfg["Cin"] // cfg["g"], *cfg["k"]))
    b = RNG.standard_normal(cfg["Cout"]) if cfg["bias"] else None
    y = ops.conv2d(x, w, b, cfg["s"], cfg["p"], cfg["g"])
    ref = F.conv2d(torch.from_numpy(x), torch.from_numpy(w),
                   None if b is None else torch.from_numpy(b),
                   stride=cfg["s"], padding=cfg["p"], groups=cfg["g"]).numpy()
    assert y.shape == ref.shape
    assert rel(y, ref) < 1e-12


@pytest.mark.parametrize("k,s,p", [(3, 2, 1), (2, 2, 0), (3, 2, 0), (3, 1, 1)])
def test_pools_vs_torch(k, s, p):
    x = RNG.standard_normal((2, 5, 15, 15))
    t = torch.from_numpy(x)
    assert np.array_equal(ops.maxpool(x, k, s, (p, p)), F.max_pool2d(t, k, s, p).numpy())
    for cip in (True, False):
        assert rel(ops.avgpool(x, k, s, (p, p), cip),
                   F.avg_pool2d(t, k, s, p, count_include_pad=cip).numpy()) < 1e-14
    assert rel(ops.gap(x), F.adaptive_avg_pool2d(t, 1).numpy()) < 1e-14


def test_linear_bn_vs_torch():
    x = RNG.standard_normal((4, 37))
    w = RNG.standard_normal((9, 37))
    b = RNG.standard_normal(9)
    assert rel(ops.linear(x, w, b), F.linear(*(torch.from_numpy(a) for a in (x, w, b))).numpy()) < 1e-13
    x = RNG.standard_normal((2, 6, 4, 4))
    g, be, m = (RNG.standard_normal(6) for _ in range(3))
    v = RNG.uniform(0.5, 1.5, 6)
    ref = F.batch_norm(torch.from_numpy(x), torch.from_numpy(m), torch.from_numpy(v),
                       torch.from_numpy(g), torch.from_numpy(be), False, 0.0, 1e-3).numpy()
    assert rel(ops.batchnorm(x, g, be, m, v, 1e-3), ref) < 1e-14


def test_hardswish_hardsigmoid_closed_forms():
    """MobileNetV3's activations ("M3"): PyTorch's
    definitions x * relu6(x + 3) / 6 and relu6(x + 3) / 6 at hand-checked
    points -- the knees (-3, 3), the saturation, the midpoint."""
    x = np.array([-5.0, -3.0, -1.5, 0.0, 1.0, 3.0, 4.5])
    assert np.array_equal(ops.hardswish(x), np.array([0.0, 0.0, -0.375, 0.0, 4.0 / 6.0, 3.0, 4.5]))
    assert np.array_equal(ops.hardsigmoid(x), np.array([0.0, 0.0, 0.25, 0.5, 4.0 / 6.0, 1.0, 1.0]))


def test_hardswish_hardsigmoid_scale_vs_torch():
    import torch.nn.functional as F
    rng = np.random.default_rng(5)
    x = rng.normal(scale=4.0, size=(3, 5, 4, 6))
    t = torch.from_numpy(x)
    assert np.max(np.abs(ops.hardswish(x) - F.hardswish(t).numpy())) < 1e-15
    assert np.max(np.abs(ops.hardsigmoid(x) - F.hardsigmoid(t).numpy())) < 1e-15
    s = rng.uniform(0, 1, size=(3, 5))
    ref = x * s[:, :, None, None]                 # numpy broadcasting (a library routine)
    assert np.array_equal(ops.scale_channels(x, s), ref)
    assert np.array_equal(ops.scale_channels(x, s.reshape(3, 5, 1, 1)), ref)
