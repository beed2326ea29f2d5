"""Pins of the training-tenant oracle (oracle/train.py).

Each backward operator is pinned by something other than itself: central
finite differences of the forward oracle (brute force; the ops are linear or
piecewise smooth), hand values at the kinks and ties (Q14), closed forms
(softmax-CE at uniform logits, SGD momentum over two steps, GAP), invariants
(BN-train dx is orthogonal to 1 and to xhat per channel), and PyTorch's own
fp64 autograd + torch.optim.SGD on a whole torchvision ResNet-50 in training
mode (a library routine, independent of the C loops).  A12: the mean of the
replicas' gradients equals the full-batch gradient for a BN-free tenant with
equal replica batches (mean loss)."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import workloads
from oracle import ops
from oracle import train as T


def _rng(seed):
    return np.random.default_rng(seed)


def _fd(f, a, idx, h=1e-6):
    a1, a2 = a.copy(), a.copy()
    a1[idx] += h
    a2[idx] -= h
    return (f(a1) - f(a2)) / (2 * h)


@pytest.mark.parametrize("stride,pad,groups,cin,cout", [(1, 1, 1, 2, 3), (2, 1, 1, 3, 2), (2, 0, 3, 3, 3)])
def test_conv_bwd_finite_differences(stride, pad, groups, cin, cout):
    rng = _rng(1)
    x = rng.normal(size=(2, cin, 5, 5))
    w = rng.normal(size=(cout, cin // groups, 3, 3))
    b = rng.normal(size=cout)
    y = ops.conv2d(x, w, b, stride, (pad, pad), groups)
    R = rng.normal(size=y.shape)                  # L = sum(R * y): dL/dy = R
    dx, dw, db = T.conv2d_bwd(x, w, R, stride, (pad, pad), groups, bias=True)
    L = lambda xx, ww, bb: float(np.sum(R * ops.conv2d(xx, ww, bb, stride, (pad, pad), groups)))
    for idx in np.ndindex(x.shape):
        assert _fd(lambda a: L(a, w, b), x, idx) == pytest.approx(dx[idx], abs=1e-6)
    for idx in np.ndindex(w.shape):
        assert _fd(lambda a: L(x, a, b), w, idx) == pytest.approx(dw[idx], abs=1e-6)
    for idx in np.ndindex(b.shape):
        assert _fd(lambda a: L(x, w, a), b, idx) == pytest.approx(db[idx], abs=1e-6)


def test_bn_train_forward_backward():
    rng = _rng(2)
    x = rng.normal(1.5, 2.0, size=(3, 4, 3, 2))
    g, be = rng.uniform(0.5, 1.5, 4), rng.normal(size=4)
    y, mean, var = T.bn_train_fwd(x, g, be, 1e-5)
    # definition: per-channel statistics over (n, h, w), biased variance
    assert np.allclose(mean, x.mean(axis=(0, 2, 3)), rtol=1e-14, atol=1e-14)
    assert np.allclose(var, x.var(axis=(0, 2, 3)), rtol=1e-13)
    # normalised output has zero mean and (var / (var + eps)) variance per channel, shifted by beta
    yn = (y - be[None, :, None, None]) / g[None, :, None, None]
    assert np.allclose(yn.mean(axis=(0, 2, 3)), 0, atol=1e-13)
    assert np.allclose(yn.var(axis=(0, 2, 3)), var / (var + 1e-5), rtol=1e-12)
    dy = rng.normal(size=x.shape)
    dx, dg, db = T.bn_train_bwd(x, dy, g, mean, var, 1e-5)
    xh = (x - mean[None, :, None, None]) / np.sqrt(var + 1e-5)[None, :, None, None]
    # invariants: the normalisation removes the mean direction, and the xhat
    # direction up to the eps term: sum(dx * xhat) = gamma/sigma * dgamma * eps/(var + eps)
    assert np.allclose(dx.sum(axis=(0, 2, 3)), 0, atol=1e-12)
    assert np.allclose((dx * xh).sum(axis=(0, 2, 3)), g / np.sqrt(var + 1e-5) * dg * 1e-5 / (var + 1e-5),
                       rtol=1e-6, atol=1e-15)
    # finite differences of L = sum(dy * bn_train(x))
    L = lambda xx, gg, bb: float(np.sum(dy * T.bn_train_fwd(xx, gg, bb, 1e-5)[0]))
    for idx in [(0, 0, 0, 0), (1, 2, 1, 1), (2, 3, 2, 0), (0, 1, 0, 1)]:
        assert _fd(lambda a: L(a, g, be), x, idx) == pytest.approx(dx[idx], abs=1e-6)
    for c in range(4):
        assert _fd(lambda a: L(x, a, be), g, (c,)) == pytest.approx(dg[c], abs=1e-6)
        assert _fd(lambda a: L(x, g, a), be, (c,)) == pytest.approx(db[c], abs=1e-6)


def test_relu_kinks_and_maxpool_ties():
    x = np.array([-1.0, 0.0, 0.5, 6.0, 7.0])
    dy = np.ones(5)
    assert T.relu_bwd(x, dy).tolist() == [0, 0, 1, 1, 1]
    assert T.relu_bwd(x, dy, six=True).tolist() == [0, 0, 1, 0, 0]
    # Q14: the first maximum in row-major window order takes the gradient
    x = np.array([[1.0, 3.0], [3.0, 2.0]]).reshape(1, 1, 2, 2)
    dx = T.maxpool_bwd(x, np.array([[[[5.0]]]]), (2, 2), 2)
    assert dx.reshape(-1).tolist() == [0, 5, 0, 0]
    # overlapping 3x3/s2/p1 windows: gradients of shared maxima accumulate
    x = np.zeros((1, 1, 3, 3))
    x[0, 0, 1, 1] = 1.0
    dx = T.maxpool_bwd(x, np.ones((1, 1, 2, 2)), (3, 3), 2, (1, 1))
    assert dx[0, 0, 1, 1] == 4.0 and dx.sum() == 4.0


def test_gap_linear_softmax_sgd_closed_forms():
    rng = _rng(3)
    dx = T.gap_bwd(np.array([[2.0, 4.0]]), (1, 2, 2, 2))
    assert np.all(dx[0, 0] == 0.5) and np.all(dx[0, 1] == 1.0)
    x, w = rng.normal(size=(3, 5)), rng.normal(size=(4, 5))
    dy = rng.normal(size=(3, 4))
    gx, gw, gb = T.linear_bwd(x, w, dy)
    L = lambda xx, ww: float(np.sum(dy * ops.linear(xx, ww)))
    for idx in np.ndindex(x.shape):
        assert _fd(lambda a: L(a, w), x, idx) == pytest.approx(gx[idx], abs=1e-6)
    for idx in np.ndindex(w.shape):
        assert _fd(lambda a: L(x, a), w, idx) == pytest.approx(gw[idx], abs=1e-6)
    assert np.allclose(gb, dy.sum(0), rtol=1e-14)
    # softmax-CE at uniform logits: loss = log C, dz = (1/C - onehot) / N
    z = np.full((2, 5), 0.7)
    loss, dz = T.softmax_ce(z, [1, 4])
    assert loss == pytest.approx(np.log(5), rel=1e-14)
    ref = np.full((2, 5), 0.2 / 2)
    ref[0, 1] -= 0.5
    ref[1, 4] -= 0.5
    assert np.allclose(dz, ref, atol=1e-15)
    z = rng.normal(size=(4, 7)) * 5
    loss, dz = T.softmax_ce(z, [0, 3, 6, 2])
    assert np.allclose(dz.sum(1), 0, atol=1e-15)
    for idx in [(0, 0), (1, 3), (2, 5), (3, 2)]:
        assert _fd(lambda a: T.softmax_ce(a, [0, 3, 6, 2])[0], z, idx) == pytest.approx(dz[idx], abs=1e-7)
    # SGD momentum, two steps: w2 = w0 - lr g0 - lr (m g0 + g1)
    w0, g0, g1 = rng.normal(size=6), rng.normal(size=6), rng.normal(size=6)
    w, buf = w0.copy(), np.zeros(6)
    T.sgd_momentum(w, g0, buf, 0.1, 0.9, True)
    T.sgd_momentum(w, g1, buf, 0.1, 0.9, False)
    assert np.allclose(w, w0 - 0.1 * g0 - 0.1 * (0.9 * g0 + g1), rtol=1e-14, atol=1e-15)


def _torch_resnet50_step(graph, params, x, labels, steps):
    """Reference via torchvision + fp64 autograd + torch.optim.SGD."""
    import torchvision
    from test_oracle_models import load_into_torch
    m = load_into_torch(graph, params, torchvision.models.resnet50()).train()
    opt = torch.optim.SGD(m.parameters(), lr=0.1, momentum=0.9)
    mods = [mm for mm in m.modules() if isinstance(mm, (torch.nn.Conv2d, torch.nn.BatchNorm2d, torch.nn.Linear))]
    losses, grads = [], None
    for _ in range(steps):
        opt.zero_grad()
        loss = F.cross_entropy(m(torch.from_numpy(x).double()), torch.from_numpy(labels).long())
        loss.backward()
        losses.append(float(loss.detach()))
        grads = [{n: p.grad.detach().clone().numpy() for n, p in mm.named_parameters(recurse=False)} for mm in mods]
        opt.step()
    return losses, grads, mods


def test_resnet50_train_steps_match_torch_autograd():
    """Two SGD-momentum steps of a whole ResNet-50 (BN training mode) at 32x32,
    B=4: loss, every gradient, updated weights and BN running statistics vs
    PyTorch fp64."""
    g = workloads.build_model("resnet50", 32)
    params = workloads.make_params(g, 11, "fp32")
    x = workloads.make_input(g, 4, 11, "fp32")
    labels = workloads.make_labels(4, 11)
    losses, grads_t, mods = _torch_resnet50_step(g, params, x, labels, steps=2)
    loss1, _, p1, st = T.train_step(g, params, x, labels)
    loss2, grads2, p2, _ = T.train_step(g, p1, x, labels, state=st)
    assert loss1 == pytest.approx(losses[0], rel=1e-10)
    assert loss2 == pytest.approx(losses[1], rel=1e-9)
    ours = [op for op in g.ops if op["kind"] in ("conv", "bn", "linear")]
    assert len(ours) == len(mods)
    worst = 0.0
    for op, mm, gt in zip(ours, mods, grads_t):
        go = grads2[op["id"]]
        names = {"weight": "gamma", "bias": "beta"} if op["kind"] == "bn" else {"weight": "w", "bias": "b"}
        for tn, arr in gt.items():
            a = go[names[tn]]
            worst = max(worst, float(np.max(np.abs(a - arr)) / max(np.max(np.abs(arr)), 1e-30)))
        with torch.no_grad():
            if op["kind"] == "bn":
                assert np.allclose(p2[op["id"]]["gamma"], mm.weight.numpy(), rtol=1e-9, atol=1e-10)
                assert np.allclose(p2[op["id"]]["mean"], mm.running_mean.numpy(), rtol=1e-9, atol=1e-10)
                assert np.allclose(p2[op["id"]]["var"], mm.running_var.numpy(), rtol=1e-9, atol=1e-10)
            else:
                assert np.allclose(p2[op["id"]]["w"], mm.weight.numpy(), rtol=1e-9, atol=1e-10)
    assert worst < 1e-7, worst


def test_allreduce_mean_equals_full_batch_gradient_without_bn():
    """A12: with a mean loss and equal replica batches, the mean of the
    replicas' gradients is the full-batch gradient (no BN: BN statistics are
    per replica by definition, so BN tenants differ)."""
    g = workloads.Graph("cnn_nobn", 3, 8, 8)
    h = g.conv(0, 3, 4, 3, 1, 1, bias=True)
    h = g.relu(h)
    h = g.maxpool(h, 2, 2)
    h = g.conv(h, 4, 6, 3, 2, 1)
    h = g.relu(h)
    h = g.gap(h)
    g.linear(h, 6, 5)
    params = workloads.make_params(g, 5, "fp32")
    x = workloads.make_input(g, 4, 5, "fp32")
    labels = workloads.make_labels(4, 5, 5)
    _, gfull, _, _ = T.train_step(g, params, x, labels)
    reps = [T.train_step(g, params, x[i:i + 2], labels[i:i + 2])[1] for i in (0, 2)]
    gmean = T.allreduce_mean(reps)
    for oid in gfull:
        for n in gfull[oid]:
            assert np.allclose(gmean[oid][n], gfull[oid][n], rtol=1e-12, atol=1e-14)
    # the hook path applies the averaged gradient
    _, gh, _, _ = T.train_step(g, params, x[:2], labels[:2], grads_hook=lambda gr: T.allreduce_mean([gr, reps[1]]))
    assert np.array_equal(gh[1]["w"], gmean[1]["w"])
