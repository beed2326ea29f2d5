"""A11 / D4 on the GPU: the training tenant's SGD step as executor work
items (gacer_graph.train = 1), alone and beside inference tenants in one
round (GACER's techniques
"are applicable to both the training and inference phases").

Pins (SURVEY §8(c) C2b readings):
  (1) per-operator parity of every training operator vs the fp64 oracle:
      tests/test_gpu_train_ops.py -- the executor runs the SAME device
      functions (train_dev.cuh) with the same thread count and virtual-block
      decomposition, and the same GEMM geometries, so
  (*) the executor's step is bit-identical to the call-by-call
      SequentialTrainer step (loss, gradients, updated weights, momentum);
  (2)/(3) loss and FC gradient within 2e-2 of the oracle's fp64 step;
  (4) gradients and updated weights bitwise identical across regulation
      plans (pointers, SM partitions, co-located inference tenants), and the
      co-located inference outputs byte-identical to inference-only rounds."""
import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu


def maxrel(y, r):
    return float(np.max(np.abs(y - r)) / max(np.max(np.abs(r)), 1e-30))


def nhwc8(x):
    B, C, H, W = x.shape
    xp = np.zeros((B, H, W, 8), np.float32)
    xp[..., :C] = x.transpose(0, 2, 3, 1)
    return xp


def train_case(name, hw, B, seed):
    g = workloads.build_model(name, hw)
    return g, workloads.make_params(g, seed, "fp32"), workloads.make_input(g, B, seed, "bf16"), \
        workloads.make_labels(B, seed)


def executor_steps(g, params, x, labels, B, steps, extra=(), plan=None, partition="priority", mode="executor",
                   num_ctas=0):
    """Run `steps` rounds with the training tenant first; returns per-step
    (loss, grads, params, momentum) numpy copies and the extra tenants'
    outputs of the last round."""
    import torch
    from paper_2304_11745_b200.runtime import Session
    ts = [(g, params, B, "bf16", {"train": True})] + [t[:4] for t in extra]
    s = Session(ts, partition=partition, num_ctas=num_ctas)
    try:
        s.set_input(0, x)
        s.set_labels(0, labels)
        for t, tt in enumerate(extra):
            s.set_input(t + 1, tt[4])
        if plan is not None:
            s.set_regulation(*plan)
        s.set_mode(mode)
        out = []
        for _ in range(steps):
            s.run()
            torch.cuda.synchronize()
            loss, p, gr, m = s.train_state(0)
            out.append((float(loss.item()), gr.cpu().numpy().copy(), p.cpu().numpy().copy(), m.cpu().numpy().copy()))
        res = s.results()[1:]
        launches = s.stats()["kernel_launches"]
    finally:
        s.close()
    return out, res, launches


def sequential_steps(g, params, x, labels, B, steps):
    import torch
    from paper_2304_11745_b200 import gacer as G
    from paper_2304_11745_b200.train_driver import SequentialTrainer
    G.gacer_init(0)
    try:
        tr = SequentialTrainer(g, params, B)
        xd = torch.from_numpy(nhwc8(x)).to(torch.bfloat16).cuda()
        lab = torch.from_numpy(labels).cuda()
        out = []
        for _ in range(steps):
            loss, _ = tr.step(xd, lab)
            torch.cuda.synchronize()
            out.append((float(loss.item()), tr.flat_g.cpu().numpy().copy(), tr.flat_p.cpu().numpy().copy(),
                        tr.flat_m.cpu().numpy().copy()))
    finally:
        G.gacer_shutdown()
    return out


@pytest.mark.parametrize("name,hw,B", [("resnet18", 64, 4), ("resnet50", 64, 4)])
def test_executor_step_bitwise_equals_sequential_trainer(cuda_ok, name, hw, B):
    g, params, x, labels = train_case(name, hw, B, 51)
    ex, _, launches = executor_steps(g, params, x, labels, B, steps=2)
    assert launches == 1                       # the whole step is ONE persistent-kernel launch
    sq = sequential_steps(g, params, x, labels, B, steps=2)
    for k, (a, b) in enumerate(zip(ex, sq)):
        assert a[0] == b[0], (k, a[0], b[0])
        for j, what in ((1, "grads"), (2, "params"), (3, "momentum")):
            assert a[j].tobytes() == b[j].tobytes(), (k, what, maxrel(a[j], b[j]))
    assert ex[1][0] < ex[0][0]                 # the update lowers the loss on the batch


def test_executor_step_vs_oracle_r50_224(cuda_ok):
    """C2b (2)/(3) at the configuration C2b measured: ResNet-50, 224^2, B=16:
    loss and FC gradient of the executor's step within 2e-2 of the oracle's
    fp64 step."""
    from oracle import train as OT
    from paper_2304_11745_b200 import gacer as G
    g, params, x, labels = train_case("resnet50", 224, 16, 41)
    ex, _, _ = executor_steps(g, params, x, labels, 16, steps=1)
    loss_o, grads_o, _, _ = OT.train_step(g, params, x, labels)
    G.gacer_init(-1)
    try:
        t = G.gacer_register_tenant(g, params, 16, "bf16", train=True)
        fc = len(g.ops)
        off, cnt = G.gacer_train_param(t, fc, 0)
    finally:
        G.gacer_shutdown()
    fc_id = g.ops[-1]["id"]
    gw = ex[0][1][off:off + cnt].reshape(grads_o[fc_id]["w"].shape)
    assert abs(ex[0][0] - loss_o) / abs(loss_o) <= 2e-2, (ex[0][0], loss_o)
    assert maxrel(gw, grads_o[fc_id]["w"]) <= 2e-2, maxrel(gw, grads_o[fc_id]["w"])


def test_mixed_round_invariance(cuda_ok):
    """D4 shape at a small size: a ResNet-18 training tenant beside VGG-16 and
    MobileNetV2 inference tenants in ONE round.  Training results are bitwise
    identical to the training tenant alone and across plans (sync pointers
    over every tenant's list, SM partitions, grid sizes, the sequential and
    multi-stream baselines); inference outputs are byte-identical to an
    inference-only round."""
    from paper_2304_11745_b200.runtime import Session
    g, params, x, labels = train_case("resnet18", 64, 8, 61)
    inf = []
    for i, (name, hw, bi) in enumerate((("vgg16", 224, 1), ("mobilenet_v2", 64, 2))):
        gi = workloads.build_model(name, hw)
        inf.append((gi, workloads.make_params(gi, 62 + i, "bf16"), bi, "bf16",
                    workloads.make_input(gi, bi, 62 + i, "bf16")))
    s = Session([t[:4] for t in inf])
    try:
        for t, tt in enumerate(inf):
            s.set_input(t, tt[4])
        s.run()
        inf_ref = s.results()
    finally:
        s.close()
    alone, _, _ = executor_steps(g, params, x, labels, 8, steps=2)
    n_tr = 2 * len(g.ops) + 1
    variants = [dict(), dict(partition="strict"), dict(partition="work_conserving"), dict(num_ctas=100),
                dict(plan=(None, [[len(g.ops), n_tr - 5], [5, 15], [10, 40]])),
                dict(plan=(None, [[3, n_tr - 20], [0, 22], [60, 60]]), partition="hybrid"),
                dict(mode="sequential"), dict(mode="multistream")]
    for v in variants:
        got, outs, _ = executor_steps(g, params, x, labels, 8, steps=2, extra=inf, **v)
        for k in range(2):
            assert got[k][0] == alone[k][0], v
            for j in (1, 2, 3):
                assert got[k][j].tobytes() == alone[k][j].tobytes(), (v, k, j)
        for a, b in zip(outs, inf_ref):
            assert a.tobytes() == b.tobytes(), v
