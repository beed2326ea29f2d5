"""A11 composition check: one SGD step of a small residual CNN (conv / BN-train
/ ReLU / max-pool / residual add / strided conv / GAP / FC / softmax-CE)
assembled from the device operators of include/gacer_train.h, vs the fp64
oracle's whole training step (oracle/train.py: train_step).  Gates (SURVEY
§8(c) C2b readings (2), (3)): loss and FC-layer gradient within 2e-2
(max-norm relative); the conv gradients are reported and held to a looser
bound (bf16 activations, bf16-rounded GEMM operands); the SGD update of the
FC weights within 2e-2 of the oracle's update.  Deeper gradients are
reported, not gated end to end (C2b: bf16 activations through small-batch
BN are ill-conditioned against an fp64 forward -- measured 0.1-0.27 here);
instead the last block's BN backward and weight gradient are gated at 2e-2
against the oracle fed the device's own saved tensors (reading (1)), with
a loose end-to-end bound that still catches layout or sign errors.  The step runs op by op on
one stream (each operator one or a few launches); running it as executor
work items is the next step of A11."""
import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu


def maxrel(a, r):
    a = np.asarray(a, np.float64)
    return float(np.max(np.abs(a - r)) / max(np.max(np.abs(r)), 1e-30))


def tiny_res():
    g = workloads.Graph("tiny_res", 8, 16, 16)
    c0 = g.conv(0, 8, 64, 3, 1, 1); b0 = g.bn(c0, 64); r0 = g.relu(b0)
    p0 = g.maxpool(r0, 3, 2, 1)
    c1 = g.conv(p0, 64, 64, 3, 1, 1); b1 = g.bn(c1, 64); r1 = g.relu(b1)
    c2 = g.conv(r1, 64, 64, 3, 1, 1); b2 = g.bn(c2, 64)
    a = g.add(b2, p0); r2 = g.relu(a)
    c3 = g.conv(r2, 64, 128, 3, 2, 1); b3 = g.bn(c3, 128); r3 = g.relu(b3)
    gp = g.gap(r3)
    g.linear(gp, 128, 10)
    g.n_classes = 10
    return g


def test_small_resnet_sgd_step_matches_oracle():
    import torch
    from oracle import train as OT
    from paper_2304_11745_b200 import gacer as G

    g = tiny_res()
    B = 4
    params = workloads.make_params(g, 31, "fp32")
    x = workloads.make_input(g, B, 31, "bf16")
    labels = workloads.make_labels(B, 31, 10)
    loss_o, grads_o, new_o, _ = OT.train_step(g, params, x, labels, lr=0.1, momentum=0.9)

    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
    bf = lambda shape: torch.empty(shape, dtype=torch.bfloat16, device="cuda")
    f32 = lambda shape: torch.empty(shape, device="cuda")
    P = lambda t: t.data_ptr()
    ids = {op["kind"] + str(i): op["id"] for i, op in enumerate(g.ops)}
    convs = [op for op in g.ops if op["kind"] == "conv"]
    bns = [op for op in g.ops if op["kind"] == "bn"]
    fc = [op for op in g.ops if op["kind"] == "linear"][0]
    W = {op["id"]: dev(params[op["id"]]["w"]) for op in convs + [fc]}
    bfc = dev(params[fc["id"]]["b"])
    GB = {op["id"]: (dev(params[op["id"]]["gamma"]), dev(params[op["id"]]["beta"])) for op in bns}
    G.gacer_init(0)
    try:
        ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
        WS = (ws.data_ptr() + 255) // 256 * 256
        NB = (64 << 20) - 256
        bnsc = f32(1 << 20)

        def conv(xin, op, Hin, stride, out):
            Cin, Cout = op["c_in"], op["c_out"]
            G.conv_fwd(P(xin), P(W[op["id"]]), B, Hin, Hin, Cin, Cout, 3, 3, stride, 1, 1, P(out), WS, NB)

        def bn_fwd(xin, op, M, relu, out):
            C = op["c"]
            mean, var = f32(C), f32(C)
            G.bn_train_fwd(P(xin), M, C, P(GB[op["id"]][0]), P(GB[op["id"]][1]), op["eps"], relu, P(out), P(mean),
                           P(var), P(bnsc))
            return mean, var

        X = torch.from_numpy(np.ascontiguousarray(x.transpose(0, 2, 3, 1))).to(torch.bfloat16).cuda()
        # ---- forward (NHWC)
        C0 = bf((B, 16, 16, 64)); conv(X, convs[0], 16, 1, C0)
        R0 = bf((B, 16, 16, 64)); st0 = bn_fwd(C0, bns[0], B * 256, 1, R0)
        P0 = bf((B, 8, 8, 64)); G.maxpool_fwd(P(R0), B, 16, 16, 64, 3, 3, 2, 1, 1, 8, 8, P(P0))
        C1 = bf((B, 8, 8, 64)); conv(P0, convs[1], 8, 1, C1)
        R1 = bf((B, 8, 8, 64)); st1 = bn_fwd(C1, bns[1], B * 64, 1, R1)
        C2 = bf((B, 8, 8, 64)); conv(R1, convs[2], 8, 1, C2)
        B2 = bf((B, 8, 8, 64)); st2 = bn_fwd(C2, bns[2], B * 64, 0, B2)
        R2 = bf((B, 8, 8, 64)); G.add(P(B2), P(P0), B * 64 * 64, 1, P(R2))
        C3 = bf((B, 4, 4, 128)); conv(R2, convs[3], 8, 2, C3)
        R3 = bf((B, 4, 4, 128)); st3 = bn_fwd(C3, bns[3], B * 16, 1, R3)
        GP = bf((B, 128)); G.gap_fwd(P(R3), B, 16, 128, P(GP))
        Z = f32((B, 10)); G.linear_fwd(P(GP), P(W[fc["id"]]), P(bfc), B, 128, 10, P(Z))
        lab = torch.from_numpy(labels).cuda()
        loss = f32(1); dZ = f32((B, 10)); G.softmax_ce(P(Z), P(lab), B, 10, P(loss), P(dZ), P(f32(B)))
        # ---- backward
        dGP = f32((B, 128)); dWfc = f32((10, 128)); dbfc = f32(10)
        G.linear_bwd(P(GP), P(W[fc["id"]]), P(dZ), B, 128, 10, P(dGP), P(dWfc), P(dbfc))
        dR3 = bf((B, 4, 4, 128)); G.gap_bwd(P(dGP), B, 16, 128, P(dR3))
        G.relu_bwd(P(R3), P(dR3), dR3.numel(), 0, P(dR3))          # mask from the ReLU output (y > 0 iff x > 0)
        dgam, dbet = {}, {}

        def bn_bwd(xin, dy, op, st, M, dx):
            C = op["c"]
            dgam[op["id"]], dbet[op["id"]] = f32(C), f32(C)
            G.bn_train_bwd(P(xin), P(dy), M, C, P(GB[op["id"]][0]), P(st[0]), P(st[1]), op["eps"], P(dx),
                           P(dgam[op["id"]]), P(dbet[op["id"]]), P(bnsc))

        dW = {}

        def conv_bwd(xin, dy, op, Hin, stride, dx):
            Cin, Cout = op["c_in"], op["c_out"]
            dW[op["id"]] = f32((Cout, Cin, 3, 3))
            G.conv_wgrad(P(xin), P(dy), B, Hin, Hin, Cin, Cout, 3, 3, stride, 1, 1, P(dW[op["id"]]), WS, NB)
            if dx is not None:
                G.conv_dgrad(P(dy), P(W[op["id"]]), B, Hin, Hin, Cin, Cout, 3, 3, stride, 1, 1, P(dx), WS, NB)

        dC3 = bf((B, 4, 4, 128)); bn_bwd(C3, dR3, bns[3], st3, B * 16, dC3)
        dR2 = bf((B, 8, 8, 64)); conv_bwd(R2, dC3, convs[3], 8, 2, dR2)
        G.relu_bwd(P(R2), P(dR2), dR2.numel(), 0, P(dR2))          # dA (gradient of the residual sum)
        dC2 = bf((B, 8, 8, 64)); bn_bwd(C2, dR2, bns[2], st2, B * 64, dC2)
        dR1 = bf((B, 8, 8, 64)); conv_bwd(R1, dC2, convs[2], 8, 1, dR1)
        G.relu_bwd(P(R1), P(dR1), dR1.numel(), 0, P(dR1))
        dC1 = bf((B, 8, 8, 64)); bn_bwd(C1, dR1, bns[1], st1, B * 64, dC1)
        dP0 = bf((B, 8, 8, 64)); conv_bwd(P0, dC1, convs[1], 8, 1, dP0)
        G.add(P(dR2), P(dP0), dP0.numel(), 0, P(dP0))             # skip path + branch
        dR0 = bf((B, 16, 16, 64))
        G.maxpool_bwd(P(R0), P(dP0), B, 16, 16, 64, 3, 3, 2, 1, 1, 8, 8, P(dR0), WS)
        G.relu_bwd(P(R0), P(dR0), dR0.numel(), 0, P(dR0))
        dC0 = bf((B, 16, 16, 64)); bn_bwd(C0, dR0, bns[0], st0, B * 256, dC0)
        conv_bwd(X, dC0, convs[0], 16, 1, None)
        # ---- SGD (first step: buf = g)
        wfc_new = W[fc["id"]].clone(); buf = torch.zeros_like(wfc_new)
        G.sgd_momentum(P(wfc_new), P(dWfc), P(buf), wfc_new.numel(), 0.1, 0.9, 1)
        torch.cuda.synchronize()
    finally:
        G.gacer_shutdown()

    errs = {"loss": abs(float(loss) - loss_o) / abs(loss_o),
            "fc_w": maxrel(dWfc.cpu().numpy(), grads_o[fc["id"]]["w"]),
            "fc_b": maxrel(dbfc.cpu().numpy(), grads_o[fc["id"]]["b"]),
            "fc_sgd": maxrel(wfc_new.cpu().numpy() - params[fc["id"]]["w"],
                             new_o[fc["id"]]["w"] - params[fc["id"]]["w"])}
    for op in convs:
        errs[f"conv{op['id']}_w"] = maxrel(dW[op["id"]].cpu().numpy(), grads_o[op["id"]]["w"])
    for op in bns:
        errs[f"bn{op['id']}_gamma"] = maxrel(dgam[op["id"]].cpu().numpy(), grads_o[op["id"]]["gamma"])
    # last block, oracle fed the device's saved tensors (well-conditioned)
    nchw = lambda t, *shape: t.float().cpu().numpy().astype(np.float64).reshape(shape).transpose(0, 3, 1, 2)
    op3, bn3 = convs[3], bns[3]
    ref_dC3 = OT.bn_train_bwd(nchw(C3, B, 4, 4, 128), nchw(dR3, B, 4, 4, 128), params[bn3["id"]]["gamma"],
                              st3[0].cpu().numpy().astype(np.float64), st3[1].cpu().numpy().astype(np.float64),
                              bn3["eps"])[0]
    errs["block_dC3"] = maxrel(nchw(dC3, B, 4, 4, 128), ref_dC3)
    ref_dW3 = OT.conv2d_bwd(nchw(R2, B, 8, 8, 64), params[op3["id"]]["w"], nchw(dC3, B, 4, 4, 128), 2, (1, 1))[1]
    errs["block_dW3"] = maxrel(dW[op3["id"]].cpu().numpy(), ref_dW3)
    print(errs)
    assert errs["loss"] <= 2e-2 and errs["fc_w"] <= 2e-2 and errs["fc_b"] <= 2e-2 and errs["fc_sgd"] <= 2e-2, errs
    assert errs["block_dC3"] <= 2e-2 and errs["block_dW3"] <= 2e-2, errs
    assert max(v for k, v in errs.items() if k.startswith(("conv", "bn"))) <= 0.5, errs


def test_nccl_gradient_mean_on_comm_stream():
    """A12 transport on the device: the bucketed NCCL all-reduce of CUDA
    gradient tensors on a dedicated stream (world size 1 here: the box has
    one GPU; the 2-rank arithmetic is checked with gloo on the CPU)."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    from paper_2304_11745_b200.grad_allreduce import GradBuckets
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        shapes = [(64, 3, 7, 7), (1000, 2048), (1000,)]
        g = [torch.randn(sh, device="cuda") for sh in shapes]
        ref = [t.clone() for t in g]
        comm = torch.cuda.Stream()
        comm.wait_stream(torch.cuda.current_stream())
        GradBuckets(shapes, bucket_bytes=1 << 20).reduce_mean(g, dist, stream=comm)
        torch.cuda.current_stream().wait_stream(comm)
        torch.cuda.synchronize()
        assert all(torch.equal(a, b) for a, b in zip(g, ref))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,hw,B", [("resnet50", 224, 16), ("resnet18", 64, 8)])
def test_sequential_trainer_resnet_step(name, hw, B):
    """The whole ResNet training step driven by train_driver.SequentialTrainer
    (every step a libgacer.so call) vs the oracle's fp64 step: loss and FC
    gradient within 2e-2 (C2b readings (2), (3)); a second step lowers the
    loss on the same batch (the SGD update is applied on the device)."""
    import torch
    from oracle import train as OT
    from paper_2304_11745_b200 import gacer as G
    from paper_2304_11745_b200.train_driver import SequentialTrainer

    g = workloads.build_model(name, hw)
    params = workloads.make_params(g, 41, "fp32")
    x = workloads.make_input(g, B, 41, "bf16")
    labels = workloads.make_labels(B, 41)
    loss_o, grads_o, _, _ = OT.train_step(g, params, x, labels)
    G.gacer_init(0)
    try:
        tr = SequentialTrainer(g, params, B)
        xp = np.zeros((B, hw, hw, 8), np.float32)
        xp[..., :3] = x.transpose(0, 2, 3, 1)
        xd = torch.from_numpy(xp).to(torch.bfloat16).cuda()
        lab = torch.from_numpy(labels).cuda()
        loss1, grads = tr.step(xd, lab)
        fc = [op for op in g.ops if op["kind"] == "linear"][0]["id"]
        gw = grads[fc]["w"].cpu().numpy()
        l1 = float(loss1)
        loss2, _ = tr.step(xd, lab)
        l2 = float(loss2)
        torch.cuda.synchronize()
    finally:
        G.gacer_shutdown()
    print(name, l1, loss_o, maxrel(gw, grads_o[fc]["w"]), l2)
    assert abs(l1 - loss_o) / abs(loss_o) <= 2e-2
    # FC gradient: 2e-2 (SURVEY §8(c) C2b reading (3)).  ResNet-50 runs at
    # 224^2, B=16, the configuration C2b measured (FC gradient ~1e-2 with
    # bf16 stores): its error vs the fp64 forward is the bf16-activation
    # conditioning of deep BN nets and grows as the BN sample count shrinks
    # (C2b), so small-image cases do not test the kernels
    assert maxrel(gw, grads_o[fc]["w"]) <= 2e-2
    assert l2 < l1


def test_training_step_is_bitwise_reproducible():
    """SURVEY §8(c) C2b reading (4): the training step's gradients and updated
    weights are bitwise identical run to run (fixed-order reductions
    everywhere, no atomics on values)."""
    import torch
    from paper_2304_11745_b200 import gacer as G
    from paper_2304_11745_b200.train_driver import SequentialTrainer

    g = workloads.build_model("resnet18", 64)
    B = 4
    params = workloads.make_params(g, 43, "fp32")
    x = workloads.make_input(g, B, 43, "bf16")
    labels = workloads.make_labels(B, 43)
    xp = np.zeros((B, 64, 64, 8), np.float32)
    xp[..., :3] = x.transpose(0, 2, 3, 1)
    outs = []
    G.gacer_init(0)
    try:
        xd = torch.from_numpy(xp).to(torch.bfloat16).cuda()
        lab = torch.from_numpy(labels).cuda()
        for _ in range(2):
            tr = SequentialTrainer(g, params, B)
            loss, _ = tr.step(xd, lab)
            torch.cuda.synchronize()
            outs.append((float(loss), tr.flat_g.clone(), tr.flat_p.clone()))
            del tr
    finally:
        G.gacer_shutdown()
    assert outs[0][0] == outs[1][0]
    assert torch.equal(outs[0][1], outs[1][1]) and torch.equal(outs[0][2], outs[1][2])
