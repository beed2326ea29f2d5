"""GPU parity of the training tenant's CUDA-core steps (include/gacer_train.h,
SURVEY §8(a) A11) against the fp64 oracle (oracle/train.py), per operator, fed
the GPU's own bf16 tensors (SURVEY §8(c) C2b reading (1)).  Gates: max-norm
relative error <= 2e-2 for bf16 outputs (Q2); fp32 statistics / parameter
gradients within their fp32 rounding; bitwise reproducibility run to run.
Shapes: ResNet-50 training tensors (B=64 replica at 56x56 / 7x7) cut down so
the oracle finishes in seconds, plus ragged row counts that leave a partial
row block."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def maxrel(a, r):
    return float(np.max(np.abs(np.asarray(a, np.float64) - r)) / max(np.max(np.abs(r)), 1e-30))


@pytest.fixture(scope="module")
def T():
    import torch
    from paper_2304_11745_b200 import gacer as G
    from oracle import train as OT
    return torch, G, OT


def _bf16(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).cuda()


def _np(t):
    return t.float().cpu().numpy().astype(np.float64)


def _nchw(a, N, H, W, C):
    return a.reshape(N, H, W, C).transpose(0, 3, 1, 2)


@pytest.mark.parametrize("N,H,W,C", [(4, 14, 14, 64), (3, 7, 5, 256), (2, 7, 7, 2048), (5, 3, 3, 24)])
def test_bn_train_fwd_bwd(T, N, H, W, C):
    torch, G, OT = T
    rng = np.random.default_rng(N * 1000 + C)
    M = N * H * W
    x = _bf16(torch, rng.normal(0.3, 1.7, size=(M, C)))
    dy = _bf16(torch, rng.normal(0.0, 1.0, size=(M, C)))
    gamma = torch.from_numpy(rng.uniform(0.5, 1.5, C).astype(np.float32)).cuda()
    beta = torch.from_numpy(rng.uniform(-0.2, 0.2, C).astype(np.float32)).cuda()
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    mean, var, dg, db = (torch.empty(C, device="cuda") for _ in range(4))
    scratch = torch.empty(G.bn_partials(M, C) * 2 * C + 4 * C, device="cuda")
    for relu in (0, 1):
        G.bn_train_fwd(x.data_ptr(), M, C, gamma.data_ptr(), beta.data_ptr(), 1e-5, relu, y.data_ptr(),
                       mean.data_ptr(), var.data_ptr(), scratch.data_ptr())
        torch.cuda.synchronize()
        xn = _nchw(_np(x), N, H, W, C)
        yo, mo, vo = OT.bn_train_fwd(xn, gamma.cpu().numpy(), beta.cpu().numpy(), 1e-5)
        if relu:
            yo = np.maximum(yo, 0)
        assert maxrel(mean.cpu().numpy(), mo) < 1e-4 and maxrel(var.cpu().numpy(), vo) < 1e-4
        assert maxrel(_nchw(_np(y), N, H, W, C), yo) <= 2e-2
    G.bn_train_bwd(x.data_ptr(), dy.data_ptr(), M, C, gamma.data_ptr(), mean.data_ptr(), var.data_ptr(), 1e-5,
                   dx.data_ptr(), dg.data_ptr(), db.data_ptr(), scratch.data_ptr())
    torch.cuda.synchronize()
    dxo, dgo, dbo = OT.bn_train_bwd(xn, _nchw(_np(dy), N, H, W, C), gamma.cpu().numpy(), mean.cpu().numpy().astype(np.float64),
                                    var.cpu().numpy().astype(np.float64), 1e-5)
    assert maxrel(dg.cpu().numpy(), dgo) < 1e-4
    assert maxrel(db.cpu().numpy(), dbo) < 1e-4
    assert maxrel(_nchw(_np(dx), N, H, W, C), dxo) <= 2e-2
    # the ReLU backward fused into the BN backward (mask = ReLU output > 0)
    yr = torch.empty_like(x)
    G.bn_train_fwd(x.data_ptr(), M, C, gamma.data_ptr(), beta.data_ptr(), 1e-5, 1, yr.data_ptr(),
                   mean.data_ptr(), var.data_ptr(), scratch.data_ptr())
    dxm = torch.empty_like(x)
    G.bn_train_bwd(x.data_ptr(), dy.data_ptr(), M, C, gamma.data_ptr(), mean.data_ptr(), var.data_ptr(), 1e-5,
                   dxm.data_ptr(), dg.data_ptr(), db.data_ptr(), scratch.data_ptr(), relu_y=yr.data_ptr())
    torch.cuda.synchronize()
    dym = OT.relu_bwd(_nchw(_np(yr), N, H, W, C), _nchw(_np(dy), N, H, W, C))
    dxo2, dgo2, _ = OT.bn_train_bwd(xn, dym, gamma.cpu().numpy(), mean.cpu().numpy().astype(np.float64),
                                    var.cpu().numpy().astype(np.float64), 1e-5)
    assert maxrel(dg.cpu().numpy(), dgo2) < 1e-4
    assert maxrel(_nchw(_np(dxm), N, H, W, C), dxo2) <= 2e-2
    # deterministic: a second backward is bitwise identical
    dx2 = torch.empty_like(dx)
    G.bn_train_bwd(x.data_ptr(), dy.data_ptr(), M, C, gamma.data_ptr(), mean.data_ptr(), var.data_ptr(), 1e-5,
                   dx2.data_ptr(), dg.data_ptr(), db.data_ptr(), scratch.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(dx, dx2)


def test_relu_bwd_exact(T):
    torch, G, OT = T
    rng = np.random.default_rng(3)
    vals = rng.normal(0, 4, size=4096)
    vals[:6] = [0.0, 6.0, -0.0, 5.999, 6.001, 1e-30]
    x = _bf16(torch, vals)
    dy = _bf16(torch, rng.normal(size=4096))
    for six in (0, 1):
        dx = torch.empty_like(x)
        G.relu_bwd(x.data_ptr(), dy.data_ptr(), 4096, six, dx.data_ptr())
        torch.cuda.synchronize()
        ref = OT.relu_bwd(_np(x), _np(dy), six=bool(six))
        assert np.array_equal(_np(dx), ref)          # a mask: exact


@pytest.mark.parametrize("N,H,W,C,k,s,p", [(2, 16, 16, 64, 3, 2, 1), (3, 9, 7, 16, 3, 2, 1), (2, 8, 8, 8, 2, 2, 0)])
def test_maxpool_bwd(T, N, H, W, C, k, s, p):
    torch, G, OT = T
    rng = np.random.default_rng(H * W + C)
    xv = rng.normal(size=(N, H, W, C))
    xv[0, :2, :2, :] = 1.0                            # ties: first maximum in row-major order wins (Q14)
    x = _bf16(torch, xv)
    Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    dy = _bf16(torch, rng.normal(size=(N, Ho, Wo, C)))
    dx = torch.empty_like(x)
    arg = torch.empty(N * Ho * Wo * C, dtype=torch.uint8, device="cuda")
    G.maxpool_bwd(x.data_ptr(), dy.data_ptr(), N, H, W, C, k, k, s, p, p, Ho, Wo, dx.data_ptr(), arg.data_ptr())
    torch.cuda.synchronize()
    ref = OT.maxpool_bwd(_nchw(_np(x), N, H, W, C), _nchw(_np(dy), N, Ho, Wo, C), (k, k), s, (p, p))
    got = _nchw(_np(dx), N, H, W, C)
    assert np.array_equal(got != 0, ref != 0)           # the routing (argmax choice) is exact
    assert maxrel(got, ref) <= 2e-2


def test_gap_bwd_and_softmax_ce_and_sgd(T):
    torch, G, OT = T
    rng = np.random.default_rng(9)
    N, HW, C = 6, 49, 2048
    dy = torch.from_numpy(rng.normal(size=(N, C)).astype(np.float32)).cuda()
    dx = torch.empty((N, HW, C), dtype=torch.bfloat16, device="cuda")
    G.gap_bwd(dy.data_ptr(), N, HW, C, dx.data_ptr())
    torch.cuda.synchronize()
    ref = OT.gap_bwd(dy.cpu().numpy(), (N, C, 7, 7))
    assert maxrel(_np(dx).transpose(0, 2, 1).reshape(N, C, 7, 7), ref) <= 2e-2
    # softmax-CE over 1000 classes (ResNet-50's head), ragged row count
    N, Cls = 13, 1000
    z = torch.from_numpy((rng.normal(size=(N, Cls)) * 4).astype(np.float32)).cuda()
    lab = rng.integers(0, Cls, size=N).astype(np.int32)
    labels = torch.from_numpy(lab).cuda()
    loss = torch.empty(1, device="cuda")
    dz = torch.empty_like(z)
    scratch = torch.empty(N, device="cuda")
    G.softmax_ce(z.data_ptr(), labels.data_ptr(), N, Cls, loss.data_ptr(), dz.data_ptr(), scratch.data_ptr())
    torch.cuda.synchronize()
    lo, dzo = OT.softmax_ce(z.cpu().numpy(), lab)
    assert abs(float(loss) - lo) / abs(lo) < 1e-5
    assert maxrel(dz.cpu().numpy(), dzo) < 1e-5
    # SGD momentum, two steps, vs the oracle's fp64 update
    n = 100003
    w0 = rng.normal(size=n).astype(np.float32)
    g0, g1 = rng.normal(size=n).astype(np.float32), rng.normal(size=n).astype(np.float32)
    w = torch.from_numpy(w0.copy()).cuda()
    buf = torch.zeros(n, device="cuda")
    for i, gg in enumerate((g0, g1)):
        gt = torch.from_numpy(gg).cuda()
        G.sgd_momentum(w.data_ptr(), gt.data_ptr(), buf.data_ptr(), n, 0.1, 0.9, int(i == 0))
    torch.cuda.synchronize()
    wr, br = w0.astype(np.float64), np.zeros(n)
    OT.sgd_momentum(wr, g0, br, 0.1, 0.9, True)
    OT.sgd_momentum(wr, g1, br, 0.1, 0.9, False)
    assert np.max(np.abs(w.cpu().numpy() - wr)) < 1e-6


@pytest.mark.parametrize("N,K,O", [(64, 2048, 1000), (5, 37, 11)])
def test_linear_bwd(T, N, K, O):
    torch, G, OT = T
    rng = np.random.default_rng(K)
    x = _bf16(torch, rng.normal(size=(N, K)))
    w = torch.from_numpy(rng.normal(0, 0.05, size=(O, K)).astype(np.float32)).cuda()
    dy = torch.from_numpy(rng.normal(size=(N, O)).astype(np.float32)).cuda()
    dx, dw, db = torch.empty((N, K), device="cuda"), torch.empty((O, K), device="cuda"), torch.empty(O, device="cuda")
    G.linear_bwd(x.data_ptr(), w.data_ptr(), dy.data_ptr(), N, K, O, dx.data_ptr(), dw.data_ptr(), db.data_ptr())
    torch.cuda.synchronize()
    rx, rw, rb = OT.linear_bwd(_np(x), w.cpu().numpy(), dy.cpu().numpy())
    assert maxrel(dx.cpu().numpy(), rx) < 1e-5
    assert maxrel(dw.cpu().numpy(), rw) < 1e-5
    assert maxrel(db.cpu().numpy(), rb) < 1e-5


@pytest.mark.parametrize("N,H,W,Cin,Cout,k,s,p", [(4, 14, 14, 64, 64, 3, 1, 1), (3, 14, 14, 256, 64, 1, 1, 0),
                                                   (2, 28, 28, 128, 128, 3, 1, 1), (2, 9, 11, 72, 128, 3, 1, 1),
                                                   (2, 7, 7, 512, 2048, 1, 1, 0),
                                                   (2, 28, 28, 128, 128, 3, 2, 1),    # R50 layer2 3x3/s2, even H
                                                   (2, 28, 28, 256, 512, 1, 2, 0),    # downsample 1x1/s2
                                                   (2, 15, 13, 64, 64, 3, 2, 1),      # odd sizes
                                                   (2, 32, 32, 8, 64, 7, 2, 3)])      # stem-like 7x7/s2
def test_conv_dgrad_tcgen05(T, N, H, W, Cin, Cout, k, s, p):
    """gacer_conv_dgrad: the data gradient as a stride-1 forward conv of the
    (zero-dilated) dy with the flipped, transposed filter on the executor's
    tcgen05 path, vs the oracle's scatter definition (oracle_conv2d_bwd_data)."""
    torch, G, OT = T
    rng = np.random.default_rng(Cin + Cout + H + s)
    Hd, Wd = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    dy = _bf16(torch, rng.normal(size=(N, Hd, Wd, Cout)))
    w = (rng.normal(size=(Cout, Cin, k, k)) * np.sqrt(2.0 / (Cin * k * k))).astype(np.float32)
    wd = torch.from_numpy(w).cuda()
    dx = torch.empty((N, H, W, Cin), dtype=torch.bfloat16, device="cuda")
    G.gacer_init(0)
    try:
        nb = G.conv_dgrad_workspace(N, H, W, Cin, Cout, k, k, s, p, p)
        ws = torch.empty(nb + 256, dtype=torch.uint8, device="cuda")
        base = (ws.data_ptr() + 255) // 256 * 256
        G.conv_dgrad(dy.data_ptr(), wd.data_ptr(), N, H, W, Cin, Cout, k, k, s, p, p, dx.data_ptr(), base, nb)
        torch.cuda.synchronize()
    finally:
        G.gacer_shutdown()
    wb = workloads_bf16(w)                       # the GEMM operand is the bf16-rounded filter
    ref, _, _ = OT.conv2d_bwd(np.zeros((N, Cin, H, W)), wb, _nchw(_np(dy), N, Hd, Wd, Cout), s, (p, p))
    assert maxrel(_nchw(_np(dx), N, H, W, Cin), ref) <= 2e-2


@pytest.mark.parametrize("N,H,W,Cin,Cout,k,s,p", [(4, 14, 14, 64, 64, 3, 1, 1), (3, 14, 14, 256, 64, 1, 1, 0),
                                                   (2, 28, 28, 128, 128, 3, 2, 1), (2, 15, 13, 64, 72, 3, 2, 1),
                                                   (2, 7, 7, 512, 2048, 1, 1, 0), (2, 32, 32, 8, 64, 7, 2, 3)])
def test_conv_wgrad_tcgen05(T, N, H, W, Cin, Cout, k, s, p):
    """gacer_conv_wgrad: dW as a GEMM over the output pixels on the
    executor's tcgen05 path (fixed split-K), vs the oracle's definition
    (oracle_conv2d_bwd_weight); deterministic run to run."""
    torch, G, OT = T
    rng = np.random.default_rng(Cin * 3 + Cout + H + s)
    Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    x = _bf16(torch, rng.normal(size=(N, H, W, Cin)))
    dy = _bf16(torch, rng.normal(size=(N, Ho, Wo, Cout)))
    dw = torch.empty((Cout, Cin, k, k), device="cuda")
    dw2 = torch.empty_like(dw)
    G.gacer_init(0)
    try:
        nb = G.conv_wgrad_workspace(N, H, W, Cin, Cout, k, k, s, p, p)
        ws = torch.empty(nb + 256, dtype=torch.uint8, device="cuda")
        base = (ws.data_ptr() + 255) // 256 * 256
        for out in (dw, dw2):
            G.conv_wgrad(x.data_ptr(), dy.data_ptr(), N, H, W, Cin, Cout, k, k, s, p, p, out.data_ptr(), base, nb)
        torch.cuda.synchronize()
    finally:
        G.gacer_shutdown()
    _, ref, _ = OT.conv2d_bwd(_nchw(_np(x), N, H, W, Cin), np.zeros((Cout, Cin, k, k)),
                              _nchw(_np(dy), N, Ho, Wo, Cout), s, (p, p))
    assert maxrel(dw.cpu().numpy(), ref) <= 1e-3       # fp32 accumulation of exact bf16 products
    assert torch.equal(dw, dw2)


def workloads_bf16(a):
    import workloads
    return workloads.bf16_round(np.asarray(a, np.float32)).astype(np.float64)


@pytest.mark.parametrize("N,H,W,Cin,Cout,k,s,p", [(4, 14, 14, 64, 64, 3, 1, 1), (2, 15, 13, 64, 72, 3, 2, 1),
                                                   (2, 7, 7, 512, 2048, 1, 1, 0),
                                                   (2, 32, 32, 8, 64, 7, 2, 3), (3, 30, 34, 8, 64, 7, 2, 3)])
def test_conv_wgrad_mn_major_matches_staged(T, N, H, W, Cin, Cout, k, s, p, monkeypatch):
    """The weight gradient read in place with MN-major UMMA operands (A = dy,
    B = the im2col TMA view of x; no staged transposes) computes the same
    products in the same K order as the staged K-major form: the two agree to
    fp32 rounding of the accumulation."""
    torch, G, OT = T
    rng = np.random.default_rng(Cin + 5 * Cout + H)
    Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    x = _bf16(torch, rng.normal(size=(N, H, W, Cin)))
    dy = _bf16(torch, rng.normal(size=(N, Ho, Wo, Cout)))
    outs = []
    for staged in ("0", "1"):
        monkeypatch.setenv("GACER_WGRAD_STAGED", staged)
        dw = torch.empty((Cout, Cin, k, k), device="cuda")
        G.gacer_init(0)
        try:
            nb = G.conv_wgrad_workspace(N, H, W, Cin, Cout, k, k, s, p, p)
            ws = torch.zeros(nb + 256, dtype=torch.uint8, device="cuda")
            base = (ws.data_ptr() + 255) // 256 * 256
            G.conv_wgrad(x.data_ptr(), dy.data_ptr(), N, H, W, Cin, Cout, k, k, s, p, p, dw.data_ptr(), base, nb)
            torch.cuda.synchronize()
        finally:
            G.gacer_shutdown()
        outs.append(dw.cpu().numpy())
    assert maxrel(outs[0], outs[1]) <= 1e-5, maxrel(outs[0], outs[1])


@pytest.mark.parametrize("N,H,W,Cin,Cout,k,s,p", [(2, 32, 32, 8, 64, 7, 2, 3), (3, 40, 36, 8, 64, 7, 2, 3),
                                                   (2, 16, 16, 64, 64, 3, 1, 1), (2, 14, 14, 8, 32, 3, 1, 1)])
def test_conv_fwd_train_tcgen05(T, N, H, W, Cin, Cout, k, s, p):
    """gacer_conv_fwd (the training tenant's forward conv on device-resident
    fp32 master weights): the 7x7 stem through the 8-channel TMA path
    (A_IM2COL8: per-tap 16-byte im2col boxes, block-packed weights), 3x3 64
    channels through TMA im2col, 8-channel 3x3 through the gather -- vs the
    oracle's direct convolution of the bf16-rounded filter, 2e-2 and 99.9%
    exact bf16 RNE."""
    torch, G, OT = T
    from oracle import ops as oops
    rng = np.random.default_rng(Cin * 7 + Cout + H)
    Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    x = _bf16(torch, rng.normal(size=(N, H, W, Cin)))
    w = (rng.normal(size=(Cout, Cin, k, k)) * np.sqrt(2.0 / (Cin * k * k))).astype(np.float32)
    wd = torch.from_numpy(w).cuda()
    y = torch.empty((N, Ho, Wo, Cout), dtype=torch.bfloat16, device="cuda")
    G.gacer_init(0)
    try:
        nb = G.conv_fwd_workspace(N, H, W, Cin, Cout, k, k, s, p, p)
        ws = torch.empty(nb + 256, dtype=torch.uint8, device="cuda")
        base = (ws.data_ptr() + 255) // 256 * 256
        G.conv_fwd(x.data_ptr(), wd.data_ptr(), N, H, W, Cin, Cout, k, k, s, p, p, y.data_ptr(), base, nb)
        torch.cuda.synchronize()
    finally:
        G.gacer_shutdown()
    ref = oops.conv2d(_nchw(_np(x), N, H, W, Cin), workloads_bf16(w), None, s, (p, p))
    got = _nchw(_np(y), N, Ho, Wo, Cout)
    assert maxrel(got, ref) <= 2e-2
    rne = workloads_bf16(ref.astype(np.float32)).astype(np.float64)
    assert np.mean(got == rne) >= 0.999, np.mean(got == rne)
