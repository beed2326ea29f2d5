"""Bandwidth of the training tenant's CUDA-core steps (include/gacer_train.h)
at ResNet-50 training shapes (B=64 replica, 224x224), against the measured HBM
copy bandwidth of MEASURED_PEAKS.json.

Algorithmic bytes per call (the two-pass algorithms' minimum traffic):
  bn_train_fwd  read x twice (statistics, normalise) + write y    = 3 * M*C*2 B
  bn_train_bwd  read x, dy twice (sums, apply) + write dx          = 5 * M*C*2 B
  relu_bwd      read x, dy + write dx                              = 3 * n*2 B
  maxpool_bwd   read x, dy + write dx (3x3/s2/p1 stem pool)        = (2*H*W + Ho*Wo)*N*C*2 B
                (the argmax bytes, N*Ho*Wo*C, are not counted)
Inputs are far larger than L2 (126 MB) except where noted; timings are CUDA
events over 20 back-to-back calls after 3 warm-up calls.

usage: python scripts/train_ops_bench.py [--json out.json]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_11745_b200 import gacer as G  # noqa: E402


def timed(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1e-3   # seconds per call


def main():
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
    rows = []
    B = 64
    for H, C in [(112, 64), (56, 256), (28, 512), (14, 1024), (7, 2048)]:
        M = B * H * H
        x = torch.randn(M, C, device="cuda").to(torch.bfloat16)
        dy = torch.randn(M, C, device="cuda").to(torch.bfloat16)
        y, dx = torch.empty_like(x), torch.empty_like(x)
        g, b = torch.ones(C, device="cuda"), torch.zeros(C, device="cuda")
        mean, var, dg, db = (torch.empty(C, device="cuda") for _ in range(4))
        sc = torch.empty(G.bn_partials(M, C) * 2 * C + 4 * C, device="cuda")
        t = timed(lambda: G.bn_train_fwd(x.data_ptr(), M, C, g.data_ptr(), b.data_ptr(), 1e-5, 1, y.data_ptr(),
                                         mean.data_ptr(), var.data_ptr(), sc.data_ptr()))
        rows.append(("bn_train_fwd", f"[{M},{C}]", 3 * M * C * 2, t))
        t = timed(lambda: G.bn_train_bwd(x.data_ptr(), dy.data_ptr(), M, C, g.data_ptr(), mean.data_ptr(),
                                         var.data_ptr(), 1e-5, dx.data_ptr(), dg.data_ptr(), db.data_ptr(),
                                         sc.data_ptr()))
        rows.append(("bn_train_bwd", f"[{M},{C}]", 5 * M * C * 2, t))
        if H == 56:
            t = timed(lambda: G.relu_bwd(x.data_ptr(), dy.data_ptr(), M * C, 0, dx.data_ptr()))
            rows.append(("relu_bwd", f"[{M},{C}]", 3 * M * C * 2, t))
        del x, dy, y, dx
    N, H, C = B, 112, 64
    x = torch.randn(N * H * H * C, device="cuda").to(torch.bfloat16)
    dy = torch.randn(N * 56 * 56 * C, device="cuda").to(torch.bfloat16)
    dx = torch.empty_like(x)
    arg = torch.empty(N * 56 * 56 * C, dtype=torch.uint8, device="cuda")
    t = timed(lambda: G.maxpool_bwd(x.data_ptr(), dy.data_ptr(), N, H, H, C, 3, 3, 2, 1, 1, 56, 56, dx.data_ptr(),
                                    arg.data_ptr()))
    rows.append(("maxpool_bwd", "[64,112,112,64] 3x3/s2/p1", (2 * H * H + 56 * 56) * N * C * 2, t))
    # conv backward GEMMs on tcgen05 at ResNet-50 B=64 layer shapes; FLOP =
    # 2 * N*Ho*Wo * Cout * Cin*KH*KW each (dgrad, wgrad), vs the measured bf16
    # peak (TFLOP/s rows: "bytes" column holds FLOP)
    G.gacer_init(0)
    tflop_rows = []
    try:
        for (H, Cin, Cout, k, st, p) in [(56, 64, 64, 3, 1, 1), (56, 256, 64, 1, 1, 0), (56, 64, 256, 1, 1, 0),
                                         (28, 128, 128, 3, 1, 1), (14, 256, 256, 3, 1, 1), (7, 512, 512, 3, 1, 1),
                                         (56, 128, 128, 3, 2, 1)]:
            Ho = (H + 2 * p - k) // st + 1
            x = torch.randn(B, H, H, Cin, device="cuda").to(torch.bfloat16)
            dy = torch.randn(B, Ho, Ho, Cout, device="cuda").to(torch.bfloat16)
            w = torch.randn(Cout, Cin, k, k, device="cuda")
            dx = torch.empty_like(x)
            dw = torch.empty_like(w)
            flop = 2.0 * B * Ho * Ho * Cout * Cin * k * k
            nb = G.conv_dgrad_workspace(B, H, H, Cin, Cout, k, k, st, p, p)
            ws = torch.empty(nb + 256, dtype=torch.uint8, device="cuda")
            base = (ws.data_ptr() + 255) // 256 * 256
            t = timed(lambda: G.conv_dgrad(dy.data_ptr(), w.data_ptr(), B, H, H, Cin, Cout, k, k, st, p, p,
                                           dx.data_ptr(), base, nb))
            tflop_rows.append(("conv_dgrad", f"{H}x{H} {Cin}->{Cout} k{k} s{st}", flop, t))
            nb = G.conv_wgrad_workspace(B, H, H, Cin, Cout, k, k, st, p, p)
            ws = torch.empty(nb + 256, dtype=torch.uint8, device="cuda")
            base = (ws.data_ptr() + 255) // 256 * 256
            t = timed(lambda: G.conv_wgrad(x.data_ptr(), dy.data_ptr(), B, H, H, Cin, Cout, k, k, st, p, p,
                                           dw.data_ptr(), base, nb))
            tflop_rows.append(("conv_wgrad", f"{H}x{H} {Cin}->{Cout} k{k} s{st}", flop, t))
            del x, dy, w, dx, dw, ws
    finally:
        G.gacer_shutdown()
    tpeak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))["bf16_tflops"]
    out = []
    print(f"{'op':14s} {'shape':28s} {'GFLOP':>8s} {'us':>8s} {'TF/s':>8s} {'frac':>6s}")
    for name, shape, flop, t in tflop_rows:
        tf = flop / t / 1e12
        print(f"{name:14s} {shape:28s} {flop / 1e9:8.2f} {t * 1e6:8.1f} {tf:8.1f} {tf / tpeak:6.3f}")
        out.append({"op": name, "shape": shape, "flop": flop, "us": t * 1e6, "tflops": tf,
                    "frac_of_measured_bf16": tf / tpeak, "includes": "operand staging kernels + GEMM"})
    print(f"{'op':14s} {'shape':28s} {'MB':>8s} {'us':>8s} {'GB/s':>8s} {'frac':>6s}")
    for name, shape, nbytes, t in rows:
        gbs = nbytes / t / 1e9
        print(f"{name:14s} {shape:28s} {nbytes / 1e6:8.1f} {t * 1e6:8.1f} {gbs:8.0f} {gbs / peak:6.2f}")
        out.append({"op": name, "shape": shape, "algorithmic_bytes": nbytes, "us": t * 1e6, "gbs": gbs,
                    "frac_of_measured_hbm": gbs / peak})
    if "--json" in sys.argv:
        json.dump({"peak_hbm_gbs": peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)", "rows": out},
                  open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
