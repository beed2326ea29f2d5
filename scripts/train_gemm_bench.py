"""Training GEMMs of ResNet-50 at B=64 on their own (standalone C-ABI calls,
CUDA events, warm L2, median of 20): conv forward, data gradient (stride 1,
and stride 2 phase-decomposed vs zero-dilated) and weight gradient (MN-major
operands in place vs staged transposes) -- algorithmic TFLOP/s (2 * MACs of
the layer) and the fraction of the measured bf16 peak.  The verdict's bars:
strided dgrad >= 0.12, layer1 wgrad >= 0.15 of peak.
Writes gpurun_out/train_gemm_bench.json (diagnostics)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402

B = 64
SHAPES = [  # name, H(in), Cin, Cout, k, stride, pad
    ("l1_3x3", 56, 64, 64, 3, 1, 1),
    ("l1_1x1_exp", 56, 64, 256, 1, 1, 0),
    ("l2_3x3_s2", 56, 128, 128, 3, 2, 1),
    ("l2_down_1x1_s2", 56, 256, 512, 1, 2, 0),
    ("l3_3x3_s2", 28, 256, 256, 3, 2, 1),
    ("l4_3x3", 7, 512, 512, 3, 1, 1),
]
peaks, _ = bench.load_peaks()
peak = peaks["bf16_tflops"]


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


out = []
G.gacer_init(0)
for name, H, Cin, Cout, k, s, p in SHAPES:
    Ho = (H + 2 * p - k) // s + 1
    flops = 2.0 * B * Ho * Ho * Cout * Cin * k * k
    x = torch.randn(B, H, H, Cin, device="cuda").to(torch.bfloat16)
    dy = torch.randn(B, Ho, Ho, Cout, device="cuda").to(torch.bfloat16)
    w = torch.randn(Cout, Cin, k, k, device="cuda") * 0.05
    y = torch.empty(B, Ho, Ho, Cout, device="cuda", dtype=torch.bfloat16)
    dx = torch.empty_like(x)
    dw = torch.empty_like(w)
    row = {"layer": name, "gflop": flops / 1e9}
    for what, env in (("fwd", None), ("dgrad", None), ("dgrad_dilated", "GACER_DGRAD_DILATE"),
                      ("wgrad", None), ("wgrad_staged", "GACER_WGRAD_STAGED")):
        if what == "dgrad_dilated" and s == 1:
            continue
        if env:
            os.environ[env] = "1"
        try:
            if what == "fwd":
                nb = G.conv_fwd_workspace(B, H, H, Cin, Cout, k, k, s, p, p)
            elif what.startswith("dgrad"):
                nb = G.conv_dgrad_workspace(B, H, H, Cin, Cout, k, k, s, p, p)
            else:
                nb = G.conv_wgrad_workspace(B, H, H, Cin, Cout, k, k, s, p, p)
            ws = torch.empty(nb + 256, dtype=torch.uint8, device="cuda")
            base = (ws.data_ptr() + 255) // 256 * 256
            if what == "fwd":
                fn = lambda: G.conv_fwd(x.data_ptr(), w.data_ptr(), B, H, H, Cin, Cout, k, k, s, p, p, y.data_ptr(),
                                        base, nb)
            elif what.startswith("dgrad"):
                fn = lambda: G.conv_dgrad(dy.data_ptr(), w.data_ptr(), B, H, H, Cin, Cout, k, k, s, p, p,
                                          dx.data_ptr(), base, nb)
            else:
                fn = lambda: G.conv_wgrad(x.data_ptr(), dy.data_ptr(), B, H, H, Cin, Cout, k, k, s, p, p,
                                          dw.data_ptr(), base, nb)
            ms = timed(fn)
            row[what] = {"ms": ms, "tflops": flops / ms / 1e9, "frac": flops / ms / 1e9 / peak}
        finally:
            if env:
                del os.environ[env]
        del ws
    out.append(row)
    print(json.dumps(row), flush=True)
G.gacer_shutdown()
os.makedirs("gpurun_out", exist_ok=True)
json.dump({"batch": B, "peak_tflops": peak, "rows": out}, open("gpurun_out/train_gemm_bench.json", "w"), indent=1)
