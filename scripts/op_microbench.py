"""Per-op microbenchmark: single-conv tenants (conv+BN+ReLU), one kernel per
round, timed with CUDA events over many rounds (L2 warm).  Shapes are D2's
characteristic layers.  Prints us/round and TFLOP/s for the executor (one
persistent launch) and the standalone single-op kernel (sequential mode)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

SHAPES = [  # name, cin, cout, k, stride, pad, hw, B
    ("r50_stem", 3, 64, 7, 2, 3, 224, 8),
    ("r50_l1_1x1", 64, 64, 1, 1, 0, 56, 8),
    ("r50_l1_3x3", 64, 64, 3, 1, 1, 56, 8),
    ("r50_l1_exp", 64, 256, 1, 1, 0, 56, 8),
    ("r50_l3_3x3", 256, 256, 3, 1, 1, 14, 8),
    ("r50_l4_3x3", 512, 512, 3, 1, 1, 7, 8),
    ("r50_l4_exp", 512, 2048, 1, 1, 0, 7, 8),
    ("v16_c1_2", 64, 64, 3, 1, 1, 224, 8),
    ("v16_c2_2", 128, 128, 3, 1, 1, 112, 8),
    ("v16_c3", 256, 256, 3, 1, 1, 56, 8),
    ("v16_c4", 512, 512, 3, 1, 1, 28, 8),
    ("v16_c5", 512, 512, 3, 1, 1, 14, 8),
    ("mv2_exp", 24, 144, 1, 1, 0, 56, 8),
    ("mv2_dw_s2", 96, 96, 3, 2, 1, 112, 8),     # depthwise (groups = C)
    ("mv2_dw_s1", 144, 144, 3, 1, 1, 56, 8),
    ("r50_maxpool", 64, 64, -3, 2, 1, 112, 8),  # k < 0: max-pool
]

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--only", default="")
a = ap.parse_args()
res = []
for name, cin, cout, k, st, pad, hw, B in SHAPES:
    if a.only and a.only not in name:
        continue
    g = workloads.Graph(name, cin, hw, hw)
    if k < 0:
        g.maxpool(0, -k, st, pad)
        k = -k
    else:
        c = g.conv(0, cin, cout, k, st, pad, groups=cin if name.startswith("mv2_dw") else 1)
        g.relu(g.bn(c, cout))
    p = workloads.make_params(g, 1)
    x = workloads.make_input(g, B, 1)
    s = Session([(g, p, B, "bf16")])
    s.set_input(0, x)
    ho = (hw + 2 * pad - k) // st + 1
    flops = 2.0 * B * ho * ho * cout * (1 if "dw" in name or "pool" in name else cin) * k * k
    byts = 2.0 * B * (hw * hw * cin + ho * ho * cout)
    row = {"name": name, "gflop": flops / 1e9}
    stream = torch.cuda.Stream()
    for mode in ("executor", "sequential"):
        s.set_mode(mode)
        for _ in range(3):
            G.gacer_run_round_async(stream.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.reps):
            G.gacer_run_round_async(stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1000 / a.reps
        row[mode + "_us"] = us
        row[mode + "_tflops"] = flops / us / 1e6
        row[mode + "_gbs"] = byts / us / 1e3
    st_ = s.stats()
    row["items"] = st_["n_items"]
    s.close()
    res.append(row)
    print(json.dumps(row), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/op_microbench.json", "w") as f:
    json.dump(res, f, indent=1)
