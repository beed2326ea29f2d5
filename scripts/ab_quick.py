"""Same-box A/B of library builds (GACER_LIB): D2 identity executor,
sequential and multi-stream medians + two single-op shapes (scratch)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import workloads
from paper_2304_11745_b200 import gacer as G
from paper_2304_11745_b200.runtime import Session
stream = torch.cuda.Stream()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda:0")
torch.cuda.set_stream(stream)
ts = bench.make_workload()
s = Session([(g, p, B, dt) for _, g, p, B, dt, _ in ts])
for t, (*_, x) in enumerate(ts):
    s.set_input(t, x)
r = {}
for mode in ("executor", "sequential", "multistream"):
    r[mode] = float(np.median(bench.time_mode(G, s, torch, stream, mode, 15, 3, flush)))
s.close()
for (cin, cout, k, st, pad, hw, B) in ((512, 512, 3, 1, 1, 28, 8), (512, 512, 3, 1, 1, 7, 8), (3, 64, 7, 2, 3, 224, 8)):
    g = workloads.Graph("op", cin, hw, hw)
    g.relu(g.bn(g.conv(0, cin, cout, k, st, pad), cout))
    s = Session([(g, workloads.make_params(g, 1), B, "bf16")])
    s.set_input(0, workloads.make_input(g, B, 1))
    r[f"op{cin}x{cout}k{k}@{hw}"] = float(np.median(bench.time_mode(G, s, torch, stream, "executor", 15, 3, flush)))
    s.close()
print(os.environ.get("GACER_LIB", "HEAD"), {k: round(v, 4) for k, v in r.items()}, flush=True)
