"""tenants-per-GPU scaling sweep on one B200.  Each point
draws T tenants with replacement from {AlexNet, VGG-16, ResNet-18, ResNet-50,
ResNet-101, Inception-v3, MobileNetV2} (seed 5000 + point id) at batch B, and
measures the executor (identity plan and the best SM partition) against the
sequential and one-stream-per-tenant baselines (same kernels; plain and
captured as CUDA graphs), L2 flushed between rounds.  Writes gpurun_out/d5_sweep.json."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
import workloads  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

POOL = ["alexnet", "vgg16", "resnet18", "resnet50", "resnet101", "inception_v3", "mobilenet_v2"]
POINTS = [(2, 4), (4, 4), (8, 4), (16, 1), (4, 16), (8, 16), (2, 64), (4, 64)]   # (tenants, batch)
stream = torch.cuda.Stream()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda:0")
torch.cuda.set_stream(stream)
out = []
for pid, (T, B) in enumerate(POINTS):
    rng = np.random.default_rng(5000 + pid)
    names = [POOL[int(i)] for i in rng.integers(0, len(POOL), size=T)]
    tenants, xs = [], []
    for i, n in enumerate(names):
        g = workloads.build_model(n)
        tenants.append((g, workloads.make_params(g, 5000 + 17 * pid + i, "bf16"), B, "bf16"))
        xs.append(workloads.make_input(g, B, 5000 + 17 * pid + i, "bf16"))
    s = Session(tenants)
    for t, x in enumerate(xs):
        s.set_input(t, x)
    row = {"point": pid, "tenants": names, "batch": B}
    for mode in ("sequential", "multistream", "sequential_graph", "multistream_graph"):
        row[f"{mode}_ms"] = float(np.median(bench.time_mode(G, s, torch, stream, mode, 5, 2, flush)))
    best = None
    for part in ("priority", "work_conserving", "hybrid"):
        G.gacer_set_partition(part)
        ms = float(np.median(bench.time_mode(G, s, torch, stream, "executor", 7, 2, flush)))
        row[f"executor_{part}_ms"] = ms
        best = ms if best is None else min(best, ms)
    row["executor_best_ms"] = best
    row["inferences_per_s"] = T * B / (best / 1000.0)
    row["speedup_vs_sequential"] = row["sequential_ms"] / best
    row["speedup_vs_multistream"] = row["multistream_ms"] / best
    row["speedup_vs_multistream_graph"] = row["multistream_graph_ms"] / best
    row["executor_identity_vs_multistream_graph"] = row["multistream_graph_ms"] / row["executor_priority_ms"]
    s.close()
    out.append(row)
    print(json.dumps(row), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/d5_sweep.json", "w") as f:
    json.dump(out, f, indent=1)
