"""Same-box A/B of an arbitrary tenant mix (identity plan, executor vs the
graphed multi-stream baseline): GACER_AB_MIX="vgg16:32,resnet18:32"
(diagnostics for the large-batch points of D5 / D6(i))."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
import workloads  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

mix = [(m.split(":")[0], int(m.split(":")[1])) for m in os.environ.get("GACER_AB_MIX", "vgg16:32,resnet18:32").split(",")]
ts = []
for i, (name, B) in enumerate(mix):
    g = workloads.build_model(name)
    ts.append((g, workloads.make_params(g, 7000 + i, "bf16"), B, "bf16", workloads.make_input(g, B, 7100 + i, "bf16")))
s = Session([t[:4] for t in ts], partition=os.environ.get("GACER_PARTITION", "priority"),
            coarse_deps=os.environ.get("GACER_AB_COARSE", "0") == "1")
for t, tt in enumerate(ts):
    s.set_input(t, tt[4])
stream = torch.cuda.Stream()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
res = {}
for mode, n in (("executor", 20), ("multistream_graph", 10), ("sequential_graph", 10), ("executor", 20)):
    res.setdefault(mode, []).append(float(np.median(bench.time_mode(G, s, torch, stream, mode, n, 3, flush))))
s.close()
print({k: [round(v, 4) for v in vs] for k, vs in res.items()})
