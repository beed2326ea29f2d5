"""Same-box A/B timing of D2 (identity plan, executor) and the sequential
baseline for the library named by GACER_LIB (diagnostics)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

ts = bench.make_workload(os.environ.get("GACER_AB_CONFIG", bench.CONFIG))
s = Session([(g, p, B, dt) for _, g, p, B, dt, _ in ts])
for t, (*_, x) in enumerate(ts):
    s.set_input(t, x)
stream = torch.cuda.Stream()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
res = {}
for mode, n in (("executor", 30), ("sequential", 10), ("executor", 30)):
    res.setdefault(mode, []).append(float(np.median(bench.time_mode(G, s, torch, stream, mode, n, 5, flush))))
s.close()
print(os.environ.get("GACER_LIB", "default"), os.environ.get("GACER_NO_STATS", ""),
      {k: [round(v, 4) for v in vs] for k, vs in res.items()})
