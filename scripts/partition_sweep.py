"""D2 mix: executor makespan across SM-partition policies x SM shares (and
dependency granularity), timed like bench.py (CUDA events, L2 flushed)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

ts = bench.make_workload()
stream = torch.cuda.Stream()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda:0")
torch.cuda.set_stream(stream)
SHARES = [None, [0.25, 0.5, 0.25], [0.2, 0.6, 0.2], [0.3, 0.4, 0.3], [0.15, 0.7, 0.15], [0.35, 0.3, 0.35]]
parts = sys.argv[1:] or ["priority", "work_conserving", "hybrid", "strict"]
for part in parts:
    s = Session([(g, p, B, dt) for _, g, p, B, dt, _ in ts], partition=part)
    for t, (*_, x) in enumerate(ts):
        s.set_input(t, x)
    for sh in SHARES:
        G.gacer_set_sm_shares(sh)
        ms = np.median(bench.time_mode(G, s, torch, stream, "executor", 7, 2, flush))
        print(f"{part:16s} shares={sh}: {ms:.3f} ms", flush=True)
    s.close()
