"""Each D2 tenant alone: executor round vs sequential per-op kernels, plus
the whole mix (us/round, CUDA events, warm)."""
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
for sel in ([0], [1], [2], [0, 2], [0, 1, 2]):
    sub = [ts[i] for i in sel]
    s = Session([(g, p, B, dt) for _, g, p, B, dt, _ in sub], partition=os.environ.get("GACER_PARTITION", "priority"))
    for t, (*_, x) in enumerate(sub):
        s.set_input(t, x)
    row = [",".join(ts[i][0] for i in sel)]
    for mode in ("executor", "sequential", "multistream"):
        s.set_mode(mode)
        for _ in range(3):
            G.gacer_run_round_async(stream.cuda_stream)
        torch.cuda.synchronize()
        tt = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            G.gacer_run_round_async(stream.cuda_stream)
            b.record(stream)
            torch.cuda.synchronize()
            tt.append(a.elapsed_time(b) * 1000)
        row.append(f"{mode} {np.median(tt):8.1f} us")
    print(" | ".join(row), flush=True)
    s.close()
