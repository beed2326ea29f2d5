"""Milestone timing of single-op kernels (GACER_DEBUG_TIMING=1)."""
import os
import sys
os.environ["GACER_DEBUG_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import workloads  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

EV = ["start", "claimed", "tma0", "tma_all", "mma_full0", "mma_done", "epi_tfull", "epi_done",
      "rel_fenced", "rel_atomics", "cluster_seen", "teardown", "epi_staged", "epi_loop_done", "epi_stores_issued", "epi_fenced", "epi_tmem0", "epi_chunk_staged", "epi_tma0_issued"]
for name, cin, cout, k, st, pad, hw, B in [("r50_l3_1x1", 256, 256, 1, 1, 0, 14, 8),
                                           ("r50_l1_1x1", 64, 64, 1, 1, 0, 56, 8)]:
    g = workloads.Graph(name, cin, hw, hw)
    c = g.conv(0, cin, cout, k, st, pad)
    g.relu(g.bn(c, cout))
    s = Session([(g, workloads.make_params(g, 1), B, "bf16")])
    s.set_input(0, workloads.make_input(g, B, 1))
    for mode in ("executor",):
        s.set_mode(mode)
        for _ in range(3):
            s.run()
        G.gacer_debug_timing(1, reset=True)
        s.run()
        d = G.gacer_debug_timing(1, reset=True)[0].astype(np.float64)
        used = d[:, 0] > 0
        d = d[used]
        t0 = d[:, 0].min()
        print(f"== {name} {mode}: ctas {used.sum()} round {s.stats()['last_round_ms']*1000:.1f} us")
        for e, en in enumerate(EV):
            col = d[:, e]
            col = col[col > 0]
            if len(col):
                print(f"   {en:10s} min {(col.min()-t0)/1e3:8.2f} med {(np.median(col)-t0)/1e3:8.2f} max {(col.max()-t0)/1e3:8.2f} us")
    s.close()
