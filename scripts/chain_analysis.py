"""Per-op latency breakdown of one tenant run alone in the executor (trace):
dependency-notice gap, claim->MMA (load), MMA->epilogue, epilogue->release,
waves.  Usage: python scripts/chain_analysis.py [tenant_index] [plan]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import bench  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

ti = int(sys.argv[1]) if len(sys.argv) > 1 else 0
ts = bench.make_workload()
name, g, p, B, dt, x = ts[ti]
s = Session([(g, p, B, dt)], trace=True)
s.set_input(0, x)
for _ in range(3):
    s.run()
st = s.stats()
tr = G.gacer_get_trace(int(st["n_items"])).astype(np.float64)
s.close()
t0 = tr[:, 6].min()
for c in (6, 7, 8, 9):
    tr[:, c] = np.where(tr[:, c] > 0, tr[:, c] - t0, np.nan)
print(f"{name} alone: round {st['last_round_ms']*1000:.1f} us, items {len(tr)}")
prev_end = 0.0
tot = {"gap": 0, "load": 0, "mma": 0, "epi": 0, "span": 0}
for op in np.unique(tr[:, 1]):
    sel = tr[tr[:, 1] == op]
    first, last = np.nanmin(sel[:, 6]) / 1e3, np.nanmax(sel[:, 7]) / 1e3
    load = np.nanmedian(sel[:, 8] - sel[:, 6]) / 1e3
    mma = np.nanmedian(sel[:, 9] - sel[:, 8]) / 1e3
    epi = np.nanmedian(sel[:, 7] - sel[:, 9]) / 1e3
    cc = np.nanmedian(sel[:, 7] - sel[:, 6]) / 1e3
    gap = first - prev_end
    print(f"op {int(op):3d} items {len(sel):4d} gap {gap:6.2f} span {last - first:7.2f} | "
          f"claim->mma {load:5.2f} mma->epi {mma:5.2f} epi->rel {epi:5.2f} claim->rel {cc:6.2f} us")
    tot["gap"] += gap
    tot["span"] += last - first
    prev_end = last
print({k: round(v, 1) for k, v in tot.items()})
