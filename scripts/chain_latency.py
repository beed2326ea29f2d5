"""One tenant alone (default MobileNetV2, B=8), executor with trace: per-op
latency anatomy of the chain (claim, start, accumulator-ready, release) to
see where a latency-bound chain spends its time."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import bench  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

which = int(sys.argv[1]) if len(sys.argv) > 1 else 2
coarse = len(sys.argv) > 2 and sys.argv[2] == "coarse"
ts = bench.make_workload()
name, g, p_, B, dt, x = ts[which]
s = Session([(g, p_, B, dt)], trace=True, coarse_deps=coarse)
s.set_input(0, x)
for _ in range(3):
    s.run()
st = s.stats()
tr = G.gacer_get_trace(int(st["n_items"])).astype(np.float64)
s.close()
t0 = tr[:, 6].min()
print(f"{name} alone, coarse_deps={coarse}: round {st['last_round_ms']*1000:.1f} us, items {len(tr)}")
prev_end = 0.0
tot = {"wait": 0.0, "claim2start": 0.0, "start2acc": 0.0, "acc2rel": 0.0}
for op in np.unique(tr[:, 1]):
    sel = tr[tr[:, 1] == op]
    c = (sel[:, 6] - t0) / 1e3
    st_ = (sel[:, 8] - t0) / 1e3
    acc = (sel[:, 9] - t0) / 1e3
    rel = (sel[:, 7] - t0) / 1e3
    edone = (sel[:, 10] - t0) / 1e3
    eloop = (sel[:, 11] - t0) / 1e3
    gemm = np.all(sel[:, 9] > 0)
    print(f"op {int(op):3d} items {len(sel):4d} claim[{c.min():7.1f},{c.max():7.1f}] "
          f"start-claim med {np.median(st_ - c):5.2f} "
          + (f"acc-start {np.median(acc - st_):5.2f} epi {np.median(edone - acc):5.2f} (loop {np.median(eloop - acc):5.2f}) rel {np.median(rel - edone):5.2f} " if gemm else
             f"rel-start med {np.median(rel - st_):5.2f}                       ")
          + f"end {rel.max():7.1f} (first claim - prev end {c.min() - prev_end:6.2f})")
    prev_end = rel.max()
