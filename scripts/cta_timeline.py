"""Per-CTA item timeline of one op (tenant alone, executor, trace): for the
items one SM ran back to back, print claim / start / acc-ready / epilogue-done
/ release, to see how consecutive tiles overlap inside a CTA."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import bench  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

which, opn = int(sys.argv[1]), int(sys.argv[2])
ts = bench.make_workload()
name, g, p_, B, dt, x = ts[which]
s = Session([(g, p_, B, dt)], trace=True)
s.set_input(0, x)
for _ in range(3):
    s.run()
tr = G.gacer_get_trace(int(s.stats()["n_items"])).astype(np.float64)
s.close()
t0 = tr[:, 6].min()
sel = tr[tr[:, 1] == opn]
for sm in np.unique(sel[:, 2])[:3]:
    rows = sel[sel[:, 2] == sm]
    rows = rows[np.argsort(rows[:, 6])]
    print(f"== {name} op {opn} SM {int(sm)}: {len(rows)} items")
    for r in rows[:8]:
        f = lambda v: (v - t0) / 1e3 if v > 0 else float("nan")
        print(f"  claim {f(r[6]):8.2f} start {f(r[8]):8.2f} acc {f(r[9]):8.2f} epi_done {f(r[10]):8.2f} rel {f(r[7]):8.2f}")
