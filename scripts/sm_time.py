"""D2 mix under a plan, executor with trace: SM time per op (release - start,
the item's own execution span) -- where the round's SM-time goes."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import bench  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

ts = bench.make_workload()
s = Session([(g, p, B, dt) for _, g, p, B, dt, _ in ts], trace=True, partition="work_conserving")
G.gacer_set_sm_shares([0.35, 0.3, 0.35])
for t, (*_, x) in enumerate(ts):
    s.set_input(t, x)
for _ in range(3):
    s.run()
st = s.stats()
tr = G.gacer_get_trace(int(st["n_items"])).astype(np.float64)
s.close()
names = [n for n, *_ in ts]
span = (tr[:, 7].max() - tr[:, 6].min()) / 1e3
busy = np.where(tr[:, 8] > 0, tr[:, 7] - tr[:, 8], tr[:, 7] - tr[:, 6]) / 1e3
print(f"makespan {span:.1f} us, SM-time (start->release) {busy.sum():.0f} SM-us = {busy.sum()/148:.1f} us of the full GPU")
for t in range(len(names)):
    print(f"  {names[t]:13s} {busy[tr[:, 0] == t].sum()/148:7.1f} us-GPU")
ops = []
for op in np.unique(tr[:, 1]):
    m = tr[:, 1] == op
    ops.append((busy[m].sum() / 148, int(op), names[int(tr[m][0, 0])], int(m.sum()), float(np.median(busy[m]))))
ops.sort(reverse=True)
for b, op, n, k, med in ops[:25]:
    m = tr[:, 1] == op
    cc = np.all(tr[m][:, 9] > 0) and np.all(tr[m][:, 10] == 0)
    extra = ""
    if cc:   # CUDA-core window item: start -> ring drained -> release
        extra = f"  drain med {np.median((tr[m][:, 9] - tr[m][:, 8]) / 1e3):5.2f} us"
    print(f"  op {op:4d} {n:13s} items {k:5d} item med {med:6.2f} us  GPU-time {b:6.1f} us{extra}")
