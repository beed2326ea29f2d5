"""Busy SM-time of a D2 executor round from the device trace: per item
active time (GEMM: first K-block landed -> release; CUDA-core: start ->
release) vs 148 x makespan; per tenant and per op kind."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import bench  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

plan = sys.argv[1] if len(sys.argv) > 1 else "identity"
ts = bench.make_workload()
s = Session([(g, p, B, dt) for _, g, p, B, dt, _ in ts], trace=True, partition=os.environ.get("GACER_PARTITION", "priority"))
for t, (*_, x) in enumerate(ts):
    s.set_input(t, x)
for nm, dec, ptr, sh, *_rest in bench.sweep_plans(ts):
    if nm == plan:
        s.set_regulation(dec, ptr)
        G.gacer_set_sm_shares(sh)
for _ in range(3):
    s.run()
st = s.stats()
tr = G.gacer_get_trace(int(st["n_items"])).astype(np.float64)
kinds = {}
s.close()
t0 = tr[:, 6].min()
span = tr[:, 7].max() - t0
start = np.where(tr[:, 8] > 0, tr[:, 8], tr[:, 6])
active = tr[:, 7] - start
queued = start - tr[:, 6]
names = [n for n, *_ in ts]
print(f"plan {plan}: makespan {span/1e3:.1f} us, items {len(tr)}")
print(f"busy SM-time {active.sum()/1e3:.0f} SM-us = {active.sum()/(148*span):.2f} of 148 x makespan; "
      f"queued(claim->start) {queued.sum()/1e3:.0f} SM-us")
for t, nm in enumerate(names):
    sel = tr[:, 0] == t
    gemm = sel & (tr[:, 9] > 0)
    cc = sel & (tr[:, 9] == 0)
    print(f"  {nm:13s} busy {active[sel].sum()/1e3:8.0f} SM-us (gemm {active[gemm].sum()/1e3:8.0f}, "
          f"cc {active[cc].sum()/1e3:7.0f}); gemm item: load {np.median(tr[gemm,8]-tr[gemm,6])/1e3:.2f} "
          f"mma {np.median(tr[gemm,9]-tr[gemm,8])/1e3:.2f} epi {np.median(tr[gemm,7]-tr[gemm,9])/1e3:.2f} us; "
          f"cc item {np.median(active[cc])/1e3 if cc.any() else 0:.2f} us; span "
          f"[{(tr[sel,6].min()-t0)/1e3:.0f},{(tr[sel,7].max()-t0)/1e3:.0f}]")

# true per-SM busy fraction: union of [start, release] intervals per SM
sm = tr[:, 2].astype(int)
busy_union = 0.0
gaps = []
for k in np.unique(sm):
    sel = np.where(sm == k)[0]
    iv = sorted(zip(start[sel], tr[sel, 7]))
    cur_s, cur_e = iv[0]
    tot = 0.0
    for a, b in iv[1:]:
        if a > cur_e:
            tot += cur_e - cur_s
            gaps.append(a - cur_e)
            cur_s, cur_e = a, b
        else:
            cur_e = max(cur_e, b)
    tot += cur_e - cur_s
    busy_union += tot
print(f"union busy fraction {busy_union / (148 * span):.2f}; idle gaps between items: n={len(gaps)} "
      f"median {np.median(gaps)/1e3 if gaps else 0:.2f} us, total {np.sum(gaps)/1e3:.0f} SM-us")
