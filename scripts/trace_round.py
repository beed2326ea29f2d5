"""Device trace of one executor round (options.trace = 1): per-op item
statistics, SM busy fraction and per-tenant SM-time share (the analog of the
paper's Fig. 8 occupancy analysis).  Writes a JSON
summary to gpurun_out/trace_summary.json."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--out", default="gpurun_out/trace_summary.json")
ap.add_argument("--partition", default="priority")
ap.add_argument("--shares", default="", help="comma-separated SM shares per tenant")
a = ap.parse_args()
ts = bench.make_workload()
s = Session([(g, p, B, dt) for _, g, p, B, dt, _ in ts], trace=True, partition=a.partition)
if a.shares:
    G.gacer_set_sm_shares([float(v) for v in a.shares.split(",")])
for t, (*_, x) in enumerate(ts):
    s.set_input(t, x)
for _ in range(a.rounds):
    s.run()
st = s.stats()
tr = G.gacer_get_trace(int(st["n_items"]))
s.close()
t0 = tr[:, 6].min()
tr[:, 6] -= t0
tr[:, 7] -= t0
span = tr[:, 7].max()
dur = tr[:, 7] - tr[:, 6]
names = [n for n, *_ in ts]
out = {"makespan_us": span / 1e3, "round_ms_events": st["last_round_ms"], "n_items": int(len(tr)),
       "sm_busy_frac": float(dur.sum() / (148 * span)),
       "tenant_sm_share": {names[t]: float(dur[tr[:, 0] == t].sum() / (148 * span)) for t in range(len(names))},
       "tenant_span_us": {names[t]: [float(tr[tr[:, 0] == t, 6].min() / 1e3), float(tr[tr[:, 0] == t, 7].max() / 1e3)]
                          for t in range(len(names))},
       "ops": []}
for op in np.unique(tr[:, 1]):
    sel = tr[tr[:, 1] == op]
    d = sel[:, 7] - sel[:, 6]
    out["ops"].append({"op": int(op), "tenant": names[int(sel[0, 0])], "items": int(len(sel)),
                       "start_us": float(sel[:, 6].min() / 1e3), "end_us": float(sel[:, 7].max() / 1e3),
                       "item_us_mean": float(d.mean() / 1e3), "item_us_max": float(d.max() / 1e3),
                       "sm_us": float(d.sum() / 1e3)})
os.makedirs(os.path.dirname(a.out), exist_ok=True)
with open(a.out, "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "ops"}, indent=1))
top = sorted(out["ops"], key=lambda o: -o["sm_us"])[:25]
for o in top:
    print(f"op {o['op']:4d} {o['tenant']:13s} items {o['items']:5d} [{o['start_us']:8.1f},{o['end_us']:8.1f}] "
          f"item mean {o['item_us_mean']:7.2f} max {o['item_us_max']:7.2f} sm_us {o['sm_us']:9.1f}")
