"""Per-op wall spans (first claim -> last release) and achieved TF/s of one
tenant alone and inside the D2 mix (executor, trace on): where does the
throughput-bound tenant (VGG-16) lose against the tensor roofline?
usage: op_spans.py [tenant index in D2 (default 1 = VGG-16)]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import bench  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

which = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ts = bench.make_workload()
for label, sel in (("alone", [which]), ("in D2", [0, 1, 2])):
    sub = [ts[i] for i in sel]
    s = Session([(g, p, B, dt) for _, g, p, B, dt, _ in sub], trace=True)
    for t, (*_, x) in enumerate(sub):
        s.set_input(t, x)
    for _ in range(3):
        s.run()
    st = s.stats()
    tr = G.gacer_get_trace(int(st["n_items"])).astype(np.float64)
    t0 = tr[:, 6].min()
    tt = sel.index(which)
    v = tr[tr[:, 0] == tt]
    print(f"== {ts[which][0]} {label}: round {st['last_round_ms'] * 1e3:.1f} us")
    tot_f = 0.0
    for op in np.unique(v[:, 1]):
        sel_ = v[v[:, 1] == op]
        info = G.gacer_describe_op(int(op))
        mflop = info["mflop"]
        a, b = (sel_[:, 6].min() - t0) / 1e3, (sel_[:, 7].max() - t0) / 1e3
        dur = (sel_[:, 7] - sel_[:, 6]) / 1e3
        tot_f += mflop
        print(f"op {int(op):3d} kind {info['kind']} bn {info['bn']:3d} kb {info['nkb']:3d} items {len(sel_):5d} "
              f"span [{a:7.1f},{b:7.1f}] {b - a:6.1f} us  item med {np.median(dur):6.2f} us  "
              f"{mflop / max(b - a, 1e-3) / 1e6:7.1f} TF/s over span  SMs {len(np.unique(sel_[:, 2])):3d}")
    print(f"   total {tot_f / 1e3:.1f} GFLOP")
    s.close()
