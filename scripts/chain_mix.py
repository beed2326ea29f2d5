"""Per-op chain latency of a tenant alone vs inside the mix (trace):
for each op of the tenant, the dependency-notice gap (first claim minus the
previous op's last release), the span (first claim -> last release), and the
median per-item claim->MMA start, MMA->epilogue, epilogue->release.
Usage: python scripts/chain_mix.py [plan]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import bench  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

plan_name = sys.argv[1] if len(sys.argv) > 1 else "identity"
ts = bench.make_workload()


def traced(idx):
    s = Session([ts[i][1:5] for i in idx], trace=True, partition=os.environ.get("GACER_PARTITION", "priority"))
    for j, i in enumerate(idx):
        s.set_input(j, ts[i][5])
    if len(idx) == len(ts):
        for nm, dec, ptr, sh, *_rest in bench.sweep_plans(ts):
            if nm == plan_name:
                s.set_regulation(dec, ptr)
                G.gacer_set_sm_shares(sh)
    for _ in range(3):
        s.run()
    st = s.stats()
    tr = G.gacer_get_trace(int(st["n_items"])).astype(np.float64)
    s.close()
    t0 = tr[:, 6].min()
    for c in (6, 7, 8, 9):
        tr[:, c] = np.where(tr[:, c] > 0, tr[:, c] - t0, np.nan)
    return st["last_round_ms"] * 1000, tr


def per_op(tr, tenant):
    sel_t = tr[tr[:, 0] == tenant]
    out = []
    prev_end = 0.0
    for op in np.unique(sel_t[:, 1]):
        sel = sel_t[sel_t[:, 1] == op]
        first, last = np.nanmin(sel[:, 6]) / 1e3, np.nanmax(sel[:, 7]) / 1e3
        row = dict(op=int(op), n=len(sel), gap=first - prev_end, span=last - first,
                   load=np.nanmedian(sel[:, 8] - sel[:, 6]) / 1e3,
                   mma=np.nanmedian(sel[:, 9] - sel[:, 8]) / 1e3,
                   epi=np.nanmedian(sel[:, 7] - sel[:, 9]) / 1e3,
                   c2r=np.nanmedian(sel[:, 7] - sel[:, 6]) / 1e3, end=last)
        out.append(row)
        prev_end = last
    return out


mix_ms, mix_tr = traced([0, 1, 2])
print(f"mix round {mix_ms:.1f} us plan {plan_name}")
for ti in (0, 2, 1):
    alone_ms, alone_tr = traced([ti])
    a = per_op(alone_tr, 0)
    m = per_op(mix_tr, ti)
    print(f"== {ts[ti][0]}: alone {alone_ms:.1f} us, in mix ends at {m[-1]['end']:.1f} us")
    tot = {k: [0.0, 0.0] for k in ("gap", "span")}
    for ra, rm in zip(a, m):
        print(f"op {ra['op']:3d} n {ra['n']:4d} | gap {ra['gap']:6.2f} -> {rm['gap']:6.2f} | span {ra['span']:7.2f} -> "
              f"{rm['span']:7.2f} | c2mma {ra['load']:5.2f}->{rm['load']:5.2f} mma {ra['mma']:5.2f}->{rm['mma']:5.2f} "
              f"epi {ra['epi']:5.2f}->{rm['epi']:5.2f} c2r {ra['c2r']:6.2f}->{rm['c2r']:6.2f}")
        for k in tot:
            tot[k][0] += ra[k]
            tot[k][1] += rm[k]
    print("totals alone->mix", {k: (round(v[0], 1), round(v[1], 1)) for k, v in tot.items()})
