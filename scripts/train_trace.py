"""Training tenant alone in the executor with the device trace: per-op span,
items and item-duration medians, grouped by operator kind, to see where the
step's time goes (scripts/, diagnostics)."""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import workloads  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
hw = int(sys.argv[3]) if len(sys.argv) > 3 else 224
g = workloads.build_model(name, hw)
p = workloads.make_params(g, 5, "fp32")
s = Session([(g, p, B, "bf16", {"train": True})], trace=True)
s.set_input(0, workloads.make_input(g, B, 5, "bf16"))
s.set_labels(0, workloads.make_labels(B, 5))
for _ in range(3):
    s.run()
st = s.stats()
tr = G.gacer_get_trace(int(st["n_items"])).astype(np.float64)
desc = {int(o): G.gacer_describe_op(int(o)) for o in np.unique(tr[:, 1])}
s.close()
VF = ["none", "bn_partial", "bn_finalize", "bn_apply", "relu_bwd", "add", "maxpool_fwd", "maxpool_argmax",
      "maxpool_bwd", "gap_fwd", "gap_bwd", "linear_fwd", "linear_dx", "linear_dw", "softmax_ce", "mean", "sgd",
      "filter", "dilate", "transpose_im2col", "wgrad_permute", "wgrad_reduce", "phase_scatter", "filter_all"]
t0 = tr[:, 6].min()
print(f"{name} B={B} {hw}^2 train step alone: {st['last_round_ms']:.2f} ms, items {len(tr)}")
# per op: span (first claim .. last release), sum of item durations (SM-us)
rows = []
for op in np.unique(tr[:, 1]).astype(int):
    sel = tr[tr[:, 1] == op]
    dur = (sel[:, 7] - sel[:, 6]) / 1e3
    rows.append((op, len(sel), (sel[:, 6].min() - t0) / 1e3, (sel[:, 7].max() - t0) / 1e3, float(np.median(dur)),
                 float(dur.sum())))
kind_of = lambda o: ("gemm(bn=%d,nkb=%d)" % (desc[o]["bn"], desc[o]["nkb"])) if desc[o]["kind"] == 1 else VF[desc[o]["vfn"]]
agg = {}
for r in rows:
    k = "gemm" if desc[r[0]]["kind"] == 1 else VF[desc[r[0]]["vfn"]]
    a = agg.setdefault(k, [0, 0.0, 0])
    a[0] += r[1]; a[1] += r[5]; a[2] += 1
rows.sort(key=lambda r: -r[5])
tot = sum(r[5] for r in rows)
print(f"total item SM-us {tot:.0f} = {tot / 148:.0f} us of the full GPU")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:18s} ops {a[2]:4d} items {a[0]:7d} SM-us {a[1]:10.0f} ({100 * a[1] / tot:4.1f}%)")
for r in rows[:40]:
    print(f"op {r[0]:4d} {kind_of(r[0]):22s} items {r[1]:5d} span [{r[2]:8.1f},{r[3]:8.1f}] item med {r[4]:7.2f} us  SM-us {r[5]:9.0f} "
          f"({100 * r[5] / tot:4.1f}%)")
json.dump([list(map(float, r)) for r in rows], open("gpurun_out/train_trace.json", "w"))
