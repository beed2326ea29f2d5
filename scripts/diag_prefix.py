"""Diagnostics: first op prefix of a model whose output differs between the
executor on all SMs and on one CTA (scratch)."""
import copy, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads
from paper_2304_11745_b200.runtime import Session
name, hw, B = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
g0 = workloads.build_model(name, hw)
p = workloads.make_params(g0, 82, "bf16")
x = workloads.make_input(g0, B, 82, "bf16")
def run(g, **kw):
    s = Session([(g, p, B, "bf16")], **kw)
    s.set_input(0, x)
    s.run()
    y = s.results()[0]
    s.close()
    return y
for k in list(range(3, len(g0.ops) + 1, 3)) + [len(g0.ops)]:
    g = copy.deepcopy(g0)
    g.ops = g.ops[:k]
    if g.ops[-1]["kind"] in ("concat", "flatten", "dropout"):
        continue
    try:
        a, b = run(g), run(g, num_ctas=1)
    except Exception as e:
        print(k, "ERR", str(e)[:80]); continue
    same = a.tobytes() == b.tobytes()
    print(k, g.ops[-1]["kind"], "identical" if same else f"DIFF max {np.abs(a.astype(np.float64) - b).max():.3e} n {(a != b).sum()}", flush=True)
    if not same:
        break
