"""One executor round (plus one sequential-mode round) of a config under
compute-sanitizer: D1 (tiny fp32 tenants) or D2 at
B=1.  The watchdog is raised: the sanitizer slows the spin loops by orders
of magnitude.  Usage: compute-sanitizer --tool X python scripts/sanitize_round.py d1|d2"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "d1"
if cfg == "d1":
    spec = [("tiny_cnn", 2, "fp32"), ("tiny_mlp", 2, "fp32")]
else:
    spec = [("resnet50", 1, "bf16"), ("vgg16", 1, "bf16"), ("mobilenet_v2", 1, "bf16")]
ts = []
for i, (name, B, dt) in enumerate(spec):
    g = workloads.build_model(name)
    ts.append((g, workloads.make_params(g, 70 + i, dt), B, dt, workloads.make_input(g, B, 70 + i, dt)))
s = Session([t[:4] for t in ts], watchdog_ms=600000)
for t, tt in enumerate(ts):
    s.set_input(t, tt[4])
s.set_regulation(None, [[len(g.ops) // 2] for g, *_ in ts])   # one sync pointer: the cluster barrier runs
s.run()
s.set_mode("sequential")
s.run()
print(cfg, "sanitized round ok", [float(abs(y).max()) for y in s.results()])
s.close()
