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
hw = None
train = False
if cfg == "d1":
    spec = [("tiny_cnn", 2, "fp32"), ("tiny_mlp", 2, "fp32")]
elif cfg == "next2":     # MobileNetV3 (SE, hardswish) + DenseNet-121 (nested concats), small
    spec = [("mobilenet_v3_large", 2, "bf16"), ("densenet121", 2, "bf16")]
    hw = 64
elif cfg == "d4s":       # a training tenant (ResNet-18, 64^2, B=4) beside an inference tenant
    spec = [("resnet18", 4, "bf16"), ("mobilenet_v2", 2, "bf16")]
    hw = 64
    train = True
else:
    spec = [("resnet50", 1, "bf16"), ("vgg16", 1, "bf16"), ("mobilenet_v2", 1, "bf16")]
ts = []
for i, (name, B, dt) in enumerate(spec):
    g = workloads.build_model(name, hw)
    is_train = train and i == 0
    ts.append((g, workloads.make_params(g, 70 + i, "fp32" if is_train else dt), B, dt,
               workloads.make_input(g, B, 70 + i, dt), is_train))
s = Session([(t[0], t[1], t[2], t[3], {"train": True}) if t[5] else t[:4] for t in ts], watchdog_ms=600000)
for t, tt in enumerate(ts):
    s.set_input(t, tt[4])
    if tt[5]:
        s.set_labels(t, workloads.make_labels(tt[2], 70 + t))
s.set_regulation(None, [[(2 * len(t[0].ops) + 1) // 2 if t[5] else len(t[0].ops) // 2] for t in ts])   # one pointer
s.run()
s.set_mode("sequential")
s.run()
print(cfg, "sanitized round ok", [float(abs(y).max()) for y in s.results()])
s.close()
