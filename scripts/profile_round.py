"""Run a few rounds of a config for ncu capture (not a bench: numbers taken
under a profiler are never reported as bench values)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--mode", default="executor")
a = ap.parse_args()
ts = bench.make_workload()
s = Session([(g, p, B, dt) for _, g, p, B, dt, _ in ts])
for t, (*_, x) in enumerate(ts):
    s.set_input(t, x)
s.set_mode(a.mode)
for _ in range(a.rounds):
    s.run()
torch.cuda.synchronize()
print("stats", s.stats())
s.close()
