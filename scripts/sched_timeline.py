"""Scheduler timeline of CTA 0 (GACER_DEBUG_TIMING=1), one tenant alone."""
import os
import sys
os.environ["GACER_DEBUG_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import bench  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

which = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ts = bench.make_workload()
name, g, p_, B, dt, x = ts[which]
s = Session([(g, p_, B, dt)])
s.set_input(0, x)
for _ in range(3):
    s.run()
G.gacer_debug_timing(1, reset=True)
s.run()
raw = G.gacer_debug_timing(500, reset=True).reshape(-1)
OFF = 400 * 148 * 24 + 1024
d = raw[OFF:OFF + 24 * 8].reshape(24, 8).astype(np.float64)
t0 = d[0, 0]
print(f"{name} CTA0 scheduler: scan_begin scan_end ring_ok claimed pushed (us) | allowed*1000+inflight | op")
for n in range(24):
    r = d[n]
    if r[0] == 0:
        continue
    print(f"{n:3d} " + " ".join(f"{(r[j]-t0)/1e3:8.2f}" if r[j] > 0 else "     -  " for j in (0, 1, 2, 3, 4)),
          f"| {int(r[5]):5d} | {int(r[6])}")
s.close()
