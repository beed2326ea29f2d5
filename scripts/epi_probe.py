"""Diagnostics (GACER_DIAG build): clock64 stamps of the epilogue of CTA 0's
first GEMM items for one conv op (scratch)."""
import os, sys
os.environ["GACER_DEBUG_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads
from paper_2304_11745_b200 import gacer as G
from paper_2304_11745_b200.runtime import Session
KDBG_OFF = 400 * 148 * 24
for (cin, cout, k, hw, B) in ((64, 64, 1, 28, 8), (64, 64, 3, 28, 8), (64, 256, 1, 28, 8), (512, 512, 3, 28, 8)):
    g = workloads.Graph("op", cin, hw, hw)
    g.gap(g.relu(g.bn(g.conv(0, cin, cout, k, 1, k // 2), cout)))   # (internal bf16 conv output)
    s = Session([(g, workloads.make_params(g, 1), B, "bf16")], num_ctas=int(os.environ.get("NCTA", "1")))
    s.set_input(0, workloads.make_input(g, B, 1))
    for _ in range(3):
        s.run()
    G.gacer_debug_timing(1, reset=True)
    s.run()
    n = KDBG_OFF + 2048
    buf = np.zeros(n, dtype=np.int64)
    G.lib().gacer_debug_timing(buf.ctypes.data_as(G.C.POINTER(G.C.c_int64)), n, 1)
    e = buf[KDBG_OFF + 768: KDBG_OFF + 768 + 8 * 16].reshape(8, 16)
    print(f"== conv {cin}->{cout} k{k} @{hw} B{B}: items {s.info[0]['n_fused_ops']}")
    for a in range(8):
        row = e[a]
        if row[0] == 0:
            continue
        pts = {p: int(row[p] - row[0]) for p in range(16) if row[p] > 0}
        print("  item", a, pts)
    s.close()
