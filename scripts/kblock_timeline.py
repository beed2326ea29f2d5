"""Per-k-block timeline of CTA 0 for single-op rounds (GACER_DEBUG_TIMING=1):
producer issue -> stage full (TMA latency), MMA cadence, epilogue span."""
import os
import sys
os.environ["GACER_DEBUG_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import workloads  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

SH = {"v16_c4": (512, 512, 3, 1, 1, 28, 8), "v16_c1_2": (64, 64, 3, 1, 1, 224, 8),
      "r50_l4_3x3": (512, 512, 3, 1, 1, 7, 8), "r50_l4_exp": (512, 2048, 1, 1, 0, 7, 8),
      "big_1x1": (1024, 1024, 1, 1, 0, 28, 8), "v16_c3": (256, 256, 3, 1, 1, 56, 8)}
OFF = 400 * 148 * 24
for name in (sys.argv[1:] or list(SH)):
    cin, cout, k, st, pad, hw, B = SH[name]
    g = workloads.Graph(name, cin, hw, hw)
    g.relu(g.bn(g.conv(0, cin, cout, k, st, pad), cout))
    s = Session([(g, workloads.make_params(g, 1), B, "bf16")])
    s.set_input(0, workloads.make_input(g, B, 1))
    for mode in ("sequential", "executor"):
        s.set_mode(mode)
        for _ in range(3):
            s.run()
        G.gacer_debug_timing(1, reset=True)
        s.run()
        raw = G.gacer_debug_timing(500, reset=True).reshape(-1)
        kd = raw[OFF:OFF + 768].astype(np.float64)
        full, issue, epi = kd[:256], kd[256:512], kd[512:768]
        n = int((full > 0).sum())
        t0 = min(issue[issue > 0].min() if (issue > 0).any() else full[0], full[0])
        if n == 0:
            print(f"== {name} {mode}: CTA0 ran no GEMM item"); continue
        lat = (full[:n] - issue[:n]) / 1e3
        cad = np.diff(full[:n]) / 1e3
        ep = epi[epi > 0]
        print(f"== {name} {mode}: round {s.stats()['last_round_ms']*1000:.1f} us, CTA0 kblocks {n}")
        print(f"   TMA issue->full us: med {np.median(lat):.3f} p90 {np.percentile(lat,90):.3f} max {lat.max():.3f}")
        if len(cad):
            print(f"   full cadence us: med {np.median(cad):.3f} p90 {np.percentile(cad,90):.3f}")
        print("   first 12 issue:", np.round((issue[:12] - t0) / 1e3, 2).tolist())
        print("   first 12 full :", np.round((full[:12] - t0) / 1e3, 2).tolist())
        print("   epi (tfull,done):", np.round((ep[:8] - t0) / 1e3, 2).tolist())
        ed = raw[OFF + 768:OFF + 768 + 128].reshape(8, 16).astype(np.float64)
        names = ["pop", "params", "tfull", "tmem0", "chunk", "tma_iss", "loop", "epi_end", "bulkw", "fenced", "done",
                 "fence_a", "pre_ld"]
        order = [0, 1, 2, 11, 12, 3, 4, 5, 6, 8, 7, 9, 10]
        for a in range(8):
            row = ed[a]
            if row[0] <= 0:
                continue
            print("   item", a, " ".join(f"{names[i]}:{(row[i]-row[0])/1.9e3:6.2f}" if row[i] > 0 else f"{names[i]}:  -   "
                                      for i in order), "us@1.9GHz")
    s.close()
