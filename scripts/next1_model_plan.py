"""NEXT-1 / NEXT-3 on the GPU: profile the lookup table (W, T, W_bw per fused
op and batch), run the model-based search (Algorithm 1 on Eq. 8, largest-
residue spatial heuristic; SM-only and bandwidth-aware), install the plans
and measure them against the identity plan and the measured-objective search.
Writes gpurun_out/next1_model_plan.json (profiles/ copy committed)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2304_11745_b200 import costmodel as CM  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200 import planner as PL  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "d2_r50_v16_mv2"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peaks, _ = bench.load_peaks()
try:
    t_sw = json.load(open(os.path.join(ROOT, "profiles", "r2_d7_overheads.json")))["T_SW_device_us"]
except Exception:
    t_sw = 2.0
ts = bench.make_workload(cfg)
graphs = [g for _, g, *_ in ts]
w_mode = sys.argv[2] if len(sys.argv) > 2 else "tiles"
t0 = time.perf_counter()
tenants = CM.build_lut(G, Session, graphs, [p for _, _, p, *_ in ts], [B for *_, B, _, _ in ts],
                       [dt for *_, dt, _ in ts], [x for *_, x in ts], hbm_gbs=peaks["hbm_gbs"], w_mode=w_mode)
lut_s = time.perf_counter() - t0
out = {"config": cfg, "w_mode": w_mode, "t_sw_us": t_sw, "lut_build_s": lut_s,
       "lut_entries": sum(len(tm.cost) for tm in tenants)}

stream = torch.cuda.Stream()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda:0")
torch.cuda.set_stream(stream)
s = Session([(g, p, B, dt) for _, g, p, B, dt, _ in ts])
for t, (*_, x) in enumerate(ts):
    s.set_input(t, x)
s.run()
ref = [y.tobytes() for y in s.results()]


def measure(dec, ptrs, tag):
    s.set_regulation(dec, ptrs)
    ms = float(np.median(bench.time_mode(G, s, torch, stream, "executor", 9, 3, flush)))
    s.set_mode("executor")
    s.run()
    assert [y.tobytes() for y in s.results()] == ref, tag
    return ms


ident_sim = CM.simulate(tenants, tuple(() for _ in tenants), {}, t_sw)
out["identity"] = {"measured_ms": measure(None, None, "identity"), "model_makespan_us": ident_sim.makespan,
                   "model_R": ident_sim.R,
                   "model_sequential_us": sum(tm.op_cost(f, tm.batch).T for tm in tenants
                                             for f in range(len(tm.last_member)))}
for bw in (False, True):
    res = CM.model_based_search(tenants, t_sw, max_pointers=3, rounds=1, stride=max(1, min(t.n_orig for t in tenants) // 12),
                                spatial_steps=8, bandwidth=bw)
    dec, ptrs = CM.plan_to_abi(tenants, res)
    tag = "model_sm_hbm" if bw else "model_sm"
    out[tag] = {"measured_ms": measure(dec, ptrs, tag), "model_makespan_us": res.makespan, "model_R": res.R,
                "search_s": res.seconds, "evals": res.evals, "evals_per_s": res.evals / max(res.seconds, 1e-9),
                "pointers": [list(p) for p in res.pointers],
                "decomposition": {f"{t}:{f}": list(v) for (t, f), v in res.decomposition.items()},
                "R_per_pointer_count": res.records}
    print(tag, json.dumps(out[tag])[:400], flush=True)
# the measured-objective search (planner.py), same evaluation budget class
ev = PL.measured_objective(G, s, graphs, [B for *_, B, _, _ in ts], torch, stream, flush, rounds=5, warmup=2)
t0 = time.perf_counter()
res = PL.granularity_aware_search(ev, [len(g.ops) for g in graphs],
                                  PL.SearchConfig(max_pointers=2, stride=max(1, min(len(g.ops) for g in graphs) // 6),
                                                  max_evals=30))
out["measured_search"] = {"ms": res.R, "search_s": time.perf_counter() - t0, "evals": res.evals,
                          "pointers": [list(p) for p in res.pointers]}
# Table 4 analog: model-search time at fixed evaluation counts
tab = {}
for n in (100, 500, 1000, 2000):
    r = CM.model_based_search(tenants, t_sw, max_pointers=6, rounds=4, stride=1, spatial_steps=16, max_evals=n)
    tab[n] = r.seconds
out["search_time_s_by_evals"] = tab
s.close()
print(json.dumps(out, indent=1)[:3000])
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open(f"gpurun_out/next1_{cfg}_{w_mode}.json", "w"), indent=1)
