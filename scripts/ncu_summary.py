"""Summarise ncu evidence into profiles/ (run here, no GPU needed).

  python scripts/ncu_summary.py --rep gpurun_out/prof_exec_d2.ncu-rep \
      --launches gpurun_out/launches_bench.csv --tag r1 --config d2_r50_v16_mv2
Writes profiles/<tag>_<config>.md and updates profiles/traffic.json
(dram read+write bytes per launch of gacer_executor, used by bench.py)."""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__cycles_active.avg",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {}
    for i, n in enumerate(hdr):
        if n in METRICS:
            res[n] = (vals[i], units[i])
    return res


def to_bytes(v, u):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = defaultdict(lambda: [0, 0.0])
    for d in data:
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[d["Metric Unit"]]
        k = d["Kernel Name"]
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"].replace(",", "")) * scale
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--config", default="d2_r50_v16_mv2")
    ap.add_argument("--bench", default="gpurun_out/bench.json")
    a = ap.parse_args()
    os.makedirs("profiles", exist_ok=True)
    md = [f"# ncu evidence — {a.tag}, {a.config}", ""]
    traffic = None
    if a.rep:
        m = raw_metrics(a.rep)
        md += ["## gacer_executor, one D2 round (`ncu --set full --clock-control none`)", "",
               "| metric | value | unit |", "|---|---|---|"]
        for k in METRICS:
            if k in m:
                md.append(f"| `{k}` | {m[k][0]} | {m[k][1]} |")
        if "dram__bytes_read.sum" in m and "dram__bytes_write.sum" in m:
            traffic = to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"])
            md += ["", f"DRAM traffic per launch (read + write): **{traffic / 1e6:.1f} MB**."]
        md.append("")
    if a.launches:
        agg = launches(a.launches)
        tot = sum(v[1] for v in agg.values())
        md += ["## Launch list of the bench command (`--metrics gpu__time_duration.sum`, cold, serialised)", "",
               "| kernel | launches | total us | share |", "|---|---|---|---|"]
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            md.append(f"| `{k}` | {n} | {t:.1f} | {t / tot:.1%} |")
        md.append("")
    if os.path.exists(a.bench):
        try:
            b = json.loads(open(a.bench).read().strip().splitlines()[-1])
            md += ["## bench.py line (same box)", "", "```json", json.dumps(b, indent=1), "```", ""]
        except Exception:
            pass
    path = f"profiles/{a.tag}_{a.config}.md"
    open(path, "w").write("\n".join(md))
    if traffic is not None:
        tp = "profiles/traffic.json"
        d = json.load(open(tp)) if os.path.exists(tp) else {}
        d[a.config] = traffic
        json.dump(d, open(tp, "w"), indent=1)
    print(path)


if __name__ == "__main__":
    main()
