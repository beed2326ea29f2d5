"""Per-source-line warp-stall hotspots of an ncu report (--import-source on).

usage: python scripts/ncu_source_hotspots.py REPORT.ncu-rep [--top 30] > profiles/....md

Reads `ncu -i REPORT --page source --csv --print-source cuda,sass`, keeps the
per-CUDA-line rows of the repo's own sources, and prints the lines with the
most warp-state samples, each with its enclosing function (inlined helpers are
attributed to the helper's own line, as ncu does) and its top stall reasons.
Idle warps are sampled too: samples on mbarrier/named-barrier waits are time
a role spent waiting, not issue pressure."""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True, check=True).stdout
    rows, path, header = [], None, None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1]
            continue
        if r[0] == "Line No":
            header = r
            continue
        if header is None or not r[0] or not r[0].isdigit():
            continue
        nm = len(header) - 4                 # metrics are the trailing fields (source text may hold stray quotes)
        rows.append((path, int(r[0]), ",".join(r[1:len(r) - nm - 2]), dict(zip(header[4:], r[-nm:]))))
    return rows


def functions(path):
    """line -> enclosing function name (a __device__/__global__ definition)."""
    names, cur = {}, "?"
    try:
        src = open(path).read().splitlines()
    except OSError:
        return names
    pat = re.compile(r"(?:__device__|__global__).*?\b([A-Za-z_]\w*)\s*\(")
    for i, line in enumerate(src, 1):
        m = pat.search(line)
        if m and not line.rstrip().endswith(";"):
            cur = m.group(1)
        names[i] = cur
    return names


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
    rows = [r for r in load(rep) if "/root/repo/" in (r[0] or "")]
    tot = sum(float(m.get("Warp Stall Sampling (All Samples)", 0) or 0) for _, _, _, m in rows)
    fn_cache, by_fn = {}, defaultdict(float)
    recs = []
    for path, ln, src, m in rows:
        if path not in fn_cache:
            fn_cache[path] = functions(path)
        fn = fn_cache[path].get(ln, "?")
        s = float(m.get("Warp Stall Sampling (All Samples)", 0) or 0)
        by_fn[fn] += s
        stalls = sorted(((float(v or 0), k[6:]) for k, v in m.items()
                         if k.startswith("stall_") and "Not Issued" not in k), reverse=True)[:3]
        recs.append((s, path.rsplit("/", 1)[-1], ln, fn, src.strip()[:70], stalls))
    print(f"# warp-state samples by source line ({rep.rsplit('/', 1)[-1]})\n")
    print(f"total samples in repo sources: {tot:.0f}\n")
    print("## by enclosing function (helpers separately)\n\n| function | samples | share |\n|---|---|---|")
    for fn, s in sorted(by_fn.items(), key=lambda z: -z[1])[:20]:
        print(f"| {fn} | {s:.0f} | {s / max(tot, 1):.1%} |")
    print(f"\n## top {top} lines\n\n| samples | share | file:line | function | source | top stalls |\n|---|---|---|---|---|---|")
    for s, f, ln, fn, src, st in sorted(recs, key=lambda z: -z[0])[:top]:
        sts = ", ".join(f"{k} {v:.0f}" for v, k in st if v > 0)
        print(f"| {s:.0f} | {s / max(tot, 1):.1%} | {f}:{ln} | {fn} | `{src.replace('|', '/')}` | {sts} |")


if __name__ == "__main__":
    main()
