"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return data


if __name__ == "__main__":
    d = load(sys.argv[1])
    n = int(sys.argv[2]) if len(sys.argv) > 2 else len(d)
    d = d[-n:]
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[d[0]["Metric Unit"]]
    tot = sum(float(x["Metric Value"]) for x in d) * scale
    print(f"launches {len(d)} total {tot:.1f} us")
    for x in d:
        print(f"{float(x['Metric Value']) * scale:9.1f} us  {x['Kernel Name'][:40]:40s} grid {x['Grid Size']}")
