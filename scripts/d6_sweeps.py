"""SURVEY §8(d) D6 (ii)/(iii) and the SM-budget sweep, on the GPU.

(ii)  Fig. 9 (§5.5 l.1033-1042): pointer counts 0..6 at
      equal-FLOP cut points on every tenant of D2 and D3, each executed with
      device-side cluster barriers (executor) and with the paper's CPU-side
      pointers (executor_hostsync: one launch per cluster, the host waits at
      every pointer -- T_SW of Eq. 8, l.780-799).
(iii) channel split: every conv with >= 74 output tiles
      (128x128) split 2- and 4-way along Cout, with and without per-chunk SM
      budgets W(O^B) (l.597-601) of 148 / n_chunks.
(iv)  SM budget sweep: VGG-16's convs (D2) as single budgeted chunks with
      b in {24, 48, 74, 111, 0 = unlimited}, and ResNet-50 batch-split in two
      budgeted halves -- the spatial knob of l.667-668 with an execution effect.
Every plan's outputs are compared byte for byte with the identity plan.
Writes gpurun_out/d6_sweeps.json (diagnostics; not a bench line)."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402


def op_shapes_flops(g, B):
    """Per original op: (C, H, W) of its output and 2*MAC FLOPs (conv/linear)."""
    shp = {0: (g.in_c, g.in_h, g.in_w)}
    fl, tiles = [], []
    for op in g.ops:
        c, h, w = shp[op["preds"][0]] if op["preds"] else shp[0]
        k = op["kind"]
        f = 0.0
        nt = 0
        if k == "conv":
            ho = (h + 2 * op["ph"] - op["kh"]) // op["stride"] + 1
            wo = (w + 2 * op["pw"] - op["kw"]) // op["stride"] + 1
            f = 2.0 * B * ho * wo * op["c_out"] * op["kh"] * op["kw"] * op["c_in"] / op.get("groups", 1)
            if op.get("groups", 1) == 1:
                nt = math.ceil(B * ho * wo / 128) * math.ceil(op["c_out"] / 128)
            c, h, w = op["c_out"], ho, wo
        elif k in ("maxpool", "avgpool"):
            h = (h + 2 * op["ph"] - op["kh"]) // op["stride"] + 1
            w = (w + 2 * op["pw"] - op["kw"]) // op["stride"] + 1
        elif k == "gap":
            h = w = 1
        elif k == "linear":
            f = 2.0 * B * op["c_in"] * op["c_out"]
            c, h, w = op["c_out"], 1, 1
        elif k == "concat":
            c = sum(shp[p][0] for p in op["preds"])
        elif k == "flatten":
            c, h, w = c * h * w, 1, 1
        shp[op["id"]] = (c, h, w)
        fl.append(f)
        tiles.append(nt)
    return fl, tiles


def equal_flop_cuts(fl, k):
    cum = np.cumsum(fl)
    tot = cum[-1]
    cuts = []
    for j in range(k):
        tgt = tot * (j + 1) / (k + 1)
        cuts.append(int(np.searchsorted(cum, tgt) + 1))   # cut after the op that crosses the target
    return sorted(min(c, len(fl)) for c in cuts)


def timed(G, s, stream, flush, mode, n=7):
    return float(np.median(bench.time_mode(G, s, torch, stream, mode, n, 2, flush)))


def run_config(cfg, stream, flush, out):
    ts = bench.make_workload(cfg)
    s = Session([(g, p, B, dt) for _, g, p, B, dt, _ in ts])
    for t, (*_, x) in enumerate(ts):
        s.set_input(t, x)
    s.run()
    ref = [y.tobytes() for y in s.results()]
    info = [op_shapes_flops(g, B) for _, g, _, B, _, _ in ts]
    res = {"identity_ms": timed(G, s, stream, flush, "executor")}

    def check(tag):
        s.set_mode("executor")
        s.run()
        got = [y.tobytes() for y in s.results()]
        assert got == ref, f"{cfg} {tag}: outputs differ from the identity plan"

    # (ii) pointer counts at equal-FLOP cuts, device vs host-synchronised
    ptr = {}
    for k in range(0, 7):
        cuts = [equal_flop_cuts(fl, k) for fl, _ in info]
        s.set_regulation(None, cuts if k else None)
        d = timed(G, s, stream, flush, "executor")
        h = timed(G, s, stream, flush, "executor_hostsync")
        check(f"pointers{k}")
        ptr[k] = {"device_ms": d, "host_sync_ms": h, "cuts": cuts}
        print(cfg, "pointers", k, f"device {d:.3f} ms host-sync {h:.3f} ms", flush=True)
    res["pointer_sweep"] = ptr
    # (iii) channel split of the wide convs, with and without SM budgets
    ch = {}
    for nway in (2, 4):
        for budget in (False, True):
            dec = []
            for t, (_, g, _, B, _, _) in enumerate(ts):
                fl, tiles = info[t]
                for i, op in enumerate(g.ops):
                    if op["kind"] == "conv" and tiles[i] >= 74 and op["c_out"] >= nway * 8:
                        C = op["c_out"]
                        sizes = [C // nway + (1 if j < C % nway else 0) for j in range(nway)]
                        ent = (t, i + 1, "channel", sizes)
                        if budget:
                            ent = ent + ([148 // nway] * nway,)
                        dec.append(ent)
            s.set_regulation(dec, None)
            ms = timed(G, s, stream, flush, "executor")
            check(f"channel{nway}")
            tag = f"channel{nway}" + ("+budget" if budget else "")
            ch[tag] = {"ms": ms, "n_ops_split": len(dec)}
            print(cfg, tag, f"{ms:.3f} ms ({len(dec)} ops)", flush=True)
    res["channel_split"] = ch
    # (iv) SM budgets W(O^B) on the largest tenant's convs
    names = [n for n, *_ in ts]
    big = max(range(len(ts)), key=lambda t: sum(info[t][0]))
    bud = {}
    for b in (24, 48, 74, 111, 0):
        g, B = ts[big][1], ts[big][3]
        dec = [(big, i + 1, "batch", [B], [b]) for i, op in enumerate(g.ops) if op["kind"] == "conv"]
        s.set_regulation(dec, None)
        ms = timed(G, s, stream, flush, "executor")
        check(f"budget{b}")
        bud[f"{names[big]}_convs_budget{b or 'inf'}"] = ms
        print(cfg, names[big], "budget", b, f"{ms:.3f} ms", flush=True)
    if "resnet50" in names:
        t = names.index("resnet50")
        g, B = ts[t][1], ts[t][3]
        for b in (16, 37, 74):
            dec = [(t, i + 1, "batch", [B // 2, B - B // 2], [b, b]) for i, op in enumerate(g.ops)
                   if op["kind"] == "conv"]
            s.set_regulation(dec, None)
            ms = timed(G, s, stream, flush, "executor")
            check(f"r50split_budget{b}")
            bud[f"resnet50_batch2_budget{b}"] = ms
            print(cfg, "resnet50 batch2 budget", b, f"{ms:.3f} ms", flush=True)
    res["sm_budget"] = bud
    s.close()
    out[cfg] = res


def main():
    cfgs = sys.argv[1:] or ["d2_r50_v16_mv2", "d3_five"]
    stream = torch.cuda.Stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda:0")
    torch.cuda.set_stream(stream)
    out = {"note": "median of 7 rounds per plan (L2 flushed between rounds); outputs byte-identical "
                   "to the identity plan for every plan"}
    for cfg in cfgs:
        run_config(cfg, stream, flush, out)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/d6_sweeps.json", "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
