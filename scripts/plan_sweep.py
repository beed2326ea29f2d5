"""Sweep regulation plans (SM shares, partition mode, sync pointers, batch
chunking) on the D2 mix and report the executor makespan of each."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402


def time_round(s, reps=10):
    stream = torch.cuda.Stream()
    for _ in range(3):
        G.gacer_run_round_async(stream.cuda_stream)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        G.gacer_run_round_async(stream.cuda_stream)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def equal_cuts(n_ops, k):
    return [round(n_ops * (j + 1) / (k + 1)) for j in range(k)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/plan_sweep.json")
    a = ap.parse_args()
    ts = bench.make_workload()
    res = []
    for partition in ("work_conserving",):
        s = Session([(g, p, B, dt) for _, g, p, B, dt, _ in ts], partition=partition)
        for t, (*_, x) in enumerate(ts):
            s.set_input(t, x)
        nops = [len(g.ops) for _, g, *_ in ts]

        def all_batch(tenants, sizes):
            dec = []
            for t in tenants:
                g = ts[t][1]
                for i, op in enumerate(g.ops):
                    if op["kind"] in ("conv", "linear", "maxpool", "avgpool", "gap", "add", "relu", "relu6"):
                        dec.append((t, i + 1, "batch", sizes))
            return dec
        plans = [("identity", None, None, None)]
        plans.append(("shares[.35,.45,.2]", None, None, [0.35, 0.45, 0.2]))
        for sizes in ([4, 4], [2, 2, 2, 2], [1] * 8):
            nm = "".join(str(v) for v in sizes)
            plans.append((f"all_b{nm}", all_batch([0, 1, 2], sizes), None, None))
            plans.append((f"r50mv2_b{nm}", all_batch([0, 2], sizes), None, None))
            plans.append((f"all_b{nm}+shares", all_batch([0, 1, 2], sizes), None, [0.35, 0.45, 0.2]))
        plans.append(("all_b2222+ptr2", all_batch([0, 1, 2], [2, 2, 2, 2]), [equal_cuts(n, 2) for n in nops], None))
        for name, dec, ptr, sh in plans:
            try:
                s.set_regulation(dec, ptr)
            except G.GacerError as e:
                print(json.dumps({"plan": name, "error": str(e)}), flush=True)
                continue
            G.gacer_set_sm_shares(sh)
            ms = time_round(s)
            res.append({"partition": partition, "plan": name, "ms": ms, "items": s.stats()["n_items"]})
            print(json.dumps(res[-1]), flush=True)
        s.close()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
