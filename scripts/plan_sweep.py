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
    parts = os.environ.get("PARTITIONS", "priority,work_conserving,hybrid").split(",")
    for partition in parts:
        s = Session([(g, p, B, dt) for _, g, p, B, dt, _ in ts], partition=partition)
        for t, (*_, x) in enumerate(ts):
            s.set_input(t, x)
        plans = bench.sweep_plans(ts)
        for name, dec, ptr, sh, *pol in plans:
            if pol and pol[0] != partition:
                continue   # the partition is swept by the outer loop
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
