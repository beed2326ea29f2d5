"""executor overhead microbenchmarks on chains of tiny ops.

  (i)   per-op dependency latency: a chain of N single-tile conv+BN+ReLU ops
        run by the executor: round time / N (notify + claim + TMA + MMA +
        epilogue + release, all on the critical path);
  (ii)  device pointer (cluster barrier) cost T_SW^dev: the same chain with a
        pointer after every op, (T - T_nopointer) / N;
  (iii) host-synchronised pointer cost T_SW^host (the paper's Fig. 6 / Eq. 8
        mechanics: one launch per cluster, CPU waits at every pointer):
        (T_hostsync - T_nopointer) / N;
  (iv)  per-op launch gap of the sequential baseline: T_sequential / N.
Writes gpurun_out/d7.json."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import workloads  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.runtime import Session  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 48
g = workloads.Graph("chain", 64, 8, 8)
x = 0
for i in range(N):
    x = g.relu(g.bn(g.conv(x, 64, 64, 1), 64))
p = workloads.make_params(g, 7)
inp = workloads.make_input(g, 2, 7)
s = Session([(g, p, 2, "bf16")])
s.set_input(0, inp)
stream = torch.cuda.Stream()
n_ops = len(g.ops)


def timed(mode, reps=30):
    s.set_mode(mode)
    for _ in range(5):
        G.gacer_run_round_async(stream.cuda_stream)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        G.gacer_run_round_async(stream.cuda_stream)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1000.0)
    return float(np.median(ts))


res = {"chain_ops": N, "op": "1x1 conv 64->64 + BN + ReLU, 2x8x8 (one 128x64 tile)"}
s.set_regulation(None, None)
res["executor_us"] = timed("executor")
res["sequential_us"] = timed("sequential")
# a pointer after every fused op: cut after every (conv, bn, relu) triple
cuts = [[3 * (i + 1) for i in range(N - 1)]]
s.set_regulation(None, cuts)
res["executor_pointers_us"] = timed("executor")
res["executor_hostsync_pointers_us"] = timed("executor_hostsync")
out = s.results()
s.close()
res["per_op_latency_us"] = res["executor_us"] / N
res["T_SW_device_us"] = (res["executor_pointers_us"] - res["executor_us"]) / (N - 1)
res["T_SW_host_us"] = (res["executor_hostsync_pointers_us"] - res["executor_us"]) / (N - 1)
res["sequential_per_op_us"] = res["sequential_us"] / N
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/d7.json", "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res, indent=1))
