"""Time one training tenant's SGD step (SURVEY D4's training tenant alone:
ResNet-50, B=64, 224x224, bf16 activations) through
paper_2304_11745_b200.train_driver.SequentialTrainer -- every step a
libgacer.so call on one stream (sequential per-op launches; the executor
integration of the step is the next step of A11).

Algorithmic FLOP per step = 3 x the forward conv/FC FLOP (forward, dgrad,
wgrad; the stem's dgrad is skipped, so this slightly over-counts), against
the measured bf16 peak of MEASURED_PEAKS.json.  CUDA events on the stream
bracket `--steps` steps after `--warmup` steps; inputs resident in HBM.

usage: python scripts/train_step_bench.py [--model resnet50] [--batch 64]
                                          [--hw 224] [--steps 5] [--warmup 2]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads  # noqa: E402
from paper_2304_11745_b200 import gacer as G  # noqa: E402
from paper_2304_11745_b200.train_driver import SequentialTrainer  # noqa: E402


def fwd_flops(g, B):
    shape = {0: (g.in_h, g.in_w, g.in_c)}
    fl = 0.0
    for op in g.ops:
        h, w, c = shape[op["preds"][0]]
        if op["kind"] == "conv":
            ho = (h + 2 * op["ph"] - op["kh"]) // op["stride"] + 1
            wo = (w + 2 * op["pw"] - op["kw"]) // op["stride"] + 1
            fl += 2.0 * B * ho * wo * op["c_out"] * op["c_in"] // op["groups"] * op["kh"] * op["kw"]
            shape[op["id"]] = (ho, wo, op["c_out"])
        elif op["kind"] == "maxpool":
            shape[op["id"]] = ((h + 2 * op["ph"] - op["kh"]) // op["stride"] + 1,
                               (w + 2 * op["pw"] - op["kw"]) // op["stride"] + 1, c)
        elif op["kind"] == "gap":
            shape[op["id"]] = (1, 1, c)
        elif op["kind"] == "linear":
            fl += 2.0 * B * op["c_in"] * op["c_out"]
            shape[op["id"]] = (1, 1, op["c_out"])
        else:
            shape[op["id"]] = (h, w, c)
    return fl


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--hw", type=int, default=224)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    g = workloads.build_model(a.model, a.hw)
    params = workloads.make_params(g, 7, "fp32")
    x = workloads.make_input(g, a.batch, 7, "bf16")
    labels = workloads.make_labels(a.batch, 7)
    G.gacer_init(0)
    try:
        tr = SequentialTrainer(g, params, a.batch)
        xp = np.zeros((a.batch, a.hw, a.hw, 8), np.float32)
        xp[..., :3] = x.transpose(0, 2, 3, 1)
        xd = torch.from_numpy(xp).to(torch.bfloat16).cuda()
        lab = torch.from_numpy(labels).cuda()
        for _ in range(a.warmup):
            tr.step(xd, lab)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        losses = []
        for _ in range(a.steps):
            loss, _ = tr.step(xd, lab)
            losses.append(loss)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        lv = [float(v) for v in losses]
    finally:
        G.gacer_shutdown()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
    flop = 3.0 * fwd_flops(g, a.batch)
    res = {"workload": f"{a.model} training step (SequentialTrainer)", "batch": a.batch, "hw": a.hw,
           "ms_per_step": ms, "images_per_s": a.batch / ms * 1e3, "algorithmic_tflop_per_step": flop / 1e12,
           "tflops": flop / ms / 1e9, "frac_of_measured_bf16": flop / ms / 1e9 / peak,
           "losses": lv, "note": "sequential per-op launches from Python on one stream; CUDA events"}
    print(json.dumps(res))
    if a.json:
        json.dump(res, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
