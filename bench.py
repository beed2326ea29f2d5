#!/usr/bin/env python
"""GACER on B200 -- benchmark of one regulated multi-tenant round.

Workload (BASELINE.json configs[1]): ResNet-50 + VGG-16 + MobileNetV2,
batch 8 each, 224x224, bf16, synthetic seeded inputs and random-init weights
(workloads/).  A *step* is one round: every tenant's forward once, through
the whole hot path (the persistent executor kernel).  Metric: aggregate
tenant inferences/s = sum_t B_t / makespan (higher is better).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gacer|reference]

N > 1 is launched by torchrun: one process per GPU, each running its own
replica of the mix (tenant placement, no data-path collective; weak scaling).
Timing: per-step CUDA events on the launching stream, L2 flushed (256 MB
write) between steps outside the events, barrier + synchronize around the
timed region, max over ranks.  --impl reference times the fp64 oracle (the
reference arm of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "aggregate tenant inferences/s per B200 + makespan/round vs sequential & multi-stream"
UNIT = "inferences/s"
CONFIG = "d2_r50_v16_mv2"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    def __init__(self, dev):
        self.dev, self.samples, self.reasons, self.stop_ev = dev, [], set(), threading.Event()
        self.max_mhz = None
        self.ok = False
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(dev)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass

    def _run(self):
        N = self.N
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
            "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        }
        while not self.stop_ev.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, v in names.items():
                    if r & v and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.002)   # the timed region is ~0.2 s: sample densely

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "note": "no NVML samples"}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "n_samples": len(self.samples)}


class _stdout_to_stderr:
    """NCCL's communicator creation prints its version on stdout; the
    bench's stdout is one JSON line, so fd 1 points at stderr meanwhile."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *a):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


# ------------------------------------------------------------------ workload
def make_workload(cfg=CONFIG, rank=0):
    """The config's tenants with seeded random-init weights; each rank (GPU
    replica) draws its own input batch."""
    import workloads
    from workloads.zoo import CONFIG_INDEX
    from paper_2304_11745_b200.placement import replica_seed
    ts = []
    for i, (name, B, dt) in enumerate(workloads.config_tenants(cfg)):
        g = workloads.build_model(name)
        seed = workloads.tenant_seed(CONFIG_INDEX[cfg], i)
        ts.append((name, g, workloads.make_params(g, seed, dt), B, dt,
                   workloads.make_input(g, B, replica_seed(seed, rank), dt)))
    return ts


def sweep_plans(ts):
    """Regulation plans tried by the bench: the identity
    plan, SM-share variants (the paper's resource share W), equal-op-count
    sync pointers (Matrix_P, Eq. 7) and VGG batch chunking (Eq. 5, cf. the
    paper's Table 3 case 2)."""
    nops = [len(g.ops) for _, g, *_ in ts]
    names = [n for n, *_ in ts]

    def cuts(n, k):
        return [round(n * (j + 1) / (k + 1)) for j in range(k)]
    plans = [("identity", None, None, None)]
    if len(ts) == 3:
        plans += [("shares[.35,.45,.2]", None, None, [0.35, 0.45, 0.2]),
                  ("shares[.25,.5,.25]", None, None, [0.25, 0.5, 0.25])]
    # SM partition policies (the paper's resource share W per tenant): each
    # CTA serves its own tenant first, then steals (work-conserving / hybrid)
    plans += [("work_conserving", None, None, None, "work_conserving"),
              ("hybrid", None, None, None, "hybrid")]
    if len(ts) == 3:
        plans += [(f"{pol}+shares[{a},{b},{a}]", None, None, [a, b, a], pol)
                  for pol in ("work_conserving", "hybrid") for a, b in ((0.3, 0.4), (0.35, 0.3))]
    plans += [(f"pointers{k}", None, [cuts(n, k) for n in nops], None) for k in (2, 4)]
    if "vgg16" in names:
        t = names.index("vgg16")
        g = ts[t][1]
        B = ts[t][3]
        half = [B // 2, B - B // 2]
        dec = [(t, i + 1, "batch", half) for i, op in enumerate(g.ops) if op["kind"] == "conv"]
        plans.append(("vgg_conv_batch_split", dec, None, None))

    # Eq. 5 on every decomposable op of every tenant: consecutive layers then
    # pipeline chunk by chunk through the chunk-granular dependencies
    def all_batch(nchunks):
        dec = []
        for t, (_, g, _, B, _, _) in enumerate(ts):
            k = min(nchunks, B)
            sizes = [B // k + (1 if j < B % k else 0) for j in range(k)]
            for i, op in enumerate(g.ops):
                if op["kind"] in ("conv", "linear", "maxpool", "avgpool", "gap", "add", "relu", "relu6", "bn"):
                    dec.append((t, i + 1, "batch", sizes))
        return dec
    for k in (2, 4, 8):
        plans.append((f"all_ops_batch_split{k}", all_batch(k), None, None))
    plans.append(("all_ops_batch_split4+pointers2", all_batch(4), [cuts(n, 2) for n in nops], None))
    return plans


def cpu_oracle_sample(ts, budget_s=30.0):
    """Time the fp64 oracle (as it stands) on one image of each tenant of the
    mix: a bounded sample of the workload.  Returns (images/s, cores, desc)."""
    from oracle import forward_graph
    from oracle import ops as oops
    oops.build()
    t0 = time.perf_counter()
    n = 0
    for name, g, p, B, dt, x in ts:
        forward_graph(g, p, x[:1])
        n += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt_s = time.perf_counter() - t0
    desc = f"1 image of each of {n} tenant(s) of the mix (fp64 oracle, OpenMP)"
    return n / dt_s, oops.num_threads(), desc, dt_s


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_oracle_single_thread(cfg, tenant="mobilenet_v2"):
    """The OMP_NUM_THREADS=1 arm of the oracle baseline (a subprocess: the
    OpenMP team size is fixed at library load): one image of one tenant of
    the mix (the smallest: the whole arm stays within seconds)."""
    import subprocess
    code = (
        "import sys, time; sys.path.insert(0, %r)\n"
        "import bench, workloads\n"
        "from oracle import forward_graph\n"
        "from oracle import ops as oops\n"
        "ts = [t for t in bench.make_workload(%r) if t[0] == %r]\n"
        "_, g, p, B, dt, x = ts[0]\n"
        "t0 = time.perf_counter(); forward_graph(g, p, x[:1]); s = time.perf_counter() - t0\n"
        "print(1.0 / s, oops.num_threads())\n" % (ROOT, cfg, tenant))
    env = dict(os.environ, OMP_NUM_THREADS="1")
    try:
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                             timeout=300).stdout.split()
        return {"value": float(out[0]), "unit": UNIT, "cores": int(out[1]),
                "sample": f"1 image of {tenant} (fp64 oracle, OMP_NUM_THREADS=1)"}
    except Exception as e:   # a baseline detail, never a reason to fail the bench
        return {"unavailable": str(e)[:200]}


# ------------------------------------------------------------------ main arms
def run_reference(args, rank):
    """The reference arm of this tier: the fp64 oracle as it stands, timed on
    the host cores.  Each step is a bounded sample of the workload: one image
    of one tenant, rotating over the mix's tenants (the whole K+W run stays
    within a few minutes).  Under torchrun only rank 0 runs."""
    if rank != 0:
        return
    from oracle import forward_graph
    from oracle import ops as oops
    oops.build()
    ts = make_workload(args.config)
    for i in range(args.warmup):
        _, g, p, B, dt, x = ts[i % len(ts)]
        if g.name == "mobilenet_v2":
            forward_graph(g, p, x[:1])
    tot_s, n_img = 0.0, 0
    for i in range(args.steps):
        _, g, p, B, dt, x = ts[i % len(ts)]
        t0 = time.perf_counter()
        forward_graph(g, p, x[:1])
        tot_s += time.perf_counter() - t0
        n_img += 1
    value = n_img / tot_s
    desc = (f"{args.steps} steps x 1 image, tenants of {args.config} in rotation "
            f"(fp64 oracle, OpenMP)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, random-init weights)",
        "config": {"workload": args.config, "sample": "one image per step, tenants in rotation"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": oops.num_threads(), "kind": "oracle",
                         "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def time_mode(G, s, torch, stream, mode, steps, warmup, flush, ar=None):
    """Per-round device times (CUDA events on `stream`, L2 flushed before
    every round outside the events).  mode "<baseline>_graph" replays the
    baseline round captured as a CUDA graph (gacer_capture_baseline)."""
    if mode.endswith("_graph"):
        G.gacer_capture_baseline(mode[:-len("_graph")])
        run = lambda: G.gacer_run_baseline_graph(stream.cuda_stream)
    elif ar is not None:          # a round with the overlapped gradient exchange (A12)
        s.set_mode(mode)
        run = lambda: ar.enqueue_round(stream)
    else:
        s.set_mode(mode)
        run = lambda: G.gacer_run_round_async(stream.cuda_stream)
    for _ in range(warmup):
        run()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in evs:
        flush.zero_()
        a.record(stream)
        run()
        b.record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def run_gacer(args, rank, world, dist):
    import torch
    from paper_2304_11745_b200 import gacer as G
    from paper_2304_11745_b200.placement import max_over_ranks
    from paper_2304_11745_b200.runtime import Session

    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    ts = make_workload(args.config, rank)
    sess = Session([(g, p, B, dt) for _, g, p, B, dt, _ in ts], device=dev)
    for t, (*_, x) in enumerate(ts):
        sess.set_input(t, x)
    n_inf = sum(B for _, _, _, B, _, _ in ts)
    stream = torch.cuda.Stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{dev}")
    torch.cuda.set_stream(stream)
    st = G.gacer_get_stats()

    # ---- regulation plan: identity, or the best of a short sweep (each rank
    #      picks on its own measurements; the result is identical math)
    plans = sweep_plans(ts) if args.plan == "sweep" else [("identity", None, None, None)]
    plans = [pl if len(pl) == 5 else (*pl, "priority") for pl in plans]
    plan_ms = {}
    for name, dec, ptr, sh, part in plans:
        sess.set_regulation(dec, ptr)
        G.gacer_set_partition(part)
        G.gacer_set_sm_shares(sh)
        plan_ms[name] = float(np.median(time_mode(G, sess, torch, stream, "executor", 5, 2, flush)))
    best = min(plan_ms, key=plan_ms.get)
    name, dec, ptr, sh, part = next(pl for pl in plans if pl[0] == best)
    search = None
    if args.plan == "sweep" and not args.no_search:
        # Algorithm 1 (§4.4): measured coordinate descent over
        # Matrix_P and batch decompositions under the chosen SM partition
        from paper_2304_11745_b200 import planner as PL
        G.gacer_set_partition(part)
        G.gacer_set_sm_shares(sh)
        graphs = [g for _, g, *_ in ts]
        n_ops = [len(g.ops) for g in graphs]
        ev = PL.measured_objective(G, sess, graphs, [B for _, _, _, B, _, _ in ts], torch, stream, flush,
                                   rounds=5, warmup=2)
        res = PL.granularity_aware_search(ev, n_ops, PL.SearchConfig(max_pointers=2, stride=max(1, min(n_ops) // 6),
                                                                     max_evals=args.search_evals))
        s_dec = ev.plan_decomposition(res.decomposition)
        s_ptr = [list(p_) for p_ in res.pointers] if any(res.pointers) else None
        search = {"evals": res.evals, "ms": res.R, "pointers": [list(p_) for p_ in res.pointers],
                  "batch_chunks": [c for _, c in res.decomposition], "ms_per_pointer_count": res.records}
        sname = f"gacer_search[{part}]"
        plans.append((sname, s_dec, s_ptr, sh, part))
        plan_ms[sname] = res.R
        if res.R < plan_ms[best]:
            best = sname
            name, dec, ptr, sh, part = plans[-1]
    sess.set_regulation(dec, ptr)
    G.gacer_set_partition(part)
    G.gacer_set_sm_shares(sh)

    # ---- main arm: the GACER executor under the chosen plan
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        times = time_mode(G, sess, torch, stream, "executor", args.steps, args.warmup, flush)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    total_ms = max_over_ranks(float(np.sum(times)), dist, f"cuda:{dev}")
    ms_step = total_ms / args.steps
    value = world * n_inf * args.steps / (total_ms / 1000.0)
    launches_per_round = G.gacer_get_stats()["kernel_launches"]

    # ---- temporal-regulation overhead: the same pointer
    #      plan with device-side cluster barriers vs the paper's CPU-side
    #      pointers (one launch per cluster, host sync in between, T_SW)
    t_sw = {}
    if args.plan == "sweep":
        nops = [len(g.ops) for _, g, *_ in ts]
        for kp in (2, 4):
            sess.set_regulation(None, [[round(n * (j + 1) / (kp + 1)) for j in range(kp)] for n in nops])
            G.gacer_set_sm_shares(None)
            G.gacer_set_partition("priority")
            dev_ms = float(np.median(time_mode(G, sess, torch, stream, "executor", 5, 2, flush)))
            host_ms = float(np.median(time_mode(G, sess, torch, stream, "executor_hostsync", 5, 2, flush)))
            t_sw[f"pointers{kp}"] = {"device_ms": dev_ms, "host_sync_ms": host_ms}
        sess.set_regulation(dec, ptr)
        G.gacer_set_partition(part)
        G.gacer_set_sm_shares(sh)
        sess.set_mode("executor")

    # ---- same-kernel baselines (makespan per round), same timing protocol
    base = {}
    for mode in ("sequential", "multistream", "sequential_graph", "multistream_graph"):
        tm = time_mode(G, sess, torch, stream, mode, args.steps, args.warmup, flush)
        m = max_over_ranks(float(np.mean(tm)), dist, f"cuda:{dev}")
        base[mode] = {"ms_per_round": m, "inferences_per_s": world * n_inf / (m / 1000.0),
                      "kernel_launches_per_round": G.gacer_get_stats()["kernel_launches"]}
    sess.set_mode("executor")

    # ---- e2e: through the public C ABI with HOST buffers (H2D + D2H inside
    #      the timed region, CUDA events on the library stream)
    host_in = [sess.host_input(t, x) for t, (*_, x) in enumerate(ts)]
    host_out = [torch.empty(o.shape, dtype=torch.float32).pin_memory() for o in sess.outputs]
    for _ in range(args.warmup):
        G.gacer_run_round_host([h.data_ptr() for h in host_in], [h.data_ptr() for h in host_out])
    e2e_ms = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        G.gacer_run_round_host([h.data_ptr() for h in host_in], [h.data_ptr() for h in host_out])
        e2e_ms.append(G.gacer_get_stats()["last_round_ms"])
    e2e_total = max_over_ranks(float(np.sum(e2e_ms)), dist, f"cuda:{dev}")
    h2d = int(sum(i["in_bytes"] for i in sess.info))
    d2h = int(sum(i["out_bytes"] for i in sess.info))

    if rank == 0:
        peaks, src = load_peaks()
        flops = st["tensor_flops"]
        peak = peaks["bf16_tflops"]
        achieved = flops / (ms_step / 1000.0) / 1e12
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                traffic = json.load(f).get(args.config)
        except Exception:
            pass
        fp32 = all(dt == "fp32" for *_, dt, _ in ts)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if fp32 else "bf16",
            "data": "synthetic (seeded inputs, random-init weights)",
            "config": {"workload": args.config, "tenants": [f"{n}(B={B})" for n, _, _, B, _, _ in ts],
                       "image": ts[0][1].in_h, "plan": best, "mode": "executor",
                       "parallelism": f"replica-per-gpu x{world}",
                       "l2": "flushed between steps (256 MB write, outside the events)"},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "gacer_executor",
                         "algorithmic": f"{flops / 1e9:.1f} GFLOP conv+FC (2*MAC) per launch",
                         "peak_source": f"{src} bf16_tflops (burst; kernel timed alone)"},
            **({"roofline_note": "D1 (tiny fp32 tenants on CUDA cores) is latency-bound: a chain of "
                                 "dependent single-tile ops; the TFLOP/s fraction is not meaningful"}
               if fp32 else {}),
            "e2e": {"value": world * n_inf * args.steps / (e2e_total / 1000.0), "unit": UNIT,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches_per_round * args.steps,
            "clocks": clk.summary(),
            "plans_ms": plan_ms,
            "pointer_sync_ms": t_sw,
            "search": search,
            "baselines": base,
            "speedup_vs_sequential": base["sequential"]["ms_per_round"] / ms_step,
            "speedup_vs_multistream": base["multistream"]["ms_per_round"] / ms_step,
            "speedup_vs_sequential_graph": base["sequential_graph"]["ms_per_round"] / ms_step,
            "speedup_vs_multistream_graph": base["multistream_graph"]["ms_per_round"] / ms_step,
            "makespan_ms": {"p10": float(np.percentile(times, 10)), "p50": float(np.median(times)),
                            "p90": float(np.percentile(times, 90))},
        }
        if world == 1 and not args.no_cpu_baseline:
            v, cores, desc, secs = cpu_oracle_sample(ts, budget_s=30.0)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                                    "sample": desc, "cpu_model": cpu_model(),
                                    "single_thread": cpu_oracle_single_thread(args.config)}
        print(json.dumps(line), flush=True)
    sess.close()


def run_d4(args, rank, world, dist):
    """D4 (BASELINE.json configs[3]): ResNet-50 TRAINING (B=64, one SGD step
    per round: forward, softmax-CE, backward, SGD-momentum update) co-located
    with VGG-16 + MobileNetV2 inference (B=8 each) in ONE executor round.
    Reports the inference aggregate (value) and the training images/s of the
    same rounds, against the sequential and multi-stream baselines of the
    same operators (plain and CUDA-graphed) and each side alone."""
    import torch
    import workloads
    from workloads.zoo import CONFIG_INDEX, TRAIN_CONFIGS
    from paper_2304_11745_b200 import gacer as G
    from paper_2304_11745_b200.placement import max_over_ranks, replica_seed
    from paper_2304_11745_b200.runtime import Session

    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    spec = TRAIN_CONFIGS["d4_mixed"]
    ts = []
    for i, (name, B, dt, train) in enumerate(spec):
        g = workloads.build_model(name)
        seed = workloads.tenant_seed(CONFIG_INDEX["d4_mixed"], i)
        ts.append((name, g, workloads.make_params(g, seed, "fp32" if train else dt), B, dt,
                   workloads.make_input(g, B, replica_seed(seed, rank), dt), train,
                   workloads.make_labels(B, replica_seed(seed, rank)) if train else None))
    stream = torch.cuda.Stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{dev}")
    torch.cuda.set_stream(stream)

    # A12: the data-parallel gradient mean of the training tenant inside the
    # round (NCCL on a communication stream, bucket waits on the executor's
    # counters, SGD behind the gradient gate); SMs left to the collective
    dp = dist is not None or args.allreduce
    reserve = 12 if dp else 0
    if dp and dist is None:            # world size 1: a one-rank NCCL group exercises the same path
        import torch.distributed as dist_mod
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29541")
        with _stdout_to_stderr():
            dist_mod.init_process_group("nccl", rank=0, world_size=1)
        dp_group = dist_mod
    else:
        dp_group = dist

    def session(sel):
        s = Session([(g, p, B, dt, {"train": True}) if tr else (g, p, B, dt)
                     for j, (_, g, p, B, dt, _, tr, _) in enumerate(ts) if j in sel], device=dev,
                    num_ctas=(148 - reserve) if (dp and 0 in sel) else 0)
        for k, j in enumerate(sel):
            s.set_input(k, ts[j][5])
            if ts[j][6]:
                s.set_labels(k, ts[j][7])
        return s

    n_inf = sum(B for _, _, _, B, _, _, tr, _ in ts if not tr)
    n_train = sum(B for _, _, _, B, _, _, tr, _ in ts if tr)
    res = {}
    # ---- each side alone (context)
    for label, sel in (("train_alone", [0]), ("inference_alone", [1, 2])):
        s = session(sel)
        res[label] = float(np.median(time_mode(G, s, torch, stream, "executor", max(3, args.steps // 2),
                                               args.warmup, flush)))
        s.close()
    # ---- the mixed round: plans (SM partition / shares), then the timed run
    s = session([0, 1, 2])
    st = G.gacer_get_stats()
    ar = None
    if dp:
        from paper_2304_11745_b200.grad_allreduce import ExecutorAllReduce
        with _stdout_to_stderr():      # (the communicator is created here)
            ar = ExecutorAllReduce(s, 0, dp_group)
    plans = {"priority": ("priority", None), "hybrid": ("hybrid", None),
             "work_conserving": ("work_conserving", None), "strict[.7,.2,.1]": ("strict", [0.7, 0.2, 0.1])}
    plan_ms = {}
    for name, (part, sh) in plans.items():
        G.gacer_set_partition(part)
        G.gacer_set_sm_shares(sh)
        plan_ms[name] = float(np.median(time_mode(G, s, torch, stream, "executor", 3, 2, flush, ar)))
    best = min(plan_ms, key=plan_ms.get)
    G.gacer_set_partition(plans[best][0])
    G.gacer_set_sm_shares(plans[best][1])
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        times = time_mode(G, s, torch, stream, "executor", args.steps, args.warmup, flush, ar)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    total_ms = max_over_ranks(float(np.sum(times)), dist, f"cuda:{dev}")
    ms_step = total_ms / args.steps
    occ = G.gacer_get_stats()
    base = {}
    # (graph baselines are not captured with the data-parallel gradient gate)
    for mode in ("sequential", "multistream") + (() if dp else ("sequential_graph", "multistream_graph")):
        tm = time_mode(G, s, torch, stream, mode, max(3, args.steps // 2), args.warmup, flush, ar)
        m = max_over_ranks(float(np.mean(tm)), dist, f"cuda:{dev}")
        base[mode] = {"ms_per_round": m, "inferences_per_s": world * n_inf / (m / 1000.0),
                      "train_images_per_s": world * n_train / (m / 1000.0),
                      "kernel_launches_per_round": G.gacer_get_stats()["kernel_launches"]}
    s.set_mode("executor")
    # ---- e2e: host buffers (images of all three tenants copied in, logits out)
    # (a blocking host-buffer round: the gradient exchange is not enqueued
    #  behind it, so the gate is switched off for this leg)
    if ar is not None:
        ar.close()
    host_in = [s.host_input(t, ts[j][5]) for t, j in enumerate([0, 1, 2])]
    host_out = [torch.empty(o.shape, dtype=torch.float32).pin_memory() for o in s.outputs]
    for _ in range(args.warmup):
        G.gacer_run_round_host([h.data_ptr() for h in host_in], [h.data_ptr() for h in host_out])
    e2e_ms = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        G.gacer_run_round_host([h.data_ptr() for h in host_in], [h.data_ptr() for h in host_out])
        e2e_ms.append(G.gacer_get_stats()["last_round_ms"])
    e2e_total = max_over_ranks(float(np.sum(e2e_ms)), dist, f"cuda:{dev}")
    loss = float(s.train_state(0)[0].item())
    if rank == 0:
        peaks, src = load_peaks()
        # algorithmic training FLOPs: forward + data gradient + weight
        # gradient = 3 x the forward conv+FC FLOPs
        g50 = ts[0][1]
        G.gacer_init(-1)
        fwd = G.gacer_get_tenant_info(G.gacer_register_tenant(g50, ts[0][2], n_train, "bf16"))["flops"]
        G.gacer_shutdown()
        flops = 3.0 * fwd + sum(i["flops"] for i in s.info[1:])
        achieved = flops / (ms_step / 1000.0) / 1e12
        peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
        line = {
            "metric": METRIC, "value": world * n_inf * args.steps / (total_ms / 1000.0), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded inputs and labels, random-init weights)",
            "config": {"workload": "d4_mixed", "tenants": ["resnet50(train, B=64)", "vgg16(B=8)",
                                                           "mobilenet_v2(B=8)"],
                       "image": 224, "plan": best, "mode": "executor",
                       "parallelism": f"replica-per-gpu x{world}",
                       "l2": "flushed between steps (256 MB write, outside the events)"},
            "train_images_per_s": world * n_train * args.steps / (total_ms / 1000.0),
            "train_loss_last": loss,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": None, "kernel": "gacer_executor_train",
                         "algorithmic": f"{flops / 1e9:.1f} GFLOP per round: 3 x ResNet-50 forward (B=64) "
                                        f"+ VGG-16 and MobileNetV2 forward (B=8)",
                         "peak_source": f"{src} bf16_tflops_sustained (seconds-long step)"},
            "e2e": {"value": world * n_inf * args.steps / (e2e_total / 1000.0), "unit": UNIT,
                    "h2d_bytes_per_step": int(sum(i["in_bytes"] for i in s.info)),
                    "d2h_bytes_per_step": int(sum(i["out_bytes"] for i in s.info))},
            "gpu_launches": args.steps,
            "clocks": clk.summary(),
            "plans_ms": plan_ms,
            "alone_ms": res,
            "baselines": base,
            "speedup_vs_sequential": base["sequential"]["ms_per_round"] / ms_step,
            "speedup_vs_multistream": base["multistream"]["ms_per_round"] / ms_step,
            **({"speedup_vs_sequential_graph": base["sequential_graph"]["ms_per_round"] / ms_step,
                "speedup_vs_multistream_graph": base["multistream_graph"]["ms_per_round"] / ms_step}
               if "sequential_graph" in base else {}),
            "speedup_vs_alone_sum": (res["train_alone"] + res["inference_alone"]) / ms_step,
            "occupancy_sm_ms": [v / 1e6 for v in occ["tenant_sm_ns"]],
            "makespan_ms": {"p10": float(np.percentile(times, 10)), "p50": float(np.median(times)),
                            "p90": float(np.percentile(times, 90))},
            "n_items_per_round": st["n_items"],
            "grad_allreduce": ({"buckets": len(ar.buckets), "bytes": int(4 * sum(n for _, n in ar.buckets)),
                                "world": world, "reserved_sms": reserve, "transport": "nccl",
                                "overlap": "bucket waits on the executor's completion counters"}
                               if ar is not None else None),
        }
        print(json.dumps(line), flush=True)
    s.close()
    if dp and dist is None:
        dp_group.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="gacer", choices=["gacer", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default=CONFIG, choices=["d1_tiny", "d2_r50_v16_mv2", "d3_five", "d4_mixed",
                                                         "t2_alex_v16_r18", "t2_r50_v16_m3", "t2_r101_d121_m3"])
    ap.add_argument("--plan", default="sweep", choices=["identity", "sweep"])
    ap.add_argument("--no-search", action="store_true", help="skip the Algorithm 1 plan search")
    ap.add_argument("--search-evals", type=int, default=30)
    ap.add_argument("--allreduce", action="store_true",
                    help="d4_mixed at N=1: run the training tenant's gradient all-reduce path anyway")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        backend = "nccl" if args.impl == "gacer" else "gloo"
        if args.impl == "gacer":
            import torch
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        with _stdout_to_stderr():
            dist_mod.init_process_group(backend)
            if backend == "nccl":
                dist_mod.barrier()     # creates the communicator (prints the NCCL version)
        dist = dist_mod
    if args.impl == "reference":
        run_reference(args, rank)
    elif args.config == "d4_mixed":
        run_d4(args, rank, world, dist)
    else:
        run_gacer(args, rank, world, dist)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
