"""Schedule invariance on the GPU (north_star: "bit-identical across
different regulation plans of the same tenant mix").

The D2 mix (ResNet-50 + VGG-16 + MobileNetV2, B=8, 224^2, bf16) runs under
the identity plan, seeded random spatial plans (batch and channel chunks),
random sync pointers, priority / strict / work-conserving / hybrid SM partitions, several grid
sizes, and the sequential / multi-stream baselines: every output must be
byte-identical.  The device trace must respect the cluster barrier
(Eq. 6, l.725: clusters are deployed in order) and chain order."""
import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu

D2 = [("resnet50", 8), ("vgg16", 8), ("mobilenet_v2", 8)]


@pytest.fixture(scope="module")
def d2():
    ts = []
    for i, (name, B) in enumerate(D2):
        g = workloads.build_model(name)
        seed = workloads.tenant_seed(2, i)
        ts.append((g, workloads.make_params(g, seed, "bf16"), B, "bf16",
                   workloads.make_input(g, B, seed, "bf16")))
    return ts


def random_plan(ts, rng, n_pointers):
    dec = []
    for t, (g, p, B, dt, x) in enumerate(ts):
        for i, op in enumerate(g.ops):
            if op["kind"] not in ("conv", "linear", "maxpool", "gap"):
                continue
            r = rng.random()
            if r < 0.25:
                k = int(rng.integers(2, 5))
                cuts = np.sort(rng.choice(np.arange(1, B), size=min(k, B) - 1, replace=False))
                sizes = np.diff(np.concatenate([[0], cuts, [B]])).astype(int).tolist()
                dec.append((t, i + 1, "batch", sizes))
            elif r < 0.35:
                C = op.get("c_out") or None
                if not C:
                    continue
                a = int(rng.integers(1, C))
                dec.append((t, i + 1, "channel", [a, C - a]))
    ptrs = []
    for g, *_ in ts:
        n = len(g.ops)
        ptrs.append(sorted(int(v) for v in rng.integers(0, n + 1, size=n_pointers)))
    return dec, ptrs


def run(ts, plan=None, mode="executor", **kw):
    from paper_2304_11745_b200.runtime import Session
    s = Session([t[:4] for t in ts], **kw)
    try:
        for t, tt in enumerate(ts):
            s.set_input(t, tt[4])
        if plan is not None:
            s.set_regulation(*plan)
        s.set_mode(mode)
        s.run()
        s.run()   # second round: counters/epochs re-armed correctly
        out = s.results()
        trace = None
        if kw.get("trace"):
            from paper_2304_11745_b200 import gacer as G
            trace = G.gacer_get_trace(int(s.stats()["n_items"]))
        return out, trace
    finally:
        s.close()


def test_bitwise_across_plans_and_modes(cuda_ok, d2):
    ref, _ = run(d2)
    variants = [dict(mode="sequential"), dict(mode="multistream"),
                dict(partition="strict"), dict(partition="work_conserving"), dict(partition="hybrid"),
                dict(num_ctas=37), dict(num_ctas=296), dict(coarse_deps=True),
                dict(coarse_deps=True, partition="strict")]
    rng = np.random.default_rng(12345)
    for k in range(6):
        variants.append(dict(plan=random_plan(d2, rng, n_pointers=k % 4)))
    variants.append(dict(plan=random_plan(d2, rng, 3), partition="strict", num_ctas=100))
    # the paper's CPU-side pointers: one launch per cluster, host sync between
    variants.append(dict(plan=random_plan(d2, rng, 3), mode="executor_hostsync"))
    for v in variants:
        out, _ = run(d2, **v)
        for t, (a, b) in enumerate(zip(ref, out)):
            assert a.tobytes() == b.tobytes(), (t, {k: v[k] for k in v if k != "plan"})


def test_trace_respects_clusters_and_chain(cuda_ok, d2):
    rng = np.random.default_rng(7)
    plan = random_plan(d2, rng, n_pointers=3)
    _, tr = run(d2, plan=plan, trace=True)
    cl, t0, t1 = tr[:, 4], tr[:, 6], tr[:, 7]
    assert np.all(t1 >= t0)
    for k in range(int(cl.max())):
        if np.any(cl == k) and np.any(cl == k + 1):
            assert t0[cl == k + 1].min() >= t1[cl == k].max(), k
    # identity plan with op-level dependencies (coarse_deps): VGG-16 is a
    # chain, so every item of fused op f+1 starts after every item of fused
    # op f has ended
    _, tr = run(d2, trace=True, coarse_deps=True)
    vgg = tr[tr[:, 0] == 1]
    ops = np.unique(vgg[:, 1])
    for a, b in zip(ops, ops[1:]):
        assert vgg[vgg[:, 1] == b, 6].min() >= vgg[vgg[:, 1] == a, 7].max()
    # tile-level dependencies (default): consecutive ops may overlap, but no
    # item of op f+1 starts before some item of op f has ended, and op f+1
    # cannot finish before op f
    _, tr = run(d2, trace=True)
    vgg = tr[tr[:, 0] == 1]
    for a, b in zip(ops, ops[1:]):
        assert vgg[vgg[:, 1] == b, 6].min() >= vgg[vgg[:, 1] == a, 7].min()
        assert vgg[vgg[:, 1] == b, 7].max() >= vgg[vgg[:, 1] == a, 7].max()


def max_concurrency(t0, t1):
    ev = sorted([(a, 1) for a in t0] + [(b, -1) for b in t1], key=lambda e: (e[0], e[1]))
    cur = best = 0
    for _, d in ev:
        cur += d
        best = max(best, cur)
    return best


def test_sm_budget_bounds_concurrency(cuda_ok, d2):
    """gacer_chunking.sm_budget (W(O^B)): a budgeted
    chunk never has more than its budget of items in flight (device trace:
    claim .. release intervals), unbudgeted it spreads over many more SMs,
    and the outputs are byte-identical either way (and with budgeted
    batch/channel chunks of every tenant)."""
    ref, _ = run(d2)
    g = d2[1][0]                      # VGG-16: every conv / pool / FC one budgeted chunk of 12 SMs
    ops = [i + 1 for i, op in enumerate(g.ops) if op["kind"] in ("conv", "maxpool", "linear")]
    b = 12
    dec = [(1, i, "batch", [8], [b]) for i in ops]
    out, tr = run(d2, plan=(dec, None), trace=True)
    for a, c in zip(ref, out):
        assert a.tobytes() == c.tobytes()
    _, tr0 = run(d2, trace=True)
    widest = 0
    for T, budget in ((tr, b), (tr0, None)):
        v = T[T[:, 0] == 1]
        for op in np.unique(v[:, 1]):
            sel = v[v[:, 1] == op]
            if len(sel) < 4 * b:
                continue
            conc = max_concurrency(sel[:, 6], sel[:, 7])
            if budget is not None:
                # claim stamps follow the semaphore wait; +1 for a stamp taken
                # on the far side of a concurrent release
                assert conc <= budget + 2, (op, conc)
            else:
                widest = max(widest, conc)
    assert widest > 3 * b, widest
    # budgeted batch and channel chunks on every tenant: bit-identical
    dec = []
    for t, (gg, p, B, dt, x) in enumerate(d2):
        for i, op in enumerate(gg.ops):
            if op["kind"] == "conv" and op.get("groups", 1) == 1:
                if i % 2:
                    dec.append((t, i + 1, "batch", [B // 2, B - B // 2], [20, 0]))
                else:
                    C = op["c_out"]
                    dec.append((t, i + 1, "channel", [C // 2, C - C // 2], [7, 30]))
    out, _ = run(d2, plan=(dec, None))
    for a, c in zip(ref, out):
        assert a.tobytes() == c.tobytes()


def test_full_size_sampled_parity(cuda_ok, d2):
    """D2 at its full bench size (B=8, executor mode): sampled outputs vs the
    oracle run one sample at a time (batch independence, C3)."""
    from oracle import forward_graph
    out, _ = run(d2)
    for t, (g, p, B, dt, x) in enumerate(d2):
        for n in ([0, B - 1] if g.name != "vgg16" else [B - 1]):
            r = forward_graph(g, p, x[n:n + 1])[0]
            err = np.max(np.abs(out[t][n] - r)) / np.max(np.abs(r))
            assert err <= 2e-2, (g.name, n, err)


def test_host_buffer_round_matches_device_round(cuda_ok, d2):
    """gacer_run_round_host (the e2e path): the input copies run on a copy
    stream behind per-tenant input gates while the round already runs; the
    outputs must be byte-identical to a round on device-resident inputs, for
    several consecutive rounds and in both executor modes."""
    import torch

    from paper_2304_11745_b200 import gacer as G
    from paper_2304_11745_b200.runtime import Session
    ref, _ = run(d2)
    s = Session([t[:4] for t in d2])
    try:
        host_in = [s.host_input(t, tt[4]) for t, tt in enumerate(d2)]
        host_out = [torch.empty(o.shape, dtype=torch.float32).pin_memory() for o in s.outputs]
        for mode in ("executor", "executor_hostsync"):
            s.set_mode(mode)
            for _ in range(3):
                for h in host_out:
                    h.fill_(float("nan"))
                G.gacer_run_round_host([h.data_ptr() for h in host_in], [h.data_ptr() for h in host_out])
                for a, b in zip(ref, host_out):
                    assert np.asarray(a).tobytes() == b.numpy().tobytes(), mode
    finally:
        s.close()


def test_graph_baselines_byte_identical(cuda_ok, d2):
    """The sequential / multi-stream baselines captured as CUDA graphs
    (gacer_capture_baseline) replay the same per-op launches: outputs
    byte-identical to the executor's, and the capture is discarded when the
    I/O is re-bound."""
    import torch
    from paper_2304_11745_b200 import gacer as G
    from paper_2304_11745_b200.runtime import Session
    ref, _ = run(d2)
    s = Session([t[:4] for t in d2])
    try:
        for t, tt in enumerate(d2):
            s.set_input(t, tt[4])
        for mode in ("sequential", "multistream"):
            G.gacer_capture_baseline(mode)
            for _ in range(2):
                for o in s.outputs:
                    o.fill_(float("nan"))
                G.gacer_run_baseline_graph(0)
                torch.cuda.synchronize()
                for a, b in zip(ref, s.results()):
                    assert a.tobytes() == b.tobytes(), mode
            assert G.gacer_get_stats()["kernel_launches"] > 100
        G.gacer_bind_io(0, s.inputs[0].data_ptr(), s.outputs[0].data_ptr())
        with pytest.raises(Exception):
            G.gacer_run_baseline_graph(0)
    finally:
        s.close()


def test_occupancy_stats(cuda_ok, d2):
    """gacer_get_stats' occupancy counters (the Fig. 8 analog, PAPER.md
    l.979-981): every tenant accumulates item time, the per-round figures are
    bounded by makespan x CTAs (x the in-flight depth), and a plan with sync
    pointers spends CTA time at cluster barriers that the identity plan does
    not."""
    from paper_2304_11745_b200.runtime import Session
    s = Session([t[:4] for t in d2])
    try:
        for t, tt in enumerate(d2):
            s.set_input(t, tt[4])
        for _ in range(3):
            s.run()
        st = s.stats()
        assert st["stat_rounds"] == 3
        ms = st["last_round_ms"]
        cap = ms * 1e6 * 148 * 4
        assert all(0 < v < cap for v in st["tenant_sm_ns"]), st
        assert st["barrier_wait_ns"] == 0
        n = [len(g.ops) for g, *_ in d2]
        s.set_regulation(None, [[x // 3, 2 * x // 3] for x in n])
        for _ in range(2):
            s.run()
        st2 = s.stats()
        assert st2["stat_rounds"] == 2 and st2["barrier_wait_ns"] > 0
    finally:
        s.close()


def test_bitwise_next2_mix(cuda_ok):
    """Table 2's R101+D121+M3 mix (at 64^2 / B=2): outputs
    byte-identical across random batch / channel plans (with SM budgets),
    pointers, partitions and the two baselines."""
    ts = []
    for i, name in enumerate(("resnet101", "densenet121", "mobilenet_v3_large")):
        g = workloads.build_model(name, 64)
        ts.append((g, workloads.make_params(g, 80 + i, "bf16"), 2, "bf16", workloads.make_input(g, 2, 80 + i, "bf16")))
    ref, _ = run(ts)
    rng = np.random.default_rng(99)
    variants = [dict(mode="sequential"), dict(mode="multistream"), dict(partition="work_conserving")]
    for k in range(3):
        dec, ptr = random_plan(ts, rng, n_pointers=k + 1)
        dec = [d + ([int(rng.integers(0, 40))] * len(d[3]),) if j % 3 == 0 else d for j, d in enumerate(dec)]
        variants.append(dict(plan=(dec, ptr)))
    for v in variants:
        out, _ = run(ts, **v)
        for t, (a, b) in enumerate(zip(ref, out)):
            assert a.tobytes() == b.tobytes(), (t, {kk: v[kk] for kk in v if kk != "plan"})


def test_buffer_reuse_is_invisible(cuda_ok, d2, monkeypatch):
    """Liveness-based activation-buffer reuse (host.cpp reuse_buffers) with
    tile-level write-after-read dependencies: outputs byte-identical to
    private buffers, also with the most aggressive reuse distance (1: a
    buffer is taken over right after its last reader's issue slot, so the
    WAR dependencies bind) under a strict partition, few CTAs, and random
    plans with pointers."""
    monkeypatch.setenv("GACER_REUSE", "0")
    ref, _ = run(d2)
    monkeypatch.setenv("GACER_REUSE", "1")
    rng = np.random.default_rng(99)
    variants = [dict(), dict(plan=random_plan(d2, rng, 2))]
    monkeypatch.setenv("GACER_REUSE_DIST", "1")
    variants += [dict(), dict(partition="strict", num_ctas=37), dict(plan=random_plan(d2, rng, 3), num_ctas=64)]
    for v in variants:
        out, _ = run(d2, **v)
        for t, (a, b) in enumerate(zip(ref, out)):
            assert a.tobytes() == b.tobytes(), (t, {k: v[k] for k in v if k != "plan"})
