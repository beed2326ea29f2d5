"""C-ABI tests that need no GPU: the library loads, exports every symbol
include/gacer.h declares, and its host logic (validation, lowering, Eq. 6/7
plan compilation) behaves as the paper and the header state.  Uses the
HOST-ONLY instance (gacer_init(-1)): no CUDA call is made."""
import os
import re

import numpy as np
import pytest

import workloads
from gacer_testutil import read_golden
from paper_2304_11745_b200 import gacer as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture()
def host():
    G.gacer_init(-1)
    yield
    G.gacer_shutdown()


def test_exports_every_declared_symbol():
    declared = set()
    for h in ("gacer.h", "gacer_train.h"):
        with open(os.path.join(ROOT, "include", h)) as f:
            hdr = f.read()
        declared |= set(re.findall(r"^\s*(?:int|int32_t|int64_t|const char\*)\s+(gacer_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 22
    lib = G.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(G.EXPORTS)


def test_train_ops_reject_bad_shapes_without_touching_the_device():
    """Argument validation of include/gacer_train.h runs on the host: bad
    shapes / null pointers return an error code before any launch."""
    with pytest.raises(G.GacerError) as e:
        G.bn_train_fwd(16, 4, 12, 16, 16, 1e-5, 0, 16, 16, 16, 16)      # C % 8 != 0
    assert e.value.name == "GACER_E_SHAPE"
    with pytest.raises(G.GacerError) as e:
        G.relu_bwd(0, 0, 8, 0, 0)
    assert e.value.name == "GACER_E_INVALID_ARG"
    with pytest.raises(G.GacerError) as e:
        G.maxpool_bwd(16, 16, 1, 4, 4, 8, 3, 3, 2, 1, 1, 3, 2, 16, 16)  # Ho inconsistent
    assert e.value.name == "GACER_E_SHAPE"
    assert G.bn_partials(100000, 64) == 148 * 4 and G.bn_partials(40, 64) == 2


def chain_graph(n_ops, c=8, hw=4):
    """conv followed by n_ops-1 ReLUs: an n_ops-long operator list."""
    g = workloads.Graph("chain", c, hw, hw)
    x = g.conv(0, c, c, 1)
    for _ in range(n_ops - 1):
        x = g.relu(x)
    return g


def register(g, B=2, dt="bf16", seed=0):
    return G.gacer_register_tenant(g, workloads.make_params(g, seed, dt), B, dt)


def test_eq6_eq7_cluster_compilation(host):
    """Eq. 7 (l.747) and Eq. 6 (l.730-732) as compiled by gacer_set_regulation."""
    lines = read_golden("eq6_clusters.txt")
    ns, cuts = (t.strip() for t in lines[0].split("|"))
    ns = [int(v) for v in ns.split(",")]
    matrix_p = [[int(v) for v in c.split(",")] for c in cuts.split("/")]
    for n in ns:
        register(chain_graph(n))
    G.gacer_set_regulation(None, matrix_p)
    got = [G.gacer_query_op_clusters(t, n) for t, n in enumerate(ns)]
    # expected: parse the golden listing back into op -> cluster
    for k, ln in enumerate(lines[1:]):
        segs = re.findall(r"\[([^\]]*)\]", ln)
        for m, seg in enumerate(segs):
            for i in re.findall(r"O_\{\d+,(\d+)\}", seg):
                assert got[m][int(i) - 1] == k
    st = G.gacer_get_stats()
    assert st["n_clusters"] == 3


def test_eq7_segments_golden(host):
    for ln in read_golden("eq7_segments.txt"):
        n, cuts, segs = (t.strip() for t in ln.split("|"))
        register(chain_graph(int(n)))
        G.gacer_set_regulation(None, [[int(c) for c in cuts.split(",")]])
        got = G.gacer_query_op_clusters(0, int(n))
        for k, seg in enumerate(segs.split(";")):
            for i in seg.split(","):
                assert got[int(i) - 1] == k


def test_error_codes_graph(host):
    g = chain_graph(3)
    g.ops[1]["id"] = 1                       # duplicate id
    with pytest.raises(G.GacerError) as e:
        register(g)
    assert e.value.name == "GACER_E_DUPLICATE_ID"
    g = chain_graph(3)
    g.ops[2]["preds"] = [42]
    with pytest.raises(G.GacerError) as e:
        register(g)
    assert e.value.name == "GACER_E_UNKNOWN_PREDECESSOR"
    g = chain_graph(3)
    g.ops[0]["preds"] = [3]                  # 1 <- 3 <- 2 <- 1
    with pytest.raises(G.GacerError) as e:
        register(g)
    assert e.value.name == "GACER_E_CYCLE"
    g = chain_graph(3)
    g.ops[0]["c_in"] = 16
    with pytest.raises(G.GacerError) as e:
        register(g)
    assert e.value.name == "GACER_E_SHAPE"


def test_error_codes_plan(host):
    register(chain_graph(6))
    register(chain_graph(4))
    cases = [
        (([(0, 1, "batch", [1, 2])], None), "GACER_E_CHUNK_SUM_MISMATCH"),     # Eq. 5: sum != B=2
        (([(0, 1, "batch", None)], None), "GACER_E_MASKED_OP_MISSING_CHUNKS"),
        (([(0, 1, "channel", [4, 3])], None), "GACER_E_CHUNK_SUM_MISMATCH"),   # C_out = 8
        ((None, [[7], [1]]), "GACER_E_CUT_OUT_OF_RANGE"),
        ((None, [[3, 2], [1, 1]]), "GACER_E_UNSORTED_CUTS"),
        ((None, [[-1], [1]]), "GACER_E_CUT_OUT_OF_RANGE"),
        (([(0, 1, "batch", [1, 1], [2, -1])], None), "GACER_E_INVALID_ARG"),  # sm_budget < 0
    ]
    for (dec, ptr), name in cases:
        with pytest.raises(G.GacerError) as e:
            G.gacer_set_regulation(dec, ptr, n_tenants=2)
        assert e.value.name == name, (dec, ptr, e.value)
    # atomic: a failed call leaves the previous plan in force
    G.gacer_set_regulation(None, [[2], [1]])
    with pytest.raises(G.GacerError):
        G.gacer_set_regulation(None, [[3, 2], [0, 0]])
    assert G.gacer_query_op_clusters(0, 6) == [0, 0, 1, 1, 1, 1]
    with pytest.raises(G.GacerError) as e:
        G.gacer_run_round()
    assert e.value.name == "GACER_E_STATE"


def test_table3_plans_accepted(host):
    """Table 3 (l.1074-1082): V16(32) || R18(32) with convs and the ReLUs after
    them batch-decomposed per the listed list_B -- all are legal plans."""
    v16, r18 = workloads.build_model("vgg16"), workloads.build_model("resnet18")
    register(v16, 32)
    register(r18, 32)
    base = G.gacer_get_stats()["n_items"]
    for ln in read_golden("table3_plans.txt"):
        _, lv, lr = (t.strip() for t in ln.split("|"))
        dec = []
        for t, (g, lst) in enumerate(((v16, lv), (r18, lr))):
            sizes = [int(v) for v in lst.split(",")]
            if len(sizes) == 1:
                continue
            for i, op in enumerate(g.ops):
                if op["kind"] == "conv" or (op["kind"] == "relu" and i > 0 and g.ops[i - 1]["kind"] == "conv"):
                    dec.append((t, i + 1, "batch", sizes))
        G.gacer_set_regulation(dec, None, n_tenants=2)
        # chunks own whole tiles: the decomposition never adds or drops work
        assert G.gacer_get_stats()["n_items"] == base


def test_sm_budgets_accepted_and_work_preserving(host):
    """gacer_chunking.sm_budget (W(O^B), l.597-601): per-chunk budgets are
    part of a legal plan, a single chunk budgets an undecomposed op, and
    budgets never add or drop work items (they only gate WHEN items run)."""
    v16, r18 = workloads.build_model("vgg16"), workloads.build_model("resnet18")
    register(v16, 8)
    register(r18, 8)
    base = G.gacer_get_stats()["n_items"]
    convs = [i + 1 for i, op in enumerate(v16.ops) if op["kind"] == "conv"]
    dec = [(0, i, "batch", [8], [24]) for i in convs]
    dec += [(1, i + 1, "batch", [4, 4], [16, 0]) for i, op in enumerate(r18.ops) if op["kind"] == "conv"]
    G.gacer_set_regulation(dec, [[len(v16.ops) // 2], [len(r18.ops) // 2]], n_tenants=2)
    assert G.gacer_get_stats()["n_items"] == base
    # a fused op whose members carry different budgets is rejected
    i = convs[0]
    with pytest.raises(G.GacerError) as e:
        G.gacer_set_regulation([(0, i, "batch", [8], [24]), (0, i + 1, "batch", [8], [12])], None, n_tenants=2)
    assert e.value.name == "GACER_E_INVALID_ARG"


def test_identity_plan_and_fusion_counts(host):
    t = register(workloads.build_model("resnet50"), 8)
    info = G.gacer_get_tenant_info(t)
    assert info["n_orig_ops"] == 175 and info["n_fused_ops"] == 56
    assert abs(info["flops"] - 65.43e9) / 65.43e9 < 1e-3
    st = G.gacer_get_stats()
    assert st["n_clusters"] == 1 and st["n_fused_ops"] == 56


def test_partition_modes_validated():
    """Every gacer_partition value opens an instance; others are rejected."""
    import ctypes
    for name in G.PARTITION:
        G.gacer_init(-1, partition=name)
        G.gacer_shutdown()
    for bad in (-1, 4, 99):
        o = G.gacer_options(num_ctas=0, partition=bad, watchdog_ms=0, trace=0)
        assert G.lib().gacer_init(-1, ctypes.byref(o)) == -1  # GACER_E_INVALID_ARG
    assert G.PARTITION["priority"] == 0   # the default (zeroed options)
    G.gacer_init(-1)
    try:
        for name in G.PARTITION:            # switchable at run time (part of the regulation)
            G.gacer_set_partition(name)
        for bad in (-1, 4, 99):
            assert G.lib().gacer_set_partition(bad) == -1
    finally:
        G.gacer_shutdown()


def test_tile_path_counts(host):
    """The per-op RNE gates of test_gpu_parity.py target specific tile
    paths; the lowering must route those shapes there: VGG-16's FC1 is a
    swap-AB linear with a fixed split-K, and the D2 mix carries M-pair
    (256-row) and 128x256 tiles."""
    g = workloads.Graph("fc_op", 512, 7, 7)
    g.linear(g.flatten(0), 512 * 49, 4096)
    t = register(g, 8)
    info = G.gacer_get_tenant_info(t)
    assert info["swap_ops"] == 1 and info["split_k_ops"] == 1 and info["gemm_ops"] == 1
    G.gacer_shutdown()
    G.gacer_init(-1)
    for cin, cout in ((64, 64), (32, 96), (64, 128)):
        g = workloads.Graph("mpair", cin, 112, 112)
        g.relu(g.bn(g.conv(0, cin, cout, 3, 1, 1), cout))
        info = G.gacer_get_tenant_info(register(g, 8))
        assert info["mpair_ops"] == 1, (cin, cout, info)
    v = G.gacer_get_tenant_info(register(workloads.build_model("vgg16"), 8))
    assert v["mpair_ops"] >= 1 and v["wide_ops"] >= 1 and v["swap_ops"] == 3


def test_next2_models_lower(host):
    """NEXT-2 tenants (the paper's M3 and D121) lower without
    copies: MobileNetV3's SE block = GAP, FC+ReLU, FC, channel scale (4 ops;
    hardswish / hardsigmoid are separate eltwise ops); DenseNet-121's nested concats are zero-copy channel
    prefixes of one buffer per block, its pre-activation BN+ReLU one CUDA-core
    op per dense layer."""
    counts = {}
    for name, want in (("mobilenet_v3_large", (187, 110)), ("densenet121", (427, 188))):
        g = workloads.build_model(name)
        t = register(g, 8)
        info = G.gacer_get_tenant_info(t)
        counts[name] = (info["n_orig_ops"], info["n_fused_ops"])
        assert counts[name] == want, (name, counts[name])
    # stem 1 + 14 expands + 15 depthwise + 8 SE x 4 + 15 projects + head 4, plus
    # the 29 hardswish / hardsigmoid activations as their own eltwise ops
    assert 1 + 14 + 15 + 8 * 4 + 15 + 4 + 29 == 110
    # conv0 + maxpool + 58 dense layers x 3 + 3 transitions x 3 + BN/ReLU, GAP, FC
    assert 2 + 58 * 3 + 3 * 3 + 3 == 188


def test_buffer_reuse_footprint(host, monkeypatch):
    """Liveness-based activation-buffer reuse: the D2
    tenants' activation footprint drops to roughly their live set (ResNet-50
    B=8: < 1/3 of one buffer per tensor), every reusing tensor records its
    predecessors for the write-after-read dependencies, concat slices and
    the graph input/output never take part, and without GACER_REUSE=1 (the
    default) every tensor keeps its own buffer."""
    monkeypatch.setenv("GACER_REUSE", "1")
    for name, frac in (("resnet50", 0.34), ("vgg16", 0.5), ("mobilenet_v2", 0.34), ("densenet121", 0.34)):
        info = G.gacer_get_tenant_info(register(workloads.build_model(name), 8))
        assert info["reused_tensors"] > 0, name
        assert info["act_bytes"] <= frac * info["act_bytes_private"], (name, info)
    monkeypatch.setenv("GACER_REUSE", "0")
    info = G.gacer_get_tenant_info(register(workloads.build_model("resnet50"), 8))
    assert info["reused_tensors"] == 0 and info["act_bytes"] == info["act_bytes_private"]
    # a chain of equal tensors: with distance 2, three buffers suffice
    monkeypatch.setenv("GACER_REUSE", "1")
    g = workloads.Graph("chain", 64, 32, 32)
    x = 0
    for _ in range(8):
        x = g.relu(g.bn(g.conv(x, 64, 64, 3, 1, 1), 64))
    g.linear(g.flatten(g.gap(x)), 64, 10)
    info = G.gacer_get_tenant_info(register(g, 2))
    one = 2 * 32 * 32 * 64 * 2
    assert info["act_bytes"] == 3 * one, info   # (the small GAP output fits a freed buffer)


def test_split_k_defaults(host, monkeypatch):
    """Split-K (a function of the layer shape and these process knobs only):
    convolutions run without it by default (the fixed-order reduction tail
    outweighs the parallelism inside a multi-tenant round), the swap-AB
    linears keep it; GACER_SPLITK_MAX re-enables it for convolutions (the
    per-op GPU gate of the deep-K case runs that way)."""
    def deep():
        g = workloads.Graph("deep", 512, 7, 7)
        g.relu(g.bn(g.conv(0, 512, 512, 3, 1, 1), 512))
        return G.gacer_get_tenant_info(register(g, 8))
    assert deep()["split_k_ops"] == 0
    monkeypatch.setenv("GACER_SPLITK_MAX", "4")
    assert deep()["split_k_ops"] == 1
    monkeypatch.delenv("GACER_SPLITK_MAX")
    v = G.gacer_get_tenant_info(register(workloads.build_model("vgg16"), 8))
    assert v["split_k_ops"] >= 1 and v["swap_ops"] == 3
