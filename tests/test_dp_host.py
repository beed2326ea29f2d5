"""A12 host logic (no GPU): gradient buckets cover the flat gradient buffer
exactly once, last layers first, within the bucket size unless a single
parameter is larger; enabling the gradient gate keeps the plan's work and
only adds the gate dependency of the SGD item."""
import pytest

import workloads
from paper_2304_11745_b200 import gacer as G


@pytest.fixture()
def r50():
    G.gacer_init(-1)
    g = workloads.build_model("resnet50", 64)
    p = workloads.make_params(g, 3, "fp32")
    t = G.gacer_register_tenant(g, p, 4, "bf16", train=True)
    yield g, t
    G.gacer_shutdown()


@pytest.mark.parametrize("mb", [1, 4, 25, 1000])
def test_buckets_partition_the_gradients(r50, mb):
    g, t = r50
    n = G.gacer_get_tenant_info(t)["n_params"]
    bks = G.gacer_train_buckets(t, mb << 20)
    cover = sorted(bks)
    pos = 0
    for off, cnt in cover:
        assert off == pos and cnt > 0
        pos += cnt
    assert pos == n                                          # exactly once, no gaps
    assert [b[0] for b in bks] == sorted([b[0] for b in bks], reverse=True)   # last layers first
    assert bks[0][0] + bks[0][1] == n                        # the buffer's tail (the FC) goes first
    biggest = max(G.gacer_train_param(t, i + 1, 0)[1] for i, op in enumerate(g.ops) if op["kind"] == "conv")
    assert all(c * 4 <= max(mb << 20, 4 * biggest) for _, c in bks)


def test_gate_keeps_the_work(r50):
    g, t = r50
    n0 = G.gacer_get_stats()["n_items"]
    G.gacer_train_set_allreduce(t, True)
    assert G.gacer_get_stats()["n_items"] == n0
    G.gacer_train_set_allreduce(t, False)
    with pytest.raises(G.GacerError):
        G.gacer_train_set_allreduce(t + 5, True)
