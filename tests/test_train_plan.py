"""Host-side plan of the training driver (paper_2304_11745_b200/train_driver.py:
plan_graph), CPU only: NHWC shapes, the ReLUs fused into their producers, and
loud refusal of operator patterns the device training path does not cover."""
import pytest

import workloads
from paper_2304_11745_b200.train_driver import plan_graph


def test_resnet50_plan_shapes_and_fusion():
    g = workloads.build_model("resnet50", 224)
    shape, fused = plan_graph(g)
    assert shape[0] == (224, 224, 8)                       # 3 channels padded to the 8-channel granule
    first_conv = g.ops[0]
    assert shape[first_conv["id"]] == (112, 112, 64)
    gap = [op for op in g.ops if op["kind"] == "gap"][0]
    assert shape[gap["id"]] == (1, 1, 2048)
    relus = [op for op in g.ops if op["kind"] == "relu"]
    assert len(fused) == len(relus) and set(fused.values()) == {r["id"] for r in relus}
    kinds = {g.ops[[o["id"] for o in g.ops].index(p)]["kind"] for p in fused}
    assert kinds == {"bn", "add"}
    assert shape[g.ops[-1]["id"]] == (1, 1, 1000)


def test_unsupported_patterns_raise():
    with pytest.raises(NotImplementedError):
        plan_graph(workloads.build_model("mobilenet_v2", 64))    # depthwise (grouped) convs, ReLU6
    g = workloads.Graph("conv_relu", 8, 8, 8)
    c = g.conv(0, 8, 16, 3, 1, 1)
    g.relu(c)                                                  # ReLU straight after a conv: not fusable
    with pytest.raises(NotImplementedError):
        plan_graph(g)
    g = workloads.Graph("flat_head", 16, 4, 4)
    c = g.bn(g.conv(0, 16, 16, 3, 1, 1), 16)
    g.linear(g.flatten(g.relu(c)), 16 * 16, 10)               # flatten -> linear over a 4x4 map
    with pytest.raises(NotImplementedError):
        plan_graph(g)
