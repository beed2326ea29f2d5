"""Whole-tenant pins: the oracle's graph interpreter vs torchvision's model
definitions run in torch-CPU fp64 with the same weights (a library routine,
independent of the oracle's C loops), plus the invariants PAPER.md relies on:
batch independence and Eq. 5 decomposition invariance ("without sacrificing
model accuracy", l.674)."""
import numpy as np
import pytest
import torch
import torchvision

import workloads
from oracle import forward_graph, chunked_forward


def load_into_torch(graph, params, tmodel):
    """Copy our per-op params into a torchvision model, matching modules in
    registration order (conv/bn/linear)."""
    ours = [op for op in graph.ops if op["kind"] in ("conv", "bn", "linear")]
    theirs = [m for m in tmodel.modules()
              if isinstance(m, (torch.nn.Conv2d, torch.nn.BatchNorm2d, torch.nn.Linear))]
    assert len(ours) == len(theirs), (len(ours), len(theirs))
    with torch.no_grad():
        for op, m in zip(ours, theirs):
            p = params[op["id"]]
            if op["kind"] == "bn":
                assert isinstance(m, torch.nn.BatchNorm2d) and m.num_features == op["c"]
                m.weight.copy_(torch.from_numpy(p["gamma"]))
                m.bias.copy_(torch.from_numpy(p["beta"]))
                m.running_mean.copy_(torch.from_numpy(p["mean"]))
                m.running_var.copy_(torch.from_numpy(p["var"]))
                m.eps = op["eps"]
            else:
                # (a linear of ours may be torchvision's 1x1 conv on a pooled
                #  map: MobileNetV3's squeeze-and-excitation FCs)
                assert m.weight.numel() == p["w"].size and m.weight.shape[0] == p["w"].shape[0], (op, m)
                m.weight.copy_(torch.from_numpy(p["w"]).reshape(m.weight.shape))
                if "b" in p:
                    m.bias.copy_(torch.from_numpy(p["b"]))
                else:
                    assert m.bias is None
    return tmodel.double().eval()


TV = {
    "resnet18": lambda: torchvision.models.resnet18(),
    "resnet34": lambda: torchvision.models.resnet34(),
    "resnet50": lambda: torchvision.models.resnet50(),
    "resnet101": lambda: torchvision.models.resnet101(),
    "mobilenet_v2": lambda: torchvision.models.mobilenet_v2(),
    "vgg16": lambda: torchvision.models.vgg16(),
    "alexnet": lambda: torchvision.models.alexnet(),
    "inception_v3": lambda: torchvision.models.inception_v3(
        aux_logits=False, init_weights=False, transform_input=False),
    "mobilenet_v3_large": lambda: torchvision.models.mobilenet_v3_large(),
    "densenet121": lambda: torchvision.models.densenet121(),
}

CASES = [("resnet18", 64, 2), ("resnet50", 64, 2), ("mobilenet_v2", 64, 2),
         ("alexnet", 224, 1), ("vgg16", 224, 1), ("inception_v3", 224, 1),
         ("resnet101", 64, 1), ("resnet34", 64, 1), ("mobilenet_v3_large", 64, 2),
         ("densenet121", 64, 1)]


@pytest.mark.parametrize("name,hw,batch", CASES)
def test_tenant_vs_torchvision(name, hw, batch):
    g = workloads.build_model(name, hw)
    params = workloads.make_params(g, seed=7, dtype="bf16")
    x = workloads.make_input(g, batch, seed=7, dtype="bf16")
    y = forward_graph(g, params, x)
    tm = load_into_torch(g, params, TV[name]())
    with torch.no_grad():
        ref = tm(torch.from_numpy(x.astype(np.float64))).numpy()
    assert y.shape == ref.shape
    err = np.max(np.abs(y - ref)) / np.max(np.abs(ref))
    assert err < 1e-10, err


def test_tiny_tenants_vs_torch():
    import torch.nn.functional as F
    g = workloads.build_model("tiny_cnn")
    p = workloads.make_params(g, 11, "fp32")
    x = workloads.make_input(g, 2, 11, "fp32")
    convs = [op for op in g.ops if op["kind"] == "conv"]
    t = torch.from_numpy(x.astype(np.float64))
    for i, op in enumerate(convs):
        t = F.relu(F.conv2d(t, torch.from_numpy(p[op["id"]]["w"].astype(np.float64)),
                            torch.from_numpy(p[op["id"]]["b"].astype(np.float64)), padding=1))
        if i < 2:
            t = F.max_pool2d(t, 2, 2)
    ref = t.mean(dim=(2, 3)).numpy()
    assert np.max(np.abs(forward_graph(g, p, x) - ref)) < 1e-12

    g = workloads.build_model("tiny_mlp")
    p = workloads.make_params(g, 12, "fp32")
    x = workloads.make_input(g, 2, 12, "fp32")
    lins = [op for op in g.ops if op["kind"] == "linear"]
    t = torch.from_numpy(x.reshape(2, -1).astype(np.float64))
    t = F.relu(F.linear(t, *(torch.from_numpy(p[lins[0]["id"]][k].astype(np.float64)) for k in "wb")))
    t = F.linear(t, *(torch.from_numpy(p[lins[1]["id"]][k].astype(np.float64)) for k in "wb"))
    assert np.max(np.abs(forward_graph(g, p, x) - t.numpy())) < 1e-12


@pytest.mark.parametrize("name,hw", [("resnet18", 32), ("mobilenet_v2", 32), ("mobilenet_v3_large", 32),
                                     ("densenet121", 32)])
def test_batch_independence(name, hw):
    g = workloads.build_model(name, hw)
    p = workloads.make_params(g, 3)
    x = workloads.make_input(g, 3, 3)
    y = forward_graph(g, p, x)
    for n in range(3):
        assert np.array_equal(y[n:n + 1], forward_graph(g, p, x[n:n + 1]))


@pytest.mark.parametrize("seed", range(4))
def test_chunked_forward_is_exact(seed):
    """Eq. 5 decomposition (batch and channel) reproduces the undecomposed
    forward bit-for-bit in fp64."""
    rng = np.random.default_rng(seed)
    name = ["resnet18", "mobilenet_v2", "mobilenet_v3_large", "densenet121"][seed % 4]
    g = workloads.build_model(name, 32)
    p = workloads.make_params(g, seed)
    B = 4
    x = workloads.make_input(g, B, seed)
    dec = {}
    for op in g.ops:
        if op["kind"] in ("flatten", "concat"):
            continue
        r = rng.random()
        if r < 0.3:
            n = int(rng.integers(1, B + 1))
            cuts = np.sort(rng.choice(np.arange(1, B), size=n - 1, replace=False)) if n > 1 else []
            sizes = np.diff(np.concatenate([[0], cuts, [B]])).astype(int).tolist()
            dec[op["id"]] = ("batch", sizes)
        elif r < 0.5 and op["kind"] in ("conv", "linear", "bn", "relu", "relu6", "hardswish"):
            C = op.get("c_out", op.get("c"))
            if C is None or C < 2:
                continue
            a = int(rng.integers(1, C))
            dec[op["id"]] = ("channel", [a, C - a])
    y = forward_graph(g, p, x)
    yc = chunked_forward(g, p, x, dec)
    assert np.array_equal(y, yc)
