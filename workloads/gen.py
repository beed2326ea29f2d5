"""Seeded synthetic tensors.  Data only.

* Generator: numpy ``Generator(PCG64(seed))``; seed = 1000*config + tenant
  index, weights use seed + 500.
* Inputs U(-1, 1), NCHW float32.
* conv / linear weights: normal with std = sqrt(gain / fan_in), gain = 2 (He)
  except MobileNetV2 (gain 1, C2a).  Biases U(-0.1, 0.1).
* BN: gamma U(0.8, 1.2) (U(0.1, 0.3) for the last BN of a residual branch),
  beta U(-0.1, 0.1), running mean U(-0.1, 0.1), running var U(0.8, 1.2).
* For bf16 tenants, inputs and conv/linear weights are rounded to bf16 (RNE)
  so that both the oracle and the GPU consume exactly the same values; BN
  parameters and biases stay float32.
"""
from __future__ import annotations

import numpy as np


def bf16_round(a) -> np.ndarray:
    """Round float32 values to the nearest bfloat16 (ties to even); returns
    float32 holding bf16-representable values.  NaN/Inf are not expected."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).reshape(a.shape)


def tenant_seed(config_index: int, tenant_index: int) -> int:
    return 1000 * config_index + tenant_index


def make_params(graph, seed: int, dtype: str = "bf16") -> dict:
    """Return {op_id: {name: float32 array}} for every parameterised op."""
    rng = np.random.Generator(np.random.PCG64(seed + 500))
    gain = graph.init_gain
    out = {}
    for op in graph.ops:
        k = op["kind"]
        if k == "conv":
            cig = op["c_in"] // op["groups"]
            fan_in = cig * op["kh"] * op["kw"]
            w = rng.normal(0.0, np.sqrt(gain / fan_in),
                           size=(op["c_out"], cig, op["kh"], op["kw"])).astype(np.float32)
            p = {"w": bf16_round(w) if dtype == "bf16" else w}
            if op["bias"]:
                p["b"] = rng.uniform(-0.1, 0.1, size=op["c_out"]).astype(np.float32)
            out[op["id"]] = p
        elif k == "linear":
            w = rng.normal(0.0, np.sqrt(gain / op["c_in"]),
                           size=(op["c_out"], op["c_in"])).astype(np.float32)
            p = {"w": bf16_round(w) if dtype == "bf16" else w}
            if op["bias"]:
                p["b"] = rng.uniform(-0.1, 0.1, size=op["c_out"]).astype(np.float32)
            out[op["id"]] = p
        elif k == "bn":
            c = op["c"]
            lo, hi = (0.1, 0.3) if op.get("res_last") else (0.8, 1.2)
            out[op["id"]] = {
                "gamma": rng.uniform(lo, hi, size=c).astype(np.float32),
                "beta": rng.uniform(-0.1, 0.1, size=c).astype(np.float32),
                "mean": rng.uniform(-0.1, 0.1, size=c).astype(np.float32),
                "var": rng.uniform(0.8, 1.2, size=c).astype(np.float32),
            }
    return out


def make_input(graph, batch: int, seed: int, dtype: str = "bf16") -> np.ndarray:
    """NCHW float32 input U(-1,1) (bf16-rounded for bf16 tenants)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    x = rng.uniform(-1.0, 1.0, size=(batch, graph.in_c, graph.in_h, graph.in_w)).astype(np.float32)
    return bf16_round(x) if dtype == "bf16" else x


def make_labels(batch: int, seed: int, n_classes: int = 1000) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed + 900))
    return rng.integers(0, n_classes, size=batch).astype(np.int32)
