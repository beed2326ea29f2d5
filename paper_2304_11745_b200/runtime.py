"""Torch plumbing around the C ABI: device buffers and layout marshalling.

PyTorch provides device memory, pinned host memory and streams only; every
step of a round runs inside libgacer.so.  ``Session`` registers a list of
tenants, allocates their NHWC input / float32 output buffers and binds them.
"""
from __future__ import annotations

import numpy as np
import torch

from . import gacer as G


def nchw_to_nhwc_padded(x: np.ndarray, c_pad: int, dtype: torch.dtype) -> torch.Tensor:
    """NCHW float32 host array -> NHWC [B,H,W,c_pad] host tensor (zero
    padding channels).  Values of bf16 tenants are already bf16-representable,
    so the cast is exact."""
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).permute(0, 2, 3, 1)
    B, H, W, C = t.shape
    out = torch.zeros((B, H, W, c_pad), dtype=torch.float32)
    out[..., :C] = t
    return out.to(dtype)


class Session:
    """One GACER instance on one GPU with its registered tenants."""

    def __init__(self, tenants, device=0, num_ctas=0, partition="priority",
                 watchdog_ms=0, trace=False, coarse_deps=False):
        """tenants: list of (graph, params, batch, dtype)."""
        self.device = device
        torch.cuda.set_device(device)
        G.gacer_init(device, num_ctas=num_ctas, partition=partition, watchdog_ms=watchdog_ms, trace=trace,
                     coarse_deps=coarse_deps)
        self.tenants = []
        self.inputs, self.outputs, self.info = [], [], []
        for graph, params, batch, dtype in tenants:
            tid = G.gacer_register_tenant(graph, params, batch, dtype)
            info = G.gacer_get_tenant_info(tid)
            tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
            x = torch.zeros((batch, info["in_h"], info["in_w"], info["in_c_pad"]), dtype=tdt,
                            device=f"cuda:{device}")
            y = torch.zeros((batch, info["out_features"]), dtype=torch.float32, device=f"cuda:{device}")
            G.gacer_bind_io(tid, x.data_ptr(), y.data_ptr())
            self.tenants.append((graph, batch, dtype))
            self.inputs.append(x)
            self.outputs.append(y)
            self.info.append(info)

    def set_input(self, t: int, x_nchw: np.ndarray):
        info = self.info[t]
        h = nchw_to_nhwc_padded(x_nchw, info["in_c_pad"], self.inputs[t].dtype)
        self.inputs[t].copy_(h.to(self.inputs[t].device))

    def host_input(self, t: int, x_nchw: np.ndarray) -> torch.Tensor:
        """Pinned host copy of tenant t's input in the device layout."""
        info = self.info[t]
        return nchw_to_nhwc_padded(x_nchw, info["in_c_pad"], self.inputs[t].dtype).pin_memory()

    def set_regulation(self, decomposition=None, pointers=None):
        return G.gacer_set_regulation(decomposition, pointers, n_tenants=len(self.tenants))

    def set_mode(self, mode: str):
        return G.gacer_set_mode(mode)

    def run(self):
        return G.gacer_run_round()

    def results(self):
        torch.cuda.synchronize(self.device)
        return [y.cpu().numpy().copy() for y in self.outputs]

    def stats(self):
        return G.gacer_get_stats()

    def close(self):
        G.gacer_shutdown()
