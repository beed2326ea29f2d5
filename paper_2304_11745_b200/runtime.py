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


def _device_view(ptr: int, count: int, device: str) -> torch.Tensor:
    """A float32 torch tensor aliasing `count` floats of library-owned device
    memory at `ptr` (no copy; the library owns the memory)."""
    class _Arr:
        __cuda_array_interface__ = {"shape": (count,), "typestr": "<f4", "data": (ptr, False), "version": 3}
    return torch.as_tensor(_Arr(), device=device)


class Session:
    """One GACER instance on one GPU with its registered tenants."""

    def __init__(self, tenants, device=0, num_ctas=0, partition="priority",
                 watchdog_ms=0, trace=False, coarse_deps=False):
        """tenants: list of (graph, params, batch, dtype) or (graph, params,
        batch, dtype, {"train": True, "lr": .., "momentum": ..}) for a
        training tenant (its round is one SGD step; labels via set_labels)."""
        self.device = device
        torch.cuda.set_device(device)
        G.gacer_init(device, num_ctas=num_ctas, partition=partition, watchdog_ms=watchdog_ms, trace=trace,
                     coarse_deps=coarse_deps)
        self.tenants = []
        self.inputs, self.outputs, self.info = [], [], []
        self.labels = {}
        for entry in tenants:
            graph, params, batch, dtype = entry[:4]
            opts = entry[4] if len(entry) > 4 else {}
            tid = G.gacer_register_tenant(graph, params, batch, dtype, train=opts.get("train", False),
                                          lr=opts.get("lr", 0.1), momentum=opts.get("momentum", 0.9))
            info = G.gacer_get_tenant_info(tid)
            tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
            x = torch.zeros((batch, info["in_h"], info["in_w"], info["in_c_pad"]), dtype=tdt,
                            device=f"cuda:{device}")
            y = torch.zeros((batch, info["out_features"]), dtype=torch.float32, device=f"cuda:{device}")
            G.gacer_bind_io(tid, x.data_ptr(), y.data_ptr())
            if info["train"]:
                lab = torch.zeros(batch, dtype=torch.int32, device=f"cuda:{device}")
                G.gacer_bind_labels(tid, lab.data_ptr())
                self.labels[tid] = lab
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

    def set_labels(self, t: int, labels: np.ndarray):
        self.labels[t].copy_(torch.from_numpy(np.ascontiguousarray(labels, np.int32)).to(self.labels[t].device))

    def train_state(self, t: int):
        """(loss, params, grads, momentum) of training tenant t as torch views
        of the library's device buffers (valid until close())."""
        st = G.gacer_get_train_state(t)
        n = st["n_params"]
        dev = f"cuda:{self.device}"

        def view(ptr, count):
            return _device_view(ptr, count, dev)
        return view(st["loss"], 1), view(st["params"], n), view(st["grads"], n), view(st["momentum"], n)

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
