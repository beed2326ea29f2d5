"""Tenant placement across the GPUs of one node.

Inference tenants are independent units: the multi-GPU path needs placement
only, no data-path collective.  One process per GPU (torchrun); each process
owns a GACER executor for the tenants placed on its GPU.

* ``replica``: every GPU runs the full mix on its own seeded inputs (weak
  scaling: per-GPU work fixed as N grows) -- maximises aggregate inf/s.
* ``lpt``: longest-processing-time-first bin packing of the tenants by
  FLOPs -- trims the round latency of one mix, capped by the largest
  tenant's chain.

torch.distributed is used for the start barrier and the max-over-ranks of
the measured device times only (off the timed region).
"""
from __future__ import annotations

from typing import List, Sequence


def place_tenants(flops: Sequence[float], world: int, mode: str = "replica") -> List[List[int]]:
    """Return, for each rank, the list of tenant indices it runs."""
    n = len(flops)
    if world < 1:
        raise ValueError("world must be >= 1")
    if mode == "replica":
        return [list(range(n)) for _ in range(world)]
    if mode == "lpt":
        load = [0.0] * world
        out: List[List[int]] = [[] for _ in range(world)]
        for t in sorted(range(n), key=lambda i: (-flops[i], i)):
            r = min(range(world), key=lambda k: (load[k], k))
            out[r].append(t)
            load[r] += flops[t]
        for lst in out:
            lst.sort()
        return out
    raise ValueError(f"unknown placement mode {mode!r}")


def replica_seed(base_seed: int, rank: int) -> int:
    """Seed of a replica's inputs: every GPU draws its own batch."""
    return base_seed + 10007 * rank


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a scalar over all ranks (the bench's timing rule)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_throughput(units_per_rank: Sequence[float], max_time_s: float) -> float:
    """Whole-job throughput: all ranks' units over the slowest rank's time."""
    return float(sum(units_per_rank)) / max_time_s
