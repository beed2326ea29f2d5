"""Data-parallel gradient exchange of a training tenant.

With G replicas (one process per GPU) each replica computes the gradients of
its own batch (BN statistics per replica); the SGD update then applies the
MEAN of the replicas' gradients (oracle/train.py: ``allreduce_mean``).  This
is the one real exchange step of the method's data-parallel path, so it is
the one collective: ``torch.distributed.all_reduce(SUM)`` over NCCL (NVLink /
NVSwitch; ``gloo`` on CPU for the tests) on flat fp32 buckets, issued on a
dedicated communication stream so buckets can overlap the rest of the
backward pass.  The 1/G scale is applied once per bucket after the sum.

Plumbing only (torch.distributed is the transport); the gradients are
produced and consumed by the library's kernels (include/gacer_train.h).
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

BUCKET_BYTES = 25 << 20      # per all-reduce call: launch latency amortised, still overlappable


class GradBuckets:
    """Static bucketing of a fixed list of gradient tensors (same order and
    shapes on every replica).  ``reduce_mean`` replaces every tensor by the
    mean over the process group, in place."""

    def __init__(self, shapes: Sequence[Tuple[int, ...]], bucket_bytes: int = BUCKET_BYTES):
        self.shapes = [tuple(s) for s in shapes]
        self.buckets: List[List[int]] = []
        cur, cur_bytes = [], 0
        # reverse order: the last layers' gradients are ready first in backward
        for i in reversed(range(len(self.shapes))):
            n = 1
            for d in self.shapes[i]:
                n *= d
            if cur and cur_bytes + 4 * n > bucket_bytes:
                self.buckets.append(cur)
                cur, cur_bytes = [], 0
            cur.append(i)
            cur_bytes += 4 * n
        if cur:
            self.buckets.append(cur)

    def reduce_mean(self, grads: List, dist, group=None, stream=None) -> None:
        """All-reduce every bucket (flattened fp32) and scale by 1/G.  With a
        CUDA ``stream`` the copies and collectives are issued on it (the
        caller orders it after the producing kernels)."""
        import torch

        G = dist.get_world_size(group)
        ctx = torch.cuda.stream(stream) if stream is not None else _null()
        with ctx:
            for b in self.buckets:
                flat = torch.cat([grads[i].reshape(-1).float() for i in b])
                dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
                flat.mul_(1.0 / G)
                off = 0
                for i in b:
                    n = grads[i].numel()
                    grads[i].copy_(flat[off:off + n].view_as(grads[i]))
                    off += n


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def grads_as_list(grads: Dict[int, Dict[str, object]]) -> Tuple[List, List[Tuple[int, str]]]:
    """Flatten {op_id: {name: tensor}} into a list in (op_id, name) order."""
    keys = [(oid, n) for oid in sorted(grads) for n in sorted(grads[oid])]
    return [grads[o][n] for o, n in keys], keys
