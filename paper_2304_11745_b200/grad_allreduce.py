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


class ExecutorAllReduce:
    """A12 inside a GACER round: the training
    tenant's gradient mean over the data-parallel group, overlapped with its
    own backward pass.

    Per round: the executor launch on the compute stream, then on a
    communication stream, bucket by bucket (last layers first,
    ``gacer_train_buckets``): a device-side wait for the ops that write the
    bucket's gradient slice (``gacer_stream_wait_grads``: stream memory waits
    on the executor's completion counters -- the collective of the last
    layers starts while the earlier layers' backward still runs), the NCCL
    all-reduce (SUM) of that slice of the library's flat fp32 gradient buffer
    and the 1/G scale; after the last bucket the tenant's gradient gate opens
    (``gacer_stream_open_grad_gate``) and the SGD item of the round, which
    waits on it, applies the mean.  The executor must leave SMs free for the
    collective's kernels (Session(num_ctas=#SMs - reserve)).

    Plumbing only: the gradients are produced and consumed by libgacer's
    kernels; torch.distributed (NCCL) is the transport."""

    def __init__(self, session, tenant: int, dist, group=None, bucket_bytes: int = BUCKET_BYTES,
                 comm_stream=None):
        import torch
        from . import gacer as G
        self.G, self.dist, self.group, self.t = G, dist, group, tenant
        G.gacer_train_set_allreduce(tenant, True)
        self.buckets = G.gacer_train_buckets(tenant, bucket_bytes)
        _, _, self.grads, _ = session.train_state(tenant)
        self.world = dist.get_world_size(group)
        self.comm = comm_stream or torch.cuda.Stream(device=session.device)
        # create the communicator now: NCCL's lazy initialisation inside a
        # round could synchronise the device while the executor waits for
        # the gradient gate (a deadlock until the watchdog fires)
        with torch.cuda.stream(self.comm):
            w = torch.zeros(8, device=self.grads.device)
            dist.all_reduce(w, group=group)
        torch.cuda.synchronize(session.device)

    def enqueue_round(self, stream) -> None:
        """One round (every tenant's step / forward) with the overlapped
        gradient exchange of this tenant; all work is enqueued, nothing
        blocks the host."""
        import torch
        G = self.G
        G.gacer_run_round_async(stream.cuda_stream)
        cs = self.comm.cuda_stream
        with torch.cuda.stream(self.comm):
            for off, n in self.buckets:
                G.gacer_stream_wait_grads(cs, self.t, off, n)
                v = self.grads[off:off + n]
                self.dist.all_reduce(v, op=self.dist.ReduceOp.SUM, group=self.group)
                if self.world > 1:
                    v.mul_(1.0 / self.world)
            G.gacer_stream_open_grad_gate(cs, self.t)

    def close(self):
        self.G.gacer_train_set_allreduce(self.t, False)
