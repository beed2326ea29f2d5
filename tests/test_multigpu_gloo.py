"""N > 1 path on CPU: world-size-2 gloo process group exercising the
placement and max-over-ranks timing logic the bench uses under torchrun
(inference tenants shard by placement, no data-path collective)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2304_11745_b200.placement import (
    aggregate_throughput, max_over_ranks, place_tenants, replica_seed)


def test_place_replica_and_lpt():
    flops = [65.4, 247.5, 4.8]
    assert place_tenants(flops, 4, "replica") == [[0, 1, 2]] * 4
    p = place_tenants(flops, 2, "lpt")
    assert sorted(sum(p, [])) == [0, 1, 2]
    assert [1] in p                       # the largest tenant alone
    five = [22.9, 58.1, 249.6, 90.8, 9.6]  # D3 at B=16 (GFLOP)
    p2 = place_tenants(five, 2, "lpt")
    assert sorted(sum(p2, [])) == [0, 1, 2, 3, 4]
    loads = sorted(sum(five[i] for i in r) for r in p2)
    assert loads[1] == 249.6              # R101 alone bounds the round
    with pytest.raises(ValueError):
        place_tenants(flops, 0)
    assert len({replica_seed(2000, r) for r in range(8)}) == 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    my_time = 1.0 + rank          # rank 1 is the slowest
    t = max_over_ranks(my_time, dist)
    units = [24.0] * world         # each replica runs the full D2 mix (24 images)
    thr = aggregate_throughput(units, t)
    placement = place_tenants([1.0, 2.0, 3.0], world, "lpt")
    q.put((rank, t, thr, placement))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_max_over_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, t, thr, placement in res:
        assert t == 2.0                    # max over ranks
        assert abs(thr - 48.0 / 2.0) < 1e-12
        assert placement == res[0][3]      # every rank computes the same placement


def _grad_worker(rank, world, port, q):
    import numpy as np
    import torch
    from paper_2304_11745_b200.grad_allreduce import GradBuckets
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shapes = [(64, 3, 7, 7), (64,), (256, 64, 1, 1), (1000, 2048), (1000,)]
    rng = np.random.default_rng(100 + rank)               # each replica's own gradients
    grads = [torch.from_numpy(rng.normal(size=s).astype(np.float32)) for s in shapes]
    mine = [g.clone().numpy() for g in grads]
    b = GradBuckets(shapes, bucket_bytes=1 << 20)         # several buckets
    b.reduce_mean(grads, dist)
    q.put((rank, mine, [g.numpy() for g in grads], len(b.buckets)))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_gradient_mean_matches_oracle():
    """A12: the bucketed all-reduce of the replicas' gradients equals the
    oracle's replica mean (oracle/train.py allreduce_mean) on every rank."""
    from oracle.train import allreduce_mean
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_grad_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    import numpy as np
    per_rank = [{i: {"g": g} for i, g in enumerate(r[1])} for r in res]
    ref = allreduce_mean(per_rank)
    for rank, _, reduced, nb in res:
        assert nb >= 3
        for i, g in enumerate(reduced):
            assert np.allclose(g, ref[i]["g"], rtol=1e-6, atol=1e-7), (rank, i)
    assert all(np.array_equal(a, b) for a, b in zip(res[0][2], res[1][2]))   # identical on every rank
