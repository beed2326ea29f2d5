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
