"""The N>1 path (replicas only) with world_size-2 gloo on CPU:
disjoint seed shards, max-over-ranks time, sum-over-ranks propagations, and
per-query results gathered in rank order."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_02846_b200 import replicas


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        seeds = replicas.shard_seeds(1000, rank, world, 4)
        # rank-dependent fake timings: the job time is the slowest rank's
        mx, total = replicas.reduce_job(10.0 + rank, 100.0 * (rank + 1), world=world)
        gathered = replicas.gather_results([{"rank": rank, "seed": s} for s in seeds], world=world)
        out.put((rank, seeds, mx, total, gathered))
    finally:
        dist.destroy_process_group()


def test_world_size_2_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    (_, s0, mx0, tot0, g0), (_, s1, mx1, tot1, g1) = res
    assert s0 == [1000, 1001, 1002, 1003] and s1 == [1004, 1005, 1006, 1007]
    assert not set(s0) & set(s1)
    assert mx0 == mx1 == 11.0
    assert tot0 == tot1 == 300.0
    assert g0 == g1 and [d["seed"] for d in g0] == s0 + s1


def test_round_robin_and_errors():
    seeds = list(range(10))
    parts = [replicas.round_robin(seeds, r, 4) for r in range(4)]
    assert sorted(sum(parts, [])) == seeds
    assert parts[1] == [1, 5, 9]
    with pytest.raises(ValueError):
        replicas.shard_seeds(0, 2, 2, 3)
    assert replicas.reduce_job(5.0, 7, world=1) == (5.0, 7.0)
