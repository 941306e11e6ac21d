"""Multi-GPU = independent replicas.

The Kino-PAX+ iteration does not shard: its three passes share one region
table and one tree with a barrier between passes.  The
unit of parallelism across GPUs is therefore the independent seeded query
(SPEC.md:485, :528): rank r of a world of N solves its own seeds, and only the
scalar results (device time, propagations, per-query outcomes) cross ranks —
never the planner's data path.
"""
from __future__ import annotations


def shard_seeds(base: int, rank: int, world: int, per_rank: int) -> list[int]:
    """Seeds of rank `rank`: base + rank * per_rank + i (disjoint across ranks)."""
    if not (0 <= rank < world) or per_rank < 0:
        raise ValueError("bad rank / world / per_rank")
    return [base + rank * per_rank + i for i in range(per_rank)]


def round_robin(seeds: list[int], rank: int, world: int) -> list[int]:
    """Query q -> rank q mod N (the batch config's assignment)."""
    return [s for i, s in enumerate(seeds) if i % world == rank]


def reduce_job(device_ms: float, props: float, *, world: int, device=None):
    """Whole-job aggregation: time = max over ranks (the slowest replica bounds
    the job), propagations = sum over ranks.  Returns (max_ms, total_props)."""
    if world <= 1:
        return float(device_ms), float(props)
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(device_ms), float(props)], dtype=torch.float64, device=device)
    mx = t.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = t.clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    return float(mx[0]), float(sm[1])


def gather_results(results: list[dict], *, world: int) -> list[dict]:
    """All ranks' per-query result dicts, concatenated in rank order (host side)."""
    if world <= 1:
        return list(results)
    import torch.distributed as dist

    out = [None] * world
    dist.all_gather_object(out, results)
    return [r for part in out for r in part]
