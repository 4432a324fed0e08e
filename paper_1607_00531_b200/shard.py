"""Host-side work partitioning for multi-GPU runs (one process per GPU).

ADMM and GN columns never couple across volume pairs, so the C4 batch (64
independent pairs) shards by pairs with no data-path collective (SURVEY
§8(e)): rank r solves a contiguous block of pairs on its own GPU through
epc_admm_solve_batch. Only timing and result gathering use the process group.
"""
from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced block [first, first + count) of n items for rank."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    count = base + (1 if rank < extra else 0)
    first = rank * base + min(rank, extra)
    return first, count


def owner_of(i: int, n: int, world: int) -> int:
    """Rank that owns item i under shard_range."""
    for r in range(world):
        f, c = shard_range(n, r, world)
        if f <= i < f + c:
            return r
    raise IndexError(i)


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (timing is reported as the slowest rank)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, dist=None, device=None) -> float:
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
