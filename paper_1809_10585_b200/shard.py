"""Sharding of independent HODLR matrices over ranks (BASELINE configs 3/4:
"batch sharded across 1/2/4/8 GPUs").  Independent factorizations need no
data-path collective; ranks only agree on timing (max over ranks)."""

from __future__ import annotations


def shard_seeds(total: int, world: int, rank: int) -> list:
    """Contiguous block of matrix indices of `rank` (ceil split)."""
    per = -(-total // world)
    return list(range(rank * per, min(total, (rank + 1) * per)))


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (the job time is the slowest rank's)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
