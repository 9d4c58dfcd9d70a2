"""Multi-GPU plumbing for the codec path: streams are
independent, so ranks shard streams with no collective on the data path.
The only collectives are the post-run timing reduction and barriers."""

from __future__ import annotations


def rank_streams(rank: int, world: int, per_rank: int) -> list:
    """Weak scaling: every rank owns ``per_rank`` streams, ids rank*per_rank + i."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return [rank * per_rank + i for i in range(per_rank)]


def strong_streams(rank: int, world: int, total: int) -> list:
    """Strong scaling alternative: stream_id % world == rank."""
    return [s for s in range(total) if s % world == rank]


def max_over_ranks(value: float, device=None) -> float:
    """Device-time of a step is the max over ranks (the slowest GPU)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
