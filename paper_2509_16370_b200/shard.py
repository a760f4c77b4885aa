"""Batch sharding across GPUs (row e): instances are independent, so ranks own contiguous
global-id ranges and no collective touches the data path.  torch.distributed is used only to
reduce the timing (max over ranks) and for barriers."""
from __future__ import annotations

from typing import Tuple


def shard_range(rank: int, world: int, total: int) -> Tuple[int, int]:
    """Contiguous [begin, end) of global instance ids owned by `rank`; the remainder is spread
    over the first ranks so shard sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world or total < 0:
        raise ValueError("bad shard request")
    base, rem = divmod(total, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar over the default process group (identity when not initialised)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
