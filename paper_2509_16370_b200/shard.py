"""Batch sharding across GPUs (row e): instances are independent, so ranks own contiguous
global-id ranges and no collective touches the data path.  torch.distributed is used only to
reduce the timing (max over ranks), for barriers, and for the final gather of per-instance
summaries to rank 0 after the solve (status, u_0, KKT residual norms; for the IPM
step α_p, D, 𝒜(0)); full trajectories stay on their device."""
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


def gather_summaries(parts, rank: int, world: int, total: int):
    """Gather per-instance summary tensors of every rank's shard to rank 0 (after the solve).

    parts: dict name -> tensor [shard_size, ...] (this rank's contiguous shard, shard_range order),
    e.g. status, u_0 and the KKT residual norms of rr_factor_solve, or status, α_p, D, 𝒜(0) of
    ipm_step.  Returns, on rank 0, dict name -> tensor [total, ...] in global-id
    order; None on the other ranks.  One dist.gather per tensor to rank 0 (NCCL point-to-point
    over NVLink / NVSwitch on GPUs, gloo on CPU): only rank 0 receives, so memory and traffic are
    O(total) there and O(shard) elsewhere.  Shards differ in size by at most one; every rank pads
    to the largest shard."""
    import torch
    import torch.distributed as dist
    if world == 1 or not (dist.is_available() and dist.is_initialized()):
        return dict(parts)
    sizes = [e - b for b, e in (shard_range(r, world, total) for r in range(world))]
    mx = max(sizes)
    out = {}
    for name in sorted(parts):          # same collective order on every rank
        t = parts[name]
        if t.shape[0] != sizes[rank]:
            raise ValueError("summary %s has %d rows, shard has %d" % (name, t.shape[0], sizes[rank]))
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[:t.shape[0]].copy_(t)
        if rank == 0:
            bufs = [torch.empty_like(pad) for _ in range(world)]
            dist.gather(pad, gather_list=bufs, dst=0)
            out[name] = torch.cat([bufs[r][:sizes[r]] for r in range(world)], dim=0)
        else:
            dist.gather(pad, dst=0)
    return out if rank == 0 else None
