"""Multi-GPU: replicas only.

The solve path has no exchange step: independent systems (graphs) shard
across ranks and each rank runs its share with no collective.  The only
cross-rank operations are the timing barrier and the max-over-ranks
reduction of the device time used to report whole-job throughput.
"""

from __future__ import annotations


def shard(items: list, rank: int, world: int) -> list:
    """Contiguous, balanced shard of ``items`` for ``rank`` (sizes differ by <= 1)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    n = len(items)
    lo = rank * n // world
    hi = (rank + 1) * n // world
    return items[lo:hi]


def aggregate_throughput(local_ms: float, local_units: int, device=None) -> tuple:
    """(units/s over all ranks, max-over-ranks ms, total units).

    Uses torch.distributed when initialised (nccl on GPUs, gloo in tests);
    the job's time is the slowest rank's device time.
    """
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(local_ms), float(local_units)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        tmax = t[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        units = t[1:].clone()
        dist.all_reduce(units, op=dist.ReduceOp.SUM)
        ms, total = float(tmax.item()), float(units.item())
    else:
        ms, total = float(t[0].item()), float(t[1].item())
    return total / (ms * 1e-3), ms, int(round(total))
