"""Multi-GPU sharding of the point pass (north star subsystem 4).

Points are independent, so the path shards by contiguous point
ranges (or per-rank batches); the approximation is built deterministically
on every rank and the per-region [R,2] int64 COUNT and float64
SUM partials are combined with ONE all-reduce of a packed float64 buffer
(NCCL over NVLink on the B200 box, gloo in CPU tests).  Counts are exact in int64; float64 sums
differ from a 1-GPU run only by summation order (rel < 1e-12).
"""
from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [begin, end) slice of n points for `rank`."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return n * rank // world, n * (rank + 1) // world


def combine(cnt, sm, group=None, force: bool = False):
    """In-place all-reduce (sum) of the per-region partials of every rank: ONE
    collective over a packed float64 [R, 4] buffer (alpha/beta COUNT, alpha/beta
    SUM).  Counts stay exact in float64 below 2^53 points.  force:
    run the collective even for a single-rank group (tests of the NCCL path)."""
    import torch
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and (force or dist.get_world_size(group) > 1):
        buf = torch.cat([cnt.to(torch.float64), sm], dim=1)
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
        cnt.copy_(buf[:, :2].to(torch.int64))
        sm.copy_(buf[:, 2:])
    return cnt, sm


__all__ = ["shard_range", "combine"]
