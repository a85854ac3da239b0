"""Multi-GPU bookkeeping of the query-sharded driver.

The path has no exchange step: each rank holds a replica of the factors and answers its own shard of
the query stream.  Two shardings (bench.py --shard):
  * index:   rank k owns the contiguous global index range [k*n/W, (k+1)*n/W);
  * spatial: rank k owns the queries whose footprint centre lies in the k-th of W vertical strips of
             the map (domain decomposition, as screen-space tiles of a renderer would give): every
             rank keeps the full stream's queries-per-row density, so binning finds the same reuse as
             one GPU with the whole batch.  The owner is a function of the record.
The only collectives run after the timed region: MAX of the per-rank step times and SUM of an fp64
result checksum.  Works with any torch.distributed backend (NCCL on the GPUs, gloo in the CPU tests).
"""
from __future__ import annotations


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced, disjoint: the shards of ranks 0..world-1 tile [0, n_total)."""
    if world < 1 or not 0 <= rank < world or n_total < 0:
        raise ValueError((n_total, rank, world))
    return rank * n_total // world, (rank + 1) * n_total // world


def spatial_owner(u, map_size: int, world: int):
    """Rank owning a query with footprint centre u (texels): the strip floor(u' W / N), u' = u wrapped
    into [0, N) (numpy arrays or scalars).  Strips are balanced for uniformly placed centres."""
    import numpy as np
    if world < 1 or map_size < 1:
        raise ValueError((map_size, world))
    uw = np.mod(np.asarray(u, np.float64), map_size)
    return np.minimum((uw * world / map_size).astype(np.int64), world - 1)


def reduce_times_and_checksum(times, checksum: float, device=None):
    """all_reduce(MAX) of a list of per-rank times and all_reduce(SUM) of the checksum.
    Returns (max_times list, total checksum).  Single-process: identity."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(times), dtype=torch.float64, device=device)
    c = torch.tensor([checksum], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
    return t.tolist(), float(c.item())
