"""Hypothesis sharding across ranks (one process per GPU).

Rank r owns the contiguous hypothesis range shard_range(n, r, world); scores
are all-gathered (torch.distributed: NCCL on GPUs, gloo in the CPU tests) in
rank order, so every rank holds the global score array in hypothesis order
and runs the same fixed-order reduction on it -- results are bitwise
independent of the GPU count.
"""
from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple:
    """[lo, hi) of rank `rank`: the first n % world ranks get one extra."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_scores(local, n_total: int, world: int, group=None):
    """All-gather per-rank score shards (torch tensors, rows = hypotheses)
    into the global array in hypothesis order.  Uneven shards are padded to
    the largest shard for the collective and compacted afterwards."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local
    sizes = [shard_range(n_total, r, world) for r in range(world)]
    m = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((m,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty((world * m,) + tuple(local.shape[1:]), dtype=local.dtype,
                      device=local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    if all(hi - lo == m for lo, hi in sizes):
        return out
    parts = [out[r * m: r * m + (hi - lo)] for r, (lo, hi) in enumerate(sizes)]
    return torch.cat(parts)
