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


class SymmetricExchange:
    """The device buffers of b3d_gpu_enumerate_shard for one process per GPU:
    every rank's global score array (2 halves of n_total x n_noise doubles,
    alternated by exchange epoch so no rank overwrites a half a slower peer
    is still reducing) and its signal pad (world x u64), allocated in
    PyTorch symmetric memory so each is mapped on every GPU over NVLink /
    NVSwitch.  `exchange(offset)` returns the next b3d_shard_exchange."""

    def __init__(self, n_total: int, n_noise: int, device, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        g = group or dist.group.WORLD
        self.world, self.rank = dist.get_world_size(g), dist.get_rank(g)
        self.n_total, self.n_noise = n_total, n_noise
        self.scores = symm_mem.empty(2 * n_total, n_noise, dtype=torch.float64, device=device)
        self._h = symm_mem.rendezvous(self.scores, g)
        self.signals = symm_mem.empty(self.world, dtype=torch.int64, device=device)
        self._hs = symm_mem.rendezvous(self.signals, g)
        self.signals.zero_()
        torch.cuda.synchronize(device)
        dist.barrier(g)
        self.score_ptrs = [int(p) for p in self._h.buffer_ptrs]
        self.signal_ptrs = [int(p) for p in self._hs.buffer_ptrs]
        self.epoch = 0

    def exchange(self, offset: int):
        from . import b3d
        self.epoch += 1
        return b3d.ShardExchange.make(self.rank, offset, self.n_total, self.score_ptrs,
                                      self.signal_ptrs, self.epoch)

    def half(self, epoch: int = None):
        """This rank's complete global array as written by exchange `epoch`."""
        e = self.epoch if epoch is None else epoch
        h = e & 1
        return self.scores[h * self.n_total:(h + 1) * self.n_total]

    def peer_ptrs(self, epoch: int, skip_self: bool = True):
        """Addresses of every (other) rank's half for `epoch` (set_score_peers)."""
        off = (epoch & 1) * self.n_total * self.n_noise * 8
        return [p + off for r, p in enumerate(self.score_ptrs) if not (skip_self and r == self.rank)]
