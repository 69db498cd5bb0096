"""Realization sharding across ranks (one process per GPU) and the final gather.

The path shards naturally: realizations / subcarriers are
independent systems, so rank r of W owns the contiguous block
[r*B/W, (r+1)*B/W) and no data-path collective exists.  The only cross-GPU
step is the final gather of the per-system statistics (NMSE, sum-rate,
iteration counts), which `gather_stats` performs with torch.distributed
(NCCL over NVLink on the GPU box, gloo in the CPU tests), preserving the
global system order even for uneven shards.
"""

from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) block of n items for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_stats(stats: dict, n_total: int, group=None) -> dict:
    """All-gather 1-D per-system tensors from every rank, concatenated in rank
    (= system) order.  Uneven shards are padded to the largest shard for the
    collective and trimmed afterwards."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return dict(stats)
    world = dist.get_world_size(group)
    sizes = [shard_range(n_total, r, world) for r in range(world)]
    cap = max(hi - lo for lo, hi in sizes)
    out = {}
    for name in sorted(stats):
        t = stats[name]
        pad = torch.zeros(cap, dtype=t.dtype, device=t.device)
        pad[:t.numel()] = t.reshape(-1)
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
        out[name] = torch.cat([p[:hi - lo] for p, (lo, hi) in zip(parts, sizes)])
    return out
