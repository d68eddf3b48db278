"""Channel sharding across GPUs.

Channels are independent ("the data processing in those channels are
naturally independent"), so rank r of G grids a contiguous channel slice and writes a
disjoint slice of the output.  No collective is on the data path; a barrier (and, for
timing, a max-reduce of one float) is the only communication.
"""
from __future__ import annotations


def channel_shard(n_channels: int, world: int, rank: int, align: int = 4):
    """Contiguous [c0, c1) of rank ``rank``: balanced, ``align``-aligned boundaries,
    covering [0, n_channels) exactly once over all ranks."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    units = (n_channels + align - 1) // align
    lo = units * rank // world
    hi = units * (rank + 1) // world
    return min(lo * align, n_channels), min(hi * align, n_channels)


def grid_sharded(grid_fn, data, world: int, rank: int, out):
    """Run ``grid_fn(data_slice) -> out_slice`` on this rank's channel slice and place it
    into ``out`` (a [C, ...] array visible to all ranks, e.g. a shared memmap)."""
    c0, c1 = channel_shard(data.shape[0], world, rank)
    if c1 > c0:
        out[c0:c1] = grid_fn(data[c0:c1])
    return c0, c1
