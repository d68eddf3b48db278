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


# ---------------------------------------------------------------- cell (map-row) sharding
# For few-channel data (e.g. cfg3: 64 channels, ~90k neighbours per cell) channel slices are
# too thin to occupy a GPU; rank r instead owns a contiguous block of map rows and grids all
# channels there.  Eq. 1 is per cell, so the row blocks are
# independent: each rank builds its own plan on the sub-map (samples that cannot reach it
# are dropped by the plan's bin keys) and writes a disjoint [C][j0:j1][nx] slice.  No
# collective on the data path.

def row_shard(ny: int, world: int, rank: int):
    """Contiguous map rows [j0, j1) of rank ``rank``, balanced, covering [0, ny) once."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    return ny * rank // world, ny * (rank + 1) // world


def sub_map(m: dict, j0: int, j1: int) -> dict:
    """Header of rows [j0, j1) of map ``m``: the same cell centres (crpix_y shifted by j0,
    so lat_j' = crval_lat + (j' + 1 - (crpix_y - j0)) cdelt_lat = lat_{j0 + j'})."""
    s = dict(m)
    s["ny"] = int(j1 - j0)
    s["crpix_y"] = float(m["crpix_y"]) - j0
    return s


def grid_cell_sharded(grid_fn, m: dict, world: int, rank: int, out):
    """Run ``grid_fn(sub_map) -> [C][rows][nx]`` on this rank's row block of map ``m`` and
    place it into ``out`` ([C][ny][nx], visible to all ranks)."""
    j0, j1 = row_shard(int(m["ny"]), world, rank)
    if j1 > j0:
        out[:, j0:j1, :] = grid_fn(sub_map(m, j0, j1))
    return j0, j1
