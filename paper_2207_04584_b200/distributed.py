"""Multi-GPU driver: channel-sharded gridding, one process per GPU.

Channels are independent ("the data processing in those channels are
naturally independent"), and the paper names a "cluster with multiple GPU accelerators" as
its next step.  Rank r of G builds the same plan from the shared
coordinates (deterministic, < 1 ms of kernels), grids the contiguous channel slice
``channel_shard(C, G, r)`` through the public host API (``hegrid_grid``: pinned staging,
H2D / permute / accumulate / D2H overlapped over CUDA streams), and writes it into a
disjoint slice of one output map shared by all ranks (a memmap, e.g. in /dev/shm).  The
only communication is a barrier; no collective is on the data path.

    torchrun --nproc-per-node G -m paper_2207_04584_b200.distributed --workload cfg4 \\
        --out /dev/shm/hegrid_cfg4.f32

Inputs are the seeded synthetic workload (``synth``); each rank generates only its own
channels.  ``grid_rank`` is the per-rank step, usable without torch.distributed (the GPU
test runs G ranks one after the other in one process and compares with G = 1).
"""
from __future__ import annotations

import argparse
import json
import os
import time

import numpy as np

from .shard import channel_shard


def grid_rank(gridder, data, out, world: int, rank: int):
    """Grid this rank's channel slice: ``out[c0:c1] = gridder(data[c0:c1])``.

    data: [C][N] (host array / memmap / tensor, original sample order); out: [C][...]
    writable and visible to every rank (e.g. np.memmap).  Returns (c0, c1)."""
    c0, c1 = channel_shard(int(data.shape[0]), world, rank)
    if c1 > c0:
        out[c0:c1] = gridder(data[c0:c1])
    return c0, c1


def open_shared_out(path: str, shape, create: bool):
    """The output map shared by all ranks: a float32 memmap ``shape`` at ``path``."""
    mode = "w+" if create else "r+"
    return np.memmap(path, dtype=np.float32, mode=mode, shape=tuple(shape))


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--workload", default="cfg4")
    ap.add_argument("--channels", type=int, default=0, help="override the workload's channel count")
    ap.add_argument("--out", default="/dev/shm/hegrid_out.f32")
    ap.add_argument("--engine", default="auto")
    a = ap.parse_args(argv)

    import torch
    import synth
    from . import Plan

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    w = synth.CONFIGS[a.workload]
    if a.channels:
        w = w.with_(channels=a.channels)
    C = w.channels
    if rank == 0:
        open_shared_out(a.out, (C, w.ny, w.nx), create=True).flush()
    if world > 1:
        dist.barrier()
    out = open_shared_out(a.out, (C, w.ny, w.nx), create=False)
    lon, lat = synth.coords(w, device=dev)
    c0, c1 = channel_shard(C, world, rank)
    # this rank's channels, generated on its GPU, staged in pinned host memory [c1-c0][N]
    vals = torch.empty((c1 - c0, w.n), dtype=torch.float32, pin_memory=True)
    for b0 in range(c0, c1, 256):
        ch = torch.arange(b0, min(b0 + 256, c1), device=dev)
        vals[b0 - c0:b0 - c0 + ch.numel()].copy_(synth.values(w, lon, lat, channels=ch).cpu())
    res = torch.empty((c1 - c0, w.ny, w.nx), dtype=torch.float32, pin_memory=True)
    lon_h, lat_h = lon.cpu().numpy(), lat.cpu().numpy()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    with Plan(lon_h, lat_h, w.map, w.fwhm_deg, w.support, device=local, engine=a.engine) as p:
        p.grid(vals, res)
    out[c0:c1] = res.numpy()
    out.flush()
    t = time.perf_counter() - t0
    if world > 1:
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
        dist.barrier()
    if rank == 0:
        print(json.dumps({"workload": w.name, "world": world, "channels": C, "out": a.out,
                          "seconds_max_over_ranks": t,
                          "samples_x_channels_per_s": w.n * C / t}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
