"""Multi-process (gloo, world_size 2) checks of the channel-sharded N>1 host logic.

On the GPU box each rank grids its own channel slice with the CUDA path; here the same
sharding, output placement and max-over-ranks timing logic run on CPU with the oracle as
the per-rank gridder, and the assembled result must equal a single-process run."""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2207_04584_b200.shard import channel_shard, grid_cell_sharded, grid_sharded, row_shard, sub_map


def _worker(rank, world, port, path, C, N, out_shape):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    w = synth.CONFIGS["cfg1"].with_(n=N, channels=C, nx=12, ny=10)
    lon, lat = synth.coords(w)
    vals = synth.values(w, lon, lat).numpy()
    out = np.memmap(path, dtype=np.float64, mode="r+", shape=out_shape)

    def grid_fn(v):
        o, _, _ = oracle.grid(lon.numpy(), lat.numpy(), v, w.map, w.fwhm_deg, w.support, nthreads=1)
        return o

    grid_sharded(grid_fn, vals, world, rank, out)
    out.flush()
    # max-over-ranks timing reduction as bench.py does it
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    assert t.item() == float(world)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_channel_sharded_grid_equals_single_process(world):
    import oracle
    import synth
    C, N = 7, 800
    w = synth.CONFIGS["cfg1"].with_(n=N, channels=C, nx=12, ny=10)
    shape = (C, w.cells)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "out.bin")
        np.memmap(path, dtype=np.float64, mode="w+", shape=shape).flush()
        port = 29500 + (os.getpid() % 2000)
        mp.spawn(_worker, args=(world, port, path, C, N, shape), nprocs=world, join=True)
        got = np.array(np.memmap(path, dtype=np.float64, mode="r", shape=shape))
    lon, lat = synth.coords(w)
    vals = synth.values(w, lon, lat).numpy()
    ref, _, _ = oracle.grid(lon.numpy(), lat.numpy(), vals, w.map, w.fwhm_deg, w.support)
    np.testing.assert_array_equal(np.isnan(got), np.isnan(ref))
    np.testing.assert_array_equal(got[~np.isnan(ref)], ref[~np.isnan(ref)])
    # every channel came from exactly one rank
    cover = np.zeros(C, int)
    for r in range(world):
        a, b = channel_shard(C, world, r)
        cover[a:b] += 1
    assert np.all(cover == 1)


def _cell_worker(rank, world, port, path, C, N, out_shape):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    w = synth.CONFIGS["cfg3"].with_(n=N, channels=C, nx=13, ny=11, field_lon=0.3, field_lat=0.3)
    lon, lat = synth.coords(w)
    vals = synth.values(w, lon, lat).numpy()
    out = np.memmap(path, dtype=np.float64, mode="r+", shape=out_shape)

    def grid_fn(sm):
        o, _, _ = oracle.grid(lon.numpy(), lat.numpy(), vals, sm, w.fwhm_deg, w.support, nthreads=1)
        return o.reshape(C, sm["ny"], sm["nx"])

    grid_cell_sharded(grid_fn, w.map, world, rank, out)
    out.flush()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_cell_sharded_grid_equals_single_process(world):
    """NEXT-3: ranks own map-row blocks (sub-map plans), the assembled map equals the
    single-process map bit for bit (same cell centres, same per-cell sums)."""
    import oracle
    import synth
    C, N = 3, 3000
    w = synth.CONFIGS["cfg3"].with_(n=N, channels=C, nx=13, ny=11, field_lon=0.3, field_lat=0.3)
    shape = (C, w.ny, w.nx)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "out.bin")
        np.memmap(path, dtype=np.float64, mode="w+", shape=shape).flush()
        port = 31500 + (os.getpid() % 2000)
        mp.spawn(_cell_worker, args=(world, port, path, C, N, shape), nprocs=world, join=True)
        got = np.array(np.memmap(path, dtype=np.float64, mode="r", shape=shape))
    lon, lat = synth.coords(w)
    vals = synth.values(w, lon, lat).numpy()
    ref, _, _ = oracle.grid(lon.numpy(), lat.numpy(), vals, w.map, w.fwhm_deg, w.support)
    ref = ref.reshape(shape)
    np.testing.assert_array_equal(np.isnan(got), np.isnan(ref))
    np.testing.assert_array_equal(got[~np.isnan(ref)], ref[~np.isnan(ref)])


def test_row_shard_covers_rows_once():
    for ny in (1, 7, 300, 512):
        for world in (1, 2, 3, 8):
            rows = [r for k in range(world) for r in range(*row_shard(ny, world, k))]
            assert rows == list(range(ny))
    m = {"nx": 5, "ny": 9, "crval_lon": 30.0, "crval_lat": 41.0, "crpix_x": 3.0,
         "crpix_y": 5.0, "cdelt_lon": 0.1, "cdelt_lat": 0.1}
    s = sub_map(m, 4, 9)
    for jp in range(5):
        lat_sub = s["crval_lat"] + (jp + 1 - s["crpix_y"]) * s["cdelt_lat"]
        lat_full = m["crval_lat"] + (jp + 4 + 1 - m["crpix_y"]) * m["cdelt_lat"]
        assert lat_sub == lat_full


def _dist_worker(rank, world, port, path, C, N, out_shape):
    """paper_2207_04584_b200.distributed.grid_rank under a gloo process group, with the
    oracle as the per-rank gridder and a shared float32 memmap as the output."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    from paper_2207_04584_b200.distributed import grid_rank, open_shared_out
    w = synth.CONFIGS["cfg1"].with_(n=N, channels=C, nx=9, ny=8)
    lon, lat = synth.coords(w)
    vals = synth.values(w, lon, lat).numpy()
    if rank == 0:
        open_shared_out(path, out_shape, create=True).flush()
    dist.barrier()
    out = open_shared_out(path, out_shape, create=False)

    def gridder(v):
        o, _, _ = oracle.grid(lon.numpy(), lat.numpy(), v, w.map, w.fwhm_deg, w.support, nthreads=1)
        return o.reshape((v.shape[0],) + tuple(out_shape[1:])).astype(np.float32)

    grid_rank(gridder, vals, out, world, rank)
    out.flush()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_distributed_driver_assembles_shared_output(world):
    """The product driver's per-rank step (distributed.grid_rank + the shared output
    memmap): G ranks together write every channel exactly once, equal to one process."""
    import oracle
    import synth
    C, N = 9, 600
    w = synth.CONFIGS["cfg1"].with_(n=N, channels=C, nx=9, ny=8)
    shape = (C, w.ny, w.nx)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "out.f32")
        port = 33500 + (os.getpid() % 2000)
        mp.spawn(_dist_worker, args=(world, port, path, C, N, shape), nprocs=world, join=True)
        got = np.array(np.memmap(path, dtype=np.float32, mode="r", shape=shape))
    lon, lat = synth.coords(w)
    vals = synth.values(w, lon, lat).numpy()
    ref, _, _ = oracle.grid(lon.numpy(), lat.numpy(), vals, w.map, w.fwhm_deg, w.support)
    ref = ref.reshape(shape).astype(np.float32)
    np.testing.assert_array_equal(np.isnan(got), np.isnan(ref))
    np.testing.assert_array_equal(got[~np.isnan(ref)], ref[~np.isnan(ref)])
