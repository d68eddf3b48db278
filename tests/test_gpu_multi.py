"""GPU checks of the channel-sharded multi-GPU driver on one GPU.

Channels are independent, so G ranks that each grid the slice
channel_shard(C, G, r) through the public host API must assemble the G = 1 map bit for bit.
Here the G "ranks" run one after the other in one process on cuda:0 (the driver's per-rank
step, distributed.grid_rank), which is exactly what each rank of a torchrun job executes.
The map has enough CTA tiles that no launch splits a tile's entry list (the split-tile mode
groups partial sums by launch shape), as at the bench's cfg4 at every G <= 8.
"""
import numpy as np
import pytest
import torch

import synth
from paper_2207_04584_b200 import Plan
from paper_2207_04584_b200.distributed import grid_rank

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def workload():
    w = synth.CONFIGS["cfg2"].with_(n=300 * 400, tracks=300, per_track=400, channels=300)
    dev = torch.device("cuda", 0)
    lon, lat = synth.coords(w, device=dev)
    vals = synth.values(w, lon, lat).cpu().contiguous()
    return w, lon.cpu().numpy(), lat.cpu().numpy(), vals


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sequential_ranks_bit_identical_to_one_rank(workload, world):
    w, lon, lat, vals = workload
    with Plan(lon, lat, w.map, w.fwhm_deg, w.support) as p:
        assert p.info()["n_used"] > 0
        ref, Wref = p.grid(vals)
        ref = np.array(ref)
        out = np.full((w.channels, w.ny, w.nx), -1.0, np.float32)

        def gridder(v):
            o, W = p.grid(np.ascontiguousarray(v))
            np.testing.assert_array_equal(W, Wref)
            return o

        for r in range(world):
            grid_rank(gridder, vals.numpy(), out, world, r)
    np.testing.assert_array_equal(np.isnan(out), np.isnan(ref))
    assert np.array_equal(out.view(np.uint32), ref.view(np.uint32))
