"""The hot path's pair set, checked exactly against the fp64 definition.

Algorithm 1 gathers, for every cell, the samples with d <= R
(line "if d(target_cell[], raw_data[i]) <= R"); north_star: "the neighbour index sets
must match bit-exactly".  Two independent views of the tensor-core engine's pairs:

* hegrid_neighbours enumerates the engine's own chunk schedule and weight expression
  (a pair counts iff its weight > 0), compared with oracle.neighbours;
* the tophat kernel with all-ones values makes every MMA product exactly 1 and every
  partial sum an exact integer, so V == 1.0f bit-exactly on every covered cell iff the
  accumulation (the schedule that feeds the MMAs) saw exactly the pairs W counted, and
  W == the oracle's neighbour count.

Plus the high-latitude domain: near a pole pairs within R have
half-longitude offsets of tens of degrees, where the fp32 series distance must keep its
higher-order terms (weight.cuh sin2_series).
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2207_04584_b200 import Plan, _binding as b
from parity_util import compare_scaled, engine_env

pytestmark = pytest.mark.gpu


def _ranges(w, k=3, width=100):
    """k cell ranges of `width` cells: the first row, the map centre, the last row."""
    cells = w.nx * w.ny
    starts = [0, (w.ny // 2) * w.nx + w.nx // 2 - width // 2, cells - width]
    return [(s, s + width) for s in starts[:k]]


@pytest.mark.parametrize("name", ["cfg3", "cfg4"])
def test_fullsize_neighbour_sets_exact(name):
    """~300 cells of the full cfg3 (4M samples, ~84k neighbours per cell) and cfg4 maps:
    the tensor-core engine's pairs equal the oracle's d <= R sets exactly."""
    w = synth.CONFIGS[name]
    lon, lat = synth.coords(w)
    lon, lat = lon.numpy(), lat.numpy()
    with Plan(lon, lat, w.map, w.fwhm_deg) as p:
        got = [p.neighbours(c0, c1) for c0, c1 in _ranges(w)]
    for (c0, c1), (off, idx) in zip(_ranges(w), got):
        ooff, oidx = oracle.neighbours(lon, lat, w.map, w.fwhm_deg, w.support,
                                       cells=np.arange(c0, c1))
        np.testing.assert_array_equal(off, ooff)
        np.testing.assert_array_equal(idx, oidx)
        assert ooff[-1] > 0


@pytest.mark.parametrize("engine", ["tc_pw", "tc_otf"])
@pytest.mark.parametrize("name", ["cfg3", "cfg4"])
def test_fullsize_tophat_all_ones_exact(name, engine, monkeypatch):
    """Tophat kernel, every value 1 (one 128-channel block, plan layout, the bench's launch
    configuration): S and W are exact integer sums, so V must be exactly 1.0f wherever
    W > 0 -- a pair dropped from the accumulation but counted in W (or vice versa) breaks
    it -- and W must equal the oracle's neighbour count on sampled cells."""
    engine = engine_env(engine, monkeypatch)
    w = synth.CONFIGS[name]
    C = min(w.channels, 128)
    lon, lat = synth.coords(w, device="cuda")
    with Plan(lon, lat, w.map, w.fwhm_deg, engine=engine, kernel="tophat") as p:
        n_used = p.info()["n_used"]
        ones = torch.ones((n_used, C), dtype=torch.float32, device="cuda")
        out = torch.empty((C, w.ny, w.nx), device="cuda")
        W = torch.empty((w.ny, w.nx), device="cuda")
        p.grid_plan_layout(ones, C, out, W)
        torch.cuda.synchronize()
    Wh = W.reshape(-1).cpu().numpy()
    cov = Wh > 0
    o = out.reshape(C, -1).cpu().numpy()
    assert cov.sum() > 0
    assert np.all(o[:, cov] == 1.0), "V != 1 on covered cells: accumulated pairs != counted pairs"
    assert np.all(np.isnan(o[:, ~cov]))
    assert np.all(Wh == np.round(Wh))
    rng = np.random.default_rng(7)
    cells = np.unique(np.concatenate([[0, w.nx - 1, w.cells - 1],
                                      rng.choice(w.cells, 60, replace=False)]))
    _, Wo, cnt = oracle.grid(lon.cpu().numpy(), lat.cpu().numpy(), None, w.map, w.fwhm_deg,
                             w.support, cells=cells, kernel="tophat")
    np.testing.assert_array_equal(Wh[cells].astype(np.int64), cnt)


def _polar_case(n=30_000, seed=11):
    """A 30 x 20 map of non-square cells (0.5 deg in lon x 0.05 deg in lat) at dec
    86.0-87.0, kernel support R = 0.9 deg (FWHM 0.7064 deg), samples uniform over the
    band dec 85.0-87.9 and +-42.5 deg of lon around the map: pairs within R reach
    half-longitude offsets of ~0.29 rad."""
    R = 0.9
    fwhm = R / 3.0 * 2.0 * math.sqrt(2.0 * math.log(2.0))
    m = dict(nx=30, ny=20, crval_lon=120.0, crval_lat=86.5, crpix_x=15.5, crpix_y=10.5,
             cdelt_lon=0.5, cdelt_lat=0.05)
    rng = np.random.default_rng(seed)
    lon = 120.0 + rng.uniform(-42.5, 42.5, n)
    lat = rng.uniform(85.0, 87.9, n)
    return m, fwhm, lon, lat


@pytest.mark.parametrize("engine", ["simt", "tc_otf", "tc_pw"])
def test_high_latitude_non_square_cells(engine, monkeypatch):
    """Zero-mean values (checked with the scale-aware rule) and the exact neighbour sets."""
    engine = engine_env(engine, monkeypatch)
    m, fwhm, lon, lat = _polar_case()
    rng = np.random.default_rng(3)
    vals = (rng.normal(0.0, 1.0, (5, lon.shape[0])) *
            (1.0 + 0.5 * np.cos(np.radians(lon - 120.0) * 8.0))).astype(np.float32)
    with Plan(lon, lat, m, fwhm, engine=engine) as p:
        out, W = p.grid(vals)
        off, idx = p.neighbours()
    st = compare_scaled(out, W, lon, lat, vals, m, fwhm)
    assert st["covered"] == m["nx"] * m["ny"]
    ooff, oidx = oracle.neighbours(lon, lat, m, fwhm)
    np.testing.assert_array_equal(off, ooff)
    np.testing.assert_array_equal(idx, oidx)


def test_high_latitude_limit_is_refused():
    """Closer to the pole the pairs' half-longitude offsets exceed 0.5 rad, the fp32 series
    distance's validated range: the lon/lat bin index refuses (EUNSUPPORTED) and AUTO builds
    the HEALPix-indexed plan instead."""
    R = 1.0
    fwhm = R / 3.0 * 2.0 * math.sqrt(2.0 * math.log(2.0))
    m = dict(nx=10, ny=10, crval_lon=0.0, crval_lat=87.7, crpix_x=5.5, crpix_y=5.5,
             cdelt_lon=0.5, cdelt_lat=0.02)
    with pytest.raises(b.HegridError) as e:
        Plan(np.array([0.0]), np.array([87.7]), m, fwhm, index="bins")
    assert e.value.code == 5
    with Plan(np.array([0.0]), np.array([87.7]), m, fwhm) as p:      # AUTO: the HEALPix index
        assert p.info()["index"] == 2
