"""GPU parity: the CUDA path through the C-ABI vs the fp64 oracle, element by element.

Sizes are chosen so the oracle finishes in seconds while the GPU path still spans many
CTA tiles, several channel blocks and ragged tails (map sizes not multiples of 8,
channel counts not multiples of 128).  Full BASELINE sizes are covered by sampled
checks in test_gpu_fullsize.py.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2207_04584_b200 import Plan, _binding as b
from parity_util import compare, engine_env, make_inputs, oracle_grid, plan_layout_values, small_workload

pytestmark = pytest.mark.gpu

ENGINES = ["simt", "tc", "tc_pw", "tc_pw_walk"]


# ------------------------------------------------------------------ plan layer
def test_radix_sort_spec_example():
    """pixel_idx [7,2,7,0,2] -> perm [3,1,4,0,2] (stable)."""
    assert b.hegrid_sort_u32(np.array([7, 2, 7, 0, 2], np.uint32)).tolist() == [3, 1, 4, 0, 2]


@pytest.mark.parametrize("n,hi", [(1, 5), (2, 1), (4095, 3), (4096, 1 << 17), (4097, 7),
                                  (1_000_003, 1 << 17), (300_000, 1 << 32 - 1)])
def test_radix_sort_matches_numpy_stable(n, hi):
    rng = np.random.default_rng(n)
    keys = rng.integers(0, hi, n, dtype=np.uint64).astype(np.uint32)
    got = b.hegrid_sort_u32(keys)
    ref = np.argsort(keys, kind="stable")
    np.testing.assert_array_equal(got, ref)


def test_radix_sort_degenerate():
    assert b.hegrid_sort_u32(np.zeros(0, np.uint32)).shape == (0,)
    keys = np.full(10_000, 42, np.uint32)
    np.testing.assert_array_equal(b.hegrid_sort_u32(keys), np.arange(10_000))
    keys = np.arange(10_000, dtype=np.uint32)[::-1].copy()
    np.testing.assert_array_equal(b.hegrid_sort_u32(keys), np.arange(10_000)[::-1])


def _cfg1():
    w = synth.CONFIGS["cfg1"]
    lon, lat, vals = make_inputs(w)
    return w, lon.numpy(), lat.numpy(), vals.numpy()


def test_neighbour_sets_exact_cfg1():
    """Algorithm 1's set {n : d <= R}, computed through the plan's candidate ranges and
    the fp32 + guard-band predicate, equals the fp64 oracle's set exactly (so the
    candidate lookup misses nothing)."""
    w, lon, lat, _ = _cfg1()
    with Plan(lon, lat, w.map, w.fwhm_deg) as p:
        off, idx = p.neighbours()
        info = p.info()
    ooff, oidx = oracle.neighbours(lon, lat, w.map, w.fwhm_deg)
    np.testing.assert_array_equal(off, ooff)
    np.testing.assert_array_equal(idx, oidx)
    assert info["n_pairs"] == ooff[-1]
    assert info["n_candidate_pairs"] >= info["n_pairs"]
    assert info["n_used"] <= w.n


def test_plan_permutation_is_stable_bin_order_cfg2_small():
    w = small_workload("cfg2", n=200 * 150, tracks=200, per_track=150)
    lon, lat = synth.coords(w)
    with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg) as p:
        perm = p.permutation()
        info = p.info()
    assert len(set(perm.tolist())) == perm.shape[0] == info["n_used"]
    # recompute each used sample's bin independently (nearest cell in the map frame)
    m = w.map
    x = (lon.numpy() - m["crval_lon"]) / m["cdelt_lon"] + m["crpix_x"] - 1
    y = (lat.numpy() - m["crval_lat"]) / m["cdelt_lat"] + m["crpix_y"] - 1
    key = (np.floor(y + 0.5) + info["mlat"]) * info["ncol"] + np.floor(x + 0.5) + info["mlon"]
    k = key[perm]
    assert np.all(np.diff(k) >= 0), "plan order is not bin order"
    same = np.diff(k) == 0
    assert np.all(np.diff(perm)[same] > 0), "ties not in original order (unstable)"


# ------------------------------------------------------------------ Eq. 1 parity
@pytest.mark.parametrize("engine", ENGINES)
def test_grid_cfg1_full_parity(engine, monkeypatch):
    engine = engine_env(engine, monkeypatch)
    """BASELINE configs[0] in full: 5000 samples, 64x64, 1 channel."""
    w, lon, lat, vals = _cfg1()
    with Plan(lon, lat, w.map, w.fwhm_deg, engine=engine) as p:
        out, W = p.grid(vals)
    o, Wo, _ = oracle_grid(w, lon, lat, vals)
    st = compare(out.reshape(1, -1), W.reshape(-1), o, Wo)
    assert st["covered"] == w.cells


@pytest.mark.parametrize("engine", ENGINES)
def test_grid_drift_scan_many_channels_ragged(engine, monkeypatch):
    engine = engine_env(engine, monkeypatch)
    """cfg2-shaped drift scan at oracle-friendly size: 70x61 map (ragged tiles), 133
    channels (two 128-channel blocks, ragged tail)."""
    w = small_workload("cfg2", n=220 * 180, tracks=220, per_track=180, nx=70, ny=61,
                       field_lon=1.2, field_lat=1.1, channels=133)
    lon, lat, vals = make_inputs(w)
    with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg, engine=engine) as p:
        out, W = p.grid(vals.numpy())
    o, Wo, _ = oracle_grid(w, lon, lat, vals)
    compare(out.reshape(133, -1), W.reshape(-1), o, Wo)


@pytest.mark.parametrize("engine", ENGINES)
def test_grid_high_density_cfg3_shape(engine, monkeypatch):
    engine = engine_env(engine, monkeypatch)
    """cfg3's density (1e6 samples/deg^2) and kernel (FWHM 6.925', ~84k neighbours per
    cell) on a 0.4 deg field, 24x24 map, 7 channels."""
    w = small_workload("cfg3", n=160_000, field_lon=0.4, field_lat=0.4, nx=24, ny=24,
                       channels=7)
    lon, lat, vals = make_inputs(w)
    with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg, engine=engine) as p:
        out, W = p.grid(vals.numpy())
        info = p.info()
    assert info["nbr_max"] > 20_000
    o, Wo, _ = oracle_grid(w, lon, lat, vals)
    compare(out.reshape(7, -1), W.reshape(-1), o, Wo)


@pytest.mark.parametrize("engine", ENGINES)
def test_device_paths_bit_identical_and_deterministic(engine, monkeypatch):
    engine = engine_env(engine, monkeypatch)
    """Host path, device USER_CN path and device PLAN_NC path give bit-identical maps;
    repeated runs are bit-identical (no atomics, fixed summation order)."""
    w = small_workload("cfg2", n=120 * 100, tracks=120, per_track=100, nx=40, ny=37,
                       field_lon=0.7, field_lat=0.6, channels=300)
    lon, lat, vals = make_inputs(w)
    with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg, n_streams=3, channel_block=64,
              engine=engine) as p:
        out_h, W_h = p.grid(vals.numpy())
        out_h2, _ = p.grid(vals.numpy())
        d = vals.cuda()
        out_d, W_d = p.grid(d)
        perm = p.permutation()
        vp = plan_layout_values(w, lon, lat, perm, list(range(300)))
        out_p = torch.empty_like(out_d)
        W_p = torch.empty_like(W_d)
        p.grid_plan_layout(vp, 300, out_p, W_p)
        torch.cuda.synchronize()
    with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg, n_streams=1, channel_block=300,
              engine=engine) as p2:
        out_h3, _ = p2.grid(vals.numpy())
    np.testing.assert_array_equal(out_h, out_h2)
    np.testing.assert_array_equal(out_h, out_d.cpu().numpy())
    np.testing.assert_array_equal(out_h, out_p.cpu().numpy())
    np.testing.assert_array_equal(out_h, out_h3)
    np.testing.assert_array_equal(W_h, W_d.cpu().numpy())
    np.testing.assert_array_equal(W_h, W_p.cpu().numpy())


def test_permute_kernel_exact():
    w = small_workload("cfg2", n=90 * 70, tracks=90, per_track=70, nx=30, ny=30,
                       field_lon=0.6, field_lat=0.6, channels=37)
    lon, lat, vals = make_inputs(w)
    with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg) as p:
        perm = torch.as_tensor(p.permutation())
        d = vals.cuda()
        vp = torch.full((perm.shape[0], 40), -1.0, device="cuda")
        p.permute(d, vp)
        torch.cuda.synchronize()
    ref = vals[:, perm].t()
    assert torch.equal(vp[:, :37].cpu(), ref)


# ------------------------------------------------------------------ edge cases
def _one_channel(lon, lat, v, m, fwhm, engine="simt"):
    with Plan(np.asarray(lon, np.float64), np.asarray(lat, np.float64), m, fwhm,
              engine=engine) as p:
        out, W = p.grid(np.asarray(v, np.float32)[None])
    o, Wo, _ = oracle.grid(np.asarray(lon), np.asarray(lat), np.asarray(v, np.float32)[None],
                           m, fwhm)
    return out.reshape(1, -1), W.reshape(-1), o, Wo


def mk_map(nx, ny, lon0, lat0, dl, dlat=None):
    return dict(nx=nx, ny=ny, crval_lon=lon0, crval_lat=lat0, crpix_x=(nx + 1) / 2,
                crpix_y=(ny + 1) / 2, cdelt_lon=dl, cdelt_lat=dl if dlat is None else dlat)


@pytest.mark.parametrize("engine", ENGINES)
def test_empty_input_all_blank(engine, monkeypatch):
    engine = engine_env(engine, monkeypatch)
    m = mk_map(9, 7, 30, 41, 1 / 60)
    with Plan(np.zeros(0), np.zeros(0), m, 0.05, engine=engine) as p:
        out, W = p.grid(np.zeros((3, 0), np.float32))
    assert np.all(np.isnan(out)) and np.all(W == 0)


@pytest.mark.parametrize("engine", ENGINES)
def test_zero_channels_writes_weight_map(engine, monkeypatch):
    engine = engine_env(engine, monkeypatch)
    rng = np.random.default_rng(0)
    lon = 30 + rng.uniform(-0.1, 0.1, 500)
    lat = 41 + rng.uniform(-0.1, 0.1, 500)
    m = mk_map(11, 13, 30, 41, 1 / 60)
    with Plan(lon, lat, m, 0.05, engine=engine) as p:
        out, W = p.grid(np.zeros((0, 500), np.float32))
    _, Wo, _ = oracle.grid(lon, lat, None, m, 0.05)
    np.testing.assert_allclose(W.reshape(-1), Wo, rtol=1e-5)


@pytest.mark.parametrize("engine", ENGINES)
def test_sample_at_cell_centre_weight_one_and_outside_samples_dropped(engine, monkeypatch):
    engine = engine_env(engine, monkeypatch)
    m = mk_map(16, 16, 30, 41, 1 / 60)
    lon_c, lat_c = oracle.cell_centre(m, 5, 9)
    lon = np.array([lon_c, 31.5, 28.0, lon_c])
    lat = np.array([lat_c, 41.0, 45.0, lat_c + 0.9 / 60])
    out, W, o, Wo = _one_channel(lon, lat, [5.0, 1.0, 2.0, 7.0], m, 0.05, engine)
    compare(out, W, o, Wo)
    with Plan(lon, lat, m, 0.05) as p:
        assert p.info()["n_used"] == 2


@pytest.mark.parametrize("engine", ENGINES)
def test_negative_cdelt_and_lon_zero_straddle(engine, monkeypatch):
    engine = engine_env(engine, monkeypatch)
    rng = np.random.default_rng(4)
    lon = (rng.uniform(-0.25, 0.25, 6000) + 360.0) % 360.0
    lat = rng.uniform(-0.2, 0.2, 6000)
    m = mk_map(29, 23, 0.0, 0.0, -1 / 60, 1 / 60)
    v = 10 + rng.normal(0, 1, 6000)
    compare(*_one_channel(lon, lat, v, m, 0.05, engine))


def test_support_edge_guard_band():
    """Samples at d = R(1 +- 1e-7) from a cell on the equator: inside the fp32 guard band,
    decided by the fp64 recheck exactly like the oracle."""
    m = mk_map(1, 1, 10.0, 0.0, 1 / 60)
    R = 3 * 0.05 / (2 * math.sqrt(2 * math.log(2)))
    lon = np.array([10 + R * (1 - 1e-7), 10 - R * (1 + 1e-7), 10.0, 10.0])
    lat = np.array([0.0, 0.0, R * (1 - 1e-9), -R * (1 + 1e-9)])
    with Plan(lon, lat, m, 0.05) as p:
        off, idx = p.neighbours()
    ooff, oidx = oracle.neighbours(lon, lat, m, 0.05)
    assert idx.tolist() == oidx.tolist() == [0, 2]


def test_domain_and_unsupported_errors():
    m = mk_map(8, 8, 30, 41, 1 / 60)
    with pytest.raises(b.HegridError) as e:
        Plan(np.array([30.0, np.nan]), np.array([41.0, 41.0]), m, 0.05)
    assert e.value.code == 2
    with pytest.raises(b.HegridError) as e:
        Plan(np.array([30.0]), np.array([91.0]), m, 0.05)
    assert e.value.code == 2
    with pytest.raises(b.HegridError) as e:
        Plan(np.array([30.0]), np.array([41.0]), m, 1.0, index="bins")        # R = 1.27 deg > 1 deg
    assert e.value.code == 5
    with pytest.raises(b.HegridError) as e:
        Plan(np.array([30.0]), np.array([88.9]), mk_map(8, 8, 30, 88.9, 1 / 60), 0.05, index="bins")
    assert e.value.code == 5
    # AUTO serves both with the HEALPix index
    for mm, fw in ((m, 1.0), (mk_map(8, 8, 30, 88.9, 1 / 60), 0.05)):
        with Plan(np.array([30.0]), np.array([41.0 if fw == 1.0 else 88.9]), mm, fw) as p:
            assert p.info()["index"] == 2
    # domain errors are domain errors for the HEALPix index too
    with pytest.raises(b.HegridError) as e:
        Plan(np.array([30.0]), np.array([91.0]), m, 0.05, index="healpix")
    assert e.value.code == 2
    opts = b.make_opts(index=7)
    with pytest.raises(b.HegridError) as e:
        b.hegrid_plan_create(np.array([30.0]), np.array([41.0]), m, 0.05, 3.0, opts)
    assert e.value.code == 1


def test_device_coordinate_plan_matches_host_plan():
    w = small_workload("cfg2", n=80 * 60, tracks=80, per_track=60, nx=24, ny=20,
                       field_lon=0.4, field_lat=0.35, channels=5)
    lon, lat, vals = make_inputs(w)
    with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg) as p1, \
            Plan(lon.cuda(), lat.cuda(), w.map, w.fwhm_deg) as p2:
        np.testing.assert_array_equal(p1.permutation(), p2.permutation())
        a, _ = p1.grid(vals.numpy())
        bb, _ = p2.grid(vals.numpy())
    np.testing.assert_array_equal(a, bb)


def test_launches_are_counted():
    before = b.hegrid_launch_count()
    w, lon, lat, vals = _cfg1()
    with Plan(lon, lat, w.map, w.fwhm_deg) as p:
        p.grid(vals)
    assert b.hegrid_launch_count() > before


def test_tc_pw_cta_order_invariant(monkeypatch):
    """The precomputed-weight engine's result does not depend on the CTA walk (channel-block
    groups, super-tiles): every (tile, channel block) is computed the same way wherever it
    runs, so the maps are bit-identical."""
    w = small_workload("cfg2", n=160 * 120, tracks=160, per_track=120, nx=45, ny=41,
                       field_lon=0.8, field_lat=0.75, channels=700)
    lon, lat, vals = make_inputs(w)
    monkeypatch.setenv("HEGRID_TC_PW", "1")
    outs = []
    for group, sup in (("1", "1"), ("3", "2"), ("6", "4")):
        monkeypatch.setenv("HEGRID_TC_GROUP", group)
        monkeypatch.setenv("HEGRID_TC_SUPER", sup)
        with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg, engine="tc") as p:
            d = vals.cuda()
            out, W = p.grid(d)
            outs.append((out.cpu().numpy(), W.cpu().numpy()))
    for o, W in outs[1:]:
        np.testing.assert_array_equal(o, outs[0][0])
        np.testing.assert_array_equal(W, outs[0][1])
    o, Wo, _ = oracle_grid(w, lon, lat, vals)
    compare(outs[0][0].reshape(700, -1), outs[0][1].reshape(-1), o, Wo)


def test_tc_pw_and_otf_bit_identical(monkeypatch):
    """The precomputed weight image holds exactly the weights the on-the-fly producers
    compute, and both modes accumulate each block in the same chunk order: the maps are
    bit-identical whichever mode a launch takes (the host path mixes them when its last
    channel block is small)."""
    w = small_workload("cfg2", n=150 * 110, tracks=150, per_track=110, nx=38, ny=35,
                       field_lon=0.7, field_lat=0.65, channels=530)
    lon, lat, vals = make_inputs(w)
    res = []
    for pw in ("0", "1"):
        monkeypatch.setenv("HEGRID_TC_PW", pw)
        with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg, engine="tc") as p:
            out, W = p.grid(vals.cuda())
            res.append((out.cpu().numpy(), W.cpu().numpy()))
    np.testing.assert_array_equal(res[0][0], res[1][0])
    np.testing.assert_array_equal(res[0][1], res[1][1])
    # host path: 512-channel blocks (precomputed weights) plus an 18-channel tail block
    monkeypatch.delenv("HEGRID_TC_PW")
    with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg, engine="tc", channel_block=512) as p:
        out_h, W_h = p.grid(vals.numpy())
    np.testing.assert_array_equal(np.asarray(out_h).reshape(res[0][0].shape), res[0][0])


@pytest.mark.parametrize("engine", ["simt", "tc_otf", "tc_pw"])
def test_tophat_kernel_parity(engine, monkeypatch):
    """SPEC.md:117-126 tophat kernel through the C-ABI (hegrid_kernel.kind = TOPHAT): W is
    the exact neighbour count, the map the neighbour mean, against the oracle."""
    engine = engine_env(engine, monkeypatch)
    w = small_workload("cfg2", n=120 * 100, tracks=120, per_track=100, nx=40, ny=37,
                       field_lon=0.7, field_lat=0.6, channels=520)
    lon, lat, vals = make_inputs(w)
    with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg, engine=engine, kernel="tophat") as p:
        out, W = p.grid(vals.cuda())
        out, W = out.cpu().numpy(), W.cpu().numpy()
    o, Wo, cnt = oracle.grid(lon.numpy(), lat.numpy(), vals.numpy(), w.map, w.fwhm_deg,
                             w.support, kernel="tophat")
    np.testing.assert_array_equal(W.reshape(-1).astype(np.int64), cnt)
    compare(out.reshape(520, -1), W.reshape(-1), o, Wo)


@pytest.mark.parametrize("engine", ["simt", "tc"])
def test_cell_sharded_plans_assemble_to_full_map(engine, monkeypatch):
    """NEXT-3 cell sharding on the GPU path: three map-row blocks, each gridded by its own
    sub-map plan (as three ranks would), assemble to the full map within the parity rule."""
    from paper_2207_04584_b200.shard import row_shard, sub_map
    engine = engine_env(engine, monkeypatch)
    w = small_workload("cfg3", n=60_000, field_lon=0.3, field_lat=0.3, nx=20, ny=19, channels=5)
    lon, lat, vals = make_inputs(w)
    out = np.empty((5, w.ny, w.nx), np.float32)
    W = np.empty((w.ny, w.nx), np.float32)
    for r in range(3):
        j0, j1 = row_shard(w.ny, 3, r)
        sm = sub_map(w.map, j0, j1)
        with Plan(lon.numpy(), lat.numpy(), sm, w.fwhm_deg, engine=engine) as p:
            o, ww = p.grid(vals.numpy())
        out[:, j0:j1] = np.asarray(o).reshape(5, j1 - j0, w.nx)
        W[j0:j1] = np.asarray(ww).reshape(j1 - j0, w.nx)
    o, Wo, _ = oracle_grid(w, lon, lat, vals)
    compare(out.reshape(5, -1), W.reshape(-1), o, Wo)


@pytest.mark.parametrize("engine", ["simt", "tc_otf", "tc_pw"])
def test_nonfinite_values_propagate_within_support(engine, monkeypatch):
    """NaN / +-Inf sample values (reading R15, nonfinite.cuh): Eq. 1's sum makes exactly the
    cells within R of such a sample NaN / +-Inf, as in the fp64 oracle; every other cell keeps
    the parity rule (no 0 * NaN leak through a block's zero weights).  Channel 7 is NaN at
    every sample, which overflows the per-launch record buffer and takes the scan path."""
    engine = engine_env(engine, monkeypatch)
    w = small_workload("cfg2", n=220 * 180, tracks=220, per_track=180, nx=70, ny=61,
                       field_lon=1.2, field_lat=1.1, channels=133)
    lon, lat, vals = make_inputs(w)
    v = vals.numpy().copy()
    rng = np.random.default_rng(5)
    pick = rng.choice(w.n, 40, replace=False)
    v[0, pick[:3]] = np.nan
    v[5, pick[3:8]] = np.inf
    v[5, pick[8:13]] = -np.inf
    v[130, pick[13:40]] = np.nan
    v[131, pick[3]] = np.inf                  # channel in the second 128-channel block
    v[7, :] = np.nan
    with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg, engine=engine) as p:
        out, W = p.grid(v)
    out = np.asarray(out, np.float64).reshape(133, -1)
    o, Wo, _ = oracle.grid(lon.numpy(), lat.numpy(), v, w.map, w.fwhm_deg, w.support)
    cov = Wo > 0
    fin = np.isfinite(o)
    assert (~fin[:, cov]).sum() > 100
    # non-finite cells: identical class (NaN, +Inf, -Inf)
    np.testing.assert_array_equal(np.isnan(out), np.isnan(o))
    np.testing.assert_array_equal(np.isposinf(out), np.isposinf(o))
    np.testing.assert_array_equal(np.isneginf(out), np.isneginf(o))
    ok = fin & cov[None, :]
    assert np.max(np.abs(out[ok] - o[ok]) / np.abs(o[ok])) <= 1e-5
    np.testing.assert_allclose(np.asarray(W).reshape(-1), Wo, rtol=1e-5)


def test_weight_image_cap_and_opt_out():
    """hegrid_opts.weight_image_max_bytes: < 0 never builds the precomputed weight image, a
    cap below its size leaves it unbuilt (weights computed per launch), the default builds
    it; the maps are bit-identical either way (same weights, same accumulation order)."""
    w = small_workload("cfg2", n=150 * 110, tracks=150, per_track=110, nx=38, ny=35,
                       field_lon=0.7, field_lat=0.65, channels=260)
    lon, lat, vals = make_inputs(w)
    d = vals.cuda()
    res = {}
    for cap in (0, -1, 1024):
        with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg, engine="tc",
                  weight_image_max_bytes=cap) as p:
            out, W = p.grid(d)
            res[cap] = (out.cpu().numpy(), W.cpu().numpy(), p.info()["weight_image_bytes"])
    assert res[0][2] > 0 and res[-1][2] == 0 and res[1024][2] == 0
    for cap in (-1, 1024):
        np.testing.assert_array_equal(res[cap][0], res[0][0])
        np.testing.assert_array_equal(res[cap][1], res[0][1])


def test_user_layout_calls_on_two_streams_concurrently():
    """USER_CN device calls on two streams of one plan: each takes its own scratch from the
    plan's stream-ordered pool, so neither corrupts the other."""
    w = small_workload("cfg2", n=120 * 100, tracks=120, per_track=100, nx=40, ny=37,
                       field_lon=0.7, field_lat=0.6, channels=600)
    lon, lat, vals = make_inputs(w)
    a = vals.cuda()
    b = (vals * 2.0 + 1.0).cuda()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg) as p:
        ref_a, _ = p.grid(a)
        ref_b, _ = p.grid(b)
        torch.cuda.synchronize()
        for _ in range(3):
            oa, _ = p.grid(a, stream=s1)
            ob, _ = p.grid(b, stream=s2)
            torch.cuda.synchronize()
            assert torch.equal(oa, ref_a) and torch.equal(ob, ref_b)


def test_pipeline_trace_stages_are_ordered():
    """hegrid_pipeline_trace after a profiled host call: one row per channel block, stages in
    order (H2D, permute + accumulate, D2H) on the block's stream, blocks of one slot
    serialised, slots used round-robin."""
    w = small_workload("cfg2", n=120 * 100, tracks=120, per_track=100, nx=40, ny=37,
                       field_lon=0.7, field_lat=0.6, channels=700)
    lon, lat, vals = make_inputs(w)
    with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg, n_streams=3, channel_block=128) as p:
        p.profile(True)
        out, W = p.grid(vals.numpy())
        tr = p.pipeline_trace()
        p.profile(False)
    assert tr.shape == (6, 5)
    assert tr[:, 0].tolist() == [0, 1, 2, 0, 1, 2]
    assert np.all(np.diff(tr[:, 1:], axis=1) >= 0)
    for s in range(3):
        rows = tr[tr[:, 0] == s]
        assert np.all(rows[1:, 1] >= rows[:-1, 4])
    o, Wo, _ = oracle_grid(w, lon, lat, vals)
    compare(out.reshape(700, -1), W.reshape(-1), o, Wo)
