"""NEXT-4 kernel/sample variants on the GPU against the fp64 oracle:
NaN/Inf masking (hegrid_opts.nonfinite = MASK, reading R24) and per-sample weights
(hegrid_plan_set_sample_weights, reading R25), for every engine and both indexes."""
import numpy as np
import pytest

import oracle
import synth
from paper_2207_04584_b200 import HegridError, Plan
from parity_util import RTOL, compare, engine_env, make_inputs, small_workload

pytestmark = pytest.mark.gpu
ENGINES = ["simt", "tc_otf", "tc_pw", "healpix"]


def _plan(lon, lat, w, engine, monkeypatch, **kw):
    if engine == "healpix":
        return Plan(lon, lat, w.map, w.fwhm_deg, index="healpix", **kw)
    return Plan(lon, lat, w.map, w.fwhm_deg, engine=engine_env(engine, monkeypatch), **kw)


def _workload():
    w = small_workload("cfg2", n=140 * 110, tracks=140, per_track=110, nx=37, ny=29,
                       field_lon=0.8, field_lat=0.6, channels=133)
    lon, lat, vals = make_inputs(w)
    return w, lon.numpy(), lat.numpy(), vals.numpy()


def _compare_nan_aware(out, W, o, Wo):
    out = np.asarray(out, np.float64).reshape(o.shape)
    W = np.asarray(W, np.float64).reshape(Wo.shape)
    assert np.array_equal(W > 0, Wo > 0)
    cov = Wo > 0
    assert np.max(np.abs(W[cov] - Wo[cov]) / Wo[cov]) <= RTOL
    assert np.array_equal(np.isnan(out), np.isnan(o)), "NaN patterns differ"
    ok = ~np.isnan(o)
    assert np.max(np.abs(out[ok] - o[ok]) / np.abs(o[ok])) <= RTOL
    return int((np.isnan(o) & cov[None, :]).sum())


@pytest.mark.parametrize("engine", ENGINES)
def test_nonfinite_mask_parity(engine, monkeypatch):
    w, lon, lat, vals = _workload()
    rng = np.random.default_rng(24)
    vals = vals.copy()
    n = lon.shape[0]
    vals[3, rng.choice(n, 300, replace=False)] = np.nan          # a flagged channel
    vals[70, rng.choice(n, 40, replace=False)] = np.inf
    vals[132, rng.choice(n, 25, replace=False)] = -np.inf
    vals[5, :] = np.nan                                          # a fully flagged channel
    with _plan(lon, lat, w, engine, monkeypatch, nonfinite="mask") as p:
        out, W = p.grid(vals)
    o, Wo, _ = oracle.grid(lon, lat, vals, w.map, w.fwhm_deg, w.support, mask=True)
    blank = _compare_nan_aware(out, W, o, Wo)
    assert blank > 0                              # the fully flagged channel is blank
    assert np.all(np.isnan(np.asarray(out).reshape(o.shape)[5]))
    # untouched channels are the propagate-mode values, bit for bit
    with _plan(lon, lat, w, engine, monkeypatch) as p:
        outp, _ = p.grid(vals)
    a = np.asarray(out).reshape(o.shape)[10]
    bb = np.asarray(outp).reshape(o.shape)[10]
    assert np.array_equal(a.view(np.uint32), bb.view(np.uint32))


@pytest.mark.parametrize("engine", ENGINES)
def test_sample_weights_parity(engine, monkeypatch):
    w, lon, lat, vals = _workload()
    rng = np.random.default_rng(25)
    om = rng.uniform(0.2, 3.0, lon.shape[0]).astype(np.float32)
    om[rng.choice(lon.shape[0], 500, replace=False)] = 0.0       # excluded samples
    with _plan(lon, lat, w, engine, monkeypatch) as p:
        out0, W0 = p.grid(vals)
        p.set_sample_weights(om)
        out, W = p.grid(vals)
        p.set_sample_weights(None)                               # back to omega = 1
        out1, W1 = p.grid(vals)
    o, Wo, _ = oracle.grid(lon, lat, vals, w.map, w.fwhm_deg, w.support,
                           sample_weights=om.astype(np.float64))
    compare(out, W, o, Wo)
    assert np.array_equal(np.asarray(out0).view(np.uint32), np.asarray(out1).view(np.uint32))
    assert np.array_equal(np.asarray(W0).view(np.uint32), np.asarray(W1).view(np.uint32))


def test_sample_weights_errors():
    w, lon, lat, vals = _workload()
    with Plan(lon, lat, w.map, w.fwhm_deg) as p:
        with pytest.raises(HegridError) as e:
            p.set_sample_weights(np.ones(lon.shape[0] - 1, np.float32))
        assert e.value.code == 1
        bad = np.ones(lon.shape[0], np.float32)
        bad[7] = -1.0
        with pytest.raises(HegridError) as e:
            p.set_sample_weights(bad)
        assert e.value.code == 2
        bad[7] = np.nan
        with pytest.raises(HegridError) as e:
            p.set_sample_weights(bad)
        assert e.value.code == 2


@pytest.mark.parametrize("proj", ["tan", "sin"])
@pytest.mark.parametrize("wide", [False, True])
def test_projected_maps(proj, wide):
    """Zenithal TAN / SIN maps (reading R26): cell centres from the projection, gridded through
    the HEALPix index (AUTO; the bin index refuses them), against the oracle's own projection
    code -- values, W, blank pattern and the exact neighbour sets."""
    rng = np.random.default_rng(26)
    if wide:      # a 40 x 40 degree field at high latitude, R = 1.7 deg
        n, cen, half, fw, cd, nx = 40000, (120.0, 62.0), 20.0, 1.33, 1.25, 33
    else:         # a 1.3 x 1 degree field, R = 3.8 arcmin
        n, cen, half, fw, cd, nx = 30000, (30.0, 41.0), 0.65, 0.05, 1 / 30, 41
    lat = cen[1] + (rng.random(n) - 0.5) * 2 * half
    lon = cen[0] + (rng.random(n) - 0.5) * 2 * half / np.cos(np.radians(cen[1]))
    m = {"nx": nx, "ny": nx - 8, "crval_lon": cen[0], "crval_lat": cen[1], "crpix_x": (nx + 1) / 2,
         "crpix_y": (nx - 7) / 2, "cdelt_lon": -cd, "cdelt_lat": cd, "projection": proj}
    vals = (10 + rng.standard_normal((3, n))).astype(np.float32)
    with pytest.raises(HegridError):
        Plan(lon, lat, m, fw, index="bins")
    with Plan(lon, lat, m, fw) as p:
        assert p.info()["index"] == 2
        out, W = p.grid(vals)
        off, idx = p.neighbours()
    o, Wo, _ = oracle.grid(lon, lat, vals, m, fw, 3.0)
    st = compare(out, W, o, Wo)
    assert st["covered"] > 0.5 * m["nx"] * m["ny"]
    ooff, oidx = oracle.neighbours(lon, lat, m, fw, 3.0)
    np.testing.assert_array_equal(off, ooff)
    np.testing.assert_array_equal(idx, oidx)
