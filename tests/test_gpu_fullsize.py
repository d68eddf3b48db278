"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(device-resident plan-layout values, hegrid_grid_device), checked on sampled outputs the
oracle computes one by one: evenly spread cells (including map corners and edges) x a
spread of channels (first, last, ragged positions)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2207_04584_b200 import Plan
from parity_util import RTOL, engine_env, plan_layout_values

pytestmark = pytest.mark.gpu


def sample_cells(w, k=40, seed=0):
    rng = np.random.default_rng(seed)
    corners = [0, w.nx - 1, (w.ny - 1) * w.nx, w.cells - 1, (w.ny // 2) * w.nx + w.nx // 2]
    return np.unique(np.concatenate([corners, rng.choice(w.cells, k, replace=False)]))


def sample_channels(C, k=12):
    ch = sorted(set([0, C - 1, C // 2, 127 % C, 128 % C] +
                    np.linspace(0, C - 1, k).astype(int).tolist()))
    return np.array(ch, np.int64)


@pytest.mark.parametrize("engine", ["simt", "tc_otf", "tc_pw"])
@pytest.mark.parametrize("name,channels", [("cfg2", None), ("cfg3", None), ("cfg4", None),
                                           ("cfg5", 260)])
def test_fullsize_sampled_parity(name, channels, engine, monkeypatch):
    engine = engine_env(engine, monkeypatch)
    w = synth.CONFIGS[name]
    C = w.channels if channels is None else channels
    lon, lat = synth.coords(w, device="cuda")
    with Plan(lon, lat, w.map, w.fwhm_deg, engine=engine) as p:
        perm = torch.as_tensor(p.permutation(), device="cuda")
        vp = plan_layout_values(w, lon, lat, perm, list(range(C)))
        out = torch.empty((C, w.ny, w.nx), device="cuda")
        W = torch.empty((w.ny, w.nx), device="cuda")
        p.grid_plan_layout(vp, C, out, W)
        torch.cuda.synchronize()
        del vp
        info = p.info()
    cells = sample_cells(w)
    chans = sample_channels(C)
    vals = synth.values(w, lon, lat, channels=torch.as_tensor(chans, device="cuda")).cpu().numpy()
    o, Wo, cnt = oracle.grid(lon.cpu().numpy(), lat.cpu().numpy(), vals, w.map, w.fwhm_deg,
                             w.support, cells=cells)
    g = out.reshape(C, -1)[torch.as_tensor(chans, device="cuda")][:, torch.as_tensor(cells, device="cuda")]
    g = g.cpu().double().numpy()
    gw = W.reshape(-1)[torch.as_tensor(cells, device="cuda")].cpu().double().numpy()
    cov = Wo > 0
    assert np.array_equal(gw > 0, cov)
    assert np.all(np.isnan(g[:, ~cov]))
    assert np.max(np.abs(gw[cov] - Wo[cov]) / Wo[cov]) <= RTOL
    assert np.max(np.abs(g[:, cov] - o[:, cov]) / np.abs(o[:, cov])) <= RTOL
    # whole-map sanity: no NaN on covered cells, W > 0 exactly where neighbours exist
    Wall = W.reshape(-1).cpu().numpy()
    assert info["n_pairs"] > 0 and (Wall > 0).sum() >= cov.sum()


def test_fullsize_zero_mean_scale_aware():
    """cfg4 at full size in the bench's launch configuration with signed, zero-mean values
    (the synthetic sky minus its 10 K baseline): the scale-aware rule of SURVEY.md 8(c) #11,
    |V - V_ora| <= 1e-5 sum_n w |v_n| / W, on sampled cells x channels (the plain relative
    rule is undefined where V ~ 0)."""
    from parity_util import compare_scaled
    w = synth.CONFIGS["cfg4"]
    C = w.channels
    lon, lat = synth.coords(w, device="cuda")
    with Plan(lon, lat, w.map, w.fwhm_deg, engine="tc") as p:
        perm = torch.as_tensor(p.permutation(), device="cuda")
        vp = plan_layout_values(w, lon, lat, perm, list(range(C)))
        vp -= 10.0
        out = torch.empty((C, w.ny, w.nx), device="cuda")
        W = torch.empty((w.ny, w.nx), device="cuda")
        p.grid_plan_layout(vp, C, out, W)
        torch.cuda.synchronize()
        del vp
    cells = sample_cells(w, k=60, seed=4)
    chans = sample_channels(C, k=16)
    vals = (synth.values(w, lon, lat, channels=torch.as_tensor(chans, device="cuda")) - 10.0).cpu().numpy()
    g = out.reshape(C, -1)[torch.as_tensor(chans, device="cuda")][:, torch.as_tensor(cells, device="cuda")]
    gw = W.reshape(-1)[torch.as_tensor(cells, device="cuda")]
    st = compare_scaled(g.cpu().numpy(), gw.cpu().numpy(), lon.cpu().numpy(), lat.cpu().numpy(), vals,
                        w.map, w.fwhm_deg, w.support, cells=cells)
    assert st["covered"] > 0
