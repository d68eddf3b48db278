"""Shared helpers of the parity tests: small workload builders and the comparison rule.

Parity rule (BASELINE.json north_star): on every cell with W_oracle > 0,
|V_gpu - V_ora| <= 1e-5 |V_ora| and |W_gpu - W_ora| <= 1e-5 W_ora; blank patterns
(W = 0 -> NaN) identical; neighbour sets identical.
"""
import numpy as np
import torch

import oracle
import synth

RTOL = 1e-5


def small_workload(name, **kw):
    return synth.CONFIGS[name].with_(**kw)


def make_inputs(w, channels=None, device="cpu"):
    lon, lat = synth.coords(w, device=device)
    vals = synth.values(w, lon, lat, channels=channels)
    return lon, lat, vals


def compare(out_gpu, w_gpu, out_ora, w_ora, rtol=RTOL):
    """Return a dict of error statistics; asserts the parity rule."""
    out_gpu = np.asarray(out_gpu, np.float64).reshape(out_ora.shape)
    w_gpu = np.asarray(w_gpu, np.float64).reshape(w_ora.shape)
    covered = w_ora > 0
    # blank pattern
    assert np.array_equal(w_gpu > 0, covered), "blank pattern differs"
    assert np.all(np.isnan(out_gpu[:, ~covered])), "blank cells must be NaN"
    assert not np.any(np.isnan(out_gpu[:, covered])), "covered cells must be finite"
    werr = np.abs(w_gpu[covered] - w_ora[covered]) / w_ora[covered]
    verr = np.abs(out_gpu[:, covered] - out_ora[:, covered]) / np.abs(out_ora[:, covered])
    stats = dict(max_rel_w=float(werr.max(initial=0)), max_rel_v=float(verr.max(initial=0)),
                 covered=int(covered.sum()))
    assert stats["max_rel_w"] <= rtol, stats
    assert stats["max_rel_v"] <= rtol, stats
    return stats


def oracle_grid(w, lon, lat, vals, channels=None, cells=None):
    return oracle.grid(np.asarray(lon), np.asarray(lat), np.asarray(vals), w.map, w.fwhm_deg,
                       w.support, channels=channels, cells=cells)


def plan_layout_values(w, lon, lat, perm, channels, ld=None, device="cuda"):
    """Values in the plan layout [n_used][ld], generated directly at the plan's sample
    order (synth regenerates any (channel, sample) subset exactly)."""
    C = len(channels)
    ld = ld or ((C + 3) // 4 * 4)
    perm_t = torch.as_tensor(perm, dtype=torch.int64, device=device)
    out = torch.zeros((perm_t.shape[0], ld), dtype=torch.float32, device=device)
    step = 256
    lon_d, lat_d = lon.to(device), lat.to(device)
    ch_all = torch.as_tensor(channels, dtype=torch.int64, device=device)
    for c0 in range(0, C, step):
        ch = ch_all[c0:c0 + step]
        blk = synth.values(w, lon_d, lat_d, channels=ch, samples=perm_t)  # [cb][n_used]
        out[:, c0:c0 + ch.shape[0]] = blk.t()
    return out


def engine_env(engine, monkeypatch):
    """Test engine names -> Plan engine.  "tc_pw" / "tc_otf" force the tensor-core engine's
    precomputed-weight image on / off (HEGRID_TC_PW); "tc" leaves the library's choice."""
    if engine in ("tc_pw", "tc_otf"):
        monkeypatch.setenv("HEGRID_TC_PW", "1" if engine == "tc_pw" else "0")
        return "tc"
    if engine == "tc_pw_walk":     # ragged channel-block groups, 3x3 super-tile walk
        monkeypatch.setenv("HEGRID_TC_PW", "1")
        monkeypatch.setenv("HEGRID_TC_GROUP", "2")
        monkeypatch.setenv("HEGRID_TC_SUPER", "3")
        monkeypatch.setenv("HEGRID_TC_SNAKE", "1")
        return "tc"
    return engine


def compare_scaled(out_gpu, w_gpu, lon, lat, vals, m, fwhm, support=3.0, rtol=RTOL, cells=None,
                   kernel="gaussian"):
    """Scale-aware parity for values of any sign: on covered cells,
    |V_gpu - V_ora| <= rtol * (sum_n w |v_n|) / W -- the error of a weighted mean whose terms
    each carry relative error rtol -- plus the W and blank-pattern rules of ``compare``.
    ``vals`` [C][N]; returns the statistics."""
    o, Wo, _ = oracle.grid(lon, lat, vals, m, fwhm, support, cells=cells, kernel=kernel)
    oa, _, _ = oracle.grid(lon, lat, np.abs(np.asarray(vals, np.float32)), m, fwhm, support,
                           cells=cells, kernel=kernel)
    out_gpu = np.asarray(out_gpu, np.float64).reshape(o.shape)
    w_gpu = np.asarray(w_gpu, np.float64).reshape(Wo.shape)
    cov = Wo > 0
    assert np.array_equal(w_gpu > 0, cov), "blank pattern differs"
    assert np.all(np.isnan(out_gpu[:, ~cov]))
    werr = np.abs(w_gpu[cov] - Wo[cov]) / Wo[cov]
    serr = np.abs(out_gpu[:, cov] - o[:, cov]) / oa[:, cov]
    st = dict(max_rel_w=float(werr.max(initial=0)), max_scaled_v=float(serr.max(initial=0)),
              covered=int(cov.sum()))
    assert st["max_rel_w"] <= rtol, st
    assert st["max_scaled_v"] <= rtol, st
    return st
