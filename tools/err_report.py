"""Max relative errors (sampled cells x channels, vs the oracle) at full sizes, per engine."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2207_04584_b200 import Plan  # noqa: E402
from parity_util import plan_layout_values  # noqa: E402
from test_gpu_fullsize import sample_cells, sample_channels  # noqa: E402

for name in sys.argv[1:] or ["cfg2", "cfg3", "cfg4"]:
    w = synth.CONFIGS[name]
    C = min(w.channels, 520)
    lon, lat = synth.coords(w, device="cuda")
    for engine in ("tc",):
        with Plan(lon, lat, w.map, w.fwhm_deg, engine=engine) as p:
            perm = torch.as_tensor(p.permutation(), device="cuda")
            vp = plan_layout_values(w, lon, lat, perm, list(range(C)))
            out = torch.empty((C, w.ny, w.nx), device="cuda")
            W = torch.empty((w.ny, w.nx), device="cuda")
            p.grid_plan_layout(vp, C, out, W)
            torch.cuda.synchronize()
            del vp
        cells = sample_cells(w, k=200)
        chans = sample_channels(C, k=24)
        vals = synth.values(w, lon, lat, channels=torch.as_tensor(chans, device="cuda")).cpu().numpy()
        o, Wo, _ = oracle.grid(lon.cpu().numpy(), lat.cpu().numpy(), vals, w.map, w.fwhm_deg, w.support, cells=cells)
        g = out.reshape(C, -1)[torch.as_tensor(chans, device="cuda")][:, torch.as_tensor(cells, device="cuda")].cpu().double().numpy()
        gw = W.reshape(-1)[torch.as_tensor(cells, device="cuda")].cpu().double().numpy()
        cov = Wo > 0
        ev = np.abs(g[:, cov] - o[:, cov]) / np.abs(o[:, cov])
        ew = np.abs(gw[cov] - Wo[cov]) / Wo[cov]
        print(f"{name} {engine}: V max {ev.max():.3e} p99 {np.quantile(ev, 0.99):.3e} mean {ev.mean():.3e} | W max {ew.max():.3e}", flush=True)
