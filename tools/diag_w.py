"""Which pair makes W (k_tc_wsum) exceed the oracle's count on a cfg3 cell?"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2207_04584_b200 import Plan  # noqa: E402

w = synth.CONFIGS["cfg3"]
lon, lat = synth.coords(w)
lon, lat = lon.numpy(), lat.numpy()
d2r = math.pi / 180
R = 3 * (oracle.sigma_deg(w.fwhm_deg) * d2r)


def rel(cell, s):
    i, j = cell % w.nx, cell // w.nx
    lc, bc = oracle.cell_centre(w.map, i, j)
    dl = (lon[s] - lc + 180) % 360 - 180
    h = np.sin(0.5 * (lat[s] - bc) * d2r) ** 2 + np.cos(bc * d2r) * np.cos(lat[s] * d2r) * np.sin(0.5 * dl * d2r) ** 2
    return (2 * np.arcsin(np.sqrt(h))) ** 2 / R ** 2 - 1


for eng in ("tc", "simt"):
    with Plan(lon, lat, w.map, w.fwhm_deg, engine=eng, kernel="tophat") as p:
        vals = torch.ones((1, w.n), device="cuda")
        out, W = p.grid(vals)
        Wh = W.reshape(-1).cpu().numpy()
        for cell in (347, 9935):
            off, idx = p.neighbours(cell, cell + 1)
            ooff, oidx = oracle.neighbours(lon, lat, w.map, w.fwhm_deg, cells=np.array([cell]))
            extra = np.setdiff1d(idx, oidx)
            miss = np.setdiff1d(oidx, idx)
            print(eng, cell, "W", Wh[cell], "nbrs", len(idx), "oracle", len(oidx), "extra", extra,
                  rel(cell, extra), "missing", miss, rel(cell, miss), flush=True)
