"""Diagnose tophat all-ones exactness at full size: cells where V != 1, with S = V W."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2207_04584_b200 import Plan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
w = synth.CONFIGS[name]
C = min(w.channels, 128)
lon, lat = synth.coords(w, device="cuda")
for env in ({}, {"HEGRID_TC_SPLIT": "1"}, {"HEGRID_TC_PW": "0"}, {"HEGRID_TC_SPLIT": "1", "HEGRID_TC_PW": "0"}):
    for k in ("HEGRID_TC_SPLIT", "HEGRID_TC_PW"):
        os.environ.pop(k, None)
    os.environ.update(env)
    with Plan(lon, lat, w.map, w.fwhm_deg, engine="tc", kernel="tophat") as p:
        n_used = p.info()["n_used"]
        ones = torch.ones((n_used, C), dtype=torch.float32, device="cuda")
        out = torch.empty((C, w.ny, w.nx), device="cuda")
        W = torch.empty((w.ny, w.nx), device="cuda")
        p.grid_plan_layout(ones, C, out, W)
        torch.cuda.synchronize()
    Wh = W.reshape(-1).cpu().numpy().astype(np.float64)
    o = out.reshape(C, -1).cpu().numpy().astype(np.float64)
    cov = Wh > 0
    bad = np.nonzero(np.any(o[:, cov] != 1.0, axis=0))[0]
    cells = np.nonzero(cov)[0][bad]
    print(env, "bad cells", len(cells), "of", cov.sum(), flush=True)
    if len(cells):
        S = o[:, cells] * Wh[cells]
        print("  first cells", cells[:10], "W", Wh[cells[:10]])
        print("  S-W ch0", (S[0, :10] - Wh[cells[:10]]), "V ch0", o[0, cells[:10]])
        print("  channels bad per cell", np.sum(o[:, cells] != 1.0, axis=0)[:10])
        print("  max |V-1|", np.max(np.abs(o[:, cells] - 1.0)))
        sub = cells[:5]
        _, Wo, cnt = oracle.grid(lon.cpu().numpy(), lat.cpu().numpy(), None, w.map, w.fwhm_deg,
                                 w.support, cells=sub, kernel="tophat")
        print("  oracle count", cnt, "gpu W", Wh[sub])
