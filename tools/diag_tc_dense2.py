import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import synth, oracle
from paper_2207_04584_b200 import Plan
from parity_util import make_inputs, oracle_grid
w = synth.CONFIGS["cfg3"].with_(n=160_000, field_lon=0.4, field_lat=0.4, nx=24, ny=24, channels=7)
lon, lat, vals = make_inputs(w)
o, Wo, _ = oracle_grid(w, lon, lat, vals)
res = {}
for eng in ("simt", "tc", "tc"):
    with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg, engine=eng) as p:
        out, W = p.grid(vals.numpy())
    e = (out.reshape(7, -1) - o) / np.abs(o)
    ew = (W.reshape(-1) - Wo) / Wo
    print(eng, os.environ.get("HEGRID_TC_PROMOTE"), "V max", np.abs(e).max(), "mean", e.mean(), "W max", np.abs(ew).max(), "W mean", ew.mean())
    k = np.unravel_index(np.abs(e).argmax(), e.shape)
    print("   worst (ch, cell)", k, "err", e[k])
