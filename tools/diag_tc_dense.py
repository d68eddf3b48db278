"""Dense-regime (cfg3-shape) TC accuracy vs promotion interval (HEGRID_TC_PROMOTE)."""
import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import synth, oracle
from paper_2207_04584_b200 import Plan
from parity_util import make_inputs, oracle_grid
w = synth.CONFIGS["cfg3"].with_(n=160_000, field_lon=0.4, field_lat=0.4, nx=24, ny=24, channels=7)
lon, lat, vals = make_inputs(w)
o, Wo, _ = oracle_grid(w, lon, lat, vals)
for eng in ("simt", "tc"):
    with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg, engine=eng) as p:
        out, W = p.grid(vals.numpy())
    e = np.abs(out.reshape(7, -1) - o) / np.abs(o)
    print(eng, os.environ.get("HEGRID_TC_PROMOTE"), "max", e.max(), "mean", e.mean(), "W", np.max(np.abs(W.reshape(-1) - Wo) / Wo))
