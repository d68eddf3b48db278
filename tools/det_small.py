import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import synth
from paper_2207_04584_b200 import Plan
from parity_util import make_inputs
cfg = sys.argv[1]
if cfg == "dense":
    w = synth.CONFIGS["cfg3"].with_(n=160_000, field_lon=0.4, field_lat=0.4, nx=24, ny=24, channels=7)
else:
    w = synth.CONFIGS["cfg2"].with_(n=220 * 180, tracks=220, per_track=180, nx=70, ny=61, field_lon=1.2, field_lat=1.1, channels=133)
lon, lat, vals = make_inputs(w)
with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg, engine="tc") as p:
    d = vals.cuda()
    outs = [p.grid(d)[0].cpu().numpy().copy() for _ in range(3)]
print(cfg, os.environ.get("HEGRID_TC_DENSE"), os.environ.get("HEGRID_TC_PROMOTE"),
      [float(np.nanmax(np.abs(o - outs[0]))) for o in outs[1:]])
