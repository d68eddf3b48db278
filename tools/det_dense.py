import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import synth
from paper_2207_04584_b200 import Plan
from parity_util import make_inputs
w = synth.CONFIGS["cfg3"].with_(n=160_000, field_lon=0.4, field_lat=0.4, nx=24, ny=24, channels=7)
lon, lat, vals = make_inputs(w)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg, engine="tc") as p:
    d = vals.cuda()
    outs = []
    for r in range(reps):
        out, W = p.grid(d)
        torch.cuda.synchronize()
        outs.append(out.cpu().numpy().copy())
for r in range(1, reps):
    diff = np.abs(outs[r] - outs[0])
    print("rep", r, "max diff", np.nanmax(diff), "n diff", int((diff > 0).sum()), "cells", np.unique(np.argwhere(diff > 0)[:, 1:], axis=0)[:5].tolist())
