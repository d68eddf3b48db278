import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import synth, oracle
from paper_2207_04584_b200 import Plan
from parity_util import make_inputs, oracle_grid
w = synth.CONFIGS["cfg2"].with_(n=220 * 180, tracks=220, per_track=180, nx=70, ny=61, field_lon=1.2, field_lat=1.1, channels=133)
lon, lat, vals = make_inputs(w)
o, Wo, _ = oracle_grid(w, lon, lat, vals)
o = o.reshape(133, 61, 70)
with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg, engine="tc") as p:
    d = vals.cuda()
    outs = [p.grid(d)[0].cpu().numpy().copy() for _ in range(3)]
for k, out in enumerate(outs):
    err = (out - o) / np.abs(o)
    bad = np.abs(err) > 1e-5
    print("rep", k, "n bad", int(bad.sum()), "max", float(np.nanmax(np.abs(err))))
    if bad.any():
        ch, j, i = np.nonzero(bad)
        print("   channels", np.unique(ch)[:20].tolist(), "...", "rows", np.unique(j)[:30].tolist())
        print("   cols", np.unique(i)[:40].tolist())
        print("   tiles (i//16, j//16)", sorted(set(zip((i // 16).tolist(), (j // 16).tolist())))[:20])
        print("   blocks-in-tile ((i%16)//4, (j%16)//4)", sorted(set(zip(((i % 16) // 4).tolist(), ((j % 16) // 4).tolist())))[:20])
        print("   channel lanes mod 128", np.unique(ch % 128)[:40].tolist())
