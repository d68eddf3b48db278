import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import synth, oracle
from paper_2207_04584_b200 import Plan
from parity_util import make_inputs, oracle_grid
w = synth.CONFIGS["cfg2"].with_(n=220 * 180, tracks=220, per_track=180, nx=70, ny=61, field_lon=1.2, field_lat=1.1, channels=133)
lon, lat, vals = make_inputs(w)
o, Wo, _ = oracle_grid(w, lon, lat, vals)
o = o.reshape(133, 61, 70); Wo = Wo.reshape(61, 70)
with Plan(lon.numpy(), lat.numpy(), w.map, w.fwhm_deg, engine="tc") as p:
    d = vals.cuda()
    outs = [p.grid(d)[0].cpu().numpy().copy() for _ in range(3)]
    os.environ["HEGRID_TC_PROMOTE"] = "1000000"
a, b = outs[0], outs[1]
diff = np.abs(a - b)
k = np.unravel_index(np.nanargmax(diff), diff.shape)
print("worst", k, "rep0", a[k], "rep1", b[k], "rep2", outs[2][k], "oracle", o[k], "W", Wo[k[1], k[2]])
# S = V*W: difference in S units
print("dS rep0-oracle", (a[k] - o[k]) * Wo[k[1], k[2]], "dS rep1-oracle", (b[k] - o[k]) * Wo[k[1], k[2]])
# pattern along channels at that cell
c = k[1], k[2]
print("errors along channels at cell (rep0):", ((a[:, c[0], c[1]] - o[:, c[0], c[1]]) * Wo[c])[:40:4])
print("errors along channels at cell (rep1):", ((b[:, c[0], c[1]] - o[:, c[0], c[1]]) * Wo[c])[:40:4])
print("values along channels:", (o[:, c[0], c[1]] * Wo[c])[:40:4])
