"""A small gridding run through the C-ABI without torch (numpy inputs, host API), for
compute-sanitizer: python tools/sanitize_case.py <simt|tc_otf|tc_pw>."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2207_04584_b200 import Plan  # noqa: E402

mode = sys.argv[1]
engine = "simt" if mode == "simt" else "tc"
if mode == "tc_otf":
    os.environ["HEGRID_TC_PW"] = "0"
elif mode == "tc_pw":
    os.environ["HEGRID_TC_PW"] = "1"
rng = np.random.default_rng(2207)
for n, C, nx, ny, fw in ((5000, 1, 64, 64, 3 / 60), (3000, 133, 21, 19, 3 / 60), (20000, 7, 17, 13, 6.925 / 60)):
    lon = 30 + (rng.random(n) - 0.5) * (nx / 60 if fw < 0.1 else 0.3)
    lat = 41 + (rng.random(n) - 0.5) * (ny / 60 if fw < 0.1 else 0.25)
    m = {"nx": nx, "ny": ny, "crval_lon": 30.0, "crval_lat": 41.0, "crpix_x": (nx + 1) / 2,
         "crpix_y": (ny + 1) / 2, "cdelt_lon": 1 / 60 if fw < 0.1 else 0.3 / nx,
         "cdelt_lat": 1 / 60 if fw < 0.1 else 0.25 / ny}
    v = (10 + rng.standard_normal((C, n))).astype(np.float32)
    with Plan(lon, lat, m, fw, engine=engine) as p:
        out, W = p.grid(v)
    assert np.isfinite(out[:, W > 0]).all()
print("ok", mode)
