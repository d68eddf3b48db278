"""Minimal driver for ncu: build the plan, generate plan-layout values, run the device
grid `--launches` times (ncu selects the accumulate launch with -k/-s/-c)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from bench import plan_layout_values  # noqa: E402
from paper_2207_04584_b200 import Plan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg4")
ap.add_argument("--channels", type=int, default=0)
ap.add_argument("--launches", type=int, default=2)
ap.add_argument("--engine", default="tc")
a = ap.parse_args()
w = synth.CONFIGS[a.workload]
C = a.channels or w.channels
lon, lat = synth.coords(w, device="cuda")
p = Plan(lon, lat, w.map, w.fwhm_deg, w.support, engine=a.engine)
perm = torch.as_tensor(p.permutation(), device="cuda")
vp = plan_layout_values(w, lon, lat, perm, list(range(C)), "cuda")
out = torch.empty((C, w.ny, w.nx), device="cuda")
W = torch.empty((w.ny, w.nx), device="cuda")
for _ in range(a.launches):
    p.grid_plan_layout(vp, C, out, W)
torch.cuda.synchronize()
print("ok", p.info())
