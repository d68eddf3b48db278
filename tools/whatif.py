"""Time the accumulate kernel under HEGRID_TC_DEBUG variants (profiling builds: load with
HEGRID_LIB=tmp_libs/lib_prof.so).  Usage: whatif.py --workload cfg4 --channels 1024 D1 D2 ..."""
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
ap.add_argument("--channels", type=int, default=1024)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("dbg", nargs="*", default=["0"])
a = ap.parse_args()
w = synth.CONFIGS[a.workload]
C = a.channels or w.channels
lon, lat = synth.coords(w, device="cuda")
p = Plan(lon, lat, w.map, w.fwhm_deg, w.support, engine="tc")
perm = torch.as_tensor(p.permutation(), device="cuda")
vp = plan_layout_values(w, lon, lat, perm, list(range(C)), "cuda")
out = torch.empty((C, w.ny, w.nx), device="cuda")
W = torch.empty((w.ny, w.nx), device="cuda")
p.grid_plan_layout(vp, C, out, W)
torch.cuda.synchronize()
for d in a.dbg:
    os.environ["HEGRID_TC_DEBUG"] = d
    p.grid_plan_layout(vp, C, out, W)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        p.grid_plan_layout(vp, C, out, W)
    e1.record()
    torch.cuda.synchronize()
    print(f"dbg={d:>8} ms/launch {e0.elapsed_time(e1) / a.reps:8.3f}", flush=True)
os.environ["HEGRID_TC_DEBUG"] = "0"
