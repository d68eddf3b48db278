"""Per-plan preparation cost of the TC engine: two plans in one process (the second one shows
the steady cost, without lazy module loading).  HEGRID_TC_TIMING=1 prints the phases."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from bench import plan_layout_values  # noqa: E402
from paper_2207_04584_b200 import Plan  # noqa: E402

w = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
C = 512
lon, lat = synth.coords(w, device="cuda")
for it in range(2):
    t0 = time.perf_counter()
    p = Plan(lon, lat, w.map, w.fwhm_deg, w.support, engine="tc")
    perm = torch.as_tensor(p.permutation(), device="cuda")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    vp = plan_layout_values(w, lon, lat, perm, list(range(C)), "cuda")
    out = torch.empty((C, w.ny, w.nx), device="cuda")
    W = torch.empty((w.ny, w.nx), device="cuda")
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    p.grid_plan_layout(vp, C, out, W)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    p.grid_plan_layout(vp, C, out, W)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"plan {it}: plan {1e3 * (t1 - t0):.1f} ms, first grid {1e3 * (t3 - t2):.1f} ms, "
          f"second grid {1e3 * (t4 - t3):.1f} ms", flush=True)
    p.close()
