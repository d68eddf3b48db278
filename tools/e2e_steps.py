"""Time the bench's e2e step (Plan from host coords + hegrid_grid + close) phase by phase."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from bench import user_layout_values_pinned  # noqa: E402
from paper_2207_04584_b200 import Plan  # noqa: E402

w = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
dev = torch.device("cuda", 0)
lon, lat = synth.coords(w, device=dev)
C = w.channels
vals = user_layout_values_pinned(w, lon, lat, list(range(C)), dev)
out = torch.empty((C, w.ny, w.nx), dtype=torch.float32, pin_memory=True)
W = torch.empty((w.ny, w.nx), dtype=torch.float32, pin_memory=True)
lon_h, lat_h = lon.cpu().numpy(), lat.cpu().numpy()
for rep in range(int(os.environ.get("REPS", "6"))):
    t0 = time.perf_counter()
    p = Plan(lon_h, lat_h, w.map, w.fwhm_deg, w.support)
    t1 = time.perf_counter()
    p.grid(vals, out, W)
    t2 = time.perf_counter()
    p.close()
    t3 = time.perf_counter()
    print(f"rep {rep}: plan {1e3 * (t1 - t0):.1f}  grid {1e3 * (t2 - t1):.1f}  close {1e3 * (t3 - t2):.1f} ms", flush=True)
