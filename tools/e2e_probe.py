"""e2e breakdown on cfg4: pinned H2D/D2H bandwidth, plan creation from host coords, one host
hegrid_grid call with the per-block pipeline trace (H2D / permute+accumulate / D2H per stream)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from bench import user_layout_values_pinned  # noqa: E402
from paper_2207_04584_b200 import Plan  # noqa: E402

w = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
dev = torch.device("cuda", 0)
# pinned copy bandwidth
h = torch.empty(1 << 28, dtype=torch.float32, pin_memory=True)
d = torch.empty(1 << 28, dtype=torch.float32, device=dev)
for name, src, dst in (("H2D", h, d), ("D2H", d, h)):
    dst.copy_(src, non_blocking=True); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    print(f"pinned {name}: {3 * 4 * (1 << 28) / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
del h, d
lon, lat = synth.coords(w, device=dev)
C = w.channels
vals = user_layout_values_pinned(w, lon, lat, list(range(C)), dev)
out = torch.empty((C, w.ny, w.nx), dtype=torch.float32, pin_memory=True)
W = torch.empty((w.ny, w.nx), dtype=torch.float32, pin_memory=True)
lon_h, lat_h = lon.cpu().numpy(), lat.cpu().numpy()
for rep in range(3):
    t0 = time.perf_counter()
    p = Plan(lon_h, lat_h, w.map, w.fwhm_deg, w.support, engine="tc")
    t1 = time.perf_counter()
    p.profile(True)
    p.grid(vals, out, W)
    t2 = time.perf_counter()
    tr = p.pipeline_trace()
    p.profile(False)
    print(f"rep {rep}: plan {1e3 * (t1 - t0):.1f} ms, grid {1e3 * (t2 - t1):.1f} ms, "
          f"blocks {len(tr)}, info {p.info()['t_plan_ms']:.2f} ms")
    t3 = time.perf_counter()
    p.grid(vals, out, W)
    t4 = time.perf_counter()
    print(f"   second grid on the same plan: {1e3 * (t4 - t3):.1f} ms")
    if rep == 0:
        for r in tr[:12]:
            print("   slot %d: h2d %.2f-%.2f  compute ..%.2f  d2h ..%.2f ms" % tuple(r))
        print("   last:", tr[-1])
    p.close()
