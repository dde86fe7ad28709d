#!/usr/bin/env python
"""Where the end-to-end step's time goes (run on the GPU box): pinned H2D / D2H bandwidth, and the
phases of bench.py's e2e step (handle init from host Gaussians, add_views with host region maps,
finalize into host codes, close), each bracketed by a device sync (host wall clock)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2605_13600_b200 import synth  # noqa: E402
from paper_2605_13600_b200.uplift import SparseUplift  # noqa: E402

dev = torch.device("cuda", 0)
out = {}
x = torch.empty(2 << 30, dtype=torch.uint8).pin_memory()
y = torch.empty(2 << 30, dtype=torch.uint8, device=dev)
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); y.copy_(x, non_blocking=True); torch.cuda.synchronize()
    out["h2d_GBps"] = (2 << 30) / (time.perf_counter() - t) / 1e9
    t = time.perf_counter(); x.copy_(y, non_blocking=True); torch.cuda.synchronize()
    out["d2h_GBps"] = (2 << 30) / (time.perf_counter() - t) / 1e9
del x, y
cfg = synth.CONFIGS["outdoor"]
scene = synth.make_scene(cfg, 0)
g = scene.gaussians
cams = scene.cameras
maps = synth.make_region_maps_torch(cfg, dev, seed=0).cpu().pin_memory()
codes = synth.make_codes(cfg, seed=0)
codes_h = synth.Codes(torch.from_numpy(codes.atoms.view(np.int32)).pin_memory(), torch.from_numpy(codes.coefs).pin_memory(),
                      codes.row0, codes.num_regions)
g_h = synth.Gaussians(*[torch.from_numpy(a).pin_memory() for a in (g.means, g.scales, g.rotations, g.opacities)])
atoms_h = torch.empty((g.count, cfg.K), dtype=torch.int32).pin_memory()
coefs_h = torch.empty((g.count, cfg.K), dtype=torch.float32).pin_memory()
for rep in range(3):
    ph = {}
    torch.cuda.synchronize(); t0 = time.perf_counter()
    u = SparseUplift(g_h, cfg.L, cfg.K, device=0, rows_padded=g.count)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    u.add_views(cams, maps, codes_h)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    u.finalize(0, g.count, out_atoms=atoms_h, out_coefs=coefs_h)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    u.close()
    torch.cuda.synchronize(); t4 = time.perf_counter()
    ph = {"init_ms": (t1 - t0) * 1e3, "add_views_ms": (t2 - t1) * 1e3, "finalize_ms": (t3 - t2) * 1e3,
          "close_ms": (t4 - t3) * 1e3, "total_ms": (t4 - t0) * 1e3}
    out[f"rep{rep}"] = ph
# device-resident add_views for reference
md = maps.to(dev)
cd = synth.Codes(codes_h.atoms.to(dev), codes_h.coefs.to(dev), codes.row0, codes.num_regions)
gd = synth.Gaussians(*[a.to(dev) for a in (g_h.means, g_h.scales, g_h.rotations, g_h.opacities)])
u = SparseUplift(gd, cfg.L, cfg.K, device=0, rows_padded=g.count)
for rep in range(2):
    u.reset(); torch.cuda.synchronize(); t = time.perf_counter(); u.add_views(cams, md, cd); torch.cuda.synchronize()
    out[f"device_add_views_ms{rep}"] = (time.perf_counter() - t) * 1e3
u.close()
print(json.dumps(out, indent=1))
