#!/usr/bin/env python
"""Warp/sub-batch statistics of the production raster on a few outdoor views (measurement build
with -DRASTER_STATS; run on the GPU box):  python scripts/raster_stats.py [views] [config]"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_13600_b200 import build  # noqa: E402

lib = build.build(out=os.path.join(ROOT, "paper_2605_13600_b200", "libscoup_stats.so"), defines=["RASTER_STATS"])
os.environ["SCOUP_LIB"] = lib
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2605_13600_b200 import abi, synth  # noqa: E402
from paper_2605_13600_b200.uplift import SparseUplift  # noqa: E402

nv = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cfg = synth.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "outdoor"]
scene = synth.make_scene(cfg, 0)
views = list(range(0, cfg.num_views, max(1, cfg.num_views // nv)))[:nv]
dev = torch.device("cuda", 0)
maps = synth.make_region_maps_torch(cfg, dev, seed=0, views=views)
codes = synth.make_codes(cfg, seed=0, views=views)
cd = synth.Codes(torch.from_numpy(codes.atoms.view(np.int32)).to(dev), torch.from_numpy(codes.coefs).to(dev),
                 codes.row0, codes.num_regions)
g = scene.gaussians
gd = synth.Gaussians(*[torch.from_numpy(a).to(dev) for a in (g.means, g.scales, g.rotations, g.opacities)])
L = abi.lib()
L.scoup_debug_raster_stats.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 16)()
with SparseUplift(gd, cfg.L, cfg.K) as up:
    up.add_views([scene.cameras[v] for v in views], maps, cd)
    torch.cuda.synchronize()
    L.scoup_debug_raster_stats(buf, 1)
    up.reset()
    up.add_views([scene.cameras[v] for v in views], maps, cd)
    torch.cuda.synchronize()
    L.scoup_debug_raster_stats(buf, 1)
s = list(buf)
ws = max(1, s[0])
out = {"config": cfg.name, "views": nv, "warp_subbatches": s[0],
       "active_groups_hist_0to4": [v / ws for v in s[1:6]],
       "grp_full_frac": s[6] / ws, "mask_records_per_warp_subbatch": s[7] / ws,
       "records_per_subbatch": s[8] / ws, "refill_rounds": s[9], "accepted_per_round": s[10] / max(1, s[9]),
       "superbatches": s[11], "records_per_superbatch": s[12] / max(1, s[11]), "ctas_nonempty": s[13],
       "list_entries_per_nonempty_cta": s[14] / max(1, s[13]),
       "superbatches_per_cta": s[11] / max(1, s[13])}
print(json.dumps(out, indent=1))
