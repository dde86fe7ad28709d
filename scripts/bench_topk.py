#!/usr/bin/env python
"""Eq. 6 finalize (Top-K + L1) on an outdoor-sized accumulator (3M x 64 fp32, ~30% non-zero),
timed with CUDA events over repeated launches: achieved HBM GB/s of the algorithmic traffic
(4 L B read + 8 K B written per row) against MEASURED_PEAKS.json.  Run on the GPU box."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2605_13600_b200 import synth  # noqa: E402
from paper_2605_13600_b200.uplift import SparseUplift  # noqa: E402

G, L, K = 3_000_000, 64, 8
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
density = float(sys.argv[2]) if len(sys.argv) > 2 else 0.3
dev = torch.device("cuda", 0)
# G real rows (a handle's rows beyond its Gaussian count are padding and skip the read)
g = synth.Gaussians(*(np.zeros((G, 3), np.float32), np.full((G, 3), 0.1, np.float32),
                      np.tile(np.array([[1, 0, 0, 0]], np.float32), (G, 1)), np.full((G,), 0.5, np.float32)))
up = SparseUplift(g, L, K, rows_padded=G)
gen = torch.Generator(device=dev).manual_seed(0)
W = torch.rand((G, L), device=dev, generator=gen)
W = torch.where(torch.rand((G, L), device=dev, generator=gen) < density, W, torch.zeros_like(W))
atoms = torch.empty((G, K), dtype=torch.int32, device=dev)
coefs = torch.empty((G, K), dtype=torch.float32, device=dev)
up.finalize(0, G, W_rows=W, out_atoms=atoms, out_coefs=coefs)  # warm-up
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = []
for _ in range(reps):
    e0.record()
    up.finalize(0, G, W_rows=W, out_atoms=atoms, out_coefs=coefs)
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
up.close()
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6546.9)
t = float(np.median(ms))
byts = G * (4 * L + 8 * K)
print(json.dumps({"kernel": "topk_tile_kernel", "rows": G, "L": L, "K": K, "density": density, "ms": t, "GB/s": byts / t / 1e6,
                  "frac_hbm": byts / t / 1e6 / peak, "peak_gbs": peak,
                  "note": "median of %d finalize calls (each includes the handle's stream sync)" % reps}))
