#!/usr/bin/env python
"""Benchmark of SURVEY.md §8(f) NEXT-2: sparse coefficient rendering (Eq. 7) and the
codebook decode (Eq. 8) on one B200.

The scene of BASELINE.json configs[3] ("outdoor": 3M Gaussians, 1600x1066, L=64) is uplifted
once (the bench.py step), then every view is rendered from the stored K-sparse codes
(W_hat_v, [H, W, L] fp32) and, per view, decoded against a random codebook C [L, D] (D=512, a
CLIP-sized feature).  Timed with CUDA events on the handle's stream, after warm-up; inputs are
far larger than L2.  Prints one JSON line.

    python scripts/bench_render.py [--views 300] [--steps 3] [--warmup 3] [--D 512]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="outdoor")
    ap.add_argument("--views", type=int, default=0)
    ap.add_argument("--batch", type=int, default=4, help="views per render call")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--D", type=int, default=512)
    args = ap.parse_args()
    import torch
    from paper_2605_13600_b200 import synth
    from paper_2605_13600_b200.uplift import SparseUplift

    dev = torch.device("cuda", 0)
    cfg = synth.CONFIGS[args.config]
    if args.views:
        cfg = cfg.with_(num_views=args.views)
    scene = synth.make_scene(cfg, 0)
    g = scene.gaussians
    gd = synth.Gaussians(*[torch.from_numpy(a).to(dev) for a in (g.means, g.scales, g.rotations, g.opacities)])
    maps = synth.make_region_maps_torch(cfg, dev, level=0, seed=0)
    ch = synth.make_codes(cfg, level=0, seed=0)
    codes = synth.Codes(torch.from_numpy(ch.atoms.view(np.int32)).to(dev), torch.from_numpy(ch.coefs).to(dev),
                        ch.row0, ch.num_regions)
    up = SparseUplift(gd, cfg.L, cfg.K)
    up.set_counters(True)  # the render evaluates exactly the uplift's fragments: count them once
    up.add_views(scene.cameras, maps, codes)
    atoms, coefs = up.finalize()
    st = up.stats()
    up.set_counters(False)
    tests_v = st["support_tests"] / cfg.num_views
    contrib_v = st["contributions"] / cfg.num_views
    del maps
    torch.cuda.synchronize()
    H, W, L, B = scene.cameras[0].height, scene.cameras[0].width, cfg.L, args.batch
    Wh = torch.empty((B, H, W, L), dtype=torch.float32, device=dev)
    F = torch.empty((H * W, args.D), dtype=torch.float32, device=dev)
    C = torch.randn((L, args.D), generator=torch.Generator().manual_seed(3)).to(dev)
    stream = up.stream

    def render_all():
        for v0 in range(0, cfg.num_views, B):
            cams = scene.cameras[v0:v0 + B]
            up.render(cams, atoms, coefs, out=Wh[:len(cams)])

    def decode_all():
        for v in range(cfg.num_views):
            up.decode(Wh[v % B], C, out=F)

    def fill_all():  # write-only stream of the same size as the decode output: HBM write reference
        for v in range(cfg.num_views):
            F.fill_(1.0)

    res = {}
    for name, fn in (("render", render_all), ("decode", decode_all), ("fill", fill_all)):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / args.steps / cfg.num_views
    up.close()
    # decode is an fp32 GEMM [HW, L] x [L, D]: flops and its operand/result bytes per view
    flops = 2.0 * H * W * L * args.D
    byts = 4.0 * (H * W * L + L * args.D + H * W * args.D)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    dec_gbs = byts / (res["decode"] * 1e-3) / 1e9
    # render (Eq. 7): the uplift's 27 lane-ops per support test plus 2 K per contribution (K
    # products coef * e and K adds into the pixel's row), against the FP32-lane peak
    peak_lane = 148 * 128 * peaks["sm_max_mhz"] * 1e6 / 1e12
    ren_ops = (27 * tests_v + 2 * cfg.K * contrib_v) / (res["render"] * 1e-3) / 1e12
    print(json.dumps({
        "metric": "Eq. 7 sparse coefficient render + Eq. 8 decode, ms per view",
        "config": {"workload": f"{args.config}: {g.count} Gaussians, {cfg.num_views} views {W}x{H}, L={L}, "
                               f"K={cfg.K}, D={args.D}", "views_per_render_call": B},
        "render_ms_per_view": res["render"], "render_fps": 1e3 / res["render"],
        "decode_ms_per_view": res["decode"], "decode_tflops": flops / (res["decode"] * 1e-3) / 1e12,
        "decode_gbps": byts / (res["decode"] * 1e-3) / 1e9,
        "fill_gbps": 4.0 * H * W * args.D / (res["fill"] * 1e-3) / 1e9,
        "render_out_gbps": 4.0 * H * W * L / (res["render"] * 1e-3) / 1e9,
        "render_roofline": {"bound": "alu", "kernel": "render_kernel", "achieved": ren_ops, "peak": peak_lane,
                            "unit": "T lane-ops/s", "frac": ren_ops / peak_lane,
                            "support_tests_per_view": tests_v, "contributions_per_view": contrib_v},
        "decode_roofline": {"bound": "hbm", "kernel": "decode_kernel (tcgen05 3xTF32)", "achieved": dec_gbs,
                            "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": dec_gbs / peaks["hbm_gbs"],
                            "bytes": "4 L read + 4 D written per pixel (+ the codebook)"},
        "dtype": "f32", "data": "synthetic",
    }))


if __name__ == "__main__":
    main()
