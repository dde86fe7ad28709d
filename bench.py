#!/usr/bin/env python
"""Benchmark: SCOUP scene uplift (weighted sparse aggregation) on B200.

One step = one full scene uplift of BASELINE.json configs[3] ("outdoor": 3M Gaussians,
300 views at 1600x1066, L=64, S=K=8): every view rasterised and aggregated (Eq. 5 /
Algorithm 1), then Eq. 6 Top-K on every Gaussian.  With N ranks the views are sharded
(v = rank mod N), the fp32 partial sums are combined by an NCCL reduce-scatter and each
rank finalises its Gaussian shard.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config outdoor] [--impl ours|reference]

Prints ONE JSON line on rank 0 (see DESIGN.md §7 for every field).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "scene uplift seconds & pixel-Gaussian contributions/s at 1/2/4/8 B200"
# algorithmic lane-ops of the spec per support test and per contribution
OPS_PER_TEST = 27


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="outdoor")
    ap.add_argument("--views", type=int, default=0, help="limit the number of views (quick runs only)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-views", type=int, default=1, help="views in the oracle cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dense", type=int, default=0,
                    help="dense feature uplift baseline (Eq. 3) with D-dim region features instead of codes")
    ap.add_argument("--exchange", default="fused", choices=["fused", "nccl"],
                    help="N > 1: fused peer-read reduction + Top-K over CUDA IPC (default), or NCCL "
                         "reduce-scatter + Top-K")
    ap.add_argument("--same-device", action="store_true",
                    help="TEST ONLY: every rank on cuda:0 with a gloo process group (the N > 1 flow on one "
                         "GPU; the fused exchange then maps same-device IPC handles).  Timings are not "
                         "meaningful in this mode")
    ap.add_argument("--dump-codes", default="",
                    help="directory: each rank saves its Gaussian shard's codes after the timed steps")
    ap.add_argument("--cpu-workers", type=int, default=0,
                    help="threads of the all-core oracle baseline (0: host cores, bounded by memory)")
    return ap.parse_args()


def relaunch(args) -> int:
    """`--gpus N` (N > 1) without a torch.distributed environment: re-launch this command as N
    ranks on this node (torch.distributed.run, rendezvous on 127.0.0.1), NCCL logging on so the
    rank/channel setup is visible in stderr.  Returns the launcher's exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    print(f"[bench] launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)
            if not any(len(ln.split(",")) >= 8 for ln in self.lines):
                # a region shorter than nvidia-smi's first sample: one sample at its end
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=20)
                    self.lines.extend(ln.strip() for ln in out.stdout.splitlines())
                except Exception:
                    pass

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


def measured_traffic():
    """DRAM bytes of the fused kernel from the committed ncu capture (profiles/raster_traffic.json),
    per view (a launch covers a batch of views), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "raster_traffic.json")) as fh:
            t = json.load(fh)
        return (t["dram_bytes_read"] + t["dram_bytes_write"]) / t["views_per_launch"], t["source"]
    except Exception:
        return None, None


def crop_band(cam, y0, y1):
    """The rows [y0, y1) of a view as a camera of its own (same rays; principal point shifted)."""
    from paper_2605_13600_b200 import synth
    return synth.Camera(cam.fx, cam.fy, cam.cx, cam.cy - y0, cam.width, y1 - y0, cam.world_to_camera)


def _band_sample(cfg, scene, views, band, seed=0, device=None):
    """Region maps, codes and band cameras of the middle 1/band of the rows of each listed view."""
    from paper_2605_13600_b200 import synth
    import torch
    dev = device if device is not None else torch.device("cpu")
    maps = synth.make_region_maps_torch(cfg, dev, seed=seed, views=views).cpu().numpy().view(np.uint32)
    y0 = cfg.height // 2 - cfg.height // (2 * band)
    y1 = y0 + cfg.height // band
    maps = np.ascontiguousarray(maps[:, y0:y1])
    codes = synth.make_codes(cfg, seed=seed, views=views)
    cams = [crop_band(scene.cameras[v], y0, y1) for v in views]
    return maps, codes, cams, y0, y1


def cpu_baseline(cfg, scene, views, seed=0, band=3, device=None):
    """The oracle as it stands, single-threaded, on a bounded sample: the middle third of the
    rows of each listed view (full Gaussian set, full width; ~12 s per outdoor view band)."""
    import oracle
    maps, codes, cams, y0, y1 = _band_sample(cfg, scene, views, band, seed, device)
    t0 = time.perf_counter()
    W, Z, frags = oracle.uplift_accumulate(scene.gaussians, cams, maps, codes.atoms,
                                           codes.coefs, codes.row0, codes.num_regions, cfg.L, cfg.K)
    dt = time.perf_counter() - t0
    per_view = dt * band / len(views)
    return {"value": float(frags.sum()) / dt, "unit": "contributions/s", "cores": 1, "kind": "oracle",
            "sample": f"rows {y0}..{y1} of views {views} of {cfg.name} ({cfg.num_gaussians} Gaussians, "
                      f"{cfg.width}x{cfg.height}), accumulation, {dt:.1f} s single-threaded",
            "seconds": dt, "contributions": int(frags.sum()),
            "scene_uplift_s_extrapolated": per_view * cfg.num_views * len(cfg.regions),
            "extrapolation": f"{dt:.1f} s x {band} bands per view / {len(views)} views x {cfg.num_views} views"
                             f" x {len(cfg.regions)} levels (labelled: extrapolated)"}


def cpu_baseline_all_cores(cfg, scene, workers=0, seed=0, band=3, device=None):
    """SURVEY.md §8(d) all-core CPU baseline: the same oracle on P host threads over view shards
    (one middle-third band of a different view per thread), fp64 partials merged in a fixed
    order.  P = host cores, bounded so that P fp64 partials of [G, L] fit in
    half of the available host memory; `cores` reports the P actually used."""
    import oracle
    ncores = len(os.sched_getaffinity(0))
    part_bytes = cfg.num_gaussians * (cfg.L + 1) * 8
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:  # noqa: BLE001
        avail = 8 << 30
    cap = max(1, int(0.5 * avail // part_bytes))
    P = max(1, min(workers or ncores, ncores, cap, cfg.num_views))
    views = list(range(0, cfg.num_views, max(1, cfg.num_views // P)))[:P]
    maps, codes, cams, y0, y1 = _band_sample(cfg, scene, views, band, seed, device)
    t0 = time.perf_counter()
    W, Z, frags = oracle.uplift_accumulate_parallel(scene.gaussians, cams, maps, codes.atoms, codes.coefs,
                                                    codes.row0, codes.num_regions, cfg.L, cfg.K, workers=P)
    dt = time.perf_counter() - t0
    return {"value": float(frags.sum()) / dt, "unit": "contributions/s", "cores": P, "kind": "oracle",
            "sample": f"rows {y0}..{y1} of {P} views ({views[0]}, {views[1] if P > 1 else ''}...) of {cfg.name}, "
                      f"one view band per thread, {dt:.1f} s wall on {P} of {ncores} host cores",
            "seconds": dt, "contributions": int(frags.sum()),
            "scene_uplift_s_extrapolated": dt * band * cfg.num_views * len(cfg.regions) / P,
            "extrapolation": f"{dt:.1f} s wall x {band} bands per view x {cfg.num_views} views x "
                             f"{len(cfg.regions)} levels / {P} views per wall (labelled: extrapolated)",
            "cpu_model": _cpu_model()}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from paper_2605_13600_b200 import synth
    cfg = synth.CONFIGS[args.config]
    if args.views:
        cfg = cfg.with_(num_views=args.views)
    scene = synth.make_scene(cfg, 0)
    vals = []
    per = []
    # the middle third of a view's rows (~17 s per outdoor step) up to 8 steps in all, thinner
    # middle bands beyond that, so that any --steps/--warmup run stays within a few minutes
    band = 3 * max(1, -(-(args.warmup + args.steps) // 8))
    for s in range(args.warmup + args.steps):
        v = [s % cfg.num_views]
        r = cpu_baseline(cfg, scene, v, band=band)
        if s >= args.warmup:
            vals.append(r["value"])
            per.append(r)
    value = statistics.median(vals)
    ms = statistics.median([r["seconds"] for r in per]) * 1e3
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "contributions/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg.name, "gaussians": cfg.num_gaussians, "views": cfg.num_views,
                       "width": cfg.width, "height": cfg.height, "L": cfg.L, "S": cfg.S, "K": cfg.K,
                       "levels": 1, "regions_per_view": list(cfg.regions[:1]), "parallelism": "CPU oracle, 1 thread",
                       "step": f"one view of the workload per step (bounded sample: the middle 1/{band} of its rows)"},
            "cpu_baseline": {"value": value, "unit": "contributions/s", "cores": 1, "kind": "oracle",
                             "sample": f"per step the middle 1/{band} of one view's rows (all Gaussians), views 0.."
                                       + str(args.warmup + args.steps - 1)},
            "e2e": {"value": value, "unit": "contributions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def measured_red_rates(dev_index: int):
    """R_red measured live through include/scoup_diag.h: float adds per second
    of red.global.add.f32 (and the v4 form) to one 32-B sector per lane, into an L2-resident
    32 MB buffer and an HBM-resident 4 GB buffer."""
    from paper_2605_13600_b200 import abi
    out = {}
    for name, nbytes in (("l2_32MB", 32 << 20), ("hbm_4GB", 4 << 30)):
        for vec in (False, True):
            rate, ms = abi.scoup_diag_red_rate(dev_index, nbytes, True, vec, 1 << 28, 5)
            out[f"{name}_{'v4' if vec else 'f32'}"] = rate / 1e9
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "RANK" not in os.environ:
        sys.exit(relaunch(args))
    import torch
    import torch.distributed as dist
    from paper_2605_13600_b200 import synth
    from paper_2605_13600_b200.uplift import SparseUplift

    rank, world, local = env_rank()
    t_start = time.perf_counter()

    def trace(msg):  # SCOUP_BENCH_TRACE=1: per-rank progress on stderr (debugging multi-rank runs)
        if os.environ.get("SCOUP_BENCH_TRACE"):
            print(f"[rank {rank} +{time.perf_counter() - t_start:.1f}s] {msg}", file=sys.stderr, flush=True)

    if world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        sys.exit(2)
    same = args.same_device
    local_dev = 0 if same else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if same:  # NCCL refuses two ranks on one GPU; the collectives here are host-side only
            import datetime
            dist.init_process_group("gloo", timeout=datetime.timedelta(seconds=300))
        else:
            dist.init_process_group("nccl", device_id=dev)
    coll_dev = torch.device("cpu") if same else dev
    cfg = synth.CONFIGS[args.config]
    if args.views:
        cfg = cfg.with_(num_views=args.views)
    scene = synth.make_scene(cfg, 0)
    g = scene.gaussians
    dense = args.dense > 0
    if dense:  # Eq. 3 baseline: D-dim features per region, one level, no Top-K (f_i = W_i / Z_i)
        cfg = cfg.with_(L=args.dense, S=args.dense, regions=cfg.regions[:1])
    G, L, K = g.count, cfg.L, cfg.K
    from paper_2605_13600_b200 import distributed as D
    my_views = D.views_for_rank(cfg.num_views, rank, world)
    cams = [scene.cameras[v] for v in my_views]
    # semantic levels (configs[2]: three nested levels) are fused into one raster pass
    nlev = len(cfg.regions)
    maps_l = [synth.make_region_maps_torch(cfg, dev, level=l, seed=0, views=my_views) for l in range(nlev)]
    codes_hl = [synth.make_dense_features(cfg, L, level=l, seed=0, views=my_views) if dense else
                synth.make_codes(cfg, level=l, seed=0, views=my_views) for l in range(nlev)]
    codes_l = [synth.Codes(None if c.atoms is None else torch.from_numpy(c.atoms.view(np.int32)).to(dev),
                           torch.from_numpy(c.coefs).to(dev), c.row0, c.num_regions) for c in codes_hl]
    gd = synth.Gaussians(*[torch.from_numpy(a).to(dev) for a in (g.means, g.scales, g.rotations, g.opacities)])
    Npad = D.padded_rows(G, world)
    first_row, shard = D.row_shard(G, rank, world)
    up = SparseUplift(gd, L, K, device=local_dev, rows_padded=Npad, levels=nlev)
    Ws = torch.empty((shard, L), dtype=torch.float32, device=dev) if world > 1 else None
    Zs = torch.empty((shard,), dtype=torch.float32, device=dev) if world > 1 else None

    def add(u, m_l, c_l):
        if nlev == 1:
            u.add_views(cams, m_l[0], c_l[0])
        else:
            u.add_views(cams, m_l, c_l)

    # N > 1: the fused exchange reads the peers' accumulators through CUDA IPC
    # mappings (set up once for the timed handle); if any rank cannot map them, every rank uses
    # the NCCL reduce-scatter + shard Top-K instead
    peers, peer_bases, exchange = None, [], "nccl" if world == 1 else args.exchange
    if same:
        exchange = "fused"  # (gloo has no CUDA reduce-scatter; same-device IPC maps fine)
    trace("inputs ready")
    if world > 1 and exchange == "fused" and not dense:
        try:
            peers, peer_bases = D.exchange_accumulators(up.W, rank, world, local_dev)
        except Exception as ex:  # noqa: BLE001 -- reported, then the NCCL path
            print(f"[rank {rank}] fused exchange unavailable ({ex}); using NCCL reduce-scatter", file=sys.stderr)
            exchange = "nccl"
        everyone = [None] * world  # the fused path only if every rank has its mappings
        dist.all_gather_object(everyone, exchange == "fused")
        if not all(everyone):
            exchange = "nccl"
    if world > 1 and rank == 0:
        print(f"[bench] {world} ranks, exchange: {exchange}", file=sys.stderr, flush=True)

    def finalize_all(u, out_atoms=None, out_coefs=None):
        if dense:  # Eq. 3 needs no Top-K: f_i = W_i / Z_i (W is the output)
            return None
        res = None
        for lvl in range(nlev):
            if world > 1 and u is up and exchange == "fused":
                res = D.fused_reduce_finalize(u, peers, first_row, shard, level=lvl, out_atoms=out_atoms,
                                              out_coefs=out_coefs)
            elif world > 1:
                Wl = u.W if nlev == 1 else u.W[lvl]
                D.reduce_scatter_accumulators(Wl, u.Z, Ws, Zs)
                res = u.finalize(first_row=first_row, num_rows=shard, W_rows=Ws, Z_rows=Zs, level=lvl,
                                 out_atoms=out_atoms, out_coefs=out_coefs)
            else:
                res = u.finalize(0, G, level=lvl, out_atoms=out_atoms, out_coefs=out_coefs)
        return res

    def step():
        up.reset()
        add(up, maps_l, codes_l)
        return finalize_all(up)

    def barrier():
        if world > 1:
            dist.barrier()

    def reduce_over_ranks(x: float, op) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=op)
        return float(t.item())

    def max_over_ranks(x: float) -> float:
        return reduce_over_ranks(x, dist.ReduceOp.MAX if world > 1 else None)

    def sum_over_ranks(x: float) -> float:
        return reduce_over_ranks(x, dist.ReduceOp.SUM if world > 1 else None)

    # first warm-up step with the instrumented kernel variant: the algorithmic work of one step
    # (support tests, contributions, global reds) for the roofline numerators; the timed steps
    # run the production kernel
    trace("counting step")
    up.set_counters(True)
    step()
    torch.cuda.synchronize()
    trace("counting step done")
    st0 = up.stats()  # one step's counters (reset at each step start)
    up.set_counters(False)
    for _ in range(args.warmup - 1):
        step()
    torch.cuda.synchronize()
    contrib_step = sum_over_ranks(st0["contributions"])
    tests_step = sum_over_ranks(st0["support_tests"])
    entries_step = sum_over_ranks(st0["tile_entries"])
    visible_step = sum_over_ranks(st0["visible"])
    lane_evals_step = sum_over_ranks(st0["lane_evaluations"])
    reds_step = sum_over_ranks(st0["global_reds"])

    trace("warm-up done")
    up.set_timing(True)
    barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_dev) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            last = step()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    trace("timed steps done")
    elapsed_ms = max_over_ranks(e0.elapsed_time(e1))
    tm = up.timing()
    st = up.stats()
    ms_per_step = elapsed_ms / args.steps
    value = contrib_step * args.steps / (elapsed_ms / 1e3)
    if args.dump_codes and last is not None:
        os.makedirs(args.dump_codes, exist_ok=True)
        np.save(os.path.join(args.dump_codes, f"atoms_rank{rank}.npy"), last[0].cpu().numpy().view(np.uint32))
        np.save(os.path.join(args.dump_codes, f"coefs_rank{rank}.npy"), last[1].cpu().numpy())
        with open(os.path.join(args.dump_codes, f"shard_rank{rank}.json"), "w") as fh:
            json.dump({"first_row": first_row, "rows": shard, "world": world, "exchange": exchange}, fh)

    # ---- roofline timing pass (untimed): one more step with ONE pipeline context, so the raster
    # launches' event times are the kernel's own durations (no overlap with the other context's
    # front); the live step above runs the two overlapping contexts
    up.set_pipeline(1)
    up.set_timing(True)
    barrier()
    step()
    torch.cuda.synchronize()
    tm1 = up.timing()
    up.set_pipeline(2)
    trace("timing pass done")
    raster_own_ms = max_over_ranks(tm1["raster_ms"])  # per step (one step in this pass)
    front_own_ms = max_over_ranks(tm1["preprocess_ms"] + tm1["binning_ms"])
    topk_own_ms = max_over_ranks(tm1["topk_ms"])
    peaks = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    alu_peak = sms * 128 * sm_max * 1e6 / 1e12  # T lane-ops/s (DESIGN.md §5 a4)
    # algorithmic lane-ops of one step (DESIGN.md §5 a4) over the raster's own time per step
    # (dense features, Eq. 3: the kernel sums e per region slot before the D-wide products, so only
    # the per-support-test alpha work is counted -- counting 2D + 1 per contribution would exceed
    # the peak)
    ops_step = OPS_PER_TEST * tests_step + (0 if dense else (2 * nlev * cfg.S + 1) * contrib_step)
    achieved = ops_step / world / (raster_own_ms / 1e3) / 1e12 if raster_own_ms > 0 else 0.0
    if raster_own_ms > ms_per_step:
        print(f"[bench] WARNING: raster own time {raster_own_ms:.2f} ms > step {ms_per_step:.2f} ms",
              file=sys.stderr)
    traffic_view, traffic_src = measured_traffic()
    try:
        red_peaks = measured_red_rates(local_dev)
    except Exception as ex:  # noqa: BLE001 -- reported in the line
        red_peaks = {"error": str(ex)}
    trace("red rates done")
    red_rate = reds_step / world / (raster_own_ms / 1e3) / 1e9 if raster_own_ms > 0 else 0.0
    red_peak = red_peaks.get("l2_32MB_f32")
    red_peak_hbm = red_peaks.get("hbm_4GB_f32")

    # ---- end to end through the C ABI with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        maps_hl = [m.cpu().pin_memory() for m in maps_l]
        g_h = synth.Gaussians(*[torch.from_numpy(a).pin_memory() for a in (g.means, g.scales, g.rotations, g.opacities)])
        nrows = G if world == 1 else shard
        atoms_h = torch.empty((nrows, K), dtype=torch.int32).pin_memory()
        coefs_h = torch.empty((nrows, K), dtype=torch.float32).pin_memory()
        codes_hpl = [synth.Codes(None if c.atoms is None else torch.from_numpy(c.atoms.view(np.int32)).pin_memory(),
                                 torch.from_numpy(c.coefs).pin_memory(), c.row0, c.num_regions) for c in codes_hl]

        def e2e_step():
            u2 = SparseUplift(g_h, L, K, device=local_dev, rows_padded=Npad, levels=nlev)
            add(u2, maps_hl, codes_hpl)
            finalize_all(u2, out_atoms=atoms_h, out_coefs=coefs_h)  # codes read back to the host
            u2.close()

        e2e_step()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(max(1, min(args.steps, 2))):
            e2e_step()
        torch.cuda.synchronize()
        barrier()
        n_e2e = max(1, min(args.steps, 2))
        e2e_s = max_over_ranks((time.perf_counter() - t0) / n_e2e)
        h2d = sum_over_ranks(sum(m.numel() for m in maps_hl) * 4 + G * 44 +
                             sum(c.coefs.numel() * (4 if c.atoms is None else 8) for c in codes_hpl))
        d2h = sum_over_ranks(0 if dense else nlev * nrows * K * 8)
        e2e = {"value": contrib_step / e2e_s, "unit": "contributions/s", "seconds_per_step": e2e_s,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, scene, list(range(args.cpu_views)), device=dev)
        try:
            cpu["all_cores"] = cpu_baseline_all_cores(cfg, scene, workers=args.cpu_workers, device=dev)
        except Exception as ex:  # noqa: BLE001 -- reported in the line
            cpu["all_cores"] = {"error": str(ex)}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": "contributions/s",
            "n_gpus": 1 if same else world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "scene_uplift_s": ms_per_step / 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": cfg.name + (f"-dense{L}" if dense else ""), "gaussians": G, "views": cfg.num_views, "width": cfg.width,
                       "height": cfg.height, "L": L, "S": cfg.S, "K": K, "levels": nlev,
                       "regions_per_view": list(cfg.regions),
                       "parallelism": (f"view-sharded x{world} + " + ("fused peer-read reduction + Top-K (CUDA IPC)"
                                       if exchange == "fused" else "NCCL reduce-scatter")) if world > 1 else "single GPU",
                       "l2": "inputs larger than L2 (region maps %.2f GB, W %.0f MB per GPU)" % (
                           sum(m.numel() for m in maps_l) * 4 / 1e9, nlev * Npad * L * 4 / 1e6)},
            "contributions_per_step": int(contrib_step),
            # atom updates = contributions x S per level (every outdoor pixel is
            # coded; dense mode: x D), and the per-GPU rate
            "atom_updates_per_s": value * cfg.S * nlev,
            "contributions_per_s_per_gpu": value / world,
            "support_tests_per_step": int(tests_step),
            "lane_evaluations_per_step": int(lane_evals_step),
            "raster_lane_use": tests_step / max(1, lane_evals_step),
            "bin_entries_per_step": int(entries_step),
            "visible_per_step": int(visible_step),
            "global_reds_per_step": int(reds_step),
            # live step (two overlapping contexts): per-stage event time summed over the launches
            "device_ms_per_step": {k: tm[k] / args.steps for k in ("preprocess_ms", "binning_ms", "raster_ms", "topk_ms")},
            # the one-context timing pass: each kernel's own duration per step
            "serial_ms_per_step": {"raster_ms": raster_own_ms, "front_ms": front_own_ms,
                                   "topk_ms": topk_own_ms},
            "roofline": {"bound": "alu", "kernel": "raster_aggregate_kernel", "achieved": achieved,
                         "peak": alu_peak, "unit": "T lane-ops/s", "frac": achieved / alu_peak,
                         "ops_per_step": ops_step,
                         "duration_ms_per_step": raster_own_ms,
                         "duration_source": "CUDA events around every raster launch of one step run with one "
                                            "pipeline context (no overlap), max over ranks",
                         "raster_own_over_step": raster_own_ms / max(1e-9, ms_per_step),
                         "avg_batch_ms": raster_own_ms / max(1, tm1["raster_launches"]),
                         "views_per_batch": tm1["views_timed"] / max(1, tm1["raster_launches"]),
                         "traffic": traffic_view, "traffic_unit": "DRAM bytes per view (ncu)",
                         "traffic_source": traffic_src,
                         "l2_red": {"achieved": red_rate, "unit": "G float adds/s (red.global.add.f32, W and Z)",
                                    "reds_per_step": int(reds_step), "peak": red_peak,
                                    "frac": (red_rate / red_peak) if red_peak else None,
                                    "peak_source": "scoup_diag_red_rate: one 32-B sector per lane into an "
                                                   "L2-resident 32 MB buffer, measured live (the fused kernel's "
                                                   "reds hit L2 ~86%, ncu)",
                                    "frac_of_hbm_resident_rate": (red_rate / red_peak_hbm) if red_peak_hbm else None,
                                    "measured_peaks": red_peaks},
                         "peak_source": f"{sms} SMs x 128 lanes x {sm_max:.0f} MHz (MEASURED_PEAKS sm_max_mhz)"},
            # the library's kernel launches in the timed region (its stats cover one step: they
            # are reset with the accumulators at each step start)
            "gpu_launches": int((st["kernel_launches"] + st["cub_launches"]) * args.steps),
            "gpu_launches_per_step": int(st["kernel_launches"] + st["cub_launches"]),
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        if same:
            line["ranks_on_one_device"] = world
        print(json.dumps(line), flush=True)
    trace("line printed")
    if peer_bases:  # every rank has finished reading every accumulator (the finalize barriers)
        from paper_2605_13600_b200 import abi
        barrier()
        trace("closing peer mappings")
        for b in peer_bases:
            abi.scoup_ipc_close(local_dev, b)
    up.close()
    trace("closed")
    if world > 1:
        dist.destroy_process_group()
    trace("exit")


if __name__ == "__main__":
    main()
