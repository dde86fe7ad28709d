"""The bench.py JSON contract the driver reads (one line on rank 0): the reference arm on the CPU
(-m "not gpu") and the GPU arm on a tiny workload (-m gpu)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"}


def _run(args, timeout=900):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_json_line():
    """--impl reference: the CPU oracle on a bounded sample, with the base keys, impl, and the
    cpu_baseline / e2e objects describing this run."""
    d = _run(["--impl", "reference", "--config", "tiny", "--steps", "1", "--warmup", "1"])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["config"]["workload"] == "tiny"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_gpu_arm_json_line():
    """The GPU arm on the tiny workload: base keys plus roofline, clocks, gpu_launches and an
    e2e object with the host<->device bytes it moved."""
    d = _run(["--config", "tiny", "--steps", "2", "--warmup", "3", "--no-cpu-baseline"])
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["value"] > 0
    rf = d["roofline"]
    assert rf["bound"] == "alu" and rf["peak"] > 0 and 0 < rf["frac"] <= 1 and rf["achieved"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["gpu_launches"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["contributions_per_step"] > 0 and d["config"]["workload"] == "tiny"


def test_world_size_must_match_gpus():
    """bench.py --gpus N under a launcher whose WORLD_SIZE differs exits non-zero (the driver's
    N must be the number of ranks that ran)."""
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "tiny"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 2 and "WORLD_SIZE=1" in out.stderr


@pytest.mark.gpu
def test_two_rank_flow_on_one_device_matches_oracle(tmp_path):
    """bench.py --gpus 2 re-launches itself as 2 ranks (torch.distributed.run); with
    --same-device both ranks share cuda:0 over a gloo group and the fused exchange maps the peer's
    accumulator through same-device CUDA IPC (no kernel waits on another rank: host barriers
    order the reads).  Each rank's shard codes, concatenated, equal the oracle's codes of the
    whole view set (SURVEY.md §8(c) comparator; Eq. 5 is a sum over views)."""
    import numpy as np
    sys.path.insert(0, ROOT)
    import oracle
    from paper_2605_13600_b200 import synth
    from helpers import compare_codes
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--same-device",
                          "--config", "tiny", "--steps", "1", "--warmup", "3", "--no-e2e", "--no-cpu-baseline",
                          "--dump-codes", str(tmp_path)], capture_output=True, text=True, timeout=400, cwd=ROOT,
                         env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["ranks_on_one_device"] == 2 and "fused peer-read" in d["config"]["parallelism"]
    cfg = synth.CONFIGS["tiny"]
    scene = synth.make_scene(cfg, 0)
    maps = synth.make_region_maps_numpy(cfg, seed=0)
    codes = synth.make_codes(cfg, seed=0)
    W = oracle.uplift(scene.gaussians, scene.cameras, maps, codes, cfg.L, cfg.K)[0]
    A = np.concatenate([np.load(tmp_path / f"atoms_rank{r}.npy") for r in range(2)])
    C = np.concatenate([np.load(tmp_path / f"coefs_rank{r}.npy") for r in range(2)])
    meta = [json.load(open(tmp_path / f"shard_rank{r}.json")) for r in range(2)]
    assert meta[0]["first_row"] == 0 and meta[1]["first_row"] == meta[0]["rows"]
    G = scene.gaussians.count
    bad, ties, worst = compare_codes(A[:G], C[:G], W, cfg.K)
    assert bad == 0, worst
