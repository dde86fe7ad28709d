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
