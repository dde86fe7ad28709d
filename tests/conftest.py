import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")


@pytest.fixture(scope="session")
def tiny_scene():
    from paper_2605_13600_b200 import synth
    cfg = synth.CONFIGS["tiny"]
    scene = synth.make_scene(cfg, seed=0)
    maps = synth.make_region_maps_numpy(cfg, seed=0)
    codes = synth.make_codes(cfg, seed=0)
    return cfg, scene, maps, codes


@pytest.fixture(scope="session")
def tiny_oracle(tiny_scene):
    import oracle
    cfg, scene, maps, codes = tiny_scene
    return oracle.uplift(scene.gaussians, scene.cameras, maps, codes, cfg.L, cfg.K)
