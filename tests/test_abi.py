"""The C-ABI library builds, loads and exports every symbol include/*.h declares.
Host-side argument validation is exercised without a GPU (no compute calls)."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2605_13600_b200 import abi, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", h) for h in sorted(os.listdir(os.path.join(ROOT, "include"))) if h.endswith(".h")]


@pytest.fixture(scope="module")
def lib():
    build.build()
    return abi.lib()


def declared_functions():
    src = "\n".join(open(h).read() for h in HEADERS)
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(scoup_\w+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    names = declared_functions()
    for n in ["scoup_uplift_init", "scoup_uplift_add_views", "scoup_uplift_finalize_topk", "scoup_uplift_free"]:
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    names = declared_functions()
    out = subprocess.run(["nm", "-D", "--defined-only", abi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (scoup_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(abi.EXPORTS) == set(names)
    for n in names:
        assert hasattr(lib, n)


def test_library_is_sm100a_only(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", abi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_version_and_empty_error(lib):
    assert "sm_100a" in abi.scoup_version()
    assert isinstance(abi.scoup_last_error(), str)


def test_host_side_validation_without_gpu(lib):
    """K > L is a config error; NULL out-pointer / negative sizes are EINVAL.
    These return before any CUDA call."""
    h = C.c_void_p()
    L = lib
    assert L.scoup_uplift_init(0, None, 0, None, None, None, None, 8, 9, None, None, 0, C.byref(h)) == 1
    assert "K > L" in abi.scoup_last_error()
    assert L.scoup_uplift_init(0, None, 10, None, None, None, None, 8, 2, None, None, 0, C.byref(h)) == 1
    assert "NULL" in abi.scoup_last_error()
    assert L.scoup_uplift_init(0, None, 0, None, None, None, None, 8, 0, None, None, 0, C.byref(h)) == 1
    assert L.scoup_uplift_init(0, None, -1, None, None, None, None, 8, 2, None, None, 0, C.byref(h)) == 1
    assert L.scoup_uplift_init(0, None, 10, None, None, None, None, 8, 2, None, None, 0, None) == 1
    assert L.scoup_uplift_init(0, None, 0, None, None, None, None, 2048, 2, None, None, 0, C.byref(h)) == 6
    assert L.scoup_uplift_add_views(None, 1, None, None, None, None, None, None, 4, None) == 1
    assert L.scoup_uplift_finalize_topk(None, 0, 1, None, None, None, None) == 1
    L.scoup_uplift_free(None)  # no-op


def test_sass_uses_global_reductions(lib):
    """The fused kernel issues fire-and-forget global reductions (REDG), not returning atomics."""
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", abi.LIB_PATH], capture_output=True,
                          text=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)
    raster = "".join(f for f in funcs if f.split("\n", 1)[0].find("raster_cu") >= 0)
    assert raster, "raster kernel not found in SASS"
    assert "REDG.E.ADD.F32" in raster
    assert "ATOMG.E.ADD.F32" not in raster


def test_raster2_slots_override_validation(lib):
    """scoup_diag_set_raster2_slots (include/scoup_diag.h): 0, 4 or 8 only, host-only state."""
    for bad in (-1, 1, 5, 16):
        assert lib.scoup_diag_set_raster2_slots(bad) == 1
    assert lib.scoup_diag_set_raster2_slots(4) == 0
    assert lib.scoup_diag_set_raster2_slots(8) == 0
    assert lib.scoup_diag_set_raster2_slots(0) == 0


def test_binsort_segment_override_validation(lib):
    """scoup_diag_set_binsort_segment (include/scoup_diag.h): range check, host-only state."""
    assert lib.scoup_diag_set_binsort_segment(-1) == 1
    assert lib.scoup_diag_set_binsort_segment((1 << 24) + 1) == 1
    assert lib.scoup_diag_set_binsort_segment(100) == 0
    assert lib.scoup_diag_set_binsort_segment(0) == 0
