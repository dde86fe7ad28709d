"""Build libscoup.so (the C-ABI CUDA library) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["api.cu", "kernels.cu", "binsort.cu", "raster.cu", "raster2.cu", "render.cu", "decode.cu", "sparse_coding.cu", "diag.cu"]
HEADERS = ["internal.cuh"]
LIB = os.path.join(HERE, "libscoup.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-warn-spills",
]
# The translation units of the parity-critical path (every fragment decision is
# bit-identical to the oracle's) use explicit _rn intrinsics AND forbid contraction; the others
# (Eq. 7 render accumulation, Eq. 8 decode, Eq. 4 sparse coding: tolerance-based parity) keep
# nvcc's default FMA contraction.  (render.cu's per-pixel fragment sequence is written with
# explicit intrinsics, which contraction never touches.)
SPEC_TUS = {"api.cu", "kernels.cu", "raster.cu", "raster2.cu"}


def tu_flags(src: str):
    return ["-fmad=false"] if src in SPEC_TUS else []


def _inputs():
    paths = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    paths.append(os.path.join(ROOT, "include", "scoup.h"))
    paths.append(os.path.join(ROOT, "include", "scoup_sparse_coding.h"))
    paths.append(os.path.join(ROOT, "include", "scoup_diag.h"))
    paths.append(os.path.abspath(__file__))
    return paths


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _inputs())


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=(), csrc: str = CSRC) -> str:
    """Compile libscoup.so (or a variant with extra -D defines, or from another source tree
    `csrc` -- A/B runs of an earlier revision -- into `out`)."""
    if not force and out == LIB and not defines and csrc == CSRC and not stale():
        return LIB
    tmp = out + f".tmp{os.getpid()}"
    flags = [*NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include")]
    if verbose:
        flags.insert(0, "-Xptxas=-v")
    with tempfile.TemporaryDirectory(prefix="scoup_build_") as td:
        def compile_one(src: str) -> str:
            obj = os.path.join(td, os.path.splitext(src)[0] + ".o")
            cmd = [NVCC, *flags, *tu_flags(src), "-c", os.path.join(csrc, src), "-o", obj]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.check_call(cmd)
            return obj
        # translation units compile in parallel, then one device-aware link
        with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
            objs = list(ex.map(compile_one, SOURCES))
        subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
                               "-o", tmp, *objs, "-lcublas"])
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
