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
SOURCES = ["api.cu", "kernels.cu", "raster.cu", "render.cu", "decode.cu", "sparse_coding.cu"]
HEADERS = ["internal.cuh"]
LIB = os.path.join(HERE, "libscoup.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    # parity-critical arithmetic uses explicit _rn intrinsics; also forbid contraction
    "-fmad=false",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-warn-spills",
]


def _inputs():
    paths = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    paths.append(os.path.join(ROOT, "include", "scoup.h"))
    paths.append(os.path.join(ROOT, "include", "scoup_sparse_coding.h"))
    paths.append(os.path.abspath(__file__))
    return paths


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _inputs())


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Compile libscoup.so (or a variant with extra -D defines into `out`)."""
    if not force and out == LIB and not defines and not stale():
        return LIB
    tmp = out + f".tmp{os.getpid()}"
    flags = [*NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include")]
    if verbose:
        flags.insert(0, "-Xptxas=-v")
    with tempfile.TemporaryDirectory(prefix="scoup_build_") as td:
        def compile_one(src: str) -> str:
            obj = os.path.join(td, os.path.splitext(src)[0] + ".o")
            cmd = [NVCC, *flags, "-c", os.path.join(CSRC, src), "-o", obj]
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
