"""CPU oracle for SCOUP's weighted sparse aggregation -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2605_13600_b200``) never imports it and shares no code with it.

Two independent implementations of DESIGN.md §3's specification live here:

* ``scoup_oracle.c`` (loaded via ctypes): Gaussian-major splat, fp64 accumulation,
  Eq. 6 Top-K.  Cites PAPER.md Eq. 2/3/5/6 and Algorithm 1 line by line.
* ``brute.py``: numpy float32 per-pixel brute force over ALL Gaussians (no support
  culling), used to pin the C oracle bit-for-bit on tiny scenes.

Parity status per function:
* projection, fragment weights e, W, Z, Top-K -- pinned by closed forms, hand cases
  (SURVEY.md §8(c) F1-F8), invariants and brute force (tests/test_oracle_*.py).
* whole-scene values at BASELINE.json sizes -- parity unpinned by the paper (it prints no
  worked example); pinned only through the cases above.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "scoup_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
NONE = 0xFFFFFFFF

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class OraCamera(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("width", C.c_int32), ("height", C.c_int32), ("w2c", C.c_float * 16)]


_lib_handle = None


def lib():
    global _lib_handle
    if _lib_handle is None:
        L = C.CDLL(build())
        P = C.c_void_p
        i64, i32 = C.c_int64, C.c_int32
        L.ora_exp2_spec.argtypes = [C.c_float]
        L.ora_exp2_spec.restype = C.c_float
        L.ora_exp2_spec_vec.argtypes = [i64, P, P]
        L.ora_project.argtypes = [i64, P, P, P, P, P, P]
        L.ora_project.restype = C.c_int
        L.ora_render_view.argtypes = [i64, P, P, P, P, P, P, i64, P, P, P, P]
        L.ora_render_view.restype = i64
        L.ora_uplift_accumulate.argtypes = [i64, P, P, P, P, i32, P, P, P, P, P, P, i32, i32, i32,
                                            P, P, P, P]
        L.ora_uplift_accumulate.restype = C.c_int
        L.ora_topk.argtypes = [i64, P, i32, i32, P, P]
        _lib_handle = L
    return _lib_handle


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def camera_struct(cam) -> OraCamera:
    c = OraCamera()
    c.fx, c.fy, c.cx, c.cy = cam.fx, cam.fy, cam.cx, cam.cy
    c.width, c.height = cam.width, cam.height
    w = np.asarray(cam.world_to_camera, dtype=np.float32).ravel()
    for k in range(16):
        c.w2c[k] = float(w[k])
    return c


def cameras_array(cams: Sequence) -> C.Array:
    arr = (OraCamera * len(cams))()
    for i, cam in enumerate(cams):
        arr[i] = camera_struct(cam)
    return arr


def exp2_spec(y) -> np.ndarray:
    y = _f32(np.atleast_1d(y))
    out = np.empty_like(y)
    lib().ora_exp2_spec_vec(y.size, _p(y), _p(out))
    return out


PROJ_FIELDS = ["visible", "depth", "mx", "my", "sxx", "sxy", "syy", "ca", "cb", "cc", "r",
               "qa", "qb", "qc", "o", "valid"]


def project(g, cam) -> dict:
    """Per-Gaussian projection records (DESIGN.md §3 G1, V1-V7) as a dict of float32 arrays."""
    G = g.count
    out = np.zeros((G, 16), dtype=np.float32)
    c = camera_struct(cam)
    lib().ora_project(G, _p(_f32(g.means)), _p(_f32(g.scales)), _p(_f32(g.rotations)),
                      _p(_f32(g.opacities)), C.byref(c), _p(out))
    return {k: out[:, i] for i, k in enumerate(PROJ_FIELDS)}


def render_view(g, cam, cap: int = 1 << 22):
    """Fragments of one view in Gaussian-major emission order.

    Returns (T_final f32 [H,W], pix int64 [n], gid int64 [n], e f32 [n])."""
    T = np.empty((cam.height, cam.width), dtype=np.float32)
    pix = np.empty(cap, dtype=np.int64)
    gid = np.empty(cap, dtype=np.int64)
    e = np.empty(cap, dtype=np.float32)
    err = np.zeros(1, dtype=np.int64)
    c = camera_struct(cam)
    n = lib().ora_render_view(g.count, _p(_f32(g.means)), _p(_f32(g.scales)), _p(_f32(g.rotations)),
                              _p(_f32(g.opacities)), C.byref(c), _p(T), cap, _p(pix), _p(gid), _p(e),
                              _p(err))
    if n < 0:
        raise ValueError(f"oracle: invalid Gaussian {int(err[0])}")
    if n > cap:
        raise ValueError(f"oracle: {n} fragments exceed cap {cap}")
    return T, pix[:n], gid[:n], e[:n]


class OracleError(ValueError):
    def __init__(self, code: int, index: int):
        kind = {-1: "bad argument", -2: "bad Gaussian", -3: "bad region id", -4: "bad code"}.get(code, "error")
        super().__init__(f"oracle: {kind} at index {index}")
        self.code, self.index = code, index


def uplift_accumulate(g, cams: Sequence, region_maps: np.ndarray, code_atoms: np.ndarray,
                      code_coefs: np.ndarray, code_row0: np.ndarray, num_regions: np.ndarray,
                      L: int, K: int, W: Optional[np.ndarray] = None, Z: Optional[np.ndarray] = None):
    """Eq. 5 accumulation over the given views.  Returns (W f64 [G,L], Z f64 [G], frags int64 [V])."""
    G = g.count
    V = len(cams)
    W = np.zeros((G, L), dtype=np.float64) if W is None else W
    Z = np.zeros(G, dtype=np.float64) if Z is None else Z
    frags = np.zeros(V, dtype=np.int64)
    ids = np.ascontiguousarray(region_maps, dtype=np.uint32)
    coefs = _f32(code_coefs)
    S = coefs.shape[1]
    # code_atoms None: dense features (Eq. 3 baseline, S = L)
    atoms = None if code_atoms is None else np.ascontiguousarray(code_atoms, dtype=np.uint32)
    row0 = np.ascontiguousarray(code_row0, dtype=np.int64)
    nreg = np.ascontiguousarray(num_regions, dtype=np.int32)
    err = np.zeros(1, dtype=np.int64)
    camarr = cameras_array(cams)
    rc = lib().ora_uplift_accumulate(G, _p(_f32(g.means)), _p(_f32(g.scales)), _p(_f32(g.rotations)),
                                     _p(_f32(g.opacities)), V, camarr, _p(ids), _p(row0), _p(nreg),
                                     None if atoms is None else _p(atoms), _p(coefs), S, L, K, _p(W), _p(Z),
                                     _p(frags), _p(err))
    if rc != 0:
        raise OracleError(rc, int(err[0]))
    return W, Z, frags


def uplift_accumulate_parallel(g, cams: Sequence, region_maps: np.ndarray, code_atoms, code_coefs, code_row0,
                               num_regions, L: int, K: int, workers: int = 0):
    """The same Eq. 5 accumulation, with the views split into `workers` contiguous shards run on
    host threads (the C oracle releases the GIL: ctypes), each into its own fp64 partial, merged
    in shard order (a fixed order, SPEC.md S:324's concurrency model).  The oracle's arithmetic
    is untouched: only the view loop is distributed.  Returns (W, Z, frags) like
    uplift_accumulate (sums equal up to fp64 reassociation)."""
    from concurrent.futures import ThreadPoolExecutor
    V = len(cams)
    workers = max(1, min(V, workers or len(os.sched_getaffinity(0))))
    bounds = [(V * k // workers, V * (k + 1) // workers) for k in range(workers)]
    row0 = np.asarray(code_row0, np.int64)
    nreg = np.asarray(num_regions, np.int32)

    def shard(b):
        v0, v1 = b
        return uplift_accumulate(g, list(cams[v0:v1]), region_maps[v0:v1], code_atoms, code_coefs,
                                 row0[v0:v1], nreg[v0:v1], L, K)

    with ThreadPoolExecutor(max_workers=workers) as ex:
        parts = list(ex.map(shard, bounds))
    W, Z, frags = parts[0]
    for Wp, Zp, _ in parts[1:]:
        W += Wp
        Z += Zp
    return W, Z, np.concatenate([p[2] for p in parts])


def uplift_parallel(g, cams, region_maps, codes, L: int, K: int, workers: int = 0):
    """uplift() with the view loop on host threads (uplift_accumulate_parallel)."""
    W, Z, frags = uplift_accumulate_parallel(g, cams, region_maps, codes.atoms, codes.coefs, codes.row0,
                                             codes.num_regions, L, K, workers)
    atoms, coefs = topk(W, K)
    return W, Z, frags, atoms, coefs


def topk(W: np.ndarray, K: int) -> Tuple[np.ndarray, np.ndarray]:
    """Eq. 6 per row (value desc, atom asc; positive only; fp64 L1 renormalisation)."""
    W = np.ascontiguousarray(W, dtype=np.float64)
    G, L = W.shape
    atoms = np.empty((G, K), dtype=np.uint32)
    coefs = np.empty((G, K), dtype=np.float64)
    lib().ora_topk(G, _p(W), L, K, _p(atoms), _p(coefs))
    return atoms, coefs


def uplift(g, cams, region_maps, codes, L: int, K: int):
    """Whole Algorithm 1: accumulate every view, then Top-K + L1 renormalise."""
    W, Z, frags = uplift_accumulate(g, cams, region_maps, codes.atoms, codes.coefs, codes.row0,
                                    codes.num_regions, L, K)
    atoms, coefs = topk(W, K)
    return W, Z, frags, atoms, coefs


def entropy(W: np.ndarray) -> np.ndarray:
    """H(w_i) = -sum_l w_il ln w_il of the aggregated coefficient
    distribution before Top-K, w_i = W_i / sum_l W_il (Z cancels); 0 ln 0 = 0; NaN for W_i = 0.
    Plain float64 numpy."""
    W = np.asarray(W, dtype=np.float64)
    S = W.sum(axis=1)
    with np.errstate(divide="ignore", invalid="ignore"):
        w = W / S[:, None]
        terms = np.where(w > 0, w * np.log(np.where(w > 0, w, 1.0)), 0.0)
        H = -terms.sum(axis=1)
    H[~(S > 0)] = np.nan
    return H
