"""Thin ctypes binding of libscoup.so (include/scoup.h) -- argument marshalling only.

Every step of the path runs in the CUDA library; this module converts torch tensors /
numpy arrays to pointers and status codes to exceptions.  There is no fallback: if the
extension is missing or fails to load, `lib()` raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# SCOUP_LIB: an alternative in-tree build of the same library (A/B kernel variants)
LIB_PATH = os.environ.get("SCOUP_LIB") or os.path.join(HERE, "libscoup.so")

SCOUP_NONE = 0xFFFFFFFF
STATUS = {0: "SCOUP_OK", 1: "SCOUP_EINVAL", 2: "SCOUP_EDATA", 3: "SCOUP_ECUDA", 4: "SCOUP_ENOMEM",
          5: "SCOUP_ESTATE", 6: "SCOUP_EUNSUPPORTED"}


class ScoupError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class scoup_camera(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("width", C.c_int32), ("height", C.c_int32), ("world_to_camera", C.c_float * 16)]


class scoup_stats(C.Structure):
    _fields_ = [("views", C.c_int64), ("contributions", C.c_int64), ("tile_entries", C.c_int64),
                ("visible", C.c_int64), ("support_tests", C.c_int64), ("kernel_launches", C.c_int64),
                ("cub_launches", C.c_int64), ("lane_evaluations", C.c_int64), ("batches", C.c_int64 * 2),
                ("near_frac_changes", C.c_int64), ("host_map_chunks", C.c_int64), ("near_frac", C.c_double),
                ("global_reds", C.c_int64), ("view_batch", C.c_int64)]


class scoup_timing(C.Structure):
    _fields_ = [("preprocess_ms", C.c_double), ("binning_ms", C.c_double), ("raster_ms", C.c_double),
                ("topk_ms", C.c_double), ("raster_launches", C.c_int64), ("views_timed", C.c_int64)]


EXPORTS = ["scoup_uplift_init", "scoup_uplift_init_levels", "scoup_uplift_add_views",
           "scoup_uplift_add_views_levels", "scoup_uplift_finalize_topk", "scoup_uplift_finalize_topk_level",
           "scoup_uplift_render_views", "scoup_uplift_decode", "scoup_uplift_finalize_topk_peers", "scoup_uplift_finalize_topk_entropy",
           "scoup_ipc_export", "scoup_ipc_import", "scoup_ipc_close",
           "scoup_uplift_reset", "scoup_uplift_get_accumulators", "scoup_uplift_get_stats",
           "scoup_uplift_set_counters", "scoup_uplift_set_timing", "scoup_uplift_get_timing",
           "scoup_uplift_set_pipeline", "scoup_uplift_free", "scoup_last_error", "scoup_version",
           # include/scoup_sparse_coding.h
           "scoup_sc_init", "scoup_sc_kmeans", "scoup_sc_set_state", "scoup_sc_get_state", "scoup_sc_train",
           "scoup_sc_encode", "scoup_sc_free",
           # include/scoup_diag.h (measurement helpers)
           "scoup_diag_red_rate", "scoup_diag_set_binsort_segment", "scoup_diag_set_raster2_slots", "scoup_diag_last_error"]

_lib = None


def lib():
    """Load libscoup.so (raises if it is missing -- there is no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libscoup.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        P, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        L.scoup_uplift_init.argtypes = [C.c_int, P, i64, P, P, P, P, i32, i32, P, P, i64, C.POINTER(P)]
        L.scoup_uplift_init_levels.argtypes = [C.c_int, P, i64, P, P, P, P, i32, i32, i32, P, P, i64, C.POINTER(P)]
        L.scoup_uplift_add_views_levels.argtypes = [P, i32, P, P, P, P, P, P, i32, P]
        L.scoup_uplift_finalize_topk_level.argtypes = [P, i32, i64, i64, P, P, P, P]
        L.scoup_uplift_render_views.argtypes = [P, i32, P, P, P, i32, P]
        L.scoup_uplift_decode.argtypes = [P, i64, P, P, i32, P]
        L.scoup_uplift_add_views.argtypes = [P, i32, P, P, P, P, P, P, i32, P]
        L.scoup_uplift_finalize_topk.argtypes = [P, i64, i64, P, P, P, P]
        L.scoup_uplift_reset.argtypes = [P]
        L.scoup_uplift_get_accumulators.argtypes = [P, C.POINTER(P), C.POINTER(P), C.POINTER(i64)]
        L.scoup_uplift_get_stats.argtypes = [P, C.POINTER(scoup_stats)]
        L.scoup_uplift_set_counters.argtypes = [P, C.c_int]
        L.scoup_uplift_set_timing.argtypes = [P, C.c_int]
        L.scoup_uplift_set_pipeline.argtypes = [P, C.c_int]
        L.scoup_uplift_get_timing.argtypes = [P, C.POINTER(scoup_timing)]
        L.scoup_uplift_free.argtypes = [P]
        L.scoup_uplift_free.restype = None
        L.scoup_last_error.restype = C.c_char_p
        L.scoup_uplift_finalize_topk_peers.argtypes = [P, i32, i64, i64, i32, P, P, P]
        L.scoup_uplift_finalize_topk_entropy.argtypes = [P, i32, i64, i64, P, P, P, P, P]
        L.scoup_ipc_export.argtypes = [P, P, C.POINTER(i64)]
        L.scoup_ipc_import.argtypes = [C.c_int, P, i64, C.POINTER(P), C.POINTER(P)]
        L.scoup_ipc_close.argtypes = [C.c_int, P]
        L.scoup_sc_init.argtypes = [C.c_int, P, i64, i32, i32, i32, P, C.POINTER(P)]
        L.scoup_sc_kmeans.argtypes = [P, P, P, i32, C.POINTER(i32)]
        L.scoup_sc_set_state.argtypes = [P, P, P, P, P, P, P, i64]
        L.scoup_sc_get_state.argtypes = [P] + [C.POINTER(P)] * 6 + [C.POINTER(i64)]
        L.scoup_sc_train.argtypes = [P, i32, C.c_float, C.c_float, C.c_float, C.c_float, P]
        L.scoup_sc_encode.argtypes = [P, P, P]
        L.scoup_sc_free.argtypes = [P]
        L.scoup_sc_free.restype = None
        L.scoup_version.restype = C.c_char_p
        L.scoup_diag_red_rate.argtypes = [C.c_int, i64, C.c_int, C.c_int, i64, C.c_int, C.POINTER(C.c_double),
                                          C.POINTER(C.c_double)]
        L.scoup_diag_red_rate.restype = C.c_int
        L.scoup_diag_last_error.restype = C.c_char_p
        L.scoup_diag_set_binsort_segment.argtypes = [C.c_int]
        L.scoup_diag_set_binsort_segment.restype = C.c_int
        L.scoup_diag_set_raster2_slots.argtypes = [C.c_int]
        L.scoup_diag_set_raster2_slots.restype = C.c_int
        for name in ["scoup_uplift_init", "scoup_uplift_init_levels", "scoup_uplift_add_views",
                     "scoup_uplift_add_views_levels", "scoup_uplift_finalize_topk", "scoup_uplift_finalize_topk_level",
                     "scoup_uplift_render_views", "scoup_uplift_decode",
                     "scoup_uplift_reset", "scoup_uplift_get_accumulators", "scoup_uplift_get_stats",
                     "scoup_uplift_set_counters", "scoup_uplift_set_timing", "scoup_uplift_get_timing",
                     "scoup_uplift_set_pipeline"]:
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        raise ScoupError(status, lib().scoup_last_error().decode())


def ptr(x) -> Optional[int]:
    """Raw pointer of a torch tensor / numpy array (must be contiguous), or None."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return x.data_ptr()
    raise TypeError(type(x))


def cameras_struct(cams: Sequence) -> C.Array:
    arr = (scoup_camera * len(cams))()
    for i, c in enumerate(cams):
        arr[i].fx, arr[i].fy, arr[i].cx, arr[i].cy = c.fx, c.fy, c.cx, c.cy
        arr[i].width, arr[i].height = c.width, c.height
        w = np.asarray(c.world_to_camera, dtype=np.float32).ravel()
        for k in range(16):
            arr[i].world_to_camera[k] = float(w[k])
    return arr


# ---- the C entry points, same names -------------------------------------------------

def scoup_uplift_init(device: int, stream: int, num_gaussians: int, means, scales, rotations, opacities,
                      L: int, K: int, W=None, Z=None, rows_padded: int = 0) -> int:
    h = C.c_void_p()
    _check(lib().scoup_uplift_init(device, stream or None, num_gaussians, ptr(means), ptr(scales),
                                   ptr(rotations), ptr(opacities), L, K, ptr(W), ptr(Z), rows_padded,
                                   C.byref(h)))
    return h.value


def scoup_uplift_init_levels(device: int, stream: int, num_gaussians: int, means, scales, rotations, opacities,
                             num_levels: int, L: int, K: int, W=None, Z=None, rows_padded: int = 0) -> int:
    h = C.c_void_p()
    _check(lib().scoup_uplift_init_levels(device, stream or None, num_gaussians, ptr(means), ptr(scales),
                                          ptr(rotations), ptr(opacities), num_levels, L, K, ptr(W), ptr(Z),
                                          rows_padded, C.byref(h)))
    return h.value


def _ptr_array(xs) -> C.Array:
    arr = (C.c_void_p * len(xs))()
    for i, x in enumerate(xs):
        arr[i] = ptr(x)
    return arr


def scoup_uplift_add_views_levels(h: int, cameras: Sequence, region_ids: Sequence, code_row0, num_regions,
                                  code_atoms: Sequence, code_coefs: Sequence, S: int, contributions_out=None) -> None:
    """region_ids / code_atoms / code_coefs: one array per level; code_row0 / num_regions: [levels, V]."""
    row0 = np.ascontiguousarray(code_row0, dtype=np.int64)
    nreg = np.ascontiguousarray(num_regions, dtype=np.int32)
    cams = cameras_struct(cameras)
    ids, ats, cfs = _ptr_array(region_ids), _ptr_array(code_atoms), _ptr_array(code_coefs)
    _check(lib().scoup_uplift_add_views_levels(h, len(cameras), cams, ids, ptr(row0), ptr(nreg), ats, cfs, S,
                                               ptr(contributions_out)))


def scoup_uplift_finalize_topk_level(h: int, level: int, first_row: int, num_rows: int, W_rows, Z_rows, out_atoms,
                                     out_coefs) -> None:
    _check(lib().scoup_uplift_finalize_topk_level(h, level, first_row, num_rows, ptr(W_rows), ptr(Z_rows),
                                                  ptr(out_atoms), ptr(out_coefs)))


def scoup_uplift_render_views(h: int, cameras: Sequence, code_atoms, code_coefs, K: int, out) -> None:
    _check(lib().scoup_uplift_render_views(h, len(cameras), cameras_struct(cameras), ptr(code_atoms), ptr(code_coefs),
                                           K, ptr(out)))


def scoup_uplift_decode(h: int, num_pixels: int, W_hat, C, D: int, F) -> None:
    _check(lib().scoup_uplift_decode(h, num_pixels, ptr(W_hat), ptr(C), D, ptr(F)))


def scoup_uplift_add_views(h: int, cameras: Sequence, region_ids, code_row0, num_regions, code_atoms,
                           code_coefs, S: int, contributions_out=None) -> None:
    row0 = np.ascontiguousarray(code_row0, dtype=np.int64)
    nreg = np.ascontiguousarray(num_regions, dtype=np.int32)
    cams = cameras_struct(cameras)
    _check(lib().scoup_uplift_add_views(h, len(cameras), cams, ptr(region_ids), ptr(row0), ptr(nreg),
                                        ptr(code_atoms), ptr(code_coefs), S, ptr(contributions_out)))


def scoup_uplift_finalize_topk(h: int, first_row: int, num_rows: int, W_rows, Z_rows, out_atoms,
                               out_coefs) -> None:
    _check(lib().scoup_uplift_finalize_topk(h, first_row, num_rows, ptr(W_rows), ptr(Z_rows),
                                            ptr(out_atoms), ptr(out_coefs)))


def scoup_uplift_reset(h: int) -> None:
    _check(lib().scoup_uplift_reset(h))


def scoup_uplift_get_accumulators(h: int):
    W, Z, n = C.c_void_p(), C.c_void_p(), C.c_int64()
    _check(lib().scoup_uplift_get_accumulators(h, C.byref(W), C.byref(Z), C.byref(n)))
    return W.value, Z.value, n.value


def scoup_uplift_get_stats(h: int) -> dict:
    s = scoup_stats()
    _check(lib().scoup_uplift_get_stats(h, C.byref(s)))
    out = {k: getattr(s, k) for k, _ in scoup_stats._fields_}
    out["batches"] = list(out["batches"])
    return out


def scoup_uplift_set_counters(h: int, enable: bool) -> None:
    _check(lib().scoup_uplift_set_counters(h, 1 if enable else 0))


def scoup_uplift_set_pipeline(h: int, contexts: int) -> None:
    _check(lib().scoup_uplift_set_pipeline(h, int(contexts)))


def scoup_uplift_set_timing(h: int, enable: bool) -> None:
    _check(lib().scoup_uplift_set_timing(h, 1 if enable else 0))


def scoup_uplift_get_timing(h: int) -> dict:
    t = scoup_timing()
    _check(lib().scoup_uplift_get_timing(h, C.byref(t)))
    return {k: getattr(t, k) for k, _ in scoup_timing._fields_}


def scoup_uplift_free(h: int) -> None:
    if h:
        lib().scoup_uplift_free(h)


def scoup_last_error() -> str:
    return lib().scoup_last_error().decode()


def scoup_version() -> str:
    return lib().scoup_version().decode()


# ---- 2D sparse coding (include/scoup_sparse_coding.h) -------------------------------------------

def scoup_sc_init(device: int, stream: int, R: int, D: int, L: int, K: int, features) -> int:
    h = C.c_void_p()
    _check(lib().scoup_sc_init(device, stream or None, R, D, L, K, ptr(features), C.byref(h)))
    return h.value


def scoup_sc_kmeans(h: int, uniforms, fallback, max_iter: int) -> int:
    import numpy as np
    u = np.ascontiguousarray(uniforms, dtype=np.float64)
    fb = fallback if hasattr(fallback, "data_ptr") else np.ascontiguousarray(fallback, dtype=np.float32)
    it = C.c_int32(0)
    _check(lib().scoup_sc_kmeans(h, u.ctypes.data, ptr(fb), max_iter, C.byref(it)))
    return it.value


def scoup_sc_set_state(h: int, C_=None, Z=None, mC=None, vC=None, mZ=None, vZ=None, t: int = 0) -> None:
    _check(lib().scoup_sc_set_state(h, ptr(C_), ptr(Z), ptr(mC), ptr(vC), ptr(mZ), ptr(vZ), t))


def scoup_sc_get_state(h: int):
    ps = [C.c_void_p() for _ in range(6)]
    t = C.c_int64(0)
    _check(lib().scoup_sc_get_state(h, *[C.byref(x) for x in ps], C.byref(t)))
    return [x.value for x in ps], t.value


def scoup_sc_train(h: int, epochs: int, lr: float, beta1: float, beta2: float, eps: float, loss_out=None) -> None:
    _check(lib().scoup_sc_train(h, epochs, lr, beta1, beta2, eps, ptr(loss_out)))


def scoup_sc_encode(h: int, atoms, coefs) -> None:
    _check(lib().scoup_sc_encode(h, ptr(atoms), ptr(coefs)))


def scoup_sc_free(h: int) -> None:
    if h:
        lib().scoup_sc_free(h)


# ---- fused cross-rank reduction + Top-K and its CUDA IPC plumbing (include/scoup.h) ------------

IPC_HANDLE_BYTES = 64


def scoup_uplift_finalize_topk_peers(h: int, level: int, first_row: int, num_rows: int, W_peers: Sequence[int],
                                     out_atoms, out_coefs) -> None:
    arr = (C.c_void_p * len(W_peers))(*W_peers)
    _check(lib().scoup_uplift_finalize_topk_peers(h, level, first_row, num_rows, len(W_peers), arr, ptr(out_atoms),
                                                  ptr(out_coefs)))


def scoup_ipc_export(dptr: int):
    """-> (handle bytes, offset of dptr inside its allocation)."""
    buf = C.create_string_buffer(IPC_HANDLE_BYTES)
    off = C.c_int64(0)
    _check(lib().scoup_ipc_export(dptr, buf, C.byref(off)))
    return bytes(buf.raw), off.value


def scoup_ipc_import(device: int, handle: bytes, offset: int):
    """-> (mapped pointer, mapping base for scoup_ipc_close)."""
    buf = C.create_string_buffer(handle, IPC_HANDLE_BYTES)
    d, b = C.c_void_p(), C.c_void_p()
    _check(lib().scoup_ipc_import(device, buf, offset, C.byref(d), C.byref(b)))
    return d.value, b.value


def scoup_ipc_close(device: int, base: int) -> None:
    _check(lib().scoup_ipc_close(device, base))


def scoup_uplift_finalize_topk_entropy(h: int, level: int, first_row: int, num_rows: int, W_rows, Z_rows, out_atoms,
                                       out_coefs, out_entropy) -> None:
    _check(lib().scoup_uplift_finalize_topk_entropy(h, level, first_row, num_rows, ptr(W_rows), ptr(Z_rows),
                                                    ptr(out_atoms), ptr(out_coefs), ptr(out_entropy)))


def scoup_diag_red_rate(device: int, buffer_bytes: int, scattered: bool, vec4: bool, reds_per_launch: int,
                        launches: int):
    """include/scoup_diag.h: (float adds per second, ms per launch) of red.global.add.f32 / v4."""
    rate, ms = C.c_double(), C.c_double()
    st = lib().scoup_diag_red_rate(device, int(buffer_bytes), int(scattered), int(vec4), int(reds_per_launch),
                                   int(launches), C.byref(rate), C.byref(ms))
    if st != 0:
        raise ScoupError(st, lib().scoup_diag_last_error().decode())
    return rate.value, ms.value


def scoup_diag_set_raster2_slots(slots: int) -> None:
    """include/scoup_diag.h: force the fused raster's 4- or 8-slot variant (0: adaptive)."""
    st = lib().scoup_diag_set_raster2_slots(int(slots))
    if st != 0:
        raise ScoupError(st, lib().scoup_diag_last_error().decode())


def scoup_diag_set_binsort_segment(entries_per_segment: int) -> None:
    """include/scoup_diag.h: force the binning sort's segment length (0: adaptive)."""
    st = lib().scoup_diag_set_binsort_segment(int(entries_per_segment))
    if st != 0:
        raise ScoupError(st, lib().scoup_diag_last_error().decode())
