"""User-facing Python API over the C ABI (torch tensors for device memory and streams).

    up = SparseUplift(gaussians, L=64, K=4)          # scoup_uplift_init
    up.add_views(cameras, region_ids, codes)         # scoup_uplift_add_views  (Eq. 5)
    atoms, coefs = up.finalize()                     # scoup_uplift_finalize_topk (Eq. 6)

PyTorch only provides device memory (the W/Z accumulators are torch tensors so they can
feed `torch.distributed.reduce_scatter_tensor` directly) and the current CUDA stream.
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from . import abi


def _torch():
    import torch
    return torch


class SparseUplift:
    """Uplift of one or several fused semantic levels on one device (Algorithm 1,
    P:347-372; levels > 1: SURVEY.md §8(f) NEXT-1, one raster pass feeds every level)."""

    def __init__(self, gaussians, L: int, K: int, device: int = 0, rows_padded: int = 0,
                 stream=None, levels: int = 1):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("SparseUplift needs a CUDA device (there is no CPU fallback)")
        self.device = torch.device("cuda", device)
        self.L, self.K = int(L), int(K)
        G = int(gaussians.means.shape[0])
        self.G = G
        self.rows_padded = int(rows_padded) if rows_padded else G
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.levels = int(levels)
        shape = (max(1, self.rows_padded), self.L) if self.levels == 1 else (self.levels, max(1, self.rows_padded), self.L)
        self.W = torch.empty(shape, dtype=torch.float32, device=self.device)
        self.Z = torch.empty((max(1, self.rows_padded),), dtype=torch.float32, device=self.device)
        keep = [self._as_input(a) for a in (gaussians.means, gaussians.scales, gaussians.rotations,
                                            gaussians.opacities)]
        self._h = abi.scoup_uplift_init_levels(device, self.stream.cuda_stream, G, *keep, self.levels, self.L,
                                               self.K, self.W, self.Z, self.rows_padded)
        self._keep = keep  # device inputs must outlive the stream point of init

    def _as_input(self, a):
        torch = _torch()
        if isinstance(a, np.ndarray):
            return np.ascontiguousarray(a, dtype=np.float32)
        return a.contiguous()

    def add_views(self, cameras: Sequence, region_ids, codes, contributions_out=None):
        """region_ids: [V,H,W] uint32 numpy (host) or int32/uint32 torch tensor (device or host).
        codes: synth.Codes-like (atoms [rows,S] u32, coefs [rows,S] f32, row0 [V], num_regions [V]).
        With levels > 1: a sequence of per-level region maps and a sequence of per-level codes."""
        def prep(c):  # c.atoms None: dense region features (Eq. 3 baseline), S == L
            atoms = c.atoms if not isinstance(c.atoms, np.ndarray) else np.ascontiguousarray(c.atoms, np.uint32)
            coefs = c.coefs if not isinstance(c.coefs, np.ndarray) else np.ascontiguousarray(c.coefs, np.float32)
            return atoms, coefs
        if self.levels == 1:
            atoms, coefs = prep(codes)
            S = int(coefs.shape[1])
            abi.scoup_uplift_add_views(self._h, list(cameras), region_ids, codes.row0, codes.num_regions,
                                       atoms, coefs, S, contributions_out)
            return
        if len(region_ids) != self.levels or len(codes) != self.levels:
            raise ValueError(f"expected {self.levels} region maps and code tables")
        pc = [prep(c) for c in codes]
        S = int(pc[0][1].shape[1])
        row0 = np.stack([np.asarray(c.row0, np.int64) for c in codes])
        nreg = np.stack([np.asarray(c.num_regions, np.int32) for c in codes])
        abi.scoup_uplift_add_views_levels(self._h, list(cameras), list(region_ids), row0, nreg,
                                          [a for a, _ in pc], [c for _, c in pc], S, contributions_out)

    def finalize(self, first_row: int = 0, num_rows: Optional[int] = None, W_rows=None, Z_rows=None,
                 out_atoms=None, out_coefs=None, level: int = 0):
        """Eq. 6 on rows [first_row, first_row+num_rows) of `level`.  Returns (atoms u32->int32 view, coefs)."""
        torch = _torch()
        if num_rows is None:
            num_rows = (W_rows.shape[0] if W_rows is not None else self.G - first_row)
        if out_atoms is None:
            out_atoms = torch.empty((num_rows, self.K), dtype=torch.int32, device=self.device)
        if out_coefs is None:
            out_coefs = torch.empty((num_rows, self.K), dtype=torch.float32, device=self.device)
        abi.scoup_uplift_finalize_topk_level(self._h, level, first_row, num_rows, W_rows, Z_rows, out_atoms,
                                             out_coefs)
        return out_atoms, out_coefs

    def finalize_with_entropy(self, first_row: int = 0, num_rows=None, level: int = 0):
        """Eq. 6 codes plus the pre-Top-K coefficient entropy H_i of each row."""
        torch = _torch()
        num_rows = self.G - first_row if num_rows is None else num_rows
        atoms = torch.empty((num_rows, self.K), dtype=torch.int32, device=self.device)
        coefs = torch.empty((num_rows, self.K), dtype=torch.float32, device=self.device)
        H = torch.empty((num_rows,), dtype=torch.float32, device=self.device)
        abi.scoup_uplift_finalize_topk_entropy(self._h, level, first_row, num_rows, None, None, atoms, coefs, H)
        return atoms, coefs, H

    def render(self, cameras: Sequence, atoms, coefs, out=None):
        """Eq. 7: per-pixel sum of the stored K-sparse codes w_hat_i e_i(v,p) -> [V, H, W, L] float32."""
        torch = _torch()
        cams = list(cameras)
        if out is None:
            out = torch.empty((len(cams), cams[0].height, cams[0].width, self.L), dtype=torch.float32,
                              device=self.device)
        abi.scoup_uplift_render_views(self._h, cams, atoms.contiguous(), coefs.contiguous(), int(atoms.shape[1]), out)
        return out

    def decode(self, W_hat, C, out=None):
        """Eq. 8: F = W_hat C (codebook C [L, D]); W_hat [..., L] -> F [..., D] float32."""
        torch = _torch()
        P = W_hat.numel() // self.L
        D = int(C.shape[1])
        if out is None:
            out = torch.empty(tuple(W_hat.shape[:-1]) + (D,), dtype=torch.float32, device=self.device)
        abi.scoup_uplift_decode(self._h, P, W_hat.contiguous(), C.contiguous(), D, out)
        return out

    def reset(self):
        abi.scoup_uplift_reset(self._h)

    def stats(self) -> dict:
        return abi.scoup_uplift_get_stats(self._h)

    def set_counters(self, enable: bool = True):
        abi.scoup_uplift_set_counters(self._h, enable)

    def set_pipeline(self, contexts: int = 2):
        """1: every batch step in order on one stream (per-kernel event times = each kernel's own
        duration); 2 (default): two overlapping pipeline contexts."""
        abi.scoup_uplift_set_pipeline(self._h, contexts)

    def set_timing(self, enable: bool = True):
        abi.scoup_uplift_set_timing(self._h, enable)

    def timing(self) -> dict:
        return abi.scoup_uplift_get_timing(self._h)

    def close(self):
        if getattr(self, "_h", None):
            abi.scoup_uplift_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
