"""Thin Python wrapper of include/scoup_sparse_coding.h: 2D sparse coding of region features
into SCOUP's region codes (Eq. 4; recipe P:97).

Argument marshalling only -- every step runs in libscoup.so's kernels (no CPU fallback)."""
from __future__ import annotations

from . import abi


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("SparseCoder needs CUDA (no CPU fallback)")
    return torch


class SparseCoder:
    """Codebook C [L, D] and per-region logits Z [R, L] for region features F [R, D] (a float32
    CUDA tensor, kept referenced by this object)."""

    def __init__(self, features, L: int, K: int, stream=None):
        torch = _torch()
        self.F = features.contiguous().float()
        self.R, self.D = self.F.shape
        self.L, self.K = int(L), int(K)
        self.device = self.F.device
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._h = abi.scoup_sc_init(self.device.index or 0, self.stream.cuda_stream, self.R, self.D, self.L, self.K,
                                    self.F)

    def kmeans(self, uniforms, fallback, max_iter: int = 100) -> int:
        """k-means++ seeding with the caller's draws (uniforms [L], fallback [L, D]) + Lloyd;
        then Z = 10 cos(f, C), Adam state zero.  Returns the Lloyd iterations run."""
        return abi.scoup_sc_kmeans(self._h, uniforms, fallback, max_iter)

    def state(self):
        """Views (torch tensors on the handle's memory) of C, Z, mC, vC, mZ, vZ and the step t."""
        torch = _torch()
        ptrs, t = abi.scoup_sc_get_state(self._h)
        shapes = [(self.L, self.D), (self.R, self.L), (self.L, self.D), (self.L, self.D), (self.R, self.L),
                  (self.R, self.L)]
        out = []
        for p, shp in zip(ptrs, shapes):
            n = shp[0] * shp[1]
            out.append(_wrap(p, n, self.device).view(*shp))
        return out, t

    def set_state(self, C=None, Z=None, mC=None, vC=None, mZ=None, vZ=None, t: int = 0):
        abi.scoup_sc_set_state(self._h, C, Z, mC, vC, mZ, vZ, t)

    def train(self, epochs: int, lr: float = 7e-4, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8):
        """`epochs` full-batch Adam epochs; returns the per-epoch loss (float32 CUDA tensor)."""
        torch = _torch()
        loss = torch.empty(max(epochs, 1), dtype=torch.float32, device=self.device)
        abi.scoup_sc_train(self._h, epochs, lr, beta1, beta2, eps, loss)
        return loss[:epochs]

    def encode(self):
        """Hard codes: atoms int32 (uint32 bit pattern) [R, K] and coefs float32 [R, K]."""
        torch = _torch()
        atoms = torch.empty((self.R, self.K), dtype=torch.int32, device=self.device)
        coefs = torch.empty((self.R, self.K), dtype=torch.float32, device=self.device)
        abi.scoup_sc_encode(self._h, atoms, coefs)
        return atoms, coefs

    def close(self):
        if getattr(self, "_h", None):
            abi.scoup_sc_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _wrap(ptr: int, n: int, device):
    """A float32 tensor view of n floats of device memory owned by the library."""
    import torch

    class _Holder:
        def __init__(self):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3,
                                             "strides": None}
    return torch.as_tensor(_Holder(), device=device)
