"""CPU oracle for SCOUP's 2D sparse coding (Eq. 4) --
TEST INFRASTRUCTURE ONLY (imported by tests/ and the benchmark's cpu_baseline leg, never by the
product path, and sharing no code with it).

The paper states the problem and the recipe in prose:

* Eq. 4: F_v(p) ~ W_v(p) C with ||W||_0 <= K, W >= 0, 1^T W = 1; codes are per SAM
  region, shared by its pixels.
* "a normalized soft top-K softmax over learnable region-wise logits, optimizing these logits
  jointly with the codebook via a cosine reconstruction loss".
* "4,000 epochs using the Adam optimizer with a learning rate of 0.0007, with codebook size
  L=64 and K=4 ... The codebook is initialized with the k-means algorithm on CLIP-encoded masked
  regions".

Everything the paper leaves open is fixed by DESIGN.md §14's readings (R-SC1..R-SC8), which
follow SPEC.md's operations:

* soft_topk (R-SC1): p = softmax(z); keep the K largest p (ties -> lower index), zero the rest,
  renormalise.  softmax is strictly increasing in z, so the kept set is the K largest *logits*;
  the selection is made on the float32 logits (the kernel's precision, so both sides take the
  same integer decision) and the weights are exp(z_k - max z) / sum over the kept set.
* loss (R-SC2): (1/R) sum_r (1 - cos(w_r C, f_r)), cos(x, f) = x.f / (|x| |f|) with |x| floored
  at 1e-12 (|f| > 0 is an input requirement).
* gradients (R-SC3) flow only through the kept support ("zeroed entries receive zero gradient").
* full-batch Adam (R-SC4): PyTorch semantics, betas (0.9, 0.999), eps 1e-8, bias-corrected, on
  every parameter (zero-gradient entries still move by their momentum); Z and C are updated
  from the gradients of the same state (one epoch = one full-batch step).
* logits initialised as 10 cos(f_r, C_l) against the k-means codebook (R-SC5).
* k-means (R-SC6): k-means++ seeding driven by caller-supplied uniforms u[0..L-1] (first centre
  = row floor(u_0 R); then the first row whose running sum of D^2 exceeds u_j sum D^2), with
  caller-supplied unit vectors for atoms that have no distinct row left (sum D^2 = 0, e.g.
  R < L); Lloyd iterations (nearest centre, ties -> lower index; a centre with no rows keeps its
  position) until the assignment is a fixpoint or 100 iterations.
* encode (R-SC7): the hard code of a region is its kept set in logit order with its weights.

Arithmetic is float64 from float32 inputs, written plainly (vectorised numpy over regions, the
formulas in the paper's notation).  Parity status: soft_topk pinned by closed forms;
the gradients pinned by central finite differences of the loss; Adam pinned by its closed form
first step; k-means pinned by brute-force optimal clustering on tiny separable sets and the
fixpoint conditions; training pinned by the planted-code recovery property.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

COS_FLOOR = 1e-12


def topk_select(z32: np.ndarray, K: int) -> np.ndarray:
    """Indices of the K largest float32 logits per row (ties -> lower index), in that order.

    z32: [R, L] float32.  Returns int64 [R, K]."""
    z32 = np.asarray(z32, dtype=np.float32)
    R, L = z32.shape
    if not 1 <= K <= L:
        raise ValueError("need 1 <= K <= L")
    # a stable sort of the negated logits: descending logit, equal logits in index order
    return np.argsort(-z32, axis=1, kind="stable")[:, :K].astype(np.int64)


def soft_topk(z: np.ndarray, K: int) -> Tuple[np.ndarray, np.ndarray]:
    """R-SC1: kept indices [R, K] and their weights [R, K] (float64, sum 1).

    The kept set is decided on float32(z); the weights use z as given (float64 logits are only
    used by the finite-difference pins)."""
    z = np.atleast_2d(np.asarray(z))
    sel = topk_select(z.astype(np.float32), K)
    zk = np.take_along_axis(z.astype(np.float64), sel, axis=1)
    ex = np.exp(zk - zk.max(axis=1, keepdims=True))
    return sel, ex / ex.sum(axis=1, keepdims=True)


def soft_topk_dense(z32: np.ndarray, K: int) -> np.ndarray:
    """soft_topk as a dense [R, L] weight matrix (zeros outside the kept set)."""
    z32 = np.atleast_2d(np.asarray(z32, dtype=np.float32))
    sel, w = soft_topk(z32, K)
    W = np.zeros(z32.shape, dtype=np.float64)
    np.put_along_axis(W, sel, w, axis=1)
    return W


def loss_and_grads(Z32: np.ndarray, C32: np.ndarray, F32: np.ndarray, K: int):
    """R-SC2/R-SC3: loss = (1/R) sum_r (1 - cos(w_r C, f_r)) and its gradients.

    Returns (loss, gZ [R, L], gC [L, D]) in float64."""
    Z = np.asarray(Z32)
    C = np.asarray(C32).astype(np.float64)
    F = np.asarray(F32).astype(np.float64)
    R, L = Z.shape
    sel, w = soft_topk(Z, K)                          # [R, K]
    Csel = C[sel]                                      # [R, K, D]
    x = np.einsum("rk,rkd->rd", w, Csel)               # reconstruction w_r C
    nx = np.maximum(np.linalg.norm(x, axis=1), COS_FLOOR)
    nf = np.linalg.norm(F, axis=1)
    if (nf <= 0).any():
        raise ValueError("region features must be non-zero")
    xf = np.einsum("rd,rd->r", x, F)
    cos = xf / (nx * nf)
    loss = float(np.mean(1.0 - cos))
    # d loss / d x_r = -(1/R) (f / (|x||f|) - cos x / |x|^2)
    g = -(F / (nx * nf)[:, None] - (cos / nx**2)[:, None] * x) / R
    gw = np.einsum("rd,rkd->rk", g, Csel)              # d loss / d w_k = g . C_k
    gz_sel = w * (gw - np.sum(w * gw, axis=1, keepdims=True))  # through the restricted softmax
    gZ = np.zeros((R, L), dtype=np.float64)
    np.put_along_axis(gZ, sel, gz_sel, axis=1)
    gC = np.zeros_like(C)
    for k in range(K):                                 # d loss / d C_a += w_k g
        np.add.at(gC, sel[:, k], w[:, k:k + 1] * g)
    return loss, gZ, gC


@dataclass
class AdamHyper:
    lr: float = 7e-4
    beta1: float = 0.9      # R-SC4 (PyTorch default)
    beta2: float = 0.999
    eps: float = 1e-8


def adam_step(theta, m, v, g, t: int, h: AdamHyper):
    """R-SC4: one bias-corrected Adam step (step number t >= 1), float64."""
    m = h.beta1 * m + (1.0 - h.beta1) * g
    v = h.beta2 * v + (1.0 - h.beta2) * g * g
    mhat = m / (1.0 - h.beta1 ** t)
    vhat = v / (1.0 - h.beta2 ** t)
    return theta - h.lr * mhat / (np.sqrt(vhat) + h.eps), m, v


def epoch(state: dict, F32: np.ndarray, K: int, h: AdamHyper) -> Tuple[dict, float]:
    """One full-batch epoch from `state` (float32 Z, C, mZ, vZ, mC, vC and int t = steps done):
    gradients at the current state, then Adam on Z and C with step t + 1.  Returns the new state
    (float64 arrays) and the loss at the old state."""
    loss, gZ, gC = loss_and_grads(state["Z"], state["C"], F32, K)
    t = int(state["t"]) + 1
    Z, mZ, vZ = adam_step(np.asarray(state["Z"], np.float64), np.asarray(state["mZ"], np.float64),
                          np.asarray(state["vZ"], np.float64), gZ, t, h)
    C, mC, vC = adam_step(np.asarray(state["C"], np.float64), np.asarray(state["mC"], np.float64),
                          np.asarray(state["vC"], np.float64), gC, t, h)
    return {"Z": Z, "C": C, "mZ": mZ, "vZ": vZ, "mC": mC, "vC": vC, "t": t, "gZ": gZ, "gC": gC}, loss


def init_logits(F32: np.ndarray, C32: np.ndarray, scale: float = 10.0) -> np.ndarray:
    """R-SC5: z_{r,l} = 10 cos(f_r, C_l)."""
    F = np.asarray(F32, np.float64)
    C = np.asarray(C32, np.float64)
    nf = np.linalg.norm(F, axis=1)
    nc = np.maximum(np.linalg.norm(C, axis=1), COS_FLOOR)
    return scale * (F @ C.T) / (nf[:, None] * nc[None, :])


def kmeans_pp(F32: np.ndarray, L: int, uniforms: np.ndarray, fallback: np.ndarray) -> np.ndarray:
    """R-SC6 seeding: L centres (float64 [L, D])."""
    F = np.asarray(F32, np.float64)
    R, D = F.shape
    u = np.asarray(uniforms, np.float64)
    centres = np.empty((L, D))
    r0 = min(int(np.floor(u[0] * R)), R - 1)
    centres[0] = F[r0]
    d2 = np.sum((F - centres[0]) ** 2, axis=1)
    for j in range(1, L):
        tot = d2.sum()
        if tot <= 0.0:
            centres[j] = fallback[j]
        else:
            cum = np.cumsum(d2)
            r = int(np.searchsorted(cum, u[j] * tot, side="right"))
            centres[j] = F[min(r, R - 1)]
        d2 = np.minimum(d2, np.sum((F - centres[j]) ** 2, axis=1))
    return centres


def assign(F: np.ndarray, centres: np.ndarray) -> np.ndarray:
    """Nearest centre per row (squared Euclidean, ties -> lower index)."""
    d = ((F[:, None, :] - centres[None, :, :]) ** 2).sum(axis=2)
    return np.argmin(d, axis=1)  # argmin returns the first minimum


def lloyd(F32: np.ndarray, centres: np.ndarray, max_iter: int = 100) -> Tuple[np.ndarray, np.ndarray, int]:
    """R-SC6 Lloyd iterations; returns (centres, assignment, iterations run)."""
    F = np.asarray(F32, np.float64)
    c = np.array(centres, np.float64)
    a = assign(F, c)
    it = 0
    for it in range(1, max_iter + 1):
        for j in range(c.shape[0]):
            rows = F[a == j]
            if len(rows):
                c[j] = rows.mean(axis=0)
        a2 = assign(F, c)
        if np.array_equal(a2, a):
            break
        a = a2
    return c, a, it


def wcss(F32: np.ndarray, centres: np.ndarray) -> float:
    F = np.asarray(F32, np.float64)
    a = assign(F, centres)
    return float(((F - centres[a]) ** 2).sum())


def kmeans_init(F32, L: int, uniforms, fallback, max_iter: int = 100) -> np.ndarray:
    return lloyd(F32, kmeans_pp(F32, L, uniforms, fallback), max_iter)[0]


def train(F32: np.ndarray, L: int, K: int, epochs: int, uniforms, fallback, h: Optional[AdamHyper] = None,
          kmeans_iters: int = 100):
    """k-means init, logits init, `epochs` full-batch Adam epochs.  Float64 state,
    rounded to float32 between epochs like the parameters the kernel keeps.  Returns
    (C, Z, losses)."""
    h = h or AdamHyper()
    C = kmeans_init(F32, L, uniforms, fallback, kmeans_iters).astype(np.float32)
    Z = init_logits(F32, C).astype(np.float32)
    st = {"Z": Z, "C": C, "mZ": np.zeros_like(Z), "vZ": np.zeros_like(Z), "mC": np.zeros_like(C),
          "vC": np.zeros_like(C), "t": 0}
    losses: List[float] = []
    for _ in range(epochs):
        new, loss = epoch(st, F32, K, h)
        losses.append(loss)
        st = {k: (v.astype(np.float32) if isinstance(v, np.ndarray) else v) for k, v in new.items()}
    return st["C"], st["Z"], np.array(losses)


def encode(Z32: np.ndarray, K: int) -> Tuple[np.ndarray, np.ndarray]:
    """R-SC7: hard codes (atoms uint32 [R, K], coefs float32 [R, K]) in logit order."""
    sel, w = soft_topk(Z32, K)
    return sel.astype(np.uint32), w.astype(np.float32)
