"""Pins for the 2D sparse-coding oracle (oracle/sparse_coding.py; Eq. 4 P:93-97, P:158;
SURVEY.md §8(f) NEXT-4; DESIGN.md §14 readings R-SC1..R-SC7).  CPU only.

Each pin checks the oracle against something other than itself: closed forms of the soft top-K
softmax, central finite differences of the loss for the analytic gradients, the
closed-form first Adam step, brute-force optimal k-means on tiny separable sets, the Lloyd
fixpoint conditions, and training properties."""
from __future__ import annotations

import itertools
import math

import numpy as np
import pytest

from oracle import sparse_coding as sc
from paper_2605_13600_b200 import synth


def test_soft_topk_closed_forms():
    """(4, 3, 0, ...) with K = 2 -> (e^4, e^3) / (e^4 + e^3); equal logits with K = L
    -> uniform; one dominant logit with K = 1 -> one-hot; the weights are softmax(z) restricted
    to the kept set and renormalised."""
    z = np.zeros((1, 8), np.float32)
    z[0, :2] = (4.0, 3.0)
    sel, w = sc.soft_topk(z, 2)
    assert sel.tolist() == [[0, 1]]
    assert np.allclose(w[0], [math.e**4 / (math.e**4 + math.e**3), math.e**3 / (math.e**4 + math.e**3)], rtol=1e-14)
    assert abs(w[0, 0] - 0.7311) < 1e-4
    W = sc.soft_topk_dense(np.full((1, 8), 0.3, np.float32), 8)
    assert np.allclose(W, 1.0 / 8, rtol=1e-14)
    z = np.zeros((1, 8), np.float32)
    z[0, 5] = 20.0
    assert np.array_equal(sc.soft_topk_dense(z, 1), np.eye(8)[5:6])
    # renormalised softmax: p = softmax(z) over all L, kept K largest, divided by their sum
    z = np.random.default_rng(0).normal(size=(3, 10)).astype(np.float32)
    p = np.exp(z.astype(np.float64))
    p /= p.sum(axis=1, keepdims=True)
    for r in range(3):
        keep = np.argsort(-p[r], kind="stable")[:4]
        ref = np.zeros(10)
        ref[keep] = p[r, keep] / p[r, keep].sum()
        assert np.allclose(sc.soft_topk_dense(z[r:r + 1], 4)[0], ref, rtol=1e-12, atol=1e-15)


def test_soft_topk_ties_lower_index():
    """R-SC1: equal logits keep the lower indices (S:218 'ties broken toward the lower index')."""
    z = np.array([[1.0, 2.0, 2.0, 0.5, 2.0, 2.0]], np.float32)
    sel, w = sc.soft_topk(z, 3)
    assert sel.tolist() == [[1, 2, 4]]
    assert np.allclose(w, 1.0 / 3)


def _problem(R=6, L=7, D=9, seed=3):
    rng = np.random.default_rng(seed)
    Z = rng.normal(scale=2.0, size=(R, L))
    C = rng.normal(size=(L, D))
    F = rng.normal(size=(R, D))
    return Z, C, F


@pytest.mark.parametrize("K", [1, 3, 7])
def test_gradients_match_finite_differences(K):
    """R-SC3: the analytic gradients of loss = mean(1 - cos(w C, f)) equal central differences
    of the loss itself (h = 1e-6, float64), for Z (through the restricted softmax; entries outside
    the kept set have zero gradient) and for C."""
    Z, C, F = _problem()
    loss, gZ, gC = sc.loss_and_grads(Z, C, F, K)
    h = 1e-6
    for (r, l) in itertools.product(range(Z.shape[0]), range(Z.shape[1])):
        Zp, Zm = Z.copy(), Z.copy()
        Zp[r, l] += h
        Zm[r, l] -= h
        fd = (sc.loss_and_grads(Zp, C, F, K)[0] - sc.loss_and_grads(Zm, C, F, K)[0]) / (2 * h)
        assert abs(fd - gZ[r, l]) < 1e-7 + 1e-5 * abs(fd), (r, l, fd, gZ[r, l])
    for (a, d) in itertools.product(range(C.shape[0]), range(C.shape[1])):
        Cp, Cm = C.copy(), C.copy()
        Cp[a, d] += h
        Cm[a, d] -= h
        fd = (sc.loss_and_grads(Z, Cp, F, K)[0] - sc.loss_and_grads(Z, Cm, F, K)[0]) / (2 * h)
        assert abs(fd - gC[a, d]) < 1e-7 + 1e-5 * abs(fd), (a, d, fd, gC[a, d])


def test_loss_closed_form_cases():
    """cos(w C, f) = 1 when f is the reconstruction itself (loss 0), = -1 for its negation
    (loss 2); the loss is invariant to scaling f."""
    rng = np.random.default_rng(1)
    C = rng.normal(size=(5, 6))
    Z = rng.normal(size=(4, 5))
    x = sc.soft_topk_dense(Z, 2) @ C
    assert abs(sc.loss_and_grads(Z, C, x, 2)[0]) < 1e-14
    assert abs(sc.loss_and_grads(Z, C, -x, 2)[0] - 2.0) < 1e-14
    F = rng.normal(size=(4, 6))
    assert abs(sc.loss_and_grads(Z, C, F, 2)[0] - sc.loss_and_grads(Z, C, 7.5 * F, 2)[0]) < 1e-14


def test_adam_first_step_closed_form():
    """R-SC4: from zero moments the bias-corrected first step is theta - lr g / (|g| + eps), and
    the second step with the same gradient is theta_1 - lr g / (|g| + eps) again."""
    h = sc.AdamHyper()
    g = np.array([0.3, -2.0, 1e-3, 0.0])
    th = np.array([1.0, 2.0, 3.0, 4.0])
    t1, m, v = sc.adam_step(th, np.zeros(4), np.zeros(4), g, 1, h)
    assert np.allclose(t1, th - h.lr * g / (np.abs(g) + h.eps), rtol=1e-15, atol=1e-18)
    t2, _, _ = sc.adam_step(t1, m, v, g, 2, h)
    assert np.allclose(t2, t1 - h.lr * g / (np.abs(g) + h.eps), rtol=1e-12, atol=1e-18)


def test_kmeans_distinct_rows_is_a_permutation():
    """R = L distinct rows -> the codebook is a permutation of the rows."""
    F = np.random.default_rng(2).normal(size=(6, 5)).astype(np.float32)
    u, E = synth.make_kmeans_draws(6, 5, seed=0)
    C = sc.kmeans_init(F, 6, u, E)
    got = sorted(map(tuple, np.round(C, 6)))
    assert got == sorted(map(tuple, np.round(F.astype(np.float64), 6)))


def test_kmeans_identical_rows_uses_fallback():
    """all rows identical, L = 2 -> one atom is the row, the other the fallback vector."""
    F = np.tile(np.array([[0.6, 0.8, 0.0]], np.float32), (5, 1))
    u, E = synth.make_kmeans_draws(2, 3, seed=0)
    C = sc.kmeans_init(F, 2, u, E)
    assert np.allclose(C[0], F[0]) and np.allclose(C[1], E[1])


def test_kmeans_separable_matches_brute_force():
    """k-means on 3 well-separated clusters of 4 points (L = 3): the result's WCSS equals the
    brute-force optimum over all 3^12 labelings (computed here directly), and the centres are
    the fixpoint (each the mean of its nearest rows)."""
    rng = np.random.default_rng(5)
    centres = np.array([[0, 0], [10, 0], [0, 10]], float)
    F = (np.repeat(centres, 4, axis=0) + rng.normal(scale=0.3, size=(12, 2))).astype(np.float32)
    u, E = synth.make_kmeans_draws(3, 2, seed=1)
    C = sc.kmeans_init(F, 3, u, E)
    best = math.inf
    Fd = F.astype(np.float64)
    for lab in itertools.product(range(3), repeat=12):
        lab = np.array(lab)
        w = 0.0
        for j in range(3):
            rows = Fd[lab == j]
            if len(rows):
                w += ((rows - rows.mean(axis=0)) ** 2).sum()
        best = min(best, w)
    assert abs(sc.wcss(F, C) - best) < 1e-9 * max(1.0, best)
    a = sc.assign(Fd, C)
    for j in range(3):
        assert np.allclose(C[j], Fd[a == j].mean(axis=0))


def test_training_properties():
    """a single region equal to a codebook row ends as a near one-hot code with cosine
    >= 0.999; on planted K-sparse data the loss decreases over every 50-epoch window."""
    F = np.array([[0.0, 0.6, 0.8, 0.0]], np.float32)
    u, E = synth.make_kmeans_draws(4, 4, seed=2)
    C, Z, losses = sc.train(F, 4, 2, 50, u, E)
    W = sc.soft_topk_dense(Z, 2)
    assert W.max() > 1 - 1e-3
    x = W @ C.astype(np.float64)
    assert float((x[0] @ F[0]) / np.linalg.norm(x[0]) / np.linalg.norm(F[0])) >= 0.999
    rf = synth.make_region_features(60, 16, 8, 2, noise=0.01, seed=4)
    u, E = synth.make_kmeans_draws(8, 16, seed=4)
    _, _, losses = sc.train(rf.F, 8, 2, 300, u, E)
    win = losses.reshape(-1, 50).mean(axis=1)
    assert np.all(np.diff(win) < 0), win
