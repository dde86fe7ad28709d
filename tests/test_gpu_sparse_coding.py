"""GPU parity of the 2D sparse coding kernels (include/scoup_sparse_coding.h; Eq. 4,
P:93-97) against oracle/sparse_coding.py (float64).

Tolerances: the kernels compute in float32 (sums over D features and over regions), the oracle
in float64 from the same float32 inputs; the kept set of every region is decided on the same
float32 logits on both sides (R-SC1), so the comparisons below are element-wise:
  loss 1e-5 relative; gradients (through the Adam moments) 1e-4 relative + 1e-9 absolute;
  parameters after an Adam step 2e-6 absolute (an update is lr m_hat / (sqrt(v_hat) + eps)
  <= ~lr, so this is ~1e-3 of a step)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import sparse_coding as sc
from paper_2605_13600_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


def _coder(F, L, K):
    from paper_2605_13600_b200.sparse_coding import SparseCoder
    return SparseCoder(torch.from_numpy(np.ascontiguousarray(F)).cuda(), L, K)


def _random_state(R, L, D, seed):
    rng = np.random.default_rng(seed)
    f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    return {"C": f32(rng.normal(size=(L, D))), "Z": f32(rng.normal(scale=3.0, size=(R, L))),
            "mC": f32(rng.normal(scale=1e-3, size=(L, D))), "vC": f32(rng.uniform(1e-8, 1e-6, size=(L, D))),
            "mZ": f32(rng.normal(scale=1e-3, size=(R, L))), "vZ": f32(rng.uniform(1e-8, 1e-6, size=(R, L))),
            "t": 5}


@pytest.mark.parametrize("R,D,L,K", [(300, 64, 16, 4), (1000, 512, 64, 4), (77, 96, 128, 8), (40, 33, 40, 32)])
def test_one_epoch_matches_oracle(dev, R, D, L, K):
    """One full-batch epoch from an identical float32 state (random codebook, logits and Adam
    moments, t = 5): loss, new logits, codebook and all four moments element-wise; ragged D
    (33, 96) and L (40), K up to 32, L = 128."""
    F = synth.make_region_features(R, D, min(L, 32), min(K, 4), noise=0.05, seed=R).F
    st = _random_state(R, L, D, seed=R + 1)
    h = sc.AdamHyper()
    ora, loss_o = sc.epoch(st, F, K, h)
    coder = _coder(F, L, K)
    try:
        t = {k: torch.from_numpy(v).cuda() for k, v in st.items() if k != "t"}
        coder.set_state(t["C"], t["Z"], t["mC"], t["vC"], t["mZ"], t["vZ"], st["t"])
        loss = coder.train(1, h.lr, h.beta1, h.beta2, h.eps).cpu().numpy()
        (C, Z, mC, vC, mZ, vZ), step = coder.state()
        got = {k: v.double().cpu().numpy() for k, v in zip(["C", "Z", "mC", "vC", "mZ", "vZ"], [C, Z, mC, vC, mZ, vZ])}
    finally:
        coder.close()
    assert step == st["t"] + 1
    assert abs(loss[0] - loss_o) <= 1e-5 * abs(loss_o) + 1e-7
    for k in ("mC", "vC", "mZ", "vZ"):
        assert np.allclose(got[k], ora[k], rtol=1e-4, atol=1e-9 if k[0] == "m" else 1e-12), k
    for k in ("C", "Z"):
        err = np.abs(got[k] - ora[k])
        assert err.max() <= 2e-6, (k, err.max())
    # entries outside every kept set get zero gradient: their first moment only decays
    kept = np.zeros((R, L), bool)
    np.put_along_axis(kept, sc.topk_select(st["Z"], K), True, axis=1)
    assert np.allclose(got["mZ"][~kept], 0.9 * st["mZ"][~kept].astype(np.float64), rtol=1e-6, atol=0)


def test_training_trajectory_matches_oracle(dev):
    """200 epochs from the oracle's k-means codebook and 10 cos logits (R-SC5): the per-epoch
    loss curve and the final codes agree; the loss decreases over every 50-epoch window."""
    rf = synth.make_region_features(200, 64, 16, 4, noise=0.02, seed=11)
    u, E = synth.make_kmeans_draws(16, 64, seed=11)
    C0 = sc.kmeans_init(rf.F, 16, u, E).astype(np.float32)
    Z0 = sc.init_logits(rf.F, C0).astype(np.float32)
    st = {"Z": Z0, "C": C0, "mZ": np.zeros_like(Z0), "vZ": np.zeros_like(Z0), "mC": np.zeros_like(C0),
          "vC": np.zeros_like(C0), "t": 0}
    h = sc.AdamHyper()
    losses_o = []
    for _ in range(200):
        new, loss = sc.epoch(st, rf.F, 4, h)
        losses_o.append(loss)
        st = {k: (v.astype(np.float32) if isinstance(v, np.ndarray) else v) for k, v in new.items()}
    coder = _coder(rf.F, 16, 4)
    try:
        coder.set_state(torch.from_numpy(C0).cuda(), torch.from_numpy(Z0).cuda(), t=0)
        (C, Z, mC, vC, mZ, vZ), _ = coder.state()
        for x in (mC, vC, mZ, vZ):
            x.zero_()
        torch.cuda.synchronize()
        losses = coder.train(200).cpu().numpy()
        atoms, coefs = coder.encode()
        atoms = atoms.cpu().numpy().view(np.uint32)
        coefs = coefs.cpu().numpy()
    finally:
        coder.close()
    assert np.allclose(losses, losses_o, rtol=1e-4, atol=1e-7)
    a_o, c_o = sc.encode(st["Z"], 4)
    assert (atoms == a_o).mean() > 0.99
    same = (atoms == a_o).all(axis=1)
    assert np.allclose(coefs[same], c_o[same], atol=1e-4)
    win = np.asarray(losses).reshape(-1, 50).mean(axis=1)
    assert np.all(np.diff(win) < 0)


def test_encode_matches_oracle(dev):
    """Hard codes (R-SC7): kept atoms in logit order (ties -> lower index; the logits include
    exact ties) and their soft top-K weights."""
    R, L, K, D = 500, 64, 4, 32
    F = synth.make_region_features(R, D, 16, 4, seed=3).F
    Z = np.round(np.random.default_rng(3).normal(scale=2.0, size=(R, L)), 1).astype(np.float32)  # many ties
    coder = _coder(F, L, K)
    try:
        coder.set_state(Z=torch.from_numpy(Z).cuda(), t=0)
        atoms, coefs = coder.encode()
        atoms = atoms.cpu().numpy().view(np.uint32)
        coefs = coefs.cpu().numpy()
    finally:
        coder.close()
    a_o, c_o = sc.encode(Z, K)
    assert np.array_equal(atoms, a_o)
    assert np.allclose(coefs, c_o, rtol=1e-6, atol=1e-7)


def test_kmeans_separable_clusters(dev):
    """k-means (R-SC6) on 8 well-separated clusters: the GPU codebook equals the oracle's (as a set
    of rows, 1e-4) and its WCSS agrees to 1e-5; then the logits are 10 cos(f, C)."""
    rng = np.random.default_rng(9)
    centres = rng.normal(scale=10.0, size=(8, 24))
    F = (np.repeat(centres, 50, axis=0) + rng.normal(size=(400, 24))).astype(np.float32)
    u, E = synth.make_kmeans_draws(8, 24, seed=9)
    C_o = sc.kmeans_init(F, 8, u, E)
    coder = _coder(F, 8, 2)
    try:
        coder.kmeans(u, E)
        (C, Z, *_), _ = coder.state()
        C = C.double().cpu().numpy()
        Z = Z.double().cpu().numpy()
    finally:
        coder.close()
    assert np.allclose(np.sort(C, axis=0), np.sort(C_o, axis=0), atol=1e-4)
    assert abs(sc.wcss(F, C) - sc.wcss(F, C_o)) <= 1e-5 * sc.wcss(F, C_o)
    assert np.allclose(Z, sc.init_logits(F, C.astype(np.float32)), atol=1e-4)


def test_kmeans_degenerate_cases(dev):
    """R = L distinct rows -> a permutation of the rows; identical rows, L = 2 -> the
    row and the fallback vector."""
    F = np.random.default_rng(2).normal(size=(6, 5)).astype(np.float32)
    u, E = synth.make_kmeans_draws(6, 5, seed=0)
    coder = _coder(F, 6, 2)
    try:
        coder.kmeans(u, E)
        C = coder.state()[0][0].cpu().numpy()
    finally:
        coder.close()
    assert sorted(map(tuple, np.round(C, 5))) == sorted(map(tuple, np.round(F, 5)))
    F = np.tile(np.array([[0.6, 0.8, 0.0]], np.float32), (5, 1))
    u, E = synth.make_kmeans_draws(2, 3, seed=0)
    coder = _coder(F, 2, 1)
    try:
        coder.kmeans(u, E)
        C = coder.state()[0][0].cpu().numpy()
    finally:
        coder.close()
    assert np.allclose(C[0], F[0]) and np.allclose(C[1], E[1])


def test_sparse_coding_errors(dev):
    """A zero feature row is a latched EDATA naming the row; K > L is EINVAL; L * D beyond the
    shared-memory accumulator is EUNSUPPORTED."""
    from paper_2605_13600_b200 import abi
    from paper_2605_13600_b200.sparse_coding import SparseCoder
    F = np.random.default_rng(0).normal(size=(50, 16)).astype(np.float32)
    F[17] = 0.0
    coder = SparseCoder(torch.from_numpy(F).cuda(), 8, 2)
    try:
        u, E = synth.make_kmeans_draws(8, 16)
        with pytest.raises(abi.ScoupError) as ei:
            coder.kmeans(u, E)
        assert ei.value.status == 2 and "17" in str(ei.value)
    finally:
        coder.close()
    with pytest.raises(abi.ScoupError) as ei:
        SparseCoder(torch.from_numpy(F).cuda(), 4, 5)
    assert ei.value.status == 1
    with pytest.raises(abi.ScoupError) as ei:
        SparseCoder(torch.zeros((10, 1024), device="cuda"), 128, 4)
    assert ei.value.status == 6


def test_pipeline_sparse_codes_into_uplift(dev, tiny_scene):
    """Eq. 4 -> Eq. 5/6: region features of the tiny scene (one CLIP-like vector per (view,
    region), R = 4 x 16) are sparse-coded on the GPU (k-means + 300 epochs, L = 64, K = 4); the
    hard codes are the code table of the uplift (S = K), whose W / Z / codes equal the oracle's
    uplift of the same codes."""
    from paper_2605_13600_b200.uplift import SparseUplift
    import oracle
    sys_path_helpers()
    from helpers import compare_codes
    cfg, scene, maps, _ = tiny_scene
    R = int(sum(synth.make_codes(cfg, seed=0).num_regions))
    rf = synth.make_region_features(R, 128, 24, 4, noise=0.05, seed=21)
    u, E = synth.make_kmeans_draws(cfg.L, 128, seed=21)
    coder = _coder(rf.F, cfg.L, 4)
    try:
        coder.kmeans(u, E)
        coder.train(300)
        atoms, coefs = coder.encode()
        atoms_np = atoms.cpu().numpy().view(np.uint32)
        coefs_np = coefs.cpu().numpy()
    finally:
        coder.close()
    assert np.allclose(coefs_np.sum(axis=1), 1.0, atol=1e-6) and (coefs_np > 0).all()
    base = synth.make_codes(cfg, seed=0)
    codes = synth.Codes(atoms_np, coefs_np, base.row0, base.num_regions)
    Wo, Zo, fo, ao, co = oracle.uplift(scene.gaussians, scene.cameras, maps, codes, cfg.L, 4)
    g = scene.gaussians
    gin = synth.Gaussians(*[torch.from_numpy(np.ascontiguousarray(a)).cuda()
                            for a in (g.means, g.scales, g.rotations, g.opacities)])
    up = SparseUplift(gin, cfg.L, 4)
    try:
        up.add_views(scene.cameras, torch.from_numpy(np.ascontiguousarray(maps).view(np.int32)).cuda(),
                     synth.Codes(atoms, coefs, base.row0, base.num_regions))
        a2, c2 = up.finalize()
        W = up.W[:g.count].double().cpu().numpy()
        Z = up.Z[:g.count].double().cpu().numpy()
    finally:
        up.close()
    assert np.all(np.abs(W - Wo) <= 1e-6 + 1e-4 * np.abs(Wo))
    assert np.all(np.abs(Z - Zo) <= 1e-6 + 1e-4 * np.abs(Zo))
    bad, _, worst = compare_codes(a2.cpu().numpy().view(np.uint32), c2.cpu().numpy(), Wo, 4)
    assert bad == 0, worst


def sys_path_helpers():
    import os
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    if here not in sys.path:
        sys.path.insert(0, here)
