"""Hand-built scenes and the parity comparator (test helpers; no method arithmetic)."""
from __future__ import annotations

import numpy as np

from paper_2605_13600_b200 import synth

NONE = 0xFFFFFFFF


def gaussians(means, scales, rots, opac) -> synth.Gaussians:
    return synth.Gaussians(np.asarray(means, np.float32).reshape(-1, 3),
                           np.asarray(scales, np.float32).reshape(-1, 3),
                           np.asarray(rots, np.float32).reshape(-1, 4),
                           np.asarray(opac, np.float32).reshape(-1))


def identity_camera(W, H, f=100.0, cx=None, cy=None) -> synth.Camera:
    return synth.Camera(f, f, W / 2.0 if cx is None else cx, H / 2.0 if cy is None else cy, W, H,
                        np.eye(4, dtype=np.float32))


def full_frame_codes(code_per_view, S=None):
    """One region (id 0) per view with the given [(atom, coef), ...] code."""
    S = S or max(len(c) for c in code_per_view)
    V = len(code_per_view)
    atoms = np.full((V, S), NONE, np.uint32)
    coefs = np.zeros((V, S), np.float32)
    for v, code in enumerate(code_per_view):
        for s, (a, c) in enumerate(code):
            atoms[v, s] = a
            coefs[v, s] = c
    return synth.Codes(atoms, coefs, np.arange(V, dtype=np.int64), np.ones(V, np.int32))


def compare_accumulators(W_gpu, Z_gpu, W_ora, Z_ora, rtol=1e-4, atol=1e-6):
    """|x_gpu - x_ora| <= atol + rtol |x_ora| for every element (north_star tolerance)."""
    W_gpu = np.asarray(W_gpu, np.float64)
    Z_gpu = np.asarray(Z_gpu, np.float64)
    dW = np.abs(W_gpu - W_ora) - (atol + rtol * np.abs(W_ora))
    dZ = np.abs(Z_gpu - Z_ora) - (atol + rtol * np.abs(Z_ora))
    bad_w = np.argwhere(dW > 0)
    bad_z = np.argwhere(dZ > 0)
    return bad_w, bad_z


def compare_codes(atoms_gpu, coefs_gpu, W_ora, K, rtol=1e-4, atol=1e-6):
    """compare_codes_rows (below) with a vectorised fast path: rows whose GPU atom set equals the
    oracle's positive Top-K set (oracle.topk: value desc, atom asc) are checked with array
    operations (same coefficient, order and padding rules); every other row goes through the
    row-by-row comparator, which decides tie exchanges."""
    import oracle
    W_ora = np.ascontiguousarray(W_ora, np.float64)
    G, L = W_ora.shape
    A = np.asarray(atoms_gpu).astype(np.int64) & 0xFFFFFFFF
    Cg = np.asarray(coefs_gpu, np.float64)
    Ao = oracle.topk(W_ora, K)[0].astype(np.int64)
    valid = A != NONE
    n_g = valid.sum(1)
    prefix = np.all(valid == (np.arange(K)[None, :] < n_g[:, None]), axis=1)
    same = np.all(np.sort(A, 1) == np.sort(Ao, 1), axis=1) & prefix
    Sg = np.sort(np.where(valid, A, NONE), 1)
    distinct = ~np.any((Sg[:, 1:] == Sg[:, :-1]) & (Sg[:, 1:] != NONE), axis=1)
    idx = np.where(valid, A, 0)
    w = np.take_along_axis(W_ora, idx, 1) * valid
    denom = w.sum(1)
    with np.errstate(divide="ignore", invalid="ignore"):
        ref = np.where(valid, w / np.where(denom > 0, denom, 1.0)[:, None], 0.0)
    coef_ok = np.all(np.where(valid, np.abs(Cg - ref) <= atol + rtol * ref, Cg == 0), axis=1)
    desc = np.all((Cg[:, :-1] >= Cg[:, 1:]) | ~valid[:, 1:], axis=1) if K > 1 else np.ones(G, bool)
    fast = same & distinct & coef_ok & desc
    slow = np.where(~fast)[0]
    bad, ties, worst = 0, 0, ""
    if len(slow):
        b, t, wst = compare_codes_rows(A[slow], Cg[slow], W_ora[slow], K, rtol, atol)
        bad, ties, worst = b, t, wst
        if wst:
            worst = f"(row index within the non-fast rows, first of {len(slow)}) " + wst
    return bad, ties, worst


def compare_codes_rows(atoms_gpu, coefs_gpu, W_ora, K, rtol=1e-4, atol=1e-6):
    """SURVEY.md §8(c) comparator, step 3.  Returns (n_mismatch, n_tie_allowance, worst_msg).

    The GPU's atom set must equal the oracle's positive-Top-K set, except that atoms whose
    oracle value is within tol = atol + rtol*v_K of v_K may be exchanged; coefficients of
    matched atoms must agree within atol + rtol*w (w recomputed from the oracle's fp64 W
    restricted to the GPU's chosen set, so an allowed exchange is not double-counted)."""
    G, L = W_ora.shape
    atoms_gpu = np.asarray(atoms_gpu).astype(np.int64) & 0xFFFFFFFF
    coefs_gpu = np.asarray(coefs_gpu, np.float64)
    bad, ties, worst = 0, 0, ""
    for i in range(G):
        w = W_ora[i]
        order = sorted([a for a in range(L) if w[a] > 0], key=lambda a: (-w[a], a))
        top = order[:K]
        sel = [int(a) for a in atoms_gpu[i] if a != NONE]
        if not top:
            if sel or np.any(coefs_gpu[i] != 0):
                bad += 1
                worst = worst or f"row {i}: expected empty code, got {sel}"
            continue
        vK = w[top[-1]]
        tol = atol + rtol * vK
        ok = len(sel) == len(top) and len(set(sel)) == len(sel)
        if ok and set(sel) != set(top):
            # exchanges only among near-ties of the K-th value
            for a in set(sel) ^ set(top):
                if abs(w[a] - vK) > tol:
                    ok = False
            if ok:
                ties += 1
        if ok:
            denom = sum(w[a] for a in sel)
            for s, a in enumerate(sel):
                ref = w[a] / denom
                if abs(coefs_gpu[i, s] - ref) > atol + rtol * ref:
                    ok = False
            # descending order of the stored coefficients
            if any(coefs_gpu[i, s] < coefs_gpu[i, s + 1] for s in range(len(sel) - 1)):
                ok = False
            if any(a != NONE for a in atoms_gpu[i, len(sel):]) or np.any(coefs_gpu[i, len(sel):] != 0):
                ok = False
        if not ok:
            bad += 1
            if not worst:
                worst = f"row {i}: gpu {list(zip(sel, coefs_gpu[i][:len(sel)]))} vs oracle top {[(a, w[a]) for a in top]}"
    return bad, ties, worst


def extreme_scene(seed=21):
    """Near-plane off-screen giants, needles, sub-pixel Gaussians, opacity 1/255 and 1.0."""
    rng = np.random.default_rng(seed)
    means, scales, rots, opac = [], [], [], []
    for k in range(40):  # near-plane giants, mostly off-screen
        z = 0.2 + rng.uniform(1e-4, 0.05)
        means.append([rng.uniform(-3, 3) * z * 8, rng.uniform(-3, 3) * z * 8, z])
        scales.append(np.exp(rng.uniform(np.log(0.01), np.log(2.0), 3)))
        rots.append(rng.normal(size=4))
        opac.append(rng.uniform(0.01, 1.0))
    for k in range(200):  # needles
        means.append(rng.uniform(-1, 1, 3) * [1, 1, 0.5] + [0, 0, 3])
        s = np.array([1e-3, 1e-3, 1e-3])
        s[rng.integers(0, 3)] = rng.uniform(0.3, 2.0)
        scales.append(s)
        rots.append(rng.normal(size=4))
        opac.append(rng.uniform(0.05, 1.0))
    for k in range(200):  # sub-pixel and generic
        means.append(rng.uniform(-1.5, 1.5, 3) + [0, 0, 4])
        scales.append(np.exp(rng.normal(np.log(0.002 if k % 2 else 0.05), 0.5, 3)))
        rots.append(rng.normal(size=4))
        opac.append([1 / 255, 1.0, 0.5][k % 3])
    g = gaussians(means, scales, rots, opac)
    cams = [identity_camera(160, 120, 150.0), synth.look_at_camera(np.array([0.5, -0.3, -1.0]), 160, 120, 75.0)]
    R = 9
    yy, xx = np.mgrid[0:120, 0:160]
    maps = np.stack([((xx // 40) + 4 * (yy // 40)) % R, ((xx // 23) * 7 + (yy // 17)) % R]).astype(np.uint32)
    codes = synth.make_codes(synth.CONFIGS["tiny"].with_(num_views=2, regions=(R,)), seed=9)
    return g, cams, maps, codes
