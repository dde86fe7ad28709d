"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU).

Every test names the passage it follows.  P:n = /root/reference/PAPER.md line n,
S:n = SPEC.md line n; DESIGN.md §3 is the arithmetic spec, §4 the readings.
A plausible mistake anywhere in the oracle (dropped term, wrong sign or index, transposed
operand) fails one of these.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import oracle.brute as brute
from paper_2605_13600_b200 import synth
from helpers import NONE, full_frame_codes, gaussians, identity_camera

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
f32 = np.float32


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


# ----------------------------------------------------------------------------- exp2_spec
def test_exp2_spec_accuracy_and_exact_points():
    """DESIGN.md §3 exp2_spec: |rel err| vs exact 2^y below 3e-7 on [-64, 0]; integers exact."""
    y = np.linspace(-64.0, 0.0, 400_001).astype(f32)
    got = oracle.exp2_spec(y).astype(np.float64)
    ref = np.exp2(y.astype(np.float64))
    assert np.max(np.abs(got / ref - 1)) < 3e-7
    ints = np.arange(-64, 1).astype(f32)
    assert np.array_equal(oracle.exp2_spec(ints), np.exp2(ints.astype(np.float64)).astype(f32))
    assert oracle.exp2_spec(np.array([-0.0, 0.0], f32)).tolist() == [1.0, 1.0]
    assert oracle.exp2_spec(np.array([-64.5, -1000.0], f32)).tolist() == [0.0, 0.0]


def test_exp2_spec_c_equals_numpy():
    """The two oracle implementations (C fmaf, numpy exact fma32) agree bit-for-bit."""
    rng = np.random.default_rng(1)
    y = np.concatenate([rng.uniform(-64, 0, 200_000), -rng.exponential(0.3, 50_000)]).astype(f32)
    y = np.concatenate([y, np.arange(-64, 0.25, 0.25).astype(f32) + f32(0.5)]).astype(f32)
    y = y[y <= 0]
    assert np.array_equal(oracle.exp2_spec(y).view(np.uint32), brute.exp2_spec(y).view(np.uint32))


def test_fma32_is_correctly_rounded():
    """brute.fma32 against exact rational arithmetic (pins the numpy emulation itself)."""
    from fractions import Fraction
    rng = np.random.default_rng(2)
    a = rng.normal(size=2000).astype(f32)
    b = rng.normal(size=2000).astype(f32)
    c = (-(a.astype(np.float64) * b.astype(np.float64)) * (1 + rng.normal(size=2000) * 1e-7)).astype(f32)
    got = brute.fma32(a, b, c)
    for k in range(2000):
        exact = Fraction(float(a[k])) * Fraction(float(b[k])) + Fraction(float(c[k]))
        lo = f32(float(exact))
        cands = [lo, np.nextafter(lo, f32(np.inf)), np.nextafter(lo, f32(-np.inf))]
        best = min(cands, key=lambda v: (abs(Fraction(float(v)) - exact), int(np.array(v).view(np.uint32)) & 1))
        assert got[k] == best, (k, a[k], b[k], c[k])


# ----------------------------------------------------------------------------- projection
def test_projection_isotropic_on_axis_closed_form():
    """isotropic Gaussian on the optical axis at depth d -> Sigma_2D = (f s/d)^2 I + 0.3 I."""
    for d, s, f in [(2.0, 0.05, 100.0), (3.0, 0.2, 250.0), (1.5, 0.01, 800.0)]:
        g = gaussians([0, 0, d], [s, s, s], [1, 0, 0, 0], [0.5])
        cam = identity_camera(64, 64, f)
        p = oracle.project(g, cam)
        ref = (f * s / d) ** 2 + 0.3
        assert p["visible"][0] == 1
        assert abs(p["sxx"][0] / ref - 1) < 2e-6 and abs(p["syy"][0] / ref - 1) < 2e-6
        assert abs(p["sxy"][0]) < 1e-6 * ref
        assert abs(p["r"][0] / (3 * math.sqrt(ref)) - 1) < 2e-6
        assert p["mx"][0] == 32.0 and p["my"][0] == 32.0


def test_projection_isotropic_rotation_invariant():
    """R diag(s)^2 R^T = s^2 I for isotropic s: the quaternion must not matter."""
    rng = np.random.default_rng(3)
    q = rng.normal(size=(50, 4))
    means = np.tile([[0.3, -0.2, 2.5]], (50, 1))
    g = gaussians(means, np.full((50, 3), 0.1), q, np.full(50, 0.5))
    p = oracle.project(g, identity_camera(64, 64, 120.0))
    for k in ["sxx", "sxy", "syy"]:
        assert np.max(np.abs(p[k] - p[k][0])) < 2e-6 * abs(p["sxx"][0])


def _sigma2d_fp64(mu, s, q, cam):
    """Independent fp64 EWA: Sigma_2D = J W R S S R^T W^T J^T + 0.3 I with a
    finite-difference Jacobian of the pinhole projection and scipy's rotation matrix."""
    from scipy.spatial.transform import Rotation
    R = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()  # scipy: (x, y, z, w)
    Sig3 = R @ np.diag(np.asarray(s, np.float64) ** 2) @ R.T
    M = np.asarray(cam.world_to_camera, np.float64)
    Wr, t = M[:3, :3], M[:3, 3]
    tc = Wr @ np.asarray(mu, np.float64) + t

    def proj(x):
        return np.array([cam.fx * x[0] / x[2] + cam.cx, cam.fy * x[1] / x[2] + cam.cy])

    J = np.zeros((2, 3))
    h = 1e-6 * max(1.0, abs(tc[2]))
    for k in range(3):
        e = np.zeros(3)
        e[k] = h
        J[:, k] = (proj(tc + e) - proj(tc - e)) / (2 * h)
    return J @ Wr @ Sig3 @ Wr.T @ J.T + 0.3 * np.eye(2), proj(tc), tc[2]


def test_projection_matches_fp64_ewa_and_inverse():
    """Random Gaussians and cameras: Sigma_2D, mean2d vs independent fp64 EWA; conic is its
    inverse; r = 3 sqrt(lambda_max)."""
    rng = np.random.default_rng(4)
    cfg = synth.CONFIGS["tiny"]
    G = 300
    g = gaussians(rng.uniform(-0.5, 0.5, (G, 3)), np.exp(rng.normal(np.log(0.05), 0.6, (G, 3))),
                  rng.normal(size=(G, 4)), rng.uniform(0.1, 0.9, G))
    for cam in synth.make_cameras(cfg, seed=7)[:3]:
        p = oracle.project(g, cam)
        for i in range(G):
            if not p["visible"][i]:
                continue
            S2, m2, z = _sigma2d_fp64(g.means[i], g.scales[i], g.rotations[i], cam)
            sc = max(abs(S2[0, 0]), abs(S2[1, 1]))
            assert abs(p["sxx"][i] - S2[0, 0]) < 2e-4 * sc
            assert abs(p["syy"][i] - S2[1, 1]) < 2e-4 * sc
            assert abs(p["sxy"][i] - S2[0, 1]) < 2e-4 * sc
            assert abs(p["mx"][i] - m2[0]) < 1e-3 and abs(p["my"][i] - m2[1]) < 1e-3
            assert abs(p["depth"][i] - z) < 1e-5
            S = np.array([[p["sxx"][i], p["sxy"][i]], [p["sxy"][i], p["syy"][i]]], np.float64)
            Cn = np.array([[p["ca"][i], p["cb"][i]], [p["cb"][i], p["cc"][i]]], np.float64)
            assert np.max(np.abs(S @ Cn - np.eye(2))) < 2e-5 * np.linalg.cond(S)
            lam = np.linalg.eigvalsh(S).max()
            assert abs(p["r"][i] / (3 * math.sqrt(lam)) - 1) < 1e-5
            # log2-domain quadratic form: q = -0.5 log2(e) d^T conic d
            assert abs(p["qa"][i] / (-0.5 * p["ca"][i] / math.log(2)) - 1) < 2e-7
            assert abs(p["qb"][i] / (-p["cb"][i] / math.log(2)) - 1) < 2e-7 or p["cb"][i] == 0


def test_projection_near_plane_cull():
    """Near plane 0.2: depth 0.2 culled, just above kept, behind camera culled."""
    g = gaussians([[0, 0, 0.2], [0, 0, 0.2001], [0, 0, -1.0]], np.full((3, 3), 0.01),
                  np.tile([1, 0, 0, 0], (3, 1)), [0.5, 0.5, 0.5])
    p = oracle.project(g, identity_camera(64, 64))
    assert p["visible"].tolist() == [0, 1, 0]


# ----------------------------------------------------------------------------- fragments
def _footprint_sum(means, s, q, o, W, H, f=100.0):
    g = gaussians(means, s, q, [o])
    cam = identity_camera(W, H, f)
    T, pix, gid, e = oracle.render_view(g, cam)
    p = oracle.project(g, cam)
    det = float(p["sxx"][0]) * float(p["syy"][0]) - float(p["sxy"][0]) ** 2
    return e.astype(np.float64).sum(), det, T, e


@pytest.mark.parametrize("case", load_golden("footprints.json")["cases"], ids=lambda c: c["name"])
def test_single_gaussian_footprint_closed_form(case):
    """Eq. 2 for one Gaussian: e = alpha (T = 1), and sum_p alpha over the
    alpha >= 1/255 set is the integral of the clipped Gaussian, 2 pi sqrt(det Sigma_2D) (o - 1/255)."""
    tot, det, T, e = _footprint_sum(case["mean"], case["scale"], case["rot"], case["opacity"],
                                    case["width"], case["height"])
    assert abs(det / case["det_sigma2d"] - 1) < 1e-5
    closed = 2 * math.pi * math.sqrt(det) * (case["opacity"] - 1 / 255)
    assert abs(closed / case["closed_form_sum"] - 1) < 1e-5
    assert abs(tot / closed - 1) < case["rtol"]
    # e <= o and every fragment passes alpha >= 1/255
    assert e.max() <= case["opacity"] and e.min() >= 1 / 255 - 1e-9


def test_two_overlapping_closed_form_at_centre():
    """S:142 / Eq. 2: coincident alpha = 0.5 -> e = 0.5, 0.25 exactly; o_A = 0.99 clamps."""
    cam = identity_camera(96, 96, 100.0, 48.5, 48.5)
    centre = 48 * 96 + 48
    for oa, ob, ea, eb in [(0.5, 0.5, f32(0.5), f32(0.25)),
                           (0.99, 0.5, f32(0.99), f32(0.5) * (f32(1) - f32(0.99)))]:
        g = gaussians([[0, 0, 2], [0, 0, 3]], np.full((2, 3), 0.2), np.tile([1, 0, 0, 0], (2, 1)), [oa, ob])
        T, pix, gid, e = oracle.render_view(g, cam)
        at = {int(gi): float(ev) for pi, gi, ev in zip(pix, gid, e) if pi == centre}
        assert at[0] == float(ea) and at[1] == float(eb)
        # order: A (front) is emitted before B at that pixel
        order = [int(gi) for pi, gi in zip(pix, gid) if pi == centre]
        assert order == [0, 1]


def test_two_overlapping_off_centre_closed_form():
    """Eq. 2 off-centre: e_B = alpha_B (1 - alpha_A), alpha = o exp(-d^T Sigma^-1 d / 2) with the
    closed-form isotropic Sigma_2D = (f s / d)^2 + 0.3."""
    cam = identity_camera(96, 96, 100.0, 48.5, 48.5)
    g = gaussians([[0, 0, 2], [0, 0, 3]], np.full((2, 3), 0.2), np.tile([1, 0, 0, 0], (2, 1)), [0.6, 0.7])
    T, pix, gid, e = oracle.render_view(g, cam)
    sA, sB = (100 * 0.2 / 2) ** 2 + 0.3, (100 * 0.2 / 3) ** 2 + 0.3
    frag = {(int(p), int(i)): float(v) for p, i, v in zip(pix, gid, e)}
    checked = 0
    for (x, y) in [(50, 48), (52, 55), (40, 44), (60, 48), (48, 33)]:
        d2 = (x + 0.5 - 48.5) ** 2 + (y + 0.5 - 48.5) ** 2
        aA = min(0.99, 0.6 * math.exp(-0.5 * d2 / sA))
        aB = min(0.99, 0.7 * math.exp(-0.5 * d2 / sB))
        p = y * 96 + x
        if aA >= 1 / 255:
            assert abs(frag[(p, 0)] / aA - 1) < 2e-6
        if aB >= 1 / 255:
            ref = aB * (1 - aA) if aA >= 1 / 255 else aB
            assert abs(frag[(p, 1)] / ref - 1) < 2e-6
            checked += 1
    assert checked >= 4


def test_rotated_anisotropic_per_pixel_alpha():
    """Eq. 2 alpha = o exp(-1/2 d^T Sigma_2D^-1 d) per pixel for one ROTATED anisotropic
    Gaussian (SURVEY F2 geometry: s = (0.3, 0.15, 0.2), 30 deg about the optical axis), against an
    independent fp64 Sigma_2D (scipy rotation, finite-difference Jacobian).  Off-axis pixels in
    all four quadrants: the mirrored pixels (dx, dy) and (dx, -dy) have different alphas only
    through the cross term b dx dy of the conic, so a flipped or dropped cross term (qb in the
    oracle's log2-domain quadratic form) fails here -- the footprint-sum pin cannot see it."""
    W = H = 128
    mu, s = [0.0, 0.0, 2.0], [0.3, 0.15, 0.2]
    th = math.radians(15.0)
    q = [math.cos(th), 0.0, 0.0, math.sin(th)]
    o = 0.25
    g = gaussians([mu], [s], [q], [o])
    cam = identity_camera(W, H, 100.0)
    T, pix, gid, e = oracle.render_view(g, cam)
    frag = {int(p): float(v) for p, v in zip(pix, e)}
    S2, m2, _ = _sigma2d_fp64(mu, s, q, cam)
    Sinv = np.linalg.inv(S2)
    assert abs(S2[0, 1]) > 0.2 * math.sqrt(S2[0, 0] * S2[1, 1])  # a strongly rotated ellipse
    checked = 0
    for ax, ay in [(6, 4), (11, 3), (4, 9), (14, 8), (9, 13)]:
        vals = {}
        for sx in (1, -1):
            for sy in (1, -1):
                x, y = int(m2[0]) + sx * ax, int(m2[1]) + sy * ay
                d = np.array([x + 0.5 - m2[0], y + 0.5 - m2[1]])
                ref = o * math.exp(-0.5 * d @ Sinv @ d)
                assert ref >= 1.5 / 255  # far from the alpha cut-off: a fragment on both sides
                got = frag[y * W + x]
                assert abs(got / ref - 1) < 1e-5, (x, y, got, ref)
                vals[(sx, sy)] = ref
                checked += 1
        # the mirror images differ by far more than the tolerance (the cross term matters)
        assert abs(vals[(1, 1)] / vals[(1, -1)] - 1) > 0.05
    assert checked == 20


def test_termination_reading():
    """DESIGN.md §4 reading R9 (3DGS): a fragment whose T(1-alpha) < 1e-4 ends the pixel
    without contributing.  Three coincident o = 0.99 Gaussians: only the front one contributes."""
    cam = identity_camera(96, 96, 100.0, 48.5, 48.5)
    g = gaussians([[0, 0, 2], [0, 0, 3], [0, 0, 4]], np.full((3, 3), 0.2), np.tile([1, 0, 0, 0], (3, 1)),
                  [0.99, 0.99, 0.99])
    T, pix, gid, e = oracle.render_view(g, cam)
    centre = 48 * 96 + 48
    at = [(int(i), float(v)) for p, i, v in zip(pix, gid, e) if p == centre]
    assert at == [(0, float(f32(0.99)))]
    assert T[48, 48] == f32(1) - f32(0.99)
    assert float(T[48, 48]) * (1 - 0.99) < 1e-4


def test_per_pixel_invariants(tiny_scene):
    """per pixel sum(e) <= 1 and 1 - sum(e) = T_final (telescoping, 1e-5 because
    T is fp32 over up to ~100 steps); T_final >= 1e-4 (reading R9)."""
    cfg, scene, maps, codes = tiny_scene
    for cam in scene.cameras[:2]:
        T, pix, gid, e = oracle.render_view(scene.gaussians, cam)
        s = np.zeros(cam.width * cam.height)
        np.add.at(s, pix, e.astype(np.float64))
        assert s.max() <= 1 + 1e-6
        assert np.max(np.abs(1 - s - T.ravel().astype(np.float64))) < 1e-5
        assert T.min() >= 1e-4


def test_brute_force_equivalence_bitwise(tiny_scene):
    """SURVEY.md F8 / S:143: numpy per-pixel brute force over ALL Gaussians in (depth, index)
    order == the C Gaussian-major oracle, bit-for-bit on every e and fragment count."""
    cfg, scene, maps, codes = tiny_scene
    cases = [(scene.gaussians, scene.cameras[0])]
    for seed in range(5):
        rng = np.random.default_rng([seed, 99])
        g = gaussians(rng.uniform(-1, 1, (50, 3)), np.exp(rng.normal(np.log(0.15), 0.5, (50, 3))),
                      rng.normal(size=(50, 4)), 1 / (1 + np.exp(-rng.normal(0, 1.5, 50))))
        cam = synth.look_at_camera(rng.normal(size=3) * 3 / np.linalg.norm(rng.normal(size=3)) + 0, 32, 32, 60.0)
        cases.append((g, cam))
    for g, cam in cases:
        T, pix, gid, e = oracle.render_view(g, cam)
        Tb, E = brute.render_view(g.means, g.scales, g.rotations, g.opacities, cam)
        assert np.array_equal(T.view(np.uint32), Tb.view(np.uint32))
        dense = {}
        for p, i, v in zip(pix, gid, e):
            dense.setdefault(int(i), np.zeros(cam.width * cam.height, f32))[p] = v
        assert set(dense) == set(E)
        for i in E:
            assert np.array_equal(dense[i].view(np.uint32), E[i].view(np.uint32))


# ----------------------------------------------------------------------------- aggregation
def _one_gaussian_view(o=0.3, W=96, H=96):
    g = gaussians([0, 0, 2], [0.2, 0.2, 0.2], [1, 0, 0, 0], [o])
    return g, identity_camera(W, H)


def test_unassigned_half_and_one_hot_code():
    """F5: NONE pixels add to Z but not to W; one-hot code {(3,1.0)} -> code {(3,1.0)}."""
    g, cam = _one_gaussian_view()
    T, pix, gid, e = oracle.render_view(g, cam)
    ids = np.zeros((1, 96, 96), np.uint32)
    ids[0, :, :48] = NONE
    codes = full_frame_codes([[(3, 1.0)]])
    W, Z, fr, atoms, coefs = oracle.uplift(g, [cam], ids, codes, 64, 4)
    right = (pix % 96) >= 48
    assert abs(Z[0] - e.astype(np.float64).sum()) < 1e-12 * Z[0]
    assert abs(W[0, 3] - e[right].astype(np.float64).sum()) < 1e-12 * W[0, 3]
    assert np.count_nonzero(W[0]) == 1
    assert atoms[0].tolist() == [3, NONE, NONE, NONE] and coefs[0].tolist() == [1.0, 0, 0, 0]
    assert fr[0] == len(e)


def test_full_frame_region_gives_code_times_z(tiny_scene):
    """F6 (S:293 analogue): one region covering all pixels with code c -> W_i = c Z_i, and
    w_hat_i = c (Eq. 6) for every observed Gaussian."""
    cfg, scene, maps, codes = tiny_scene
    cams = scene.cameras[:2]
    ids = np.zeros((2, 64, 64), np.uint32)
    code = [(3, 0.7), (10, 0.3)]
    W, Z, fr, atoms, coefs = oracle.uplift(scene.gaussians, cams, ids, full_frame_codes([code, code]), 64, 4)
    seen = Z > 0
    assert seen.sum() > 100
    c = np.zeros(64)
    c[3], c[10] = float(f32(0.7)), float(f32(0.3))
    assert np.allclose(W[seen], np.outer(Z[seen], c), rtol=1e-6, atol=0)
    assert np.all(atoms[seen, 0] == 3) and np.all(atoms[seen, 1] == 10)
    assert np.allclose(coefs[seen, 0], 0.7, atol=1e-6) and np.allclose(coefs[seen, 1], 0.3, atol=1e-6)
    assert np.all(atoms[~seen] == NONE)


def test_multi_view_vote():
    """F7 (S:294, P:114 'semantic voting'): same Gaussian seen in 3 identical views voting
    atom 1, atom 1, atom 2 -> K=1 gives {(1,1.0)}; K=2 gives {(1,2/3),(2,1/3)}."""
    g, cam = _one_gaussian_view(o=0.5)
    ids = np.zeros((3, 96, 96), np.uint32)
    codes = full_frame_codes([[(1, 1.0)], [(1, 1.0)], [(2, 1.0)]])
    for K, exp in [(1, [(1, 1.0)]), (2, [(1, 2 / 3), (2, 1 / 3)])]:
        W, Z, fr, atoms, coefs = oracle.uplift(g, [cam] * 3, ids, codes, 64, K)
        got = [(int(a), float(c)) for a, c in zip(atoms[0], coefs[0]) if a != NONE]
        assert [a for a, _ in got] == [a for a, _ in exp]
        assert all(abs(c - ce) < 1e-12 for (_, c), (_, ce) in zip(got, exp))


def test_topk_hand_cases():
    """Eq. 6: one-hot fixed point; (0.4,0.3,0.2,0.1), K=2 -> {(0,4/7),(1,3/7)};
    ties -> lower atom; zero row -> empty code (Alg. 1 line 15)."""
    W = np.zeros((5, 8))
    W[0, 5] = 2.5
    W[1, :4] = [0.4, 0.3, 0.2, 0.1]
    W[2, [6, 2, 4]] = [0.5, 0.5, 0.5]
    W[4, [7]] = 1e-30
    atoms, coefs = oracle.topk(W, 2)
    assert atoms[0].tolist() == [5, NONE] and coefs[0].tolist() == [1.0, 0.0]
    assert atoms[1].tolist() == [0, 1] and np.allclose(coefs[1], [4 / 7, 3 / 7], rtol=0, atol=1e-15)
    assert atoms[2].tolist() == [2, 4] and coefs[2].tolist() == [0.5, 0.5]
    assert atoms[3].tolist() == [NONE, NONE] and coefs[3].tolist() == [0.0, 0.0]
    assert atoms[4].tolist() == [7, NONE] and coefs[4].tolist() == [1.0, 0.0]


def test_topk_matches_sort_oracle():
    """1000 random sparse non-negative vectors; kept set equals a sort-based selection
    (value desc, atom asc); coefs > 0, <= K entries, L1 = 1 +- 1e-12."""
    rng = np.random.default_rng(5)
    L, K = 64, 4
    W = rng.exponential(size=(1000, L)) * (rng.uniform(size=(1000, L)) < 0.2)
    W[::17, 5] = W[::17, 9] = 0.75  # exact ties
    atoms, coefs = oracle.topk(W, K)
    for i in range(1000):
        order = sorted([a for a in range(L) if W[i, a] > 0], key=lambda a: (-W[i, a], a))[:K]
        assert [int(a) for a in atoms[i] if a != NONE] == order
        kept = coefs[i][: len(order)]
        if order:
            assert np.all(kept > 0) and abs(kept.sum() - 1) < 1e-12
            assert np.allclose(kept, W[i, order] / W[i, order].sum(), rtol=1e-14)


def test_mass_conservation_and_counts(tiny_scene, tiny_oracle):
    """sum_{i,a} W = sum over coded fragments of e * (code L1 = 1) = sum_i Z (Voronoi maps
    cover every pixel); fragment counts equal an independent count of the fragment lists."""
    cfg, scene, maps, codes = tiny_scene
    W, Z, frags, atoms, coefs = tiny_oracle
    code_l1 = codes.coefs.astype(np.float64).sum(axis=1)
    assert np.max(np.abs(code_l1 - 1)) < 1e-6
    assert abs(W.sum() / Z.sum() - 1) < 2e-6
    for v, cam in enumerate(scene.cameras):
        T, pix, gid, e = oracle.render_view(scene.gaussians, cam)
        assert frags[v] == len(e)
        assert abs(Z.sum() > 0)
    # storage bound: <= K entries per Gaussian
    assert np.all((atoms != NONE).sum(axis=1) <= cfg.K)


def test_view_order_and_gaussian_permutation_invariance(tiny_scene, tiny_oracle):
    """permuting views changes W only by fp64 reassociation; permuting the input Gaussians
    permutes the rows (per-pixel sequences are identical because depths are continuous)."""
    cfg, scene, maps, codes = tiny_scene
    W, Z, frags, atoms, coefs = tiny_oracle
    perm_v = [2, 0, 3, 1]
    cod = synth.Codes(codes.atoms, codes.coefs, codes.row0[perm_v], codes.num_regions[perm_v])
    W2, Z2, fr2, _, _ = oracle.uplift(scene.gaussians, [scene.cameras[v] for v in perm_v], maps[perm_v], cod,
                                      cfg.L, cfg.K)
    assert np.allclose(W2, W, rtol=1e-12, atol=1e-15) and np.allclose(Z2, Z, rtol=1e-12, atol=1e-15)
    assert fr2.tolist() == [frags[v] for v in perm_v]
    g = scene.gaussians
    perm = np.random.default_rng(6).permutation(g.count)
    gp = synth.Gaussians(g.means[perm], g.scales[perm], g.rotations[perm], g.opacities[perm])
    W3, Z3, fr3, _, _ = oracle.uplift(gp, scene.cameras, maps, codes, cfg.L, cfg.K)
    assert np.array_equal(W3, W[perm]) and np.array_equal(Z3, Z[perm])


def test_linearity_against_dense_uplift(tiny_scene):
    """Eq. 5 is Eq. 3 applied to W_v(p).  With K = L (no filtering) and a random
    codebook C, (W_i / Z_i) C equals the dense uplift f_i = (1/Z_i) sum e F_v(p) of the decoded
    maps F_v = W_v C (Eq. 8), computed here directly from the fragment lists."""
    cfg, scene, maps, codes = tiny_scene
    L, D = cfg.L, 16
    C = np.random.default_rng(8).normal(size=(L, D))
    cams = scene.cameras[:2]
    W, Z, fr, atoms, coefs = oracle.uplift(scene.gaussians, cams, maps[:2], codes, L, L)
    F = np.zeros((scene.gaussians.count, D))
    Zd = np.zeros(scene.gaussians.count)
    for v, cam in enumerate(cams):
        T, pix, gid, e = oracle.render_view(scene.gaussians, cam)
        rid = maps[v].ravel()[pix].astype(np.int64)
        rows = codes.row0[v] + rid
        Wp = np.zeros((len(pix), L))
        for s in range(codes.atoms.shape[1]):
            np.add.at(Wp, (np.arange(len(pix)), codes.atoms[rows, s].astype(np.int64)),
                      codes.coefs[rows, s].astype(np.float64))
        np.add.at(F, gid, e.astype(np.float64)[:, None] * (Wp @ C))
        np.add.at(Zd, gid, e.astype(np.float64))
    seen = Zd > 0
    f_dense = F[seen] / Zd[seen, None]
    f_sparse = (W[seen] / Z[seen, None]) @ C
    assert np.allclose(Z, Zd, rtol=1e-12)
    assert np.max(np.abs(f_sparse - f_dense)) < 1e-5 * np.max(np.abs(f_dense))
    # with K = L the stored code is w_i / ||w_i||_1 exactly (Eq. 6 without truncation)
    dense_codes = np.zeros((seen.sum(), L))
    idx = np.nonzero(seen)[0]
    for r, i in enumerate(idx):
        for a, c in zip(atoms[i], coefs[i]):
            if a != NONE:
                dense_codes[r, a] = c
    assert np.allclose(dense_codes, W[seen] / W[seen].sum(axis=1, keepdims=True), atol=1e-12)


def test_code_truncation_alg1_topk():
    """Algorithm 1 line 7: a region code with more than K slots is cut to its K largest
    (ties -> lower atom) before aggregation, without renormalisation."""
    g, cam = _one_gaussian_view(o=0.4)
    ids = np.zeros((1, 96, 96), np.uint32)
    codes = full_frame_codes([[(9, 0.1), (2, 0.4), (5, 0.2), (7, 0.2), (1, 0.1)]])
    W, Z, fr, atoms, coefs = oracle.uplift(g, [cam], ids, codes, 16, 3)
    nz = np.nonzero(W[0])[0].tolist()
    assert nz == [2, 5, 7]
    assert np.allclose(W[0, [2, 5, 7]] / Z[0], [0.4, 0.2, 0.2], rtol=1e-6)


def test_oracle_errors():
    """bad region id and bad code are data errors; K > L is a config error."""
    g, cam = _one_gaussian_view()
    ids = np.zeros((1, 96, 96), np.uint32)
    ids[0, 40, 40] = 5
    with pytest.raises(oracle.OracleError) as ei:
        oracle.uplift(g, [cam], ids, full_frame_codes([[(1, 1.0)]]), 8, 2)
    assert ei.value.code == -3 and ei.value.index == 40 * 96 + 40
    ids[0, 40, 40] = 0
    with pytest.raises(oracle.OracleError) as ei:
        oracle.uplift(g, [cam], ids, full_frame_codes([[(8, 1.0)]]), 8, 2)
    assert ei.value.code == -4
    with pytest.raises(oracle.OracleError):
        oracle.uplift(g, [cam], ids, full_frame_codes([[(1, 1.0)]]), 8, 9)


def test_dense_feature_path(tiny_scene):
    """Eq. 3, the dense-uplift baseline (code_atoms = None: every region carries a full
    feature vector of L values, any sign): (a) S:301, a constant feature u gives W_i = u Z_i
    exactly up to rounding; (b) decoded features F_v(r) = W_v(r) C accumulate to the same
    sum over fragments as the fragment lists, which pins the dense path independently."""
    cfg, scene, maps, codes = tiny_scene
    cams = scene.cameras[:2]
    g = scene.gaussians
    rng = np.random.default_rng(12)
    D = 24
    u = rng.normal(size=D).astype(np.float32)
    R = int(codes.num_regions[0])
    feats = np.tile(u, (2 * R, 1))
    row0 = np.array([0, R], np.int64)
    nreg = np.array([R, R], np.int32)
    W, Z, fr = oracle.uplift_accumulate(g, cams, maps[:2], None, feats, row0, nreg, D, 1)
    seen = Z > 0
    assert seen.sum() > 100
    assert np.allclose(W[seen], np.outer(Z[seen], u.astype(np.float64)), rtol=1e-6, atol=1e-9)
    # (b) decoded codes as dense features
    C = rng.normal(size=(cfg.L, D))
    Fr = np.zeros((2 * R, D), np.float32)
    for v in range(2):
        for r in range(R):
            row = codes.row0[v] + r
            w = np.zeros(cfg.L)
            for a, c in zip(codes.atoms[row], codes.coefs[row]):
                if a != NONE:
                    w[a] += c
            Fr[v * R + r] = (w @ C).astype(np.float32)
    Wd, Zd, _ = oracle.uplift_accumulate(g, cams, maps[:2], None, Fr, row0, nreg, D, 1)
    F = np.zeros((g.count, D))
    for v, cam in enumerate(cams):
        T, pix, gid, e = oracle.render_view(g, cam)
        rid = maps[v].ravel()[pix].astype(np.int64)
        prod = (Fr[v * R + rid] * e[:, None]).astype(np.float32)  # the spec's fp32 products c * e
        np.add.at(F, gid, prod.astype(np.float64))
    assert np.allclose(Wd, F, rtol=1e-9, atol=1e-12)
    assert np.allclose(Z, Zd)


def test_entropy_closed_forms():
    """P:445-448 entropy pins: uniform over L atoms -> ln L; one-hot -> 0; two atoms p, 1-p ->
    -p ln p - (1-p) ln(1-p); scaling a row (Z) does not change it; an empty row -> NaN."""
    W = np.zeros((5, 8))
    W[0] = 3.0
    W[1, 5] = 0.2
    W[2, :2] = (0.3, 0.7)
    W[3, :2] = (30.0, 70.0)
    H = oracle.entropy(W)
    assert abs(H[0] - np.log(8)) < 1e-15
    assert H[1] == 0.0
    assert abs(H[2] - (-0.3 * np.log(0.3) - 0.7 * np.log(0.7))) < 1e-15
    assert abs(H[3] - H[2]) < 1e-15
    assert np.isnan(H[4])
