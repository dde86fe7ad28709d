"""numpy float32 per-pixel brute force -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

An independent second implementation of DESIGN.md §3 used to pin the C oracle
bit-for-bit on tiny scenes (SURVEY.md §8(c) case F8, "brute-force per-pixel
evaluation").  It differs from the C oracle in traversal (every pixel tests EVERY visible
Gaussian, no support-range culling: pixels are a vector, Gaussians a sequential loop in
(depth, index) order) and in language; numpy float32 ops are single IEEE roundings, and
the spec's fused multiply-adds are emulated exactly by ``fma32``.
"""
from __future__ import annotations

import numpy as np

f32 = np.float32
NONE = 0xFFFFFFFF

K_NEAR = f32(float.fromhex("0x1.99999ap-3"))
K_LOWPASS = f32(float.fromhex("0x1.333334p-2"))
K_ACLAMP = f32(float.fromhex("0x1.fae148p-1"))
K_AMIN = f32(float.fromhex("0x1.010102p-8"))
K_TMIN = f32(float.fromhex("0x1.a36e2ep-14"))
K_HALF_LOG2E = f32(float.fromhex("-0x1.715476p-1"))
K_LOG2E_NEG = f32(float.fromhex("-0x1.715476p+0"))
_POLY = [f32(float.fromhex(h)) for h in
         ["0x1.5bba14p-10", "0x1.3cea88p-7", "0x1.c6b752p-5", "0x1.ebf9bcp-3",
          "0x1.62e42ap-1", "0x1p0"]]


def fma32(a, b, c):
    """Correctly rounded float32 fused multiply-add (IEEE 754 fusedMultiplyAdd)."""
    a = np.asarray(a, dtype=f32)
    b = np.asarray(b, dtype=f32)
    c = np.asarray(c, dtype=f32)
    p = a.astype(np.float64) * b.astype(np.float64)     # exact (48-bit product)
    c64 = c.astype(np.float64)
    s = p + c64
    bb = s - p
    err = (p - (s - bb)) + (c64 - bb)                    # TwoSum: s + err == p + c exactly
    with np.errstate(over="ignore"):
        r = s.astype(f32)
    r64 = r.astype(np.float64)
    # double rounding can only go wrong when s sits exactly on a float32 midpoint
    toward = np.where(s > r64, f32(np.inf), f32(-np.inf)).astype(f32)
    r2 = np.nextafter(r, toward)
    mid = (r64 + r2.astype(np.float64)) * 0.5
    on_mid = (s != r64) & (s == mid) & (err != 0)
    # true value lies beyond the midpoint in the direction of err
    pick_r2 = on_mid & (np.sign(err) == np.sign(r2.astype(np.float64) - r64))
    out = np.where(pick_r2, r2, r)
    # s is exactly representable as the other side's midpoint case: s == r64 never double-rounds
    return out.astype(f32)


def exp2_spec(y):
    y = np.asarray(y, dtype=f32)
    magic = f32(float.fromhex("0x1.8p23"))
    t = (y + magic).astype(f32)
    kf = (t - magic).astype(f32)
    f = (y - kf).astype(f32)
    p = np.full_like(y, _POLY[0])
    for c in _POLY[1:]:
        p = fma32(p, f, c)
    out = np.ldexp(p, kf.astype(np.int32)).astype(f32)
    return np.where(y < f32(-64.0), f32(0.0), out).astype(f32)


def project_all(means, scales, rots, opac, cam):
    """Vectorised DESIGN.md §3 G1 + V1-V7 over all Gaussians (float32)."""
    q = np.asarray(rots, dtype=f32)
    s = np.asarray(scales, dtype=f32)
    mu = np.asarray(means, dtype=f32)
    o = np.asarray(opac, dtype=f32)
    n = np.sqrt(((q[:, 0] * q[:, 0] + q[:, 1] * q[:, 1]) + q[:, 2] * q[:, 2]) + q[:, 3] * q[:, 3])
    w, x, y, z = q[:, 0] / n, q[:, 1] / n, q[:, 2] / n, q[:, 3] / n
    one, two = f32(1), f32(2)
    R = [[one - two * (y * y + z * z), two * (x * y - w * z), two * (x * z + w * y)],
         [two * (x * y + w * z), one - two * (x * x + z * z), two * (y * z - w * x)],
         [two * (x * z - w * y), two * (y * z + w * x), one - two * (x * x + y * y)]]
    M = [[R[a][b] * s[:, b] for b in range(3)] for a in range(3)]
    V = [[None] * 3 for _ in range(3)]
    for a in range(3):
        for b in range(a, 3):
            V[a][b] = (M[a][0] * M[b][0] + M[a][1] * M[b][1]) + M[a][2] * M[b][2]
            V[b][a] = V[a][b]
    P = np.asarray(cam.world_to_camera, dtype=f32).reshape(4, 4)
    t = [((P[a, 0] * mu[:, 0] + P[a, 1] * mu[:, 1]) + P[a, 2] * mu[:, 2]) + P[a, 3] for a in range(3)]
    fx, fy, cx, cy = f32(cam.fx), f32(cam.fy), f32(cam.cx), f32(cam.cy)
    vis = t[2] > K_NEAR
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        u = t[0] / t[2]
        v = t[1] / t[2]
        mx = fx * u + cx
        my = fy * v + cy
        j00 = fx / t[2]
        j02 = -(fx * u) / t[2]
        j11 = fy / t[2]
        j12 = -(fy * v) / t[2]
        Q = [[j00 * P[0, b] + j02 * P[2, b] for b in range(3)],
             [j11 * P[1, b] + j12 * P[2, b] for b in range(3)]]
        U = [[(Q[a][0] * V[0][b] + Q[a][1] * V[1][b]) + Q[a][2] * V[2][b] for b in range(3)] for a in range(2)]
        sxx = ((U[0][0] * Q[0][0] + U[0][1] * Q[0][1]) + U[0][2] * Q[0][2]) + K_LOWPASS
        sxy = (U[0][0] * Q[1][0] + U[0][1] * Q[1][1]) + U[0][2] * Q[1][2]
        syy = ((U[1][0] * Q[1][0] + U[1][1] * Q[1][1]) + U[1][2] * Q[1][2]) + K_LOWPASS
        det = sxx * syy - sxy * sxy
        vis = vis & (det > 0)
        ca = syy / det
        cb = -sxy / det
        cc = sxx / det
        mid = f32(0.5) * (sxx + syy)
        lam = mid + np.sqrt(np.maximum(f32(0), mid * mid - det))
        r = f32(3) * np.sqrt(lam)
        qa = ca * K_HALF_LOG2E
        qb = cb * K_LOG2E_NEG
        qc = cc * K_HALF_LOG2E
    return dict(visible=vis, depth=t[2], mx=mx, my=my, sxx=sxx, sxy=sxy, syy=syy, ca=ca, cb=cb, cc=cc,
                r=r, qa=qa, qb=qb, qc=qc, o=o)


def render_view(means, scales, rots, opac, cam):
    """Per-pixel brute force.  Returns (T_final [H,W], E dict gaussian -> float32 [H*W] e)."""
    pr = project_all(means, scales, rots, opac, cam)
    H, W = cam.height, cam.width
    order = np.lexsort((np.arange(len(pr["depth"])), pr["depth"]))  # (depth, index)
    order = [i for i in order if pr["visible"][i]]
    ys, xs = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    px = (xs.ravel().astype(f32) + f32(0.5)).astype(f32)
    py = (ys.ravel().astype(f32) + f32(0.5)).astype(f32)
    T = np.ones(H * W, dtype=f32)
    done = np.zeros(H * W, dtype=bool)
    frags = {}
    for i in order:
        dx = (px - pr["mx"][i]).astype(f32)
        dy = (py - pr["my"][i]).astype(f32)
        r = pr["r"][i]
        ok = (~done) & (np.abs(dx) <= r) & (np.abs(dy) <= r)
        q = fma32(dx, fma32(pr["qa"][i], dx, (pr["qb"][i] * dy).astype(f32)),
                  ((pr["qc"][i] * dy).astype(f32) * dy).astype(f32))
        ok &= ~(q > 0)
        with np.errstate(over="ignore", invalid="ignore"):
            a = np.minimum(K_ACLAMP, (pr["o"][i] * exp2_spec(q)).astype(f32)).astype(f32)
        ok &= ~(a < K_AMIN)
        Tn = (T * (f32(1) - a).astype(f32)).astype(f32)
        stop = ok & (Tn < K_TMIN)
        done |= stop
        ok &= ~stop
        if ok.any():
            e = np.zeros(H * W, dtype=f32)
            e[ok] = (a[ok] * T[ok]).astype(f32)
            frags[int(i)] = e
            T = np.where(ok, Tn, T).astype(f32)
    return T.reshape(H, W), frags


def uplift_accumulate(g, cams, region_maps, code_atoms, code_coefs, code_row0, L):
    """Eq. 5 by brute force (fp64 sums of fp32 products).  Codes are used as given."""
    G = g.count
    W = np.zeros((G, L), dtype=np.float64)
    Z = np.zeros(G, dtype=np.float64)
    frags = []
    for v, cam in enumerate(cams):
        _, E = render_view(g.means, g.scales, g.rotations, g.opacities, cam)
        ids = region_maps[v].ravel()
        nf = 0
        for i, e in E.items():
            nz = e > 0
            nf += int(nz.sum())
            Z[i] += e[nz].astype(np.float64).sum()
            for pix in np.nonzero(nz)[0]:
                rid = int(ids[pix])
                if rid == NONE:
                    continue
                row = int(code_row0[v]) + rid
                for a, c in zip(code_atoms[row], code_coefs[row]):
                    if int(a) == NONE:
                        continue
                    W[i, int(a)] += float(f32(c) * e[pix])
        frags.append(nf)
    return W, Z, np.array(frags, dtype=np.int64)
