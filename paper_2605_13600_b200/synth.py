"""Seeded synthetic inputs shaped like the paper's workloads (BASELINE.json ``configs``).

This module is the ONE piece shared by the CUDA path and the CPU oracle (`oracle/`).
It holds none of the method's arithmetic: no projection, no alpha blending, no
aggregation, no Top-K.  It only draws Gaussians, cameras, region-id maps and
per-region sparse codes, following the recipe in DESIGN.md §"Input recipe"
(SURVEY.md §8(d) "Common generator rules" + the per-config readings).

The paper's datasets (LERF-OVS, Mip-NeRF360, 3D-OVS) and its
pretrained 3DGS scenes / SAM+CLIP outputs are not available; these synthetic
scenes stand in for them.  Every array is drawn in float64 with
``numpy.random.default_rng([seed, component, index, ...])`` and cast to float32
once, so both sides read bit-identical inputs.

Region maps are integer Voronoi partitions (ties -> lower seed index), which are
exact, so the numpy generator (small configs, tests) and the torch generator
(large configs on the GPU box, plumbing only) produce identical maps.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import List, Optional, Sequence, Tuple

import numpy as np

NONE = 0xFFFFFFFF  # unassigned pixel / empty code slot

# RNG component ids (SURVEY.md §8(d) "RNG")
_C_GAUSS, _C_CAM, _C_SEEDS, _C_CODES = 0, 1, 2, 3


@dataclass(frozen=True)
class SceneConfig:
    name: str
    num_gaussians: int
    layout: str                    # uniform | clusters | indoor | outdoor
    n_clusters: int
    scale_mu: float                # scales = exp(N(ln scale_mu, scale_sigma))
    scale_sigma: float
    num_views: int
    width: int
    height: int
    fov_deg: float                 # horizontal field of view
    camera: str                    # sphere | orbit
    radius: Tuple[float, float]
    regions: Tuple[int, ...]       # regions per view, one entry per semantic level
    L: int
    S: int                         # nonzeros per region code
    K: int                         # output Top-K
    beta: float                    # Dirichlet concentration of region codes
    unassigned_frac: float = 0.0   # fraction of regions marked NONE (parity variant)

    def with_(self, **kw) -> "SceneConfig":
        return replace(self, **kw)


# BASELINE.json configs[0..4]; readings flagged in DESIGN.md §"Input recipe".
CONFIGS = {
    "tiny": SceneConfig("tiny", 2000, "uniform", 0, 0.03, 0.5, 4, 64, 64, 60.0,
                        "sphere", (3.0, 3.0), (16,), 64, 4, 4, 1.0),
    "small": SceneConfig("small", 100_000, "clusters", 20, 0.01, 0.6, 50, 512, 384, 55.0,
                         "orbit", (2.5, 3.5), (64,), 64, 4, 4, 1.0),
    "indoor": SceneConfig("indoor", 1_000_000, "indoor", 100, 0.01, 0.6, 200, 988, 731, 60.0,
                          "orbit", (2.5, 3.5), (32, 128, 512), 64, 4, 4, 0.5),
    "outdoor": SceneConfig("outdoor", 3_000_000, "outdoor", 100, 0.02, 0.8, 300, 1600, 1066, 70.0,
                           "orbit", (4.0, 4.0), (128,), 64, 8, 8, 1.0),
    "stress": SceneConfig("stress", 6_000_000, "clusters", 100, 0.05, 0.6, 800, 1920, 1080, 60.0,
                          "orbit", (3.0, 4.0), (128,), 128, 8, 8, 1.0),
}


@dataclass
class Gaussians:
    means: np.ndarray      # f32 [G,3]
    scales: np.ndarray     # f32 [G,3] activated (>0)
    rotations: np.ndarray  # f32 [G,4] (w,x,y,z), unnormalised
    opacities: np.ndarray  # f32 [G]   activated, in (0,1)

    @property
    def count(self) -> int:
        return int(self.means.shape[0])


@dataclass
class Camera:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    world_to_camera: np.ndarray  # f32 [4,4] row-major rigid [R|t], OpenCV axes


@dataclass
class ViewSeeds:
    """Voronoi seeds of one view and one semantic level."""
    sx: np.ndarray                     # int64 [R]
    sy: np.ndarray                     # int64 [R]
    parent: Optional[np.ndarray] = None  # int64 [R]: parent region at the coarser level
    parent_seeds: Optional["ViewSeeds"] = None


@dataclass
class Codes:
    atoms: np.ndarray   # u32 [R_total, S]
    coefs: np.ndarray   # f32 [R_total, S]
    row0: np.ndarray    # int64 [V]
    num_regions: np.ndarray  # int32 [V]


def _rng(seed: int, *idx: int) -> np.random.Generator:
    return np.random.default_rng([seed, *idx])


def make_gaussians(cfg: SceneConfig, seed: int = 0) -> Gaussians:
    rng = _rng(seed, _C_GAUSS, 0)
    G = cfg.num_gaussians
    if cfg.layout == "uniform":
        means = rng.uniform(-1.0, 1.0, size=(G, 3))
    else:
        frac_cluster = {"clusters": 1.0, "indoor": 0.9, "outdoor": 0.7}[cfg.layout]
        n_cl = int(round(G * frac_cluster))
        centres = rng.uniform(-1.0, 1.0, size=(cfg.n_clusters, 3))
        member = rng.integers(0, cfg.n_clusters, size=n_cl)
        cl = centres[member] + rng.normal(0.0, 0.1, size=(n_cl, 3))
        n_bg = G - n_cl
        d = rng.normal(size=(n_bg, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        if cfg.layout == "indoor":
            r = rng.uniform(4.0, 5.0, size=n_bg)
        elif cfg.layout == "outdoor":
            r = np.exp(rng.uniform(math.log(1.0), math.log(50.0), size=n_bg))
        else:
            r = np.zeros(n_bg)
        means = np.concatenate([cl, d * r[:, None]], axis=0)
        means = means[rng.permutation(G)]
    scales = np.exp(rng.normal(math.log(cfg.scale_mu), cfg.scale_sigma, size=(G, 3)))
    rots = rng.normal(size=(G, 4))
    opac = 1.0 / (1.0 + np.exp(-rng.normal(0.0, 1.5, size=G)))
    return Gaussians(means.astype(np.float32), scales.astype(np.float32),
                     rots.astype(np.float32), opac.astype(np.float32))


def look_at_camera(pos: np.ndarray, width: int, height: int, fov_deg: float) -> Camera:
    """Pinhole camera at `pos` looking at the origin; +z up (fallback +y); OpenCV axes."""
    pos = np.asarray(pos, dtype=np.float64)
    f = -pos / np.linalg.norm(pos)
    up = np.array([0.0, 0.0, 1.0])
    if abs(float(f @ up)) > 0.99:
        up = np.array([0.0, 1.0, 0.0])
    right = np.cross(f, up)
    right /= np.linalg.norm(right)
    down = np.cross(f, right)
    R = np.stack([right, down, f], axis=0)
    t = -R @ pos
    M = np.eye(4)
    M[:3, :3] = R
    M[:3, 3] = t
    fx = (width / 2.0) / math.tan(math.radians(fov_deg) / 2.0)
    return Camera(float(np.float32(fx)), float(np.float32(fx)), width / 2.0, height / 2.0,
                  width, height, M.astype(np.float32))


def make_cameras(cfg: SceneConfig, seed: int = 0) -> List[Camera]:
    rng = _rng(seed, _C_CAM, 0)
    V = cfg.num_views
    cams = []
    for v in range(V):
        if cfg.camera == "sphere":
            d = rng.normal(size=3)
            pos = d / np.linalg.norm(d) * cfg.radius[0]
        else:
            az = 2 * math.pi * v / V + rng.uniform(-0.5, 0.5) * 2 * math.pi / V
            el = math.radians(rng.uniform(-10.0, 40.0))
            r = rng.uniform(cfg.radius[0], cfg.radius[1])
            pos = r * np.array([math.cos(el) * math.cos(az), math.cos(el) * math.sin(az), math.sin(el)])
        cams.append(look_at_camera(pos, cfg.width, cfg.height, cfg.fov_deg))
    return cams


def make_view_seeds(cfg: SceneConfig, view: int, seed: int = 0) -> List[ViewSeeds]:
    """Seeds for every level of one view.  Level l>0 keeps the level-(l-1) seeds and adds
    new uniform seeds; each child's parent is the coarse region at the child's seed pixel,
    so levels are nested (reading: BASELINE.json configs[2] "each split into 4 then 16")."""
    levels: List[ViewSeeds] = []
    for lvl, R in enumerate(cfg.regions):
        rng = _rng(seed, _C_SEEDS, view, lvl)
        if lvl == 0:
            sx = rng.integers(0, cfg.width, size=R)
            sy = rng.integers(0, cfg.height, size=R)
            levels.append(ViewSeeds(sx.astype(np.int64), sy.astype(np.int64)))
        else:
            prev = levels[-1]
            Rp = len(prev.sx)
            nx = rng.integers(0, cfg.width, size=R - Rp)
            ny = rng.integers(0, cfg.height, size=R - Rp)
            sx = np.concatenate([prev.sx, nx]).astype(np.int64)
            sy = np.concatenate([prev.sy, ny]).astype(np.int64)
            parent = _voronoi_points_numpy(prev, sx, sy)
            levels.append(ViewSeeds(sx, sy, parent, prev))
    return levels


def _voronoi_points_numpy(seeds: ViewSeeds, px: np.ndarray, py: np.ndarray) -> np.ndarray:
    """Region id (at the level of `seeds`) of the given pixel coordinates."""
    d = (px[:, None] - seeds.sx[None, :]) ** 2 + (py[:, None] - seeds.sy[None, :]) ** 2
    if seeds.parent is not None:
        par = _voronoi_points_numpy(seeds.parent_seeds, px, py)
        d = np.where(seeds.parent[None, :] == par[:, None], d, np.iinfo(np.int64).max)
    return np.argmin(d, axis=1).astype(np.int64)


def voronoi_map_numpy(seeds: ViewSeeds, width: int, height: int) -> np.ndarray:
    """u32 [H,W] region map (exact integer arithmetic; ties -> lower seed index)."""
    out = np.empty((height, width), dtype=np.uint32)
    xs = np.arange(width, dtype=np.int64)
    rows = max(1, (1 << 22) // max(1, width * len(seeds.sx)))
    for y0 in range(0, height, rows):
        ys = np.arange(y0, min(height, y0 + rows), dtype=np.int64)
        px = np.broadcast_to(xs[None, :], (len(ys), width)).ravel()
        py = np.broadcast_to(ys[:, None], (len(ys), width)).ravel()
        out[y0:y0 + len(ys)] = _voronoi_points_numpy(seeds, px, py).reshape(len(ys), width)
    return out


def voronoi_map_torch(seeds: ViewSeeds, width: int, height: int, device, out=None):
    """Same map as `voronoi_map_numpy`, evaluated with torch on `device` (input plumbing
    for configs whose maps are too large to ship; exact integer arithmetic)."""
    import torch

    def pts_region(s: ViewSeeds, px, py):
        sx = torch.as_tensor(s.sx, device=device, dtype=torch.int32)
        sy = torch.as_tensor(s.sy, device=device, dtype=torch.int32)
        dx = px[:, None] - sx[None, :]
        dy = py[:, None] - sy[None, :]
        d = dx * dx + dy * dy
        if s.parent is not None:
            par = pts_region(s.parent_seeds, px, py)
            pp = torch.as_tensor(s.parent, device=device, dtype=torch.int64)
            d = torch.where(pp[None, :] == par[:, None], d, torch.iinfo(torch.int32).max)
        return torch.argmin(d, dim=1)

    if out is None:
        out = torch.empty((height, width), dtype=torch.int32, device=device)
    xs = torch.arange(width, device=device, dtype=torch.int32)
    rows = max(1, (1 << 25) // max(1, width * len(seeds.sx)))
    for y0 in range(0, height, rows):
        y1 = min(height, y0 + rows)
        ys = torch.arange(y0, y1, device=device, dtype=torch.int32)
        px = xs[None, :].expand(y1 - y0, width).reshape(-1)
        py = ys[:, None].expand(y1 - y0, width).reshape(-1)
        out[y0:y1] = pts_region(seeds, px, py).reshape(y1 - y0, width).to(torch.int32)
    return out


def unassigned_regions(cfg: SceneConfig, view: int, level: int, R: int, seed: int = 0) -> np.ndarray:
    """Boolean [R]: regions whose pixels are marked NONE (parity variant with unassigned pixels)."""
    if cfg.unassigned_frac <= 0:
        return np.zeros(R, dtype=bool)
    rng = _rng(seed, 4, view, level)
    return rng.uniform(size=R) < cfg.unassigned_frac


def apply_unassigned(idmap, mask: np.ndarray):
    """Set pixels of masked regions to NONE.  Works on numpy u32 or torch int32 maps."""
    if not mask.any():
        return idmap
    if isinstance(idmap, np.ndarray):
        idmap[mask[idmap.astype(np.int64)]] = NONE
        return idmap
    import torch
    m = torch.as_tensor(mask, device=idmap.device)
    idmap[m[idmap.long()]] = -1
    return idmap


def make_codes(cfg: SceneConfig, level: int = 0, seed: int = 0,
               views: Optional[Sequence[int]] = None) -> Codes:
    """Per-(view, region) sparse convex codes: S distinct atoms, Dirichlet(beta) coefficients."""
    views = list(range(cfg.num_views)) if views is None else list(views)
    R = cfg.regions[level]
    atoms_all, coefs_all = [], []
    for v in views:
        rng = _rng(seed, _C_CODES, v, level)
        atoms = np.argsort(rng.uniform(size=(R, cfg.L)), axis=1)[:, :cfg.S]
        coefs = rng.dirichlet(np.full(cfg.S, cfg.beta), size=R).astype(np.float32)
        bad = (coefs == 0).any(axis=1)
        while bad.any():
            coefs[bad] = rng.dirichlet(np.full(cfg.S, cfg.beta), size=int(bad.sum())).astype(np.float32)
            bad = (coefs == 0).any(axis=1)
        atoms_all.append(atoms.astype(np.uint32))
        coefs_all.append(coefs)
    row0 = np.arange(len(views), dtype=np.int64) * R
    return Codes(np.concatenate(atoms_all), np.concatenate(coefs_all), row0,
                 np.full(len(views), R, dtype=np.int32))


def make_dense_features(cfg: SceneConfig, D: int, level: int = 0, seed: int = 0,
                        views: Optional[Sequence[int]] = None) -> Codes:
    """Dense per-(view, region) features in R^D (unit-norm normal vectors, CLIP-like), for the
    dense feature uplift of Eq. 3, the baseline sparse codes replace.
    Returned as Codes with atoms=None (S = D slots, slot s = feature dimension s)."""
    views = list(range(cfg.num_views)) if views is None else list(views)
    R = cfg.regions[level]
    out = []
    for v in views:
        rng = _rng(seed, 5, v, level)
        f = rng.normal(size=(R, D))
        f /= np.linalg.norm(f, axis=1, keepdims=True)
        out.append(f.astype(np.float32))
    row0 = np.arange(len(views), dtype=np.int64) * R
    return Codes(None, np.concatenate(out), row0, np.full(len(views), R, dtype=np.int32))


def make_region_maps_numpy(cfg: SceneConfig, level: int = 0, seed: int = 0,
                           views: Optional[Sequence[int]] = None) -> np.ndarray:
    views = list(range(cfg.num_views)) if views is None else list(views)
    out = np.empty((len(views), cfg.height, cfg.width), dtype=np.uint32)
    for i, v in enumerate(views):
        s = make_view_seeds(cfg, v, seed)[level]
        out[i] = voronoi_map_numpy(s, cfg.width, cfg.height)
        apply_unassigned(out[i], unassigned_regions(cfg, v, level, cfg.regions[level], seed))
    return out


def make_region_maps_torch(cfg: SceneConfig, device, level: int = 0, seed: int = 0,
                           views: Optional[Sequence[int]] = None):
    import torch
    views = list(range(cfg.num_views)) if views is None else list(views)
    out = torch.empty((len(views), cfg.height, cfg.width), dtype=torch.int32, device=device)
    for i, v in enumerate(views):
        s = make_view_seeds(cfg, v, seed)[level]
        voronoi_map_torch(s, cfg.width, cfg.height, device, out=out[i])
        apply_unassigned(out[i], unassigned_regions(cfg, v, level, cfg.regions[level], seed))
    return out


@dataclass
class Scene:
    cfg: SceneConfig
    gaussians: Gaussians
    cameras: List[Camera]
    seed: int = 0


def make_scene(cfg: SceneConfig, seed: int = 0) -> Scene:
    return Scene(cfg, make_gaussians(cfg, seed), make_cameras(cfg, seed), seed)


# ---- 2D sparse coding inputs (Eq. 4) ----------

@dataclass
class RegionFeatures:
    """Per-region feature rows (CLIP stand-ins) and, for tests, the planted structure."""
    F: np.ndarray          # [R, D] float32, unit rows
    C_true: np.ndarray     # [L_true, D] float32 unit rows
    atoms: np.ndarray      # [R, K] planted atoms
    coefs: np.ndarray      # [R, K] planted convex weights


def make_region_features(R: int, D: int, L_true: int, K: int, noise: float = 0.01,
                         seed: int = 0) -> RegionFeatures:
    """R region features that are K-sparse convex combinations of a random unit codebook plus
    Gaussian noise (SPEC S:225's generator), normalised to unit length like CLIP embeddings."""
    rng = _rng(seed, 77)
    C = rng.normal(size=(L_true, D))
    C /= np.linalg.norm(C, axis=1, keepdims=True)
    atoms = np.stack([rng.choice(L_true, size=K, replace=False) for _ in range(R)])
    coefs = rng.dirichlet(np.ones(K), size=R)
    F = np.einsum("rk,rkd->rd", coefs, C[atoms]) + noise * rng.normal(size=(R, D))
    F /= np.linalg.norm(F, axis=1, keepdims=True)
    return RegionFeatures(F.astype(np.float32), C.astype(np.float32), atoms, coefs)


def make_kmeans_draws(L: int, D: int, seed: int = 0):
    """The random numbers k-means++ draws (R-SC6): L uniforms in [0, 1) and L unit fallback
    vectors, generated here and passed to both implementations."""
    rng = _rng(seed, 78)
    u = rng.uniform(size=L)
    E = rng.normal(size=(L, D))
    E /= np.linalg.norm(E, axis=1, keepdims=True)
    return u, E.astype(np.float32)
