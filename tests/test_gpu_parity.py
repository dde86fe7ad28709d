"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star): W and Z within 1e-4 relative / 1e-6 absolute element by
element; per-view contribution counts bit-exact (the fragment weights are bit-identical by
DESIGN.md §3, so a single flipped threshold decision fails the count); Top-K codes equal
except among near-ties of the K-th value (tests/helpers.compare_codes).
"""
import numpy as np
import pytest

import oracle
from paper_2605_13600_b200 import synth
from helpers import NONE, compare_accumulators, compare_codes, full_frame_codes, gaussians, identity_camera

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-4, 1e-6


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_13600_b200 import build
    build.build()
    return torch.device("cuda", 0)


def run_gpu(g, cams, maps, codes, L, K, *, host_inputs=False, split=None, rows_padded=0):
    from paper_2605_13600_b200.uplift import SparseUplift
    V = len(cams)
    if host_inputs:
        gin = g
        ids = np.ascontiguousarray(maps, np.uint32)
        cod = codes
    else:
        gin = synth.Gaussians(*[torch.from_numpy(np.ascontiguousarray(a)).cuda()
                                for a in (g.means, g.scales, g.rotations, g.opacities)])
        ids = torch.from_numpy(np.ascontiguousarray(maps).view(np.int32)).cuda()
        cod = synth.Codes(torch.from_numpy(np.ascontiguousarray(codes.atoms).view(np.int32)).cuda(),
                          torch.from_numpy(np.ascontiguousarray(codes.coefs)).cuda(), codes.row0, codes.num_regions)
    contrib = torch.zeros(V, dtype=torch.int64, device="cuda")
    up = SparseUplift(gin, L, K, rows_padded=rows_padded)
    try:
        chunks = [list(range(V))] if split is None else split
        for ch in chunks:
            sub_ids = ids[ch] if not host_inputs else np.ascontiguousarray(ids[ch])
            sub_codes = synth.Codes(cod.atoms, cod.coefs, codes.row0[ch], codes.num_regions[ch])
            out = contrib[ch[0]:ch[-1] + 1] if ch == list(range(ch[0], ch[-1] + 1)) else None
            up.add_views([cams[v] for v in ch], sub_ids.contiguous() if not host_inputs else sub_ids, sub_codes,
                         contributions_out=out)
        atoms, coefs = up.finalize()
        torch.cuda.synchronize()
        W = up.W[:g.count].double().cpu().numpy()
        Z = up.Z[:g.count].double().cpu().numpy()
        st = up.stats()
        return dict(W=W, Z=Z, atoms=atoms.cpu().numpy().view(np.uint32), coefs=coefs.cpu().numpy(),
                    contrib=contrib.cpu().numpy(), stats=st)
    finally:
        up.close()


def assert_parity(res, ora, K, check_counts=True):
    W, Z, frags, oatoms, ocoefs = ora
    bad_w, bad_z = compare_accumulators(res["W"], res["Z"], W, Z, RTOL, ATOL)
    assert len(bad_w) == 0, f"{len(bad_w)} W mismatches, first {bad_w[:3]}: gpu {res['W'][tuple(bad_w[0])]} ora {W[tuple(bad_w[0])]}"
    assert len(bad_z) == 0, f"{len(bad_z)} Z mismatches, first {bad_z[:3]}"
    if check_counts:
        assert res["contrib"].tolist() == frags.tolist()
        assert res["stats"]["contributions"] == int(frags.sum())
    bad, ties, worst = compare_codes(res["atoms"], res["coefs"], W, K, RTOL, ATOL)
    assert bad == 0, worst
    return ties


def test_tiny_full_parity(dev, tiny_scene, tiny_oracle):
    cfg, scene, maps, codes = tiny_scene
    res = run_gpu(scene.gaussians, scene.cameras, maps, codes, cfg.L, cfg.K)
    assert_parity(res, tiny_oracle, cfg.K)


def test_tiny_host_buffers_match_device_buffers(dev, tiny_scene, tiny_oracle):
    """The C ABI accepts host arrays (copied inside the call): same results."""
    cfg, scene, maps, codes = tiny_scene
    res = run_gpu(scene.gaussians, scene.cameras, maps, codes, cfg.L, cfg.K, host_inputs=True)
    assert_parity(res, tiny_oracle, cfg.K)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_tiny_other_seeds_with_unassigned(dev, seed):
    """Seeds 1-3; 10% of regions unassigned (NONE pixels add to Z only)."""
    cfg = synth.CONFIGS["tiny"].with_(unassigned_frac=0.1)
    scene = synth.make_scene(cfg, seed)
    maps = synth.make_region_maps_numpy(cfg, seed=seed)
    codes = synth.make_codes(cfg, seed=seed)
    assert (maps == NONE).any()
    ora = oracle.uplift(scene.gaussians, scene.cameras, maps, codes, cfg.L, cfg.K)
    res = run_gpu(scene.gaussians, scene.cameras, maps, codes, cfg.L, cfg.K)
    assert_parity(res, ora, cfg.K)


def test_streaming_add_views_equals_one_call(dev, tiny_scene, tiny_oracle):
    """add_views may be called repeatedly (checkpoint-friendly accumulation)."""
    cfg, scene, maps, codes = tiny_scene
    res = run_gpu(scene.gaussians, scene.cameras, maps, codes, cfg.L, cfg.K, split=[[0], [1, 2], [3]])
    assert_parity(res, tiny_oracle, cfg.K)


def test_small_config_view_subset(dev):
    """configs[1] (100k clustered Gaussians, 512x384, 64 regions) on 6 of its 50 views."""
    cfg = synth.CONFIGS["small"]
    scene = synth.make_scene(cfg, 0)
    views = [0, 9, 17, 25, 33, 41]
    maps = synth.make_region_maps_numpy(cfg, seed=0, views=views)
    codes = synth.make_codes(cfg, seed=0, views=views)
    cams = [scene.cameras[v] for v in views]
    ora = oracle.uplift(scene.gaussians, cams, maps, codes, cfg.L, cfg.K)
    res = run_gpu(scene.gaussians, cams, maps, codes, cfg.L, cfg.K)
    ties = assert_parity(res, ora, cfg.K)
    assert ties < 0.01 * scene.gaussians.count


def test_ragged_image_and_many_regions_fallback(dev):
    """Image 70x45 (ragged tiles on both axes) and a region map of per-pixel noise: tiles hold
    more than MAX_SLOTS distinct regions, exercising the per-pixel reduction path."""
    rng = np.random.default_rng(11)
    G = 3000
    g = gaussians(rng.uniform(-1, 1, (G, 3)), np.exp(rng.normal(np.log(0.04), 0.5, (G, 3))),
                  rng.normal(size=(G, 4)), 1 / (1 + np.exp(-rng.normal(0, 1.5, G))))
    cams = [synth.look_at_camera(np.array(p) * 3.0, 70, 45, 60.0) for p in
            ([1, 0.2, 0.3], [-0.3, 1, 0.1], [0.2, -0.5, 1])]
    R = 300
    maps = rng.integers(0, R, size=(3, 45, 70)).astype(np.uint32)
    maps[1, :, :35] = rng.integers(0, 3, size=(45, 35))  # half the view few regions
    maps[2, 10:20, 10:20] = NONE
    codes = synth.make_codes(synth.CONFIGS["tiny"].with_(num_views=3, regions=(R,)), seed=4)
    ora = oracle.uplift(g, cams, maps, codes, 64, 4)
    res = run_gpu(g, cams, maps, codes, 64, 4)
    assert_parity(res, ora, 4)


@pytest.mark.parametrize("L,K,S", [(16, 1, 4), (63, 5, 3), (32, 16, 6), (128, 8, 12)])
def test_code_shapes_and_truncation(dev, tiny_scene, L, K, S):
    """L not a multiple of 4 (scalar Top-K loads), K = 1 and K = 16, S > K codes (Algorithm 1
    per-pixel TopK truncation), L = 128 (stress config)."""
    cfg, scene, maps, _ = tiny_scene
    c2 = cfg.with_(L=L, S=S, K=K)
    codes = synth.make_codes(c2, seed=5)
    cams = scene.cameras[:2]
    ora = oracle.uplift(scene.gaussians, cams, maps[:2], codes, L, K)
    res = run_gpu(scene.gaussians, cams, maps[:2], codes, L, K)
    assert_parity(res, ora, K)


def test_edge_cases_empty_and_culled(dev):
    """No Gaussian visible (all behind the camera), a single Gaussian, and padded rows."""
    cam = identity_camera(40, 30, 50.0)
    g = gaussians([[0, 0, -2], [0.1, 0, -3]], np.full((2, 3), 0.1), np.tile([1, 0, 0, 0], (2, 1)), [0.5, 0.9])
    codes = full_frame_codes([[(1, 1.0)]])
    ids = np.zeros((1, 30, 40), np.uint32)
    res = run_gpu(g, [cam], ids, codes, 8, 2, rows_padded=5)
    assert res["stats"]["contributions"] == 0 and np.all(res["W"] == 0) and np.all(res["Z"] == 0)
    assert np.all(res["atoms"] == NONE) and np.all(res["coefs"] == 0)
    g1 = gaussians([[0, 0, 2]], [[0.1, 0.05, 0.1]], [[1, 0.2, 0, 0]], [0.7])
    ora = oracle.uplift(g1, [cam], ids, codes, 8, 2)
    res = run_gpu(g1, [cam], ids, codes, 8, 2, rows_padded=4)
    assert_parity(res, ora, 2)


def test_closed_form_cases_on_gpu(dev):
    """F3/F4 on the GPU path: exact e values at the centre pixel (alpha = 0.5 -> 0.5, 0.25) and the
    termination reading, visible through W with a per-pixel one-hot region code."""
    cam = identity_camera(96, 96, 100.0, 48.5, 48.5)
    g = gaussians([[0, 0, 2], [0, 0, 3], [0, 0, 4]], np.full((3, 3), 0.2), np.tile([1, 0, 0, 0], (3, 1)),
                  [0.99, 0.99, 0.99])
    ids = np.full((1, 96, 96), 1, np.uint32)
    ids[0, 48, 48] = 0
    codes = synth.Codes(np.array([[5], [6]], np.uint32), np.array([[1.0], [1.0]], np.float32),
                        np.array([0], np.int64), np.array([2], np.int32))
    res = run_gpu(g, [cam], ids, codes, 8, 2)
    assert res["W"][0, 5] == np.float32(0.99)
    assert res["W"][1, 5] == 0.0 and res["W"][2, 5] == 0.0
    ora = oracle.uplift(g, [cam], ids, codes, 8, 2)
    assert_parity(res, ora, 2)


def test_data_errors_are_latched(dev, tiny_scene):
    """Region id >= R_v and atom >= L are data errors, reported at the next
    synchronising call with the offending index; reset clears them."""
    from paper_2605_13600_b200 import abi
    from paper_2605_13600_b200.uplift import SparseUplift
    cfg, scene, maps, codes = tiny_scene
    bad = maps[:1].copy()
    bad[0, 10, 20] = 999
    up = SparseUplift(scene.gaussians, cfg.L, cfg.K)
    try:
        up.add_views(scene.cameras[:1], bad, codes)
        with pytest.raises(abi.ScoupError) as ei:
            up.finalize()
        assert ei.value.status == 2 and str(10 * 64 + 20) in str(ei.value)
        with pytest.raises(abi.ScoupError) as ei:
            up.add_views(scene.cameras[:1], maps[:1], codes)
        assert ei.value.status == 5
        up.reset()
        bad_codes = synth.Codes(codes.atoms.copy(), codes.coefs, codes.row0, codes.num_regions)
        bad_codes.atoms[3, 1] = 64
        up.add_views(scene.cameras[:1], maps[:1], bad_codes)
        with pytest.raises(abi.ScoupError) as ei:
            up.finalize()
        assert ei.value.status == 2 and str(3 * 4 + 1) in str(ei.value)
        up.reset()
        cam = scene.cameras[0]
        skew = synth.Camera(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height,
                            cam.world_to_camera * np.float32(1.01))
        with pytest.raises(abi.ScoupError) as ei:
            up.add_views([skew], maps[:1], codes)
        assert ei.value.status == 2
    finally:
        up.close()
    with pytest.raises(abi.ScoupError) as ei:
        SparseUplift(scene.gaussians, 8, 9)
    assert ei.value.status == 1


def test_nonfinite_gaussian_latched(dev, tiny_scene):
    from paper_2605_13600_b200 import abi
    from paper_2605_13600_b200.uplift import SparseUplift
    cfg, scene, maps, codes = tiny_scene
    g = scene.gaussians
    m = g.means.copy()
    m[17, 1] = np.nan
    up = SparseUplift(synth.Gaussians(m, g.scales, g.rotations, g.opacities), cfg.L, cfg.K)
    try:
        up.add_views(scene.cameras[:1], maps[:1], codes)
        with pytest.raises(abi.ScoupError) as ei:
            up.finalize()
        assert ei.value.status == 2 and "17" in str(ei.value)
    finally:
        up.close()


def test_outdoor_full_size_sampled_views(dev):
    """configs[3] at full size (3M Gaussians, 1600x1066, L=64, S=K=8) in the launch configuration
    bench.py times, on 2 sampled views the oracle can compute: element-wise W/Z parity over all
    3M rows, exact per-view contribution counts, and Top-K code parity."""
    cfg = synth.CONFIGS["outdoor"]
    scene = synth.make_scene(cfg, 0)
    views = [0, 150]
    maps = synth.make_region_maps_torch(cfg, torch.device("cuda"), seed=0, views=views).cpu().numpy().view(np.uint32)
    codes = synth.make_codes(cfg, seed=0, views=views)
    cams = [scene.cameras[v] for v in views]
    ora = oracle.uplift(scene.gaussians, cams, maps, codes, cfg.L, cfg.K)
    res = run_gpu(scene.gaussians, cams, maps, codes, cfg.L, cfg.K)
    ties = assert_parity(res, ora, cfg.K)
    assert ties < 1e-3 * scene.gaussians.count


def test_extreme_gaussians(dev):
    """Degenerate footprints: near-plane off-screen giants (huge conics, strong fp32 cancellation
    in q), needle-thin rotated Gaussians, sub-pixel Gaussians, opacity at 1/255 and 1.0 -- the
    conservative tile/warp filters must not drop a single fragment (exact counts)."""
    from helpers import extreme_scene
    g, cams, maps, codes = extreme_scene()
    ora = oracle.uplift(g, cams, maps, codes, 64, 4)
    assert ora[2].sum() > 1000
    res = run_gpu(g, cams, maps, codes, 64, 4)
    assert_parity(res, ora, 4)


@pytest.mark.parametrize("near_frac", ["0.01", "0.3", "1.0"])
def test_depth_chunk_split_is_exact(dev, tiny_scene, tiny_oracle, near_frac, monkeypatch):
    """DESIGN.md §5 a3: the near/far depth split (any fraction; 1.0 = a single chunk) changes
    which Gaussians are binned when, never the per-pixel fragment sequence: exact counts and
    W/Z/code parity for every split."""
    monkeypatch.setenv("SCOUP_NEAR_FRAC", near_frac)
    cfg, scene, maps, codes = tiny_scene
    res = run_gpu(scene.gaussians, scene.cameras, maps, codes, cfg.L, cfg.K)
    assert_parity(res, tiny_oracle, cfg.K)


def _band(cam, y0, y1):
    """Rows [y0, y1) of a view as a camera of its own (same rays, principal point shifted)."""
    return synth.Camera(cam.fx, cam.fy, cam.cx, cam.cy - y0, cam.width, y1 - y0, cam.world_to_camera)


def run_gpu_levels(g, cams, maps_by_level, codes_by_level, L, K, host_maps=False):
    """Fused multi-level uplift (one raster pass for every level) through the C ABI (host_maps:
    the region maps stay host arrays; the library copies them up front on its copy stream)."""
    from paper_2605_13600_b200.uplift import SparseUplift
    V, M = len(cams), len(maps_by_level)
    gin = synth.Gaussians(*[torch.from_numpy(np.ascontiguousarray(a)).cuda()
                            for a in (g.means, g.scales, g.rotations, g.opacities)])
    ids = [torch.from_numpy(np.ascontiguousarray(m).view(np.int32)) for m in maps_by_level]
    ids = [i.pin_memory() if host_maps else i.cuda() for i in ids]
    cods = [synth.Codes(torch.from_numpy(np.ascontiguousarray(c.atoms).view(np.int32)).cuda(),
                        torch.from_numpy(np.ascontiguousarray(c.coefs)).cuda(), c.row0, c.num_regions)
            for c in codes_by_level]
    contrib = torch.zeros(V, dtype=torch.int64, device="cuda")
    up = SparseUplift(gin, L, K, levels=M)
    try:
        up.add_views(cams, ids, cods, contributions_out=contrib)
        out = []
        for lvl in range(M):
            atoms, coefs = up.finalize(level=lvl)
            out.append((atoms.cpu().numpy().view(np.uint32), coefs.cpu().numpy()))
        torch.cuda.synchronize()
        W = up.W[:, :g.count].double().cpu().numpy()
        Z = up.Z[:g.count].double().cpu().numpy()
        return dict(W=W, Z=Z, codes=out, contrib=contrib.cpu().numpy(), stats=up.stats())
    finally:
        up.close()


def assert_levels_parity(res, oras, K):
    for lvl, ora in enumerate(oras):
        r = dict(W=res["W"][lvl], Z=res["Z"], atoms=res["codes"][lvl][0], coefs=res["codes"][lvl][1],
                 contrib=res["contrib"], stats=res["stats"])
        assert_parity(r, ora, K)


def test_fused_levels_tiny(dev):
    """three nested region levels (8 / 32 / 128 regions, 10% of them
    unassigned) fused into one raster pass equal three separate oracle uplifts: W per level, one
    shared Z (it counts every fragment), codes per level, exact counts."""
    cfg = synth.CONFIGS["tiny"].with_(regions=(8, 32, 128), unassigned_frac=0.1)
    scene = synth.make_scene(cfg, 7)
    maps = [synth.make_region_maps_numpy(cfg, level=l, seed=7) for l in range(3)]
    codes = [synth.make_codes(cfg, level=l, seed=7) for l in range(3)]
    oras = [oracle.uplift(scene.gaussians, scene.cameras, maps[l], codes[l], cfg.L, cfg.K) for l in range(3)]
    res = run_gpu_levels(scene.gaussians, scene.cameras, maps, codes, cfg.L, cfg.K)
    assert_levels_parity(res, oras, cfg.K)
    # host (pinned) maps: chunked up-front copies on the library's copy stream, same results
    res = run_gpu_levels(scene.gaussians, scene.cameras, maps, codes, cfg.L, cfg.K, host_maps=True)
    assert_levels_parity(res, oras, cfg.K)


def test_fused_levels_odd_code_length(dev):
    """Two fused levels with S = 3 codes (nlev * S = 6 and S not powers of two: the flush's
    index arithmetic by multiply-high instead of shifts) equal two separate oracle uplifts."""
    cfg = synth.CONFIGS["tiny"].with_(regions=(8, 64), S=3, K=3, unassigned_frac=0.1)
    scene = synth.make_scene(cfg, 11)
    maps = [synth.make_region_maps_numpy(cfg, level=l, seed=11) for l in range(2)]
    codes = [synth.make_codes(cfg, level=l, seed=11) for l in range(2)]
    oras = [oracle.uplift(scene.gaussians, scene.cameras, maps[l], codes[l], cfg.L, cfg.K) for l in range(2)]
    res = run_gpu_levels(scene.gaussians, scene.cameras, maps, codes, cfg.L, cfg.K)
    assert_levels_parity(res, oras, cfg.K)


def test_fused_levels_indoor_full_size(dev):
    """configs[2] at full size (1M Gaussians: 100 clusters + 10% shell, 988x731, Dirichlet(0.5)
    codes), its three nested levels (32 / 128 / 512 regions) fused in one pass, on 2 sampled
    views: element-wise W/Z parity for every level, exact contribution counts, Top-K parity."""
    cfg = synth.CONFIGS["indoor"]
    scene = synth.make_scene(cfg, 0)
    views = [3, 101]
    maps = [synth.make_region_maps_torch(cfg, torch.device("cuda"), level=l, seed=0, views=views)
            .cpu().numpy().view(np.uint32) for l in range(3)]
    codes = [synth.make_codes(cfg, level=l, seed=0, views=views) for l in range(3)]
    cams = [scene.cameras[v] for v in views]
    oras = [oracle.uplift(scene.gaussians, cams, maps[l], codes[l], cfg.L, cfg.K) for l in range(3)]
    res = run_gpu_levels(scene.gaussians, cams, maps, codes, cfg.L, cfg.K)
    assert_levels_parity(res, oras, cfg.K)
    # the single-level path on the finest level agrees too
    single = run_gpu(scene.gaussians, cams, maps[2], codes[2], cfg.L, cfg.K)
    assert_parity(single, oras[2], cfg.K)


def test_fused_levels_errors(dev, tiny_scene):
    """A bad region id names its level; the level count is bounded (SCOUP_MAX_LEVELS = 4,
    levels * S <= SCOUP_MAX_S); finalize on a missing level is EINVAL."""
    from paper_2605_13600_b200 import abi
    from paper_2605_13600_b200.uplift import SparseUplift
    cfg, scene, maps, codes = tiny_scene
    up = SparseUplift(scene.gaussians, cfg.L, cfg.K, levels=2)
    try:
        bad = maps[:1].copy()
        bad[0, 5, 7] = 777
        up.add_views(scene.cameras[:1], [maps[:1], bad], [codes, codes])
        with pytest.raises(abi.ScoupError) as ei:
            up.finalize()
        assert ei.value.status == 2 and "level 1" in str(ei.value) and str(5 * 64 + 7) in str(ei.value)
        with pytest.raises(abi.ScoupError) as ei:
            up.finalize(level=2)
        assert ei.value.status == 1
    finally:
        up.close()
    with pytest.raises(abi.ScoupError) as ei:
        SparseUplift(scene.gaussians, cfg.L, cfg.K, levels=5)
    assert ei.value.status == 6


def test_stress_full_size_row_band(dev):
    """configs[4] at full scene size (6M heavily overlapping Gaussians, L=128, S=K=8, 1920-px
    rows): the oracle's cost per full 1920x1080 view is minutes, so the sample is a 48-row band
    of one view (the same rays; principal point shifted), run through the same batched, chunked
    GPU path.  Element-wise parity over all 6M rows and exact counts."""
    cfg = synth.CONFIGS["stress"]
    scene = synth.make_scene(cfg, 0)
    v, y0, y1 = 5, 516, 564
    full = synth.make_region_maps_torch(cfg, torch.device("cuda"), seed=0, views=[v]).cpu().numpy().view(np.uint32)
    maps = np.ascontiguousarray(full[:, y0:y1])
    codes = synth.make_codes(cfg, seed=0, views=[v])
    cams = [_band(scene.cameras[v], y0, y1)]
    ora = oracle.uplift(scene.gaussians, cams, maps, codes, cfg.L, cfg.K)
    assert ora[2].sum() > 1_000_000
    res = run_gpu(scene.gaussians, cams, maps, codes, cfg.L, cfg.K)
    assert_parity(res, ora, cfg.K)


def run_gpu_dense(g, cams, maps, feats, D):
    from paper_2605_13600_b200.uplift import SparseUplift
    gin = synth.Gaussians(*[torch.from_numpy(np.ascontiguousarray(a)).cuda()
                            for a in (g.means, g.scales, g.rotations, g.opacities)])
    ids = torch.from_numpy(np.ascontiguousarray(maps).view(np.int32)).cuda()
    fd = synth.Codes(None, torch.from_numpy(np.ascontiguousarray(feats.coefs)).cuda(), feats.row0, feats.num_regions)
    up = SparseUplift(gin, D, 1)
    try:
        up.add_views(cams, ids, fd)
        torch.cuda.synchronize()
        return up.W[:g.count].double().cpu().numpy(), up.Z[:g.count].double().cpu().numpy()
    finally:
        up.close()


@pytest.mark.parametrize("D", [48, 64, 512])
def test_dense_feature_uplift(dev, tiny_scene, D):
    """the dense feature uplift of Eq. 3 that SCOUP's sparse
    uplift replaces -- every region carries a full D-vector of CLIP-like features (both signs),
    D = 64 and the paper's D = 512 -- through the same raster path (code_atoms = NULL): W and Z
    element-wise against the oracle's dense path."""
    cfg, scene, maps, _ = tiny_scene
    feats = synth.make_dense_features(cfg, D, seed=3)
    Wo, Zo, fo = oracle.uplift_accumulate(scene.gaussians, scene.cameras, maps, None, feats.coefs, feats.row0,
                                          feats.num_regions, D, 1)
    W, Z = run_gpu_dense(scene.gaussians, scene.cameras, maps, feats, D)
    # Z has no cancellation: the north star's bar as it stands (1e-4 rel, 1e-6 abs)
    bad_w, bad_z = compare_accumulators(W, Z, Wo, Zo, RTOL, ATOL)
    assert len(bad_z) == 0, len(bad_z)
    # W: features of both signs cancel, so |W| can be far below the magnitude sum M = sum |c e|
    # of its terms.  Cancellation-aware bound: the north star's 1e-6 + 1e-4 |W| plus the
    # forward error of an fp32 sum of n terms in any order, |err| <= (n - 1) u sum|x_i|
    # (Higham, Accuracy and Stability of Numerical Algorithms, 2nd ed., Thm 4.1 / eq. 4.4;
    # u = 2^-24), with n = the Gaussian's fragment count and M from the oracle run on |features|
    # (the products |c| e are the same fp32 numbers up to sign).
    Mo, _, _ = oracle.uplift_accumulate(scene.gaussians, scene.cameras, maps, None, np.abs(feats.coefs),
                                        feats.row0, feats.num_regions, D, 1)
    n = np.zeros(scene.gaussians.count)
    for cam in scene.cameras:
        n += np.bincount(oracle.render_view(scene.gaussians, cam)[2], minlength=scene.gaussians.count)
    err = np.abs(W - Wo)
    strict = ATOL + RTOL * np.abs(Wo)
    bound = strict + np.maximum(n - 1, 0)[:, None] * 2.0 ** -24 * Mo
    assert np.all(err <= bound), (int((err > bound).sum()), float((err - bound).max()))
    # only cancelled elements (|W| well below M) may use the extra term
    used = err > strict
    assert np.all(np.abs(Wo[used]) < 1e-2 * Mo[used]), int(used.sum())
    assert (Wo < 0).any()  # the features have both signs


def oracle_render(g, cams, atoms, coefs, L, cap=1 << 22):
    """Eq. 7 from the oracle's fragment lists: W_hat_v(p) = sum_i w_hat_i e_i(v,p) (fp64)."""
    out = np.zeros((len(cams), cams[0].height, cams[0].width, L))
    K = atoms.shape[1]
    for v, cam in enumerate(cams):
        T, pix, gid, e = oracle.render_view(g, cam, cap=cap)
        flat = out[v].reshape(-1, L)
        for k in range(K):
            a = atoms[gid, k].astype(np.int64) & 0xFFFFFFFF
            ok = a != NONE
            # the spec's fp32 products coef * e, summed in fp64
            prod = (coefs[gid[ok], k].astype(np.float32) * e[ok]).astype(np.float64)
            np.add.at(flat, (pix[ok], a[ok]), prod)
    return out


def test_render_and_decode(dev, tiny_scene):
    """sparse coefficient rendering (Eq. 7) with the uplifted
    K-sparse codes, on the same fragments as the uplift, against the oracle's fragment lists;
    then the codebook decode F = W_hat C (Eq. 8) against a float64 product."""
    from paper_2605_13600_b200.uplift import SparseUplift
    cfg, scene, maps, codes = tiny_scene
    g = scene.gaussians
    gin = synth.Gaussians(*[torch.from_numpy(np.ascontiguousarray(a)).cuda()
                            for a in (g.means, g.scales, g.rotations, g.opacities)])
    up = SparseUplift(gin, cfg.L, cfg.K)
    try:
        up.add_views(scene.cameras, maps, codes)
        atoms, coefs = up.finalize()
        Wh = up.render(scene.cameras, atoms, coefs)
        C = torch.from_numpy(np.random.default_rng(4).normal(size=(cfg.L, 512)).astype(np.float32)).cuda()
        F = up.decode(Wh, C)
        torch.cuda.synchronize()
        a_np = atoms.cpu().numpy().view(np.uint32)
        c_np = coefs.cpu().numpy()
        ref = oracle_render(g, scene.cameras, a_np, c_np, cfg.L)
        got = Wh.double().cpu().numpy()
        assert np.abs(ref).max() > 0.1
        bad = np.abs(got - ref) > 1e-6 + 1e-5 * np.abs(ref)
        assert not bad.any(), (bad.sum(), np.abs(got - ref).max())
        # rendered coefficients of a pixel sum to its accumulated alpha (codes are L1-normalised)
        Fref = ref.reshape(-1, cfg.L) @ C.double().cpu().numpy()
        Fg = F.double().cpu().numpy().reshape(-1, 512)
        assert np.allclose(Fg, Fref, rtol=1e-4, atol=1e-4)
    finally:
        up.close()


def test_render_full_size_outdoor_view(dev):
    """Eq. 7 at configs[3] full size (3M Gaussians, K = 8) through the depth-chunked GPU path on
    three row bands of a 1600-wide view: per-pixel parity with the oracle's fragment lists."""
    from paper_2605_13600_b200.uplift import SparseUplift
    cfg = synth.CONFIGS["outdoor"]
    scene = synth.make_scene(cfg, 0)
    g = scene.gaussians
    rng = np.random.default_rng(2)
    K = cfg.K
    atoms = rng.integers(0, cfg.L, size=(g.count, K)).astype(np.uint32)  # repeats allowed: Eq. 7 sums them
    atoms[rng.uniform(size=(g.count, K)) < 0.1] = NONE
    coefs = rng.dirichlet(np.ones(K), size=g.count).astype(np.float32)
    # row bands of view 17 (top edge, middle, ragged bottom edge) as cameras of their own, on
    # both sides, so every fragment the oracle lists is the GPU's exact sequence
    cam = scene.cameras[17]
    cams = [_band(cam, 0, 24), _band(cam, 520, 544), _band(cam, 1048, 1066)]
    gin = synth.Gaussians(*[torch.from_numpy(np.ascontiguousarray(a)).cuda()
                            for a in (g.means, g.scales, g.rotations, g.opacities)])
    up = SparseUplift(gin, cfg.L, K)
    try:
        got = []
        for c in cams:
            Wh = up.render([c], torch.from_numpy(atoms.view(np.int32)).cuda(), torch.from_numpy(coefs).cuda())
            got.append(Wh.double().cpu().numpy())
    finally:
        up.close()
    for c, gv in zip(cams, got):
        ref = oracle_render(g, [c], atoms, coefs, cfg.L, cap=1 << 26)
        assert np.abs(ref).max() > 0.1
        bad = np.abs(gv - ref) > 1e-6 + 1e-5 * np.abs(ref)
        assert not bad.any(), (bad.sum(), np.abs(gv - ref).max())


def test_render_errors(dev, tiny_scene):
    """Render input checks: an atom >= L (not SCOUP_NONE) or a non-finite coefficient is a latched
    EDATA naming the flat code slot; L > 128 is EUNSUPPORTED; K outside [1, 32] is EINVAL."""
    from paper_2605_13600_b200 import abi
    from paper_2605_13600_b200.uplift import SparseUplift
    cfg, scene, maps, codes = tiny_scene
    g = scene.gaussians
    K = 4
    atoms = torch.zeros((g.count, K), dtype=torch.int32, device="cuda")
    coefs = torch.full((g.count, K), 0.25, dtype=torch.float32, device="cuda")
    up = SparseUplift(g, cfg.L, K)
    try:
        up.render(scene.cameras[:1], atoms, coefs)
        up.stats()  # all rows valid (atom 0 four times: merged)
        # a slot of a Gaussian that surely renders: the one with the largest opacity
        gi = int(np.argmax(g.opacities))
        atoms[gi, 2] = cfg.L
        up.render(scene.cameras, atoms, coefs)
        with pytest.raises(abi.ScoupError) as ei:
            up.stats()
        assert ei.value.status == 2 and str(gi * K + 2) in str(ei.value)
        up.reset()
        with pytest.raises(abi.ScoupError) as ei:
            up.render(scene.cameras[:1], atoms[:, :0], coefs[:, :0])
        assert ei.value.status == 1
    finally:
        up.close()
    up = SparseUplift(g, 256, K)
    try:
        with pytest.raises(abi.ScoupError) as ei:
            up.render(scene.cameras[:1], atoms, coefs)
        assert ei.value.status == 6
    finally:
        up.close()


@pytest.mark.parametrize("L,D,P", [(64, 512, 1000), (8, 64, 129), (16, 192, 4096), (64, 768, 300),
                                   (40, 128, 7), (72, 512, 500)])
def test_decode_matches_fp64(dev, L, D, P):
    """Eq. 8 F = W_hat C against a float64 product.  L % 8 == 0, L <= 64 and D % 64
    == 0 run the tcgen05 3xTF32 kernel (ragged last 128-row tile, 1-4 N tiles of 64/128/256
    columns); L = 72 takes the cuBLAS SGEMM path.  Bound: fp32-GEMM accuracy, |F - F64| <=
    1e-5 (|W_hat| |C|) + 1e-30, i.e. ~40 ulp of the magnitude sum (3xTF32 drops terms below
    2^-20 relative per product; fp32 accumulation adds <= L 2^-24)."""
    from paper_2605_13600_b200.uplift import SparseUplift
    g = synth.Gaussians(*(np.zeros((1, 3), np.float32), np.full((1, 3), 0.1, np.float32),
                          np.array([[1, 0, 0, 0]], np.float32), np.full((1,), 0.5, np.float32)))
    rng = np.random.default_rng(L * 1000 + D)
    W = rng.normal(size=(P, L)).astype(np.float32) * rng.choice([1e-3, 1.0, 1e3], size=(P, 1)).astype(np.float32)
    C = rng.normal(size=(L, D)).astype(np.float32)
    up = SparseUplift(g, L, 1)
    try:
        n0 = up.stats()["kernel_launches"]
        F = up.decode(torch.from_numpy(W).cuda(), torch.from_numpy(C).cuda())
        torch.cuda.synchronize()
        got = F.double().cpu().numpy()
        # the library's own kernels (prep + tcgen05 decode) ran, or none (cuBLAS)
        assert up.stats()["kernel_launches"] - n0 == (2 if L <= 64 and L % 8 == 0 else 0)
    finally:
        up.close()
    ref = W.astype(np.float64) @ C.astype(np.float64)
    bound = 1e-5 * (np.abs(W.astype(np.float64)) @ np.abs(C.astype(np.float64))) + 1e-30
    err = np.abs(got - ref)
    assert (err <= bound).all(), (int((err > bound).sum()), float((err / bound).max()))


@pytest.mark.parametrize("world", [2, 3])
def test_fused_peer_reduce_topk_matches_oracle(dev, tiny_scene, world):
    """SURVEY.md §8(e) fused exchange, with the ranks emulated as `world` accumulators on one GPU
    (one kernel reads every rank's data, as the ranks' kernels would over NVLink): each rank
    accumulates the views v = r (mod P) into its own W; finalize_topk_peers then sums each rank's
    row shard over all partials and runs Eq. 6.  The concatenated shard codes equal the oracle's
    codes of the whole view set (Top-K comparator, fp32 reassociation only)."""
    from helpers import compare_codes
    from paper_2605_13600_b200 import abi
    from paper_2605_13600_b200 import distributed as D
    from paper_2605_13600_b200.uplift import SparseUplift
    cfg, scene, maps, codes = tiny_scene
    g = scene.gaussians
    Wo = oracle.uplift(g, scene.cameras, maps, codes, cfg.L, cfg.K)[0]
    gin = synth.Gaussians(*[torch.from_numpy(np.ascontiguousarray(a)).cuda()
                            for a in (g.means, g.scales, g.rotations, g.opacities)])
    Npad = D.padded_rows(g.count, world)
    ups = [SparseUplift(gin, cfg.L, cfg.K, rows_padded=Npad) for _ in range(world)]
    try:
        ids = torch.from_numpy(np.ascontiguousarray(maps).view(np.int32)).cuda()
        for r, up in enumerate(ups):
            vs = D.views_for_rank(len(scene.cameras), r, world)
            sub = synth.Codes(torch.from_numpy(np.ascontiguousarray(codes.atoms).view(np.int32)).cuda(),
                              torch.from_numpy(np.ascontiguousarray(codes.coefs)).cuda(),
                              np.ascontiguousarray(codes.row0[vs]), np.ascontiguousarray(codes.num_regions[vs]))
            up.add_views([scene.cameras[v] for v in vs], ids[vs].contiguous(), sub)
        torch.cuda.synchronize()
        peers = [up.W.data_ptr() for up in ups]
        atoms, coefs = [], []
        for r, up in enumerate(ups):
            first, n = D.row_shard(g.count, r, world)
            a = torch.empty((n, cfg.K), dtype=torch.int32, device="cuda")
            c = torch.empty((n, cfg.K), dtype=torch.float32, device="cuda")
            abi.scoup_uplift_finalize_topk_peers(up._h, 0, first, n, peers, a, c)
            atoms.append(a.cpu().numpy())
            coefs.append(c.cpu().numpy())
    finally:
        for up in ups:
            up.close()
    A = np.concatenate(atoms)[:g.count].view(np.uint32)
    Cc = np.concatenate(coefs)[:g.count]
    bad, ties, worst = compare_codes(A, Cc, Wo, cfg.K)
    assert bad == 0, worst


def test_finalize_entropy_matches_oracle(dev, tiny_scene, tiny_oracle):
    """the pre-Top-K coefficient entropy, computed in the Top-K pass,
    equals the oracle's from its fp64 W (fp32 sums and logf: 1e-5 relative + 1e-6 absolute);
    uncoded Gaussians get NaN on both sides; the codes of this entry point equal finalize's."""
    from paper_2605_13600_b200.uplift import SparseUplift
    cfg, scene, maps, codes = tiny_scene
    Wo = tiny_oracle[0]
    g = scene.gaussians
    gin = synth.Gaussians(*[torch.from_numpy(np.ascontiguousarray(a)).cuda()
                            for a in (g.means, g.scales, g.rotations, g.opacities)])
    up = SparseUplift(gin, cfg.L, cfg.K)
    try:
        up.add_views(scene.cameras, torch.from_numpy(np.ascontiguousarray(maps).view(np.int32)).cuda(),
                     synth.Codes(torch.from_numpy(codes.atoms.view(np.int32)).cuda(),
                                 torch.from_numpy(codes.coefs).cuda(), codes.row0, codes.num_regions))
        a1, c1 = up.finalize()
        a2, c2, H = up.finalize_with_entropy()
        H = H.double().cpu().numpy()
        assert torch.equal(a1, a2) and torch.equal(c1, c2)
    finally:
        up.close()
    Ho = oracle.entropy(Wo)
    assert np.array_equal(np.isnan(H), np.isnan(Ho))
    ok = ~np.isnan(Ho)
    assert ok.sum() > 100
    assert np.all(np.abs(H[ok] - Ho[ok]) <= 1e-6 + 1e-5 * np.abs(Ho[ok]))


def test_peer_finalize_single_peer_equals_finalize(dev, tiny_scene):
    """finalize_topk_peers with one peer (the handle's own W) reproduces finalize_topk bit for bit
    (the same row sums, the same Top-K), also on a ragged sub-range of rows."""
    from paper_2605_13600_b200 import abi
    from paper_2605_13600_b200.uplift import SparseUplift
    cfg, scene, maps, codes = tiny_scene
    g = scene.gaussians
    gin = synth.Gaussians(*[torch.from_numpy(np.ascontiguousarray(a)).cuda()
                            for a in (g.means, g.scales, g.rotations, g.opacities)])
    up = SparseUplift(gin, cfg.L, cfg.K)
    try:
        up.add_views(scene.cameras, torch.from_numpy(np.ascontiguousarray(maps).view(np.int32)).cuda(),
                     synth.Codes(torch.from_numpy(codes.atoms.view(np.int32)).cuda(),
                                 torch.from_numpy(codes.coefs).cuda(), codes.row0, codes.num_regions))
        a1, c1 = up.finalize(37, 1001)
        a2 = torch.empty_like(a1)
        c2 = torch.empty_like(c1)
        abi.scoup_uplift_finalize_topk_peers(up._h, 0, 37, 1001, [up.W.data_ptr()], a2, c2)
        assert torch.equal(a1, a2) and torch.equal(c1, c2)
        with pytest.raises(abi.ScoupError) as ei:  # more than SCOUP's 16 peers
            abi.scoup_uplift_finalize_topk_peers(up._h, 0, 0, 10, [up.W.data_ptr()] * 17, a2, c2)
        assert ei.value.status == 1
    finally:
        up.close()


@pytest.mark.parametrize("K", [1, 32])
def test_render_code_lengths(dev, tiny_scene, K):
    """Eq. 7 with stored codes of K = 1 and K = 32 slots (half of them empty), against the oracle's
    fragment lists."""
    from paper_2605_13600_b200.uplift import SparseUplift
    cfg, scene, _, _ = tiny_scene
    g = scene.gaussians
    rng = np.random.default_rng(K)
    atoms = rng.integers(0, cfg.L, size=(g.count, K)).astype(np.uint32)
    if K > 1:
        atoms[:, K // 2:] = NONE
    coefs = rng.uniform(0.1, 1.0, size=(g.count, K)).astype(np.float32)
    gin = synth.Gaussians(*[torch.from_numpy(np.ascontiguousarray(a)).cuda()
                            for a in (g.means, g.scales, g.rotations, g.opacities)])
    up = SparseUplift(gin, cfg.L, min(K, 8))
    try:
        Wh = up.render(scene.cameras[:2], torch.from_numpy(atoms.view(np.int32)).cuda(),
                       torch.from_numpy(coefs).cuda()).double().cpu().numpy()
    finally:
        up.close()
    ref = oracle_render(g, scene.cameras[:2], atoms, coefs, cfg.L)
    assert np.abs(ref).max() > 0.05
    assert np.all(np.abs(Wh - ref) <= 1e-6 + 1e-5 * np.abs(ref))


@pytest.mark.parametrize("L,K,density,levels", [(64, 8, 1.0, 6), (64, 8, 0.3, 0), (64, 4, 1.0, 3), (10, 4, 0.7, 4),
                                                (100, 16, 1.0, 5), (64, 1, 1.0, 2), (8, 8, 1.0, 3)])
def test_topk_kernel_exact_on_dense_rows_with_ties(dev, L, K, density, levels):
    """Eq. 6 selection on finalize_topk's own rows: dense and sparse random rows, some
    drawn from a few discrete levels so that exact ties at the K-th value are common, plus all-zero,
    single-positive and all-equal rows and negative entries.  The atoms must equal oracle.topk's
    (value desc, atom asc, positive only) EXACTLY -- the candidate bound (minimum of K group
    maxima) may not change the tie rule -- and the coefficients its fp64 L1 renormalisation to
    fp32 rounding."""
    from paper_2605_13600_b200.uplift import SparseUplift
    rng = np.random.default_rng([L, K, levels])
    G = 20_000
    if levels:
        W = rng.integers(0, levels, size=(G, L)).astype(np.float32) * np.float32(0.25)
    else:
        W = rng.random((G, L), dtype=np.float32)
    W = np.where(rng.random((G, L)) < density, W, 0.0).astype(np.float32)
    W[0] = 0.0
    W[1] = 0.0
    W[1, L - 1] = 1.0
    W[2] = 0.5
    W[3] = -rng.random(L).astype(np.float32)
    W[4, : L // 2] = -1.0
    g = synth.Gaussians(np.zeros((G, 3), np.float32), np.full((G, 3), 0.1, np.float32),
                        np.tile(np.array([[1, 0, 0, 0]], np.float32), (G, 1)), np.full((G,), 0.5, np.float32))
    with SparseUplift(g, L, K, rows_padded=G) as up:
        a, c = up.finalize(0, G, W_rows=torch.from_numpy(W).to(dev))
        torch.cuda.synchronize()
        a = a.cpu().numpy().view(np.uint32)
        c = c.cpu().numpy().astype(np.float64)
    ao, co = oracle.topk(W, K)
    assert np.array_equal(a, ao), np.argwhere(np.any(a != ao, axis=1))[:5].ravel()
    assert np.all(np.abs(c - co) <= 1e-6 * np.abs(co) + 1e-7)
