"""GPU parity: the sm_100a path through the C ABI vs the reference outputs.

Bars (north star / SURVEY §8d): projections and tile bins bit-exact; images within
1e-4 rel / 1e-3 abs (asserted) and in practice <= 1e-12; n_missing exact;
entropy_sum within 1e-11 relative; i_total within 1e-3 relative with the same argmax.
"""
import math

import numpy as np
import pytest

from conftest import golden_scene, random_map

import paper_2506_00225_b200 as sgm
from paper_2506_00225_b200 import scenes
from paper_2506_00225_b200.splatmap import (CameraModel, Pose, RenderChannels, RenderOptions,
                                            look_at)

pytestmark = pytest.mark.gpu

IMG_RTOL, IMG_ATOL = 1e-4, 1e-3  # north-star image tolerance
TIGHT = 1e-10                     # what the fp64 kernels actually achieve
ENT_RTOL = 1e-11


@pytest.fixture(scope="module")
def ctx():
    return sgm.Context(0)


def assert_planes(out, ref, keys=("silhouette", "color", "depth", "sem")):
    for key in keys:
        r = ref[key]
        if r is None:
            continue
        g = getattr(out, key)
        assert g.shape == r.shape, key
        np.testing.assert_allclose(g, r, rtol=IMG_RTOL, atol=IMG_ATOL, err_msg=key)
        assert np.max(np.abs(g - r), initial=0.0) <= TIGHT, (key, np.max(np.abs(g - r)))


def assert_projections(out, proj):
    assert len(out.projections) == len(proj)
    for f in ("mx", "my", "rad_px", "z", "alpha", "index"):
        np.testing.assert_array_equal(out.projections[f], proj[f], err_msg=f)


def assert_bins(ctx, orc, gm, cam, pose, opts, out):
    tiles = ((cam.width + opts.tile_size - 1) // opts.tile_size) * \
            ((cam.height + opts.tile_size - 1) // opts.tile_size)
    off, ids, probe = sgm.bins_of_last_render(tiles, ctx)
    o_off, o_ids, o_probe = orc.bins(orc.project(gm, cam, pose, opts), cam, opts)
    np.testing.assert_array_equal(off, o_off)
    np.testing.assert_array_equal(ids, o_ids)
    np.testing.assert_array_equal(probe, o_probe)


GOLDEN = ["saturated", "two_half", "sparse_scatter", "kM_11", "kM_22", "kM_33", "mass_5",
          "mass_6", "mass_7", "mass_8", "perm_19", "tiled_91", "early_55", "noearly_55",
          "score_8", "multi_2024"]


@pytest.mark.parametrize("name", GOLDEN)
def test_render_matches_reference_golden(ctx, orc, golden, name):
    gm, cam, pose, opts, ch, outs = golden_scene(golden, name)
    out = sgm.render(gm, cam, pose, RenderChannels.all(), opts, ctx=ctx)
    assert_projections(out, outs["projections"])
    assert_planes(out, outs)
    assert_bins(ctx, orc, gm, cam, pose, opts, out)
    h = sgm.render_entropy(gm, cam, pose, opts, ctx=ctx)
    np.testing.assert_allclose(h, outs["entropy"], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("name", ["kM_11", "tiled_91", "early_55", "noearly_55", "perm_19",
                                  "score_8", "saturated"])
def test_retained_contributors_match_reference(ctx, golden, name):
    """RenderOutput.contrib / contrib_offset (splat_render.cpp:215-216, 310, 125-137)."""
    gm, cam, pose, opts, _, outs = golden_scene(golden, name)
    out = sgm.render(gm, cam, pose, RenderChannels.all(True), opts, ctx=ctx)
    np.testing.assert_array_equal(out.contrib_offset, outs["contrib_offset"])
    np.testing.assert_array_equal(out.contrib, outs["contrib"])
    assert_planes(out, outs)


def test_retained_contributors_random_vs_reference(ctx, ref):
    cam = CameraModel(77, 53, 0, 0, 61.0, 59.5, 38.3, 26.1)
    pose = look_at([0.2, -0.1, -0.4], [0.0, 0.2, 2.5])
    gm = random_map(21, 500, cam, pose, k=4, num_classes=9)
    gm.opacity_logits[::17] = -1e4  # alpha == 0 contributors stay in the lists
    for opts in (RenderOptions(), RenderOptions(early_exit=False)):
        out = sgm.render(gm, cam, pose, RenderChannels.all(True), opts, ctx=ctx)
        r = ref.render(gm, cam, pose, 15, opts)
        np.testing.assert_array_equal(out.contrib_offset, r["contrib_offset"])
        np.testing.assert_array_equal(out.contrib, r["contrib"])


@pytest.mark.parametrize("name", ["tiled_91", "kM_11", "kM_22", "kM_33", "early_55", "perm_19"])
def test_render_reference_matches_reference(ctx, ref, golden, name):
    """render_reference (splat_render.cpp:330-358) against the reference's own: planes within
    1e-12 (test_splat_render.cpp:143-158 holds the tiled path to that bar), identical
    projections and contributor lists."""
    gm, cam, pose, _, _, _ = golden_scene(golden, name)
    out = sgm.render_reference(gm, cam, pose, RenderChannels.all(True), ctx=ctx)
    r = ref.render(gm, cam, pose, 15, which=1)
    for key in ("silhouette", "color", "depth", "sem"):
        assert np.max(np.abs(getattr(out, key) - r[key]), initial=0.0) < 1e-12, key
    assert_projections(out, r["projections"])
    np.testing.assert_array_equal(out.contrib_offset, r["contrib_offset"])
    np.testing.assert_array_equal(out.contrib, r["contrib"])


def test_render_reference_skips_zero_footprints(ctx, ref):
    """composite_pixel's `f <= 0` skip (:92): alpha == 0 splats are contributors of render()
    (it has no such test) but not of render_reference()."""
    cam = CameraModel(61, 47, 0, 0, 52.0, 50.5, 30.2, 23.4)
    pose = look_at([0.1, 0.0, -0.3], [0.0, 0.1, 2.0])
    gm = random_map(33, 400, cam, pose, k=3, num_classes=7)
    gm.opacity_logits[::9] = -1e4  # sigmoid -> exactly 0
    out = sgm.render_reference(gm, cam, pose, RenderChannels.all(True), ctx=ctx)
    r = ref.render(gm, cam, pose, 15, which=1)
    np.testing.assert_array_equal(out.contrib_offset, r["contrib_offset"])
    np.testing.assert_array_equal(out.contrib, r["contrib"])
    for key in ("silhouette", "color", "depth", "sem"):
        assert np.max(np.abs(getattr(out, key) - r[key]), initial=0.0) < 1e-12, key
    tiled = sgm.render(gm, cam, pose, RenderChannels.all(True), RenderOptions(early_exit=False),
                       ctx=ctx)
    assert len(tiled.contrib) > len(out.contrib)  # the alpha == 0 splats listed by render()
    np.testing.assert_allclose(tiled.silhouette, out.silhouette, rtol=0, atol=1e-12)


def test_reference_kats_on_gpu(ctx, golden):
    gm, cam, pose, opts, _, _ = golden_scene(golden, "saturated")
    out = sgm.render(gm, cam, pose, ctx=ctx)
    assert out.silhouette_at(8, 6) == pytest.approx(1.0, rel=1e-5)
    assert out.depth_at(8, 6) == pytest.approx(1.5, rel=1e-5)
    np.testing.assert_allclose(out.color_at(8, 6), [0.2, 0.6, 0.9], rtol=1e-5)
    gm, cam, pose, opts, _, _ = golden_scene(golden, "two_half")
    out = sgm.render(gm, cam, pose, ctx=ctx)
    assert out.silhouette_at(8, 6) == pytest.approx(0.75, rel=1e-9)
    assert out.depth_at(8, 6) == pytest.approx(1.0, rel=1e-9)
    gm, cam, pose, opts, _, _ = golden_scene(golden, "sparse_scatter")
    out = sgm.render(gm, cam, pose, ctx=ctx)
    p = out.sem_at(8, 6)
    assert p[3] == pytest.approx(0.9, rel=1e-5) and p[7] == pytest.approx(0.1, rel=1e-5)
    assert all(p[m] == 0.0 for m in range(out.channels) if m not in (3, 7))
    # mass conservation (test_splat_render.cpp:100-117)
    for seed in (5, 6, 7, 8):
        gm, cam, pose, opts, _, _ = golden_scene(golden, f"mass_{seed}")
        out = sgm.render(gm, cam, pose, ctx=ctx)
        s = out.sem.reshape(-1, out.channels).sum(axis=1)
        assert np.max(np.abs(s - out.silhouette)) < 1e-5


@pytest.mark.parametrize("name", ["score_8", "multi_2024"])
def test_scores_match_reference_golden(ctx, golden, name):
    gm, cam, pose, opts, _, outs = golden_scene(golden, name)
    cands = [sgm.CandidatePose(position=p, direction=d, id=i)
             for i, (p, d) in enumerate(zip(outs["cand_pos"], outs["cand_dir"]))]
    sgm.refresh_candidate_scores(cands, gm, cam, ctx=ctx)
    nm = np.array([c.n_missing for c in cands])
    es = np.array([c.entropy_sum for c in cands])
    np.testing.assert_array_equal(nm, outs["n_missing"])
    np.testing.assert_allclose(es, outs["entropy_sum"], rtol=ENT_RTOL, atol=0)
    if "i_total" in outs:
        sgm.combine_scores(cands, outs["current"])
        tot = np.array([c.i_total for c in cands])
        ref = outs["i_total"]
        both_tiny = (tot < 1e-300) & (ref < 1e-300)
        np.testing.assert_allclose(tot[~both_tiny], ref[~both_tiny], rtol=1e-3)
        assert int(np.argmax(tot)) == int(np.argmax(ref))


CASES = [
    dict(seed=1, n=400, k=5, nc=11, opts=RenderOptions()),
    dict(seed=2, n=400, k=5, nc=11, opts=RenderOptions(early_exit=False)),
    dict(seed=3, n=300, k=3, nc=6, opts=RenderOptions(truncation_sigmas=2.0, tile_size=16)),
    dict(seed=4, n=300, k=4, nc=9, opts=RenderOptions(), dup=True),
    dict(seed=5, n=200, k=10, nc=9, opts=RenderOptions(transmittance_eps=1e-2)),  # k = C
    dict(seed=6, n=600, k=16, nc=101, opts=RenderOptions()),
    dict(seed=7, n=150, k=1, nc=3, opts=RenderOptions(z_near=1.0)),
    dict(seed=8, n=200, k=40, nc=60, opts=RenderOptions()),  # k > 32: rows sorted per thread
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"seed{c['seed']}")
def test_random_scenes_vs_oracle(ctx, orc, case):
    cam = CameraModel(77, 53, 0, 0, 61.0, 59.5, 38.3, 26.1)  # partial tiles on both axes
    pose = look_at([0.2, -0.1, -0.4], [0.0, 0.2, 2.5])
    gm = random_map(case["seed"], case["n"], cam, pose, k=case["k"], num_classes=case["nc"],
                    dup=case.get("dup", False))
    opts = case["opts"]
    out = sgm.render(gm, cam, pose, RenderChannels.all(), opts, ctx=ctx)
    ref = orc.render(gm, cam, pose, 7, opts)
    assert_projections(out, orc.project(gm, cam, pose, opts))
    assert_planes(out, ref)
    assert_bins(ctx, orc, gm, cam, pose, opts, out)
    # scoring of a few nearby poses, batched
    rng = np.random.default_rng(case["seed"])
    poses = [look_at(rng.normal(0, 0.1, 3) + [0.2, -0.1, -0.4], [0.0, 0.2, 2.5] + rng.normal(0, .3, 3))
             for _ in range(5)]
    nm, es = sgm.score_poses(gm, cam, poses, opts, ctx=ctx)
    nm_o, es_o, _ = orc.score_views(gm, cam, poses, opts)
    np.testing.assert_array_equal(nm, nm_o)
    np.testing.assert_allclose(es, es_o, rtol=ENT_RTOL, atol=0)


def test_channel_subsets(ctx, orc):
    cam = CameraModel(40, 24, 0, 0, 35.0, 35.0, 20.0, 12.0)
    gm = random_map(8, 120, cam, k=3, num_classes=5)
    for ch, flags in ((RenderChannels(True, False, False), 1), (RenderChannels(False, True, False), 2),
                      (RenderChannels.scoring(), 4)):
        out = sgm.render(gm, cam, Pose(), ch, ctx=ctx)
        ref = orc.render(gm, cam, Pose(), flags)
        assert_planes(out, ref, keys=[k for k, f in (("color", 1), ("depth", 2), ("sem", 4))
                                      if flags & f] + ["silhouette"])


def test_empty_and_fully_culled_maps(ctx):
    cam = CameraModel.from_fov(8, 6, 60, 70)
    empty = sgm.GaussianMap(4, 9)
    h = sgm.render_entropy(empty, cam, Pose(), ctx=ctx)
    np.testing.assert_allclose(h, math.log(10.0), rtol=1e-12)  # test_splat_render.cpp:260
    out = sgm.render(empty, cam, Pose(), ctx=ctx)
    assert not out.silhouette.any() and not out.sem.any() and len(out.projections) == 0
    nm, es = sgm.score_poses(empty, cam, [Pose(), Pose()], ctx=ctx)
    assert list(nm) == [48.0, 48.0]
    np.testing.assert_allclose(es, 48 * sgm.clipped_entropy(np.zeros(10)), rtol=1e-12)
    behind = random_map(3, 50, cam, k=2, num_classes=4, depth=(-3.0, -1.0))
    out = sgm.render(behind, cam, Pose(), ctx=ctx)
    assert len(out.projections) == 0 and not out.silhouette.any()


def test_facing_away_candidate(ctx, golden):
    gm, cam, _, _, _, outs = golden_scene(golden, "score_8")
    c = [sgm.CandidatePose(position=np.array([0.0, 0, -1]), direction=np.array([0.0, 0, -1]))]
    sgm.refresh_candidate_scores(c, gm, cam, ctx=ctx)
    assert c[0].n_missing == cam.pixel_count()  # test_explorer.cpp:375
    assert c[0].entropy_sum == pytest.approx(cam.pixel_count() * math.log(6.0), rel=1e-9)


def test_storage_permutation_bit_identical(ctx):
    # test_splat_render.cpp:119-141
    cam = CameraModel(48, 36, 0, 0, 40.0, 40.0, 24.0, 18.0)
    gm = random_map(19, 200, cam, k=2, num_classes=5)
    perm = np.random.default_rng(4).permutation(gm.size())
    sh = sgm.GaussianMap.from_arrays(2, 5, gm.centers[perm], gm.log_radii[perm],
                                     gm.opacity_logits[perm], gm.colors[perm],
                                     gm.sem_indices[perm], gm.sem_probs[perm])
    a = sgm.render(gm, cam, Pose(), ctx=ctx)
    b = sgm.render(sh, cam, Pose(), ctx=ctx)
    for key in ("silhouette", "depth", "color", "sem"):
        np.testing.assert_array_equal(getattr(a, key), getattr(b, key))


def test_exact_depth_ties_resolved_like_reference(ctx, orc):
    # many Gaussians at identical depth: order must follow (z, mx, my, alpha)
    cam = CameraModel(32, 32, 0, 0, 30.0, 30.0, 16.0, 16.0)
    n = 64
    rng = np.random.default_rng(0)
    centers = np.stack([rng.choice([-0.2, 0.0, 0.2], n), rng.choice([-0.1, 0.1], n),
                        np.full(n, 1.5)], axis=1)
    gm = sgm.GaussianMap.from_arrays(2, 3, centers, np.full(n, -2.5), rng.choice([-1.0, 0.5], n),
                                     rng.uniform(0, 1, (n, 3)), np.tile([0, 2], (n, 1)),
                                     np.tile([0.6, 0.4], (n, 1)))
    out = sgm.render(gm, cam, Pose(), ctx=ctx)
    assert_projections(out, orc.project(gm, cam, Pose()))
    assert_planes(out, orc.render(gm, cam, Pose(), 7))


def test_batched_scoring_equals_one_by_one_and_is_deterministic(ctx):
    gm = scenes.make_map(0, n=5000)
    cam = scenes.CONFIGS[0].camera()
    poses = scenes.render_poses(0, 8)
    nm, es = sgm.score_poses(gm, cam, poses, ctx=ctx)
    nm2, es2 = sgm.score_poses(gm, cam, poses, ctx=ctx)
    np.testing.assert_array_equal(es, es2)
    for i, p in enumerate(poses):
        a, b = sgm.score_poses(gm, cam, [p], ctx=ctx)
        assert a[0] == nm[i] and b[0] == es[i]


def test_invalid_inputs_raise(ctx):
    cam = CameraModel.from_fov(8, 6, 60, 70)
    bad = sgm.GaussianMap.from_arrays(1, 3, [[0, 0, 1.0]], [-2.0], [0.0], [[0, 0, 0]], [[4]], [[1.0]])
    with pytest.raises(RuntimeError, match="semantic index"):
        sgm.render(bad, cam, Pose(), ctx=ctx)
    ok = sgm.GaussianMap.from_arrays(1, 3, [[0, 0, 1.0]], [-2.0], [0.0], [[0, 0, 0]], [[2]], [[1.0]])
    with pytest.raises(RuntimeError, match="tile_size"):
        sgm.render(ok, cam, Pose(), options=RenderOptions(tile_size=12), ctx=ctx)


def test_cfg0_full_scene_scoring_vs_oracle(ctx, orc):
    gm = scenes.make_map(0)
    cam = scenes.CONFIGS[0].camera()
    cands = scenes.make_candidates(0)
    sgm.refresh_candidate_scores(cands, gm, cam, ctx=ctx)
    poses = [c.camera_pose() for c in cands]
    nm_o, es_o, _ = orc.score_views(gm, cam, poses, threads=8)
    np.testing.assert_array_equal([c.n_missing for c in cands], nm_o)
    np.testing.assert_allclose([c.entropy_sum for c in cands], es_o, rtol=ENT_RTOL, atol=0)
    out = sgm.render(gm, cam, scenes.render_poses(0, 1)[0], ctx=ctx)
    ref = orc.render(gm, cam, scenes.render_poses(0, 1)[0], 7)
    assert_planes(out, ref)


def test_cfg1_full_size_properties(ctx, orc):
    """Full config-1 size (500k Gaussians, 1200x680): parity on 2 views vs the oracle
    plus size-independent properties (mass conservation, S in [0,1])."""
    gm = scenes.make_map(1)
    cam = scenes.CONFIGS[1].camera()
    poses = scenes.render_poses(1, 2)
    nm, es = sgm.score_poses(gm, cam, poses, ctx=ctx)
    nm_o, es_o, _ = orc.score_views(gm, cam, poses, threads=8)
    np.testing.assert_array_equal(nm, nm_o)
    np.testing.assert_allclose(es, es_o, rtol=ENT_RTOL, atol=0)
    out = sgm.render(gm, cam, poses[0], RenderChannels.scoring(), ctx=ctx)
    s = out.sem.reshape(-1, out.channels).sum(axis=1)
    # probs are f32-rounded (SGMP precision), so each Gaussian's k probs sum to 1 +- ~1e-7
    assert np.max(np.abs(s - out.silhouette)) < 1e-6
    assert out.silhouette.min() >= 0.0 and out.silhouette.max() <= 1.0
    h = np.array([sgm.clipped_entropy(out.sem[i * out.channels:(i + 1) * out.channels])
                  for i in range(0, cam.pixel_count(), 997)])
    assert np.all(h > 0) and np.all(h <= math.log(out.channels) + 1e-12)


def test_fronto_parallel_plane_long_depth_run(ctx, orc):
    """300 Gaussians at one exact depth: a single run of equal depth keys far longer
    than the insertion-sort limit (heapsort path of k_tiefix)."""
    cam = CameraModel(64, 48, 0, 0, 50.0, 50.0, 32.0, 24.0)
    rng = np.random.default_rng(12)
    n = 300
    centers = np.stack([rng.uniform(-0.6, 0.6, n), rng.uniform(-0.45, 0.45, n), np.full(n, 1.25)],
                       axis=1)
    centers[::7, :2] = centers[1::7, :2][: len(centers[::7])]  # some exact (z, mx, my) ties too
    gm = sgm.GaussianMap.from_arrays(3, 6, centers, np.full(n, -3.0), rng.normal(0, 1, n),
                                     rng.uniform(0, 1, (n, 3)),
                                     np.stack([rng.choice(7, 3, replace=False) for _ in range(n)]),
                                     rng.dirichlet(np.ones(3), n))
    out = sgm.render(gm, cam, Pose(), ctx=ctx)
    assert_projections(out, orc.project(gm, cam, Pose()))
    assert_planes(out, orc.render(gm, cam, Pose(), 7))
    nm, es = sgm.score_poses(gm, cam, [Pose()], ctx=ctx)
    nm_o, es_o, _ = orc.score_views(gm, cam, [Pose()])
    assert nm[0] == nm_o[0]
    np.testing.assert_allclose(es, es_o, rtol=ENT_RTOL)


def test_cfg3_full_size_vs_oracle(ctx, orc):
    """Config 3 at full size (2M Gaussians, k=8 of 42 channels, 1920x1080): two candidate
    views against the oracle, plus the batched == one-by-one property."""
    gm = scenes.make_map(3)
    cam = scenes.CONFIGS[3].camera()
    poses = [c.camera_pose() for c in scenes.make_candidates(3, 2)]
    nm, es = sgm.score_poses(gm, cam, poses, ctx=ctx)
    nm_o, es_o, _ = orc.score_views(gm, cam, poses, threads=2)
    np.testing.assert_array_equal(nm, nm_o)
    np.testing.assert_allclose(es, es_o, rtol=ENT_RTOL, atol=0)
    a, b = sgm.score_poses(gm, cam, [poses[1]], ctx=ctx)
    assert a[0] == nm[1] and b[0] == es[1]


def test_cfg4_dense_overlap_vs_oracle(ctx, orc):
    """Config 4's dense-overlap shape (1 m^3 cube, log-scales N(-2.5, 0.3), opacity
    sigmoid(N(1, 1)), k=32): long per-tile lists and early-exit divergence. A 60k-Gaussian
    prefix keeps the oracle's bins in memory; a render checks the planes too."""
    gm = scenes.make_map(4, n=60_000)
    cam = scenes.CONFIGS[4].camera()
    poses = [c.camera_pose() for c in scenes.make_candidates(4, 2)]
    nm, es = sgm.score_poses(gm, cam, poses, ctx=ctx)
    nm_o, es_o, st = orc.score_views(gm, cam, poses, threads=2)
    assert st["pairs"] > 50 * cam.pixel_count() // 64  # > 50 splats per tile on average
    np.testing.assert_array_equal(nm, nm_o)
    np.testing.assert_allclose(es, es_o, rtol=ENT_RTOL, atol=0)
    out = sgm.render(gm, cam, poses[0], RenderChannels.all(), ctx=ctx)
    assert_planes(out, orc.render(gm, cam, poses[0], 7))


def test_wide_image_bins_exact(ctx, orc):
    """More than 256 bin columns (the row scatter's column blocks span two CTA groups) and
    more than one 1024-entry segment per tile row: bins bit-exact, planes vs the oracle."""
    cam = CameraModel(2200, 48, 0, 0, 400.0, 400.0, 1100.0, 24.0)
    pose = Pose()
    gm = random_map(41, 5000, cam, pose, k=3, num_classes=5, rad_px=(0.5, 30.0), spread=1.0)
    opts = RenderOptions()
    out = sgm.render(gm, cam, pose, RenderChannels.all(), opts, ctx=ctx)
    assert_projections(out, orc.project(gm, cam, pose, opts))
    assert_bins(ctx, orc, gm, cam, pose, opts, out)
    assert_planes(out, orc.render(gm, cam, pose, 7, opts))


@pytest.mark.parametrize("seed", range(100, 124))
def test_randomised_scenes_vs_oracle(ctx, orc, seed):
    """Seeded random cameras, poses, options and maps (sizes, radii, opacities, k, C, tile
    size, truncation, early exit): projections and bins bit-exact, planes within the bar,
    scores exact / within 1e-11."""
    rng = np.random.default_rng(seed)
    W, H = int(rng.integers(9, 140)), int(rng.integers(7, 100))
    f = float(rng.uniform(0.4, 1.6)) * max(W, H)
    cam = CameraModel(W, H, 0, 0, f, f * float(rng.uniform(0.8, 1.25)),
                      float(rng.uniform(0.3, 0.7)) * W, float(rng.uniform(0.3, 0.7)) * H)
    pose = look_at(rng.normal(0, 0.3, 3), [rng.normal(0, 0.3), rng.normal(0, 0.3), 2.5])
    nc = int(rng.integers(1, 40))
    k = int(rng.integers(1, min(nc + 1, 20) + 1))
    gm = random_map(seed, int(rng.integers(1, 700)), cam, pose, k=k, num_classes=nc,
                    rad_px=(float(rng.uniform(0.2, 2.0)), float(rng.uniform(2.0, 25.0))),
                    logit=(float(rng.uniform(-6, 0)), float(rng.uniform(0, 8))),
                    dup=bool(rng.integers(0, 2)) and k >= 2)
    opts = RenderOptions(early_exit=bool(rng.integers(0, 4)),
                         transmittance_eps=float(10 ** rng.uniform(-6, -1)),
                         z_near=float(rng.uniform(0.01, 0.5)),
                         truncation_sigmas=float(rng.uniform(1.5, 4.0)),
                         tile_size=int(rng.choice([8, 16, 24])))
    out = sgm.render(gm, cam, pose, RenderChannels.all(), opts, ctx=ctx)
    assert_projections(out, orc.project(gm, cam, pose, opts))
    assert_bins(ctx, orc, gm, cam, pose, opts, out)
    assert_planes(out, orc.render(gm, cam, pose, 7, opts))
    nm, es = sgm.score_poses(gm, cam, [pose], options=opts, ctx=ctx)
    nm_o, es_o, _ = orc.score_views(gm, cam, [pose], opts)
    assert nm[0] == nm_o[0]
    np.testing.assert_allclose(es, es_o, rtol=ENT_RTOL, atol=1e-300)


@pytest.mark.parametrize("wh", [(21, 13), (48, 8), (9, 9)], ids=["6-blocks", "6-row", "4-blocks"])
def test_block_items_cross_views(ctx, orc, wh):
    """A raster CTA blends 4 consecutive (view, block) items, so with 6 blocks per view one CTA
    spans two views: every view's scores and renders must still match the oracle, and the
    batched results must equal the one-at-a-time ones (the block a CTA starts on differs)."""
    w, h = wh
    cam = CameraModel(w, h, 0, 0, 0.9 * w, 0.9 * w, 0.47 * w, 0.52 * h)
    pose = look_at([0.0, 0.0, -0.4], [0.0, 0.1, 2.5])
    gm = random_map(11, 300, cam, pose, k=4, num_classes=9)
    rng = np.random.default_rng(5)
    poses = [look_at(rng.normal(0, 0.1, 3) + [0.0, 0.0, -0.4], [0.0, 0.1, 2.5] + rng.normal(0, .3, 3))
             for _ in range(7)]
    nm, es = sgm.score_poses(gm, cam, poses, ctx=ctx)
    nm_o, es_o, _ = orc.score_views(gm, cam, poses, RenderOptions())
    np.testing.assert_array_equal(nm, nm_o)
    np.testing.assert_allclose(es, es_o, rtol=ENT_RTOL, atol=0)
    for i in (0, 3, 6):
        a, b = sgm.score_poses(gm, cam, [poses[i]], ctx=ctx)
        assert a[0] == nm[i] and b[0] == es[i]
    out = sgm.render(gm, cam, poses[2], RenderChannels.all(), ctx=ctx)
    assert_planes(out, orc.render(gm, cam, poses[2], 7))


def test_many_classes_and_the_shared_memory_limit(ctx, orc):
    """The per-block fp64 accumulator holds C channels: 300 classes still fit (one block per SM)
    and match the oracle; 1000 classes exceed the shared memory and fail loudly."""
    cam = CameraModel(40, 24, 0, 0, 36.0, 36.0, 20.1, 11.9)
    pose = look_at([0.0, 0.0, -0.4], [0.0, 0.1, 2.5])
    gm = random_map(21, 120, cam, pose, k=12, num_classes=300)
    out = sgm.render(gm, cam, pose, RenderChannels.all(), ctx=ctx)
    assert_planes(out, orc.render(gm, cam, pose, 7))
    nm, es = sgm.score_poses(gm, cam, [pose], ctx=ctx)
    nm_o, es_o, _ = orc.score_views(gm, cam, [pose], RenderOptions())
    np.testing.assert_array_equal(nm, nm_o)
    np.testing.assert_allclose(es, es_o, rtol=ENT_RTOL, atol=0)
    big = random_map(22, 50, cam, pose, k=4, num_classes=1000)
    with pytest.raises(RuntimeError, match="shared memory"):
        sgm.score_poses(big, cam, [pose], ctx=ctx)


@pytest.mark.parametrize("k", [1, 2, 3, 5, 8, 9, 16, 17, 31, 32, 33])
def test_row_sort_widths_vs_oracle(ctx, orc, k):
    """Rows are class-sorted on the GPU at upload by groups of lanes (the power of two >= k,
    k <= 32) or per thread (k > 32); duplicate class ids keep their order. Every width gives
    the oracle's planes and scores."""
    cam = CameraModel(30, 22, 0, 0, 27.0, 27.0, 15.2, 10.9)
    pose = look_at([0.0, 0.0, -0.4], [0.0, 0.1, 2.5])
    gm = random_map(40 + k, 90, cam, pose, k=k, num_classes=max(k, 40), dup=k >= 2)
    out = sgm.render(gm, cam, pose, RenderChannels.all(), ctx=ctx)
    assert_planes(out, orc.render(gm, cam, pose, 7))
    nm, es = sgm.score_poses(gm, cam, [pose], ctx=ctx)
    nm_o, es_o, _ = orc.score_views(gm, cam, [pose], RenderOptions())
    np.testing.assert_array_equal(nm, nm_o)
    np.testing.assert_allclose(es, es_o, rtol=ENT_RTOL, atol=0)


def test_bins_mixed_sparse_and_dense_rows(ctx, orc):
    """Tile rows where some 32-entry chunks are sparse (Gaussians a few tiles wide: walked
    entry by entry) and others dense (splats 30-120 px wide: walked column by column) give the
    reference's bins bit-exactly."""
    cam = CameraModel(600, 120, 0, 0, 300.0, 300.0, 299.5, 59.5)
    pose = look_at([0.0, 0.0, -0.4], [0.0, 0.0, 2.5])
    small = random_map(51, 1500, cam, pose, k=3, num_classes=7, rad_px=(0.5, 4.0))
    big = random_map(52, 400, cam, pose, k=3, num_classes=7, rad_px=(10.0, 40.0))
    gm = sgm.GaussianMap.from_arrays(
        3, 7, np.concatenate([small.centers, big.centers]),
        np.concatenate([small.log_radii, big.log_radii]),
        np.concatenate([small.opacity_logits, big.opacity_logits]),
        np.concatenate([small.colors, big.colors]),
        np.concatenate([small.sem_indices, big.sem_indices]),
        np.concatenate([small.sem_probs, big.sem_probs]))
    opts = RenderOptions()
    out = sgm.render(gm, cam, pose, RenderChannels.all(), opts, ctx=ctx)
    assert_projections(out, orc.project(gm, cam, pose, opts))
    assert_bins(ctx, orc, gm, cam, pose, opts, out)
    assert_planes(out, orc.render(gm, cam, pose, 7, opts))


def test_map_edits_reach_the_device_snapshot(ctx):
    """The cached device snapshot follows the map: reassigning an array bumps the version by
    itself; an in-place edit is picked up after touch()."""
    cam = CameraModel(40, 30, 0, 0, 35.0, 35.0, 20.0, 15.0)
    gm = random_map(4, 60, cam, k=2, num_classes=4)
    a = sgm.render(gm, cam, Pose(), ctx=ctx)
    gm.colors = np.clip(gm.colors, 0.0, 1.0) * 0.5  # reassignment
    b = sgm.render(gm, cam, Pose(), ctx=ctx)
    assert not np.array_equal(a.color, b.color)
    np.testing.assert_allclose(b.color, 0.5 * a.color, rtol=1e-12, atol=1e-15)
    gm.opacity_logits[:] = -1e4  # in place: every splat transparent once touched
    gm.touch()
    c = sgm.render(gm, cam, Pose(), ctx=ctx)
    assert np.all(c.silhouette == 0.0)
