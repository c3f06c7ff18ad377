"""GPU parity at the BASELINE configs' own sizes against the reference itself.

The checker here is `oracle/_ref` (the reference's splat_render.cpp / explorer.cpp compiled
unmodified), not the C restatement: full cfg1 planes, cfg1 scores, tile bins of a cfg1 and
a cfg3 view (bins are local to the reference's render(), so they are restated over the
reference's own projections, splat_render.cpp:205-212), and the combine_scores decision on
candidate sets whose n_missing varies (every make_candidates(1..3) view sees the cloud at
every pixel, so its i_total is 0 and the argmax there is only the id tie-break).
"""
import numpy as np
import pytest

import paper_2506_00225_b200 as sgm
from paper_2506_00225_b200 import scenes
from paper_2506_00225_b200.splatmap import RenderChannels, RenderOptions

pytestmark = pytest.mark.gpu

IMG_RTOL, IMG_ATOL = 1e-4, 1e-3  # north-star image tolerance
TIGHT = 1e-10
ENT_RTOL = 1e-11
CURRENT = np.array([4.0, 1.5, 3.0])


@pytest.fixture(scope="module")
def ctx():
    return sgm.Context(0)


@pytest.fixture(scope="module")
def cfg1():
    return scenes.make_map(1), scenes.CONFIGS[1].camera()


def _bins_vs_reference(ctx, orc, cam, projections, opts=None):
    opts = opts or RenderOptions()
    ts = opts.tile_size
    tiles = ((cam.width + ts - 1) // ts) * ((cam.height + ts - 1) // ts)
    off, ids, probe = sgm.bins_of_last_render(tiles, ctx)
    # the restatement's record carries the per-axis reach (its anisotropic extension); the
    # reference's isotropic reach is truncation_sigmas * rad_px (splat_render.cpp:205)
    proj = projections.copy()
    proj["rx"] = proj["ry"] = opts.truncation_sigmas * proj["rad_px"]
    o_off, o_ids, o_probe = orc.bins(proj, cam, opts)
    np.testing.assert_array_equal(off, o_off)
    np.testing.assert_array_equal(ids, o_ids)
    np.testing.assert_array_equal(probe, o_probe)
    return int(off[-1])


def _assert_projections(out, proj):
    assert len(out.projections) == len(proj)
    for f in ("mx", "my", "rad_px", "z", "alpha", "index"):
        np.testing.assert_array_equal(out.projections[f], proj[f], err_msg=f)


def test_cfg1_full_render_vs_reference(ctx, ref, orc, cfg1):
    """One cfg1 frame, every channel (1200x680x102 fp64 planes), against the reference's
    render(): planes, projections and the tile bins."""
    gm, cam = cfg1
    pose = scenes.render_poses(1, 1)[0]
    out = sgm.render(gm, cam, pose, RenderChannels.all(), ctx=ctx)
    r = ref.render(gm, cam, pose, 7)
    for key in ("silhouette", "color", "depth", "sem"):
        g = getattr(out, key)
        np.testing.assert_allclose(g, r[key], rtol=IMG_RTOL, atol=IMG_ATOL, err_msg=key)
        assert np.max(np.abs(g - r[key])) <= TIGHT, key
    _assert_projections(out, r["projections"])
    P = _bins_vs_reference(ctx, orc, cam, r["projections"])
    assert P > 1_000_000  # a config-scale bin set, not a micro-scene


def test_cfg1_scores_vs_reference(ctx, ref, cfg1):
    """refresh_candidate_scores on 4 cfg1 candidate views: the reference's own loop."""
    gm, cam = cfg1
    cands = scenes.make_candidates(1, 4)
    nm, es = sgm.score_poses(gm, cam, [c.camera_pose() for c in cands], ctx=ctx)
    rnm, res = ref.refresh_scores(gm, cam, [c.position for c in cands],
                                  [c.direction for c in cands], threads=4)
    np.testing.assert_array_equal(nm, rnm)
    np.testing.assert_allclose(es, res, rtol=ENT_RTOL, atol=0)


def test_cfg3_view_bins_vs_reference(ctx, ref, orc):
    """cfg3 (2M Gaussians, 1920x1080, k=8 of 42 channels): projections and bins of one view,
    and its score, against the reference."""
    gm = scenes.make_map(3)
    cam = scenes.CONFIGS[3].camera()
    cand = scenes.make_candidates(3, 1)[0]
    pose = cand.camera_pose()
    out = sgm.render(gm, cam, pose, RenderChannels(color=False, depth=False, semantics=True),
                     ctx=ctx)
    r = ref.render(gm, cam, pose, 4)
    _assert_projections(out, r["projections"])
    np.testing.assert_allclose(out.silhouette, r["silhouette"], rtol=0, atol=TIGHT)
    np.testing.assert_allclose(out.sem, r["sem"], rtol=0, atol=TIGHT)
    assert _bins_vs_reference(ctx, orc, cam, r["projections"]) > 1_000_000
    nm, es = sgm.score_poses(gm, cam, [pose], ctx=ctx)
    rnm, res = ref.refresh_scores(gm, cam, [cand.position], [cand.direction], threads=1)
    assert nm[0] == rnm[0]
    np.testing.assert_allclose(es, res, rtol=ENT_RTOL, atol=0)


def _decision(ctx, ref, gm, cam, cands, current):
    """Our scores + combine_scores vs the reference's refresh + combine on the same views."""
    for c in cands:
        c.n_missing = c.entropy_sum = 0.0
    sgm.refresh_candidate_scores(cands, gm, cam, ctx=ctx)
    nm = np.array([c.n_missing for c in cands])
    es = np.array([c.entropy_sum for c in cands])
    pos = np.array([c.position for c in cands])
    rnm, res = ref.refresh_scores(gm, cam, pos, [c.direction for c in cands], threads=16)
    np.testing.assert_array_equal(nm, rnm)
    np.testing.assert_allclose(es, res, rtol=ENT_RTOL, atol=0)
    any_ours = sgm.combine_scores(cands, current)
    any_ref, _, _, rt = ref.combine_scores(rnm, res, pos, current)
    assert any_ours == any_ref
    tot = np.array([c.i_total for c in cands])
    tiny = (np.abs(tot) < 1e-300) & (np.abs(rt) < 1e-300)
    np.testing.assert_allclose(tot[~tiny], rt[~tiny], rtol=1e-3)
    # the planning order: i_total descending, id ascending (episode.cpp:410-414)
    order = lambda t: sorted(range(len(t)), key=lambda i: (-t[i], i))
    assert order(tot) == order(rt)
    # the decision is not an id tie-break: n_missing varies and the winner has i_total > 0
    assert len(set(rnm.tolist())) > 3 and rt[order(rt)[0]] > 0.0
    srt = np.sort(res)[::-1]
    gap = srt[0] - srt[1]
    err = np.max(np.abs(es - res))
    assert gap > 1e3 * err  # top-2 gap far above the error
    return order(rt)[0], gap, err


def test_cfg1_decision_argmax_vs_reference(ctx, ref, cfg1):
    """The cfg1 map from 16 viewpoints that see it in part (n_missing 0 .. 4.6e5)."""
    gm, cam = cfg1
    _decision(ctx, ref, gm, cam, scenes.make_decision_candidates(1), CURRENT)


def test_cfg0_decision_argmax_vs_reference(ctx, ref):
    gm = scenes.make_map(0)
    cam = scenes.CONFIGS[0].camera()
    _decision(ctx, ref, gm, cam, scenes.make_decision_candidates(0, 24), np.array([2.0, 1.5, 2.0]))


def test_cfg4_prefix_decision_vs_reference(ctx, ref):
    """cfg4's dense cube from its own candidate poses (1.2 m away: the cube fills the
    centre of the image, so n_missing varies), on a 30k-Gaussian prefix of the map
    (the reference holds 16 B per tile pair per view: the full map needs ~19 GB per view)."""
    gm = scenes.make_map(4, n=30_000)
    cam = scenes.CONFIGS[4].camera()
    _decision(ctx, ref, gm, cam, scenes.make_candidates(4, 16), np.array([0.5, 0.5, 0.5]))


def _dense_scene():
    """A dense-overlap scene (cfg4's cube and poses, 100k Gaussians, 240x136 px): bins average
    several thousand entries, so scoring takes the depth-prefix binning path."""
    from paper_2506_00225_b200.splatmap import CameraModel
    gm = scenes.make_map(4, n=100_000)
    cam = CameraModel(240, 136, 0, 0, 120.0, 120.0, 119.5, 67.5)
    return gm, cam, scenes.make_candidates(4, 6)


@pytest.mark.parametrize("cap", [None, "256", "64"])
def test_depth_prefix_binning_is_exact(ctx, monkeypatch, cap):
    """Dense views: scores from depth-prefix bins (with the redo of incomplete tiles: small
    caps leave many) are bit-identical to scores from the full bins."""
    gm, cam, cands = _dense_scene()
    poses = [c.camera_pose() for c in cands]
    monkeypatch.setenv("SGM_PREFIX_BINNING", "0")
    nm2, es2 = sgm.score_poses(gm, cam, poses, ctx=ctx)
    ctx.reset_stats()
    monkeypatch.setenv("SGM_PREFIX_BINNING", "1")  # (by default from 65536 entries per bin)
    if cap:
        monkeypatch.setenv("SGM_PREFIX_CAP", cap)
    nm, es = sgm.score_poses(gm, cam, poses, ctx=ctx)
    st = ctx.stats()
    assert st["pairs"] / len(poses) > 4096 * 30 * 17  # dense: > 4096 entries per bin
    if cap:  # the second pass ran (one more raster launch per view with incomplete tiles)
        assert st["raster_launches"] > len(poses)
    assert np.array_equal(nm, nm2) and np.array_equal(es, es2)
    assert len(set(nm.tolist())) > 1  # some views see the background (tiles that never exit)


def test_dense_scene_scores_vs_reference(ctx, ref, monkeypatch):
    monkeypatch.setenv("SGM_PREFIX_BINNING", "1")
    gm, cam, cands = _dense_scene()
    nm, es = sgm.score_poses(gm, cam, [c.camera_pose() for c in cands], ctx=ctx)
    rnm, res = ref.refresh_scores(gm, cam, [c.position for c in cands],
                                  [c.direction for c in cands], threads=6)
    np.testing.assert_array_equal(nm, rnm)
    np.testing.assert_allclose(es, res, rtol=ENT_RTOL, atol=0)


def test_cfg4_full_size_modes_bit_identical(ctx, monkeypatch):
    """cfg4 at its full size (1M Gaussians, 1200x680, 1.19 G tile pairs per view): the default
    path (depth-prefix binning of 8,192 entries per bin, row pairs only for ranks that can reach
    a prefix, channel groups 4-7 in tensor memory) scores bit-identically to full bins and to the
    shared-memory accumulator; the reference cannot hold these views (16 B per tile pair)."""
    gm = scenes.make_map(4)
    cam = scenes.CONFIGS[4].camera()
    poses = [c.camera_pose() for c in scenes.make_candidates(4, 3)]
    ctx.reset_stats()
    nm, es = sgm.score_poses(gm, cam, poses, ctx=ctx)
    assert ctx.stats()["pairs"] / len(poses) > 1.0e9
    monkeypatch.setenv("SGM_PREFIX_BINNING", "0")
    nm_full, es_full = sgm.score_poses(gm, cam, poses, ctx=ctx)
    monkeypatch.setenv("SGM_TM_FIRST", "8")
    nm_smem, es_smem = sgm.score_poses(gm, cam, poses, ctx=ctx)
    assert np.array_equal(nm, nm_full) and np.array_equal(es, es_full)
    assert np.array_equal(nm, nm_smem) and np.array_equal(es, es_smem)
    assert np.all(es > 0)
