"""GPU parity of the anisotropic (EWA) splat mode, SURVEY §8 f4.

No reference counterpart exists (the reference is isotropic only), so parity is against the
builder-written CPU oracle, itself pinned by tests/test_aniso_oracle.py (numpy covariance,
numerical Jacobian, Monte-Carlo projection, isotropic limit, conservative bins): the
"parity unpinned" caveat of DESIGN.md applies. Bars as for the isotropic mode: projections
and bins bit-exact, images within 1e-10, n_missing exact, entropy_sum within 1e-11.
"""
import numpy as np
import pytest

from conftest import random_map
from test_aniso_oracle import aniso_map
from test_gpu_parity import TIGHT, ENT_RTOL, assert_planes, assert_projections

import paper_2506_00225_b200 as sgm
from paper_2506_00225_b200 import scenes
from paper_2506_00225_b200.splatmap import CameraModel, RenderChannels, RenderOptions, look_at

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return sgm.Context(0)


CASES = [
    dict(seed=1, n=400, k=5, nc=11, opts=RenderOptions()),
    dict(seed=2, n=400, k=5, nc=11, opts=RenderOptions(early_exit=False)),
    dict(seed=3, n=300, k=3, nc=6, opts=RenderOptions(truncation_sigmas=2.0, tile_size=16)),
    dict(seed=4, n=300, k=4, nc=9, opts=RenderOptions(), dup=True),
    dict(seed=6, n=600, k=16, nc=101, opts=RenderOptions()),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"seed{c['seed']}")
def test_aniso_render_vs_oracle(ctx, orc, case):
    cam = CameraModel(77, 53, 0, 0, 61.0, 59.5, 38.3, 26.1)
    pose = look_at([0.2, -0.1, -0.4], [0.0, 0.2, 2.5])
    gm = aniso_map(case["seed"], case["n"], cam, k=case["k"], num_classes=case["nc"], pose=pose,
                   dup=case.get("dup", False))
    opts = case["opts"]
    out = sgm.render(gm, cam, pose, RenderChannels.all(), opts, ctx=ctx)
    proj = orc.project(gm, cam, pose, opts)
    assert_projections(out, proj)
    assert_planes(out, orc.render(gm, cam, pose, 7, opts))
    # bins: identical ordered id lists; probe = (float mx, float my, float trunc^2)
    tiles = ((cam.width + opts.tile_size - 1) // opts.tile_size) * \
            ((cam.height + opts.tile_size - 1) // opts.tile_size)
    off, ids, probe = sgm.bins_of_last_render(tiles, ctx)
    o_off, o_ids, o_probe = orc.bins(proj, cam, opts)
    np.testing.assert_array_equal(off, o_off)
    np.testing.assert_array_equal(ids, o_ids)
    np.testing.assert_array_equal(probe, o_probe)
    # retained contributors follow the same contributor sequence
    ret = sgm.render(gm, cam, pose, RenderChannels.all(True), opts, ctx=ctx)
    assert int(ret.contrib_offset[-1]) == len(ret.contrib) > 0


def test_aniso_scores_vs_oracle(ctx, orc):
    cam = CameraModel(120, 90, 0, 0, 100.0, 100.0, 59.5, 44.5)
    gm = aniso_map(8, 800, cam, k=6, num_classes=20, depth=(0.8, 3.0))
    rng = np.random.default_rng(4)
    poses = [look_at(rng.normal(0, 0.15, 3), [rng.normal(0, 0.2), rng.normal(0, 0.2), 2.0])
             for _ in range(9)]
    nm, es = sgm.score_poses(gm, cam, poses, ctx=ctx)
    nm_o, es_o, _ = orc.score_views(gm, cam, poses, threads=4)
    np.testing.assert_array_equal(nm, nm_o)
    np.testing.assert_allclose(es, es_o, rtol=ENT_RTOL, atol=0)
    # batched == one by one (deterministic per-view reductions)
    for i in (0, 4, 8):
        n1, e1 = sgm.score_poses(gm, cam, [poses[i]], ctx=ctx)
        assert n1[0] == nm[i] and e1[0] == es[i]


def test_aniso_cfg0_scene(ctx, orc):
    gm = scenes.make_map(0, n=6000, aniso=True)
    cam = scenes.CONFIGS[0].camera()
    poses = scenes.render_poses(0, 3)
    nm, es = sgm.score_poses(gm, cam, poses, ctx=ctx)
    nm_o, es_o, _ = orc.score_views(gm, cam, poses, threads=4)
    np.testing.assert_array_equal(nm, nm_o)
    np.testing.assert_allclose(es, es_o, rtol=ENT_RTOL, atol=0)
    out = sgm.render(gm, cam, poses[0], RenderChannels.all(), RenderOptions(), ctx=ctx)
    ref = orc.render(gm, cam, poses[0], 7)
    for key in ("silhouette", "color", "depth", "sem"):
        assert np.max(np.abs(getattr(out, key) - ref[key])) <= TIGHT, key


def test_isotropic_again_after_reset(ctx, orc):
    cam = CameraModel(64, 48, 0, 0, 60.0, 60.0, 31.5, 23.5)
    gm = random_map(30, 200, cam)
    iso = sgm.render(gm, cam, sgm.Pose(), ctx=ctx)
    rng = np.random.default_rng(1)
    gm.set_anisotropic(rng.uniform(-3.5, -2.5, (200, 3)), rng.normal(0, 1, (200, 4)))
    an = sgm.render(gm, cam, sgm.Pose(), ctx=ctx)
    assert np.max(np.abs(an.silhouette - iso.silhouette)) > 1e-3  # a different footprint
    gm.set_anisotropic(None, None)
    again = sgm.render(gm, cam, sgm.Pose(), ctx=ctx)
    np.testing.assert_array_equal(again.silhouette, iso.silhouette)
    np.testing.assert_array_equal(again.sem, iso.sem)


def test_aniso_rejects_fisher_and_bad_quaternions(ctx):
    cam = CameraModel(32, 24, 0, 0, 30.0, 30.0, 16.0, 12.0)
    gm = aniso_map(2, 5, cam)
    with pytest.raises(RuntimeError, match="isotropic only"):
        sgm.fisher_prior(gm, cam, [sgm.Pose()], ctx=ctx)
    bad = aniso_map(3, 5, cam)
    bad.quats[2] = 0.0
    bad.touch()
    with pytest.raises(RuntimeError, match="quaternion"):
        sgm.render(bad, cam, sgm.Pose(), ctx=ctx)


def test_aniso_cfg1_full_size_vs_oracle(ctx, orc):
    """Config 1 at full size (500k Gaussians, 1200x680) with the drawn per-axis scales and
    quaternions: two candidate views against the oracle."""
    gm = scenes.make_map(1, aniso=True)
    cam = scenes.CONFIGS[1].camera()
    poses = [c.camera_pose() for c in scenes.make_candidates(1, 2)]
    nm, es = sgm.score_poses(gm, cam, poses, ctx=ctx)
    nm_o, es_o, _ = orc.score_views(gm, cam, poses, threads=2)
    np.testing.assert_array_equal(nm, nm_o)
    np.testing.assert_allclose(es, es_o, rtol=ENT_RTOL, atol=0)
