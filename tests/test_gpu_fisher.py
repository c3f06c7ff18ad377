"""Fisher-information gain on the GPU (sgm_fisher_prior / sgm_score_views_fisher) vs the
FD-pinned CPU oracle (tests/test_fisher_oracle.py). The prior uses fp64 atomics, so it is
compared with a tolerance; the per-view gain is deterministic."""
import numpy as np
import pytest

from conftest import random_map

import paper_2506_00225_b200 as sgm
from paper_2506_00225_b200 import scenes
from paper_2506_00225_b200.splatmap import CameraModel, RenderOptions, look_at

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return sgm.Context(0)


@pytest.mark.parametrize("opts", [RenderOptions(), RenderOptions(early_exit=False, truncation_sigmas=12.0)],
                         ids=["default", "fd-options"])
def test_fisher_prior_and_gain_vs_oracle(ctx, orc, opts):
    cam = CameraModel(45, 37, 0, 0, 40.0, 41.0, 22.3, 18.1)
    pose = look_at([0.1, -0.05, -0.4], [0.0, 0.1, 2.5])
    gm = random_map(3, 250, cam, pose, k=3, num_classes=7)
    gm.colors[::5] = np.clip(gm.colors[::5], 0.0, 1.0)
    gm.opacity_logits[::11] = 12.0  # some clamped footprints (alpha ~ 1)
    prior_poses = [look_at([0.05 * i, 0.02 * i, -0.4], [0.0, 0.1, 2.5]) for i in range(4)]
    H = sgm.fisher_prior(gm, cam, prior_poses, lam=0.5, options=opts, ctx=ctx)
    H_o = orc.fisher_accumulate(gm, cam, prior_poses, opts)
    np.testing.assert_allclose(H, H_o, rtol=1e-9, atol=1e-12 * H_o.max())
    cands = [look_at([0.1 * i - 0.2, 0.0, -0.4], [0.0, 0.1, 2.5]) for i in range(6)]
    nm, es, g = sgm.score_poses_fisher(gm, cam, cands, opts, ctx=ctx)
    nm2, es2 = sgm.score_poses(gm, cam, cands, opts, ctx=ctx)
    np.testing.assert_array_equal(nm, nm2)
    np.testing.assert_array_equal(es, es2)
    g_o = orc.fisher_gain(gm, cam, cands, H_o, 0.5, opts)
    np.testing.assert_allclose(g, g_o, rtol=1e-9)
    # deterministic: the gain does not depend on batching
    _, _, g1 = sgm.score_poses_fisher(gm, cam, cands[:1], opts, ctx=ctx)
    assert g1[0] == g[0]


def test_fisher_requires_prior_and_positive_lambda(ctx):
    cam = CameraModel(16, 12, 0, 0, 14.0, 14.0, 8.0, 6.0)
    gm = random_map(1, 20, cam, k=2, num_classes=3)
    with pytest.raises(RuntimeError, match="prior"):
        sgm.score_poses_fisher(gm, cam, [sgm.Pose()], ctx=ctx)
    with pytest.raises(RuntimeError, match="lambda"):
        sgm.fisher_prior(gm, cam, [sgm.Pose()], lam=0.0, ctx=ctx)


def test_fisher_cfg0_scene_vs_oracle(ctx, orc):
    gm = scenes.make_map(0, n=3000)
    cam = scenes.CONFIGS[0].camera()
    poses = scenes.render_poses(0, 8)
    H = sgm.fisher_prior(gm, cam, poses[:4], lam=1.0, ctx=ctx)
    H_o = orc.fisher_accumulate(gm, cam, poses[:4])
    np.testing.assert_allclose(H, H_o, rtol=1e-9, atol=1e-12 * H_o.max())
    _, _, g = sgm.score_poses_fisher(gm, cam, poses[4:], ctx=ctx)
    np.testing.assert_allclose(g, orc.fisher_gain(gm, cam, poses[4:], H_o, 1.0), rtol=1e-9)


def test_prior_from_summed_shards_equals_full_prior():
    """sgm_fisher_set_prior with the sum of two shards' priors (what the multi-GPU C2
    all-reduce produces) gives the same gains as the prior over all poses."""
    import paper_2506_00225_b200 as sgm
    from paper_2506_00225_b200 import scenes
    ctx = sgm.Context(0)
    gm = scenes.make_map(0, n=3000)
    cam = scenes.CONFIGS[0].camera()
    prior = [c.camera_pose() for c in scenes.make_candidates(0, 6, stream=2)]
    views = scenes.render_poses(0, 3)
    H_all = sgm.fisher_prior(gm, cam, prior, lam=1.0, ctx=ctx)
    _, _, g_all = sgm.score_poses_fisher(gm, cam, views, ctx=ctx)
    H_sum = sgm.fisher_prior(gm, cam, prior[:2], ctx=ctx) + sgm.fisher_prior(gm, cam, prior[2:], ctx=ctx)
    np.testing.assert_allclose(H_sum, H_all, rtol=1e-12, atol=1e-300)
    sgm.fisher_set_prior(gm, H_sum, lam=1.0, ctx=ctx)
    _, _, g_sum = sgm.score_poses_fisher(gm, cam, views, ctx=ctx)
    np.testing.assert_allclose(g_sum, g_all, rtol=1e-12)


def test_combined_gain_ranking_vs_oracle(ctx, orc):
    """The a14 scalar gain (fisher_gain + w_sem * entropy_sum) and its ranking
    (score_candidates_fisher) from GPU scores vs the same criterion on the oracle's scores:
    same gains (1e-9) and the same planning order."""
    gm = scenes.make_map(0, n=3000)
    cam = scenes.CONFIGS[0].camera()
    prior = scenes.render_poses(0, 8)[:3]
    sgm.fisher_prior(gm, cam, prior, lam=1.0, ctx=ctx)
    H_o = orc.fisher_accumulate(gm, cam, prior)
    cands = scenes.make_decision_candidates(0, 10)
    cur = np.array([2.0, 1.5, 2.0])
    for w in (1.0, 0.01):
        mine = [sgm.CandidatePose(position=c.position, direction=c.direction, id=c.id) for c in cands]
        sgm.score_candidates_fisher(mine, gm, cam, cur, w_sem=w, ctx=ctx)
        poses = [c.camera_pose() for c in cands]
        nm_o, es_o, _ = orc.score_views(gm, cam, poses)
        g_o = orc.fisher_gain(gm, cam, poses, H_o, 1.0)
        theirs = [sgm.CandidatePose(position=c.position, entropy_sum=es_o[i], fisher_gain=g_o[i],
                                    id=c.id) for i, c in enumerate(cands)]
        sgm.combine_scores_fisher(theirs, cur, w_sem=w)
        theirs.sort(key=lambda c: (-c.i_gain, c.id))
        assert [c.id for c in mine] == [c.id for c in theirs]
        np.testing.assert_allclose([c.gain for c in mine], [c.gain for c in theirs], rtol=1e-9)
        np.testing.assert_allclose([c.i_gain for c in mine], [c.i_gain for c in theirs], rtol=1e-6)
        assert mine[0].i_gain > mine[-1].i_gain > 0.0
