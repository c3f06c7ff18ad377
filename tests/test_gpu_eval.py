"""semantic_metrics + photometric_metrics on device render planes
(sgm_eval_*) against the reference's evaluator (proj/src/evaluator.cpp:93-297) over its own
render of the same map. Counts (confusion, top-1/3) and everything derived from them on the
host are exact; AP and PSNR/depth sums are reduced in a different (fixed) order, so they
are compared at 1e-9 relative."""
import numpy as np
import pytest

from conftest import random_map
from test_gpu_backward import random_frame

import paper_2506_00225_b200 as sgm
from paper_2506_00225_b200._native import SgmError
from paper_2506_00225_b200.splatmap import CameraModel, look_at

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return sgm.Context(0)


def compare(rep, ref_out):
    summary, pvm, pvp, pc = ref_out
    np.testing.assert_allclose([rep.miou_pct, rep.top1_pct, rep.top3_pct, rep.f1_pct],
                               summary[[0, 1, 2, 4]], rtol=1e-13)
    np.testing.assert_allclose(rep.map_pct, summary[3], rtol=1e-9)
    np.testing.assert_allclose([rep.psnr_db, rep.depth_l1_cm], summary[5:], rtol=1e-9)
    np.testing.assert_allclose(rep.per_view_miou, pvm, rtol=1e-13)
    np.testing.assert_allclose(rep.per_view_psnr, pvp, rtol=1e-9)
    assert len(rep.per_class) == len(pc)
    got = np.array([[p.class_id, p.iou_pct, p.ap_pct, p.f1_pct, p.gt_pixels] for p in rep.per_class])
    assert np.array_equal(got[:, [0, 4]], pc[:, [0, 4]])
    np.testing.assert_allclose(got[:, [1, 3]], pc[:, [1, 3]], rtol=1e-13)
    np.testing.assert_allclose(got[:, 2], pc[:, 2], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_metrics_match_reference(ctx, ref, seed):
    cam = CameraModel(40, 30, 0, 0, 34.0, 34.0, 20.5, 14.5)
    poses = [look_at([0.05, -0.02, -0.4], [0.0, 0.05, 2.5]),
             look_at([-0.06, 0.03, -0.35], [0.02, 0.0, 2.5]),
             look_at([0.2, 0.1, -0.5], [0.0, 0.0, 2.5])]
    gm = random_map(seed, 260, cam, poses[0], k=4, num_classes=6, logit=(-1.5, 4.5))
    frames = [random_frame(seed * 10 + i, cam, p, 6) for i, p in enumerate(poses)]
    rep = sgm.evaluate(gm, cam, frames, ctx=ctx)
    compare(rep, ref.evaluate(gm, cam, frames))
    assert 0.0 <= rep.top1_pct <= rep.top3_pct <= 100.0


def test_cfg0_scene(ctx, ref):
    from paper_2506_00225_b200 import scenes
    gm = scenes.make_map(0, n=6000)
    cam = scenes.CONFIGS[0].camera()
    poses = scenes.render_poses(0, 2)
    frames = [scenes.make_frame(0, p, seed=i) for i, p in enumerate(poses)]
    rep = sgm.evaluate(gm, cam, frames, ctx=ctx)
    compare(rep, ref.evaluate(gm, cam, frames))


def test_errors(ctx):
    ev = sgm.Evaluator(6, ctx=ctx)
    with pytest.raises(SgmError, match="view count mismatch"):
        ev.report()
    cam = CameraModel(40, 30, 0, 0, 34.0, 34.0, 20.5, 14.5)
    gm = random_map(4, 50, cam, look_at([0, 0, -0.4], [0, 0, 2.5]), k=4, num_classes=6)
    small = random_frame(5, CameraModel(20, 10, 0, 0, 10.0, 10.0, 10.0, 5.0),
                         look_at([0, 0, -0.4], [0, 0, 2.5]), 6)
    with pytest.raises(SgmError, match="resolution mismatch"):
        ev.add_view(gm, cam, small)
