"""the mapping step (render + mapping_loss + semantic_loss + analytic backward,
proj/src/losses.cpp:40-362) on the GPU vs the reference's own code (oracle/_ref). Gradients
use fp64 atomics, so they are compared with a tolerance; the reference's backward itself is
pinned by its finite-difference tests (proj/tests/test_losses.cpp:226-239, run in
tests/test_oracle.py)."""
import numpy as np
import pytest

from conftest import random_map

import paper_2506_00225_b200 as sgm
from paper_2506_00225_b200.splatmap import CameraModel, LossWeights, RenderOptions, look_at

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return sgm.Context(0)


def random_frame(seed, cam, pose, num_classes, invalid=0.1):
    """Like testutil::random_frame (proj/tests/test_helpers.hpp:69-96), numpy RNG."""
    rng = np.random.default_rng(seed)
    px = cam.width * cam.height
    Cn = num_classes + 1
    rgb = (0.1 + 0.8 * rng.uniform(0, 1, (px, 3))).astype(np.float32)
    depth = np.where(rng.uniform(0, 1, px) < invalid, 0.0,
                     0.5 + 2.5 * rng.uniform(0, 1, px)).astype(np.float32)
    p = 0.05 + rng.uniform(0, 1, (px, Cn))
    p /= p.sum(axis=1, keepdims=True)
    hot = rng.integers(0, Cn, px)
    sem = 0.3 * p
    sem[np.arange(px), hot] += 0.7
    return sgm.Frame(cam.width, cam.height, num_classes, pose, rgb.reshape(-1), depth,
                     sem.astype(np.float32).reshape(-1))


def compare(rep_g, g, rep_r, g_r):
    np.testing.assert_allclose([rep_g.photometric, rep_g.depth, rep_g.semantic], rep_r[:3], rtol=1e-10)
    assert [rep_g.photometric_px, rep_g.depth_px, rep_g.semantic_px, rep_g.uncovered_px] == \
        [int(v) for v in rep_r[3:]]
    for name in ("center", "log_radius", "opacity_logit", "color", "sem"):
        a, b = getattr(g, name), g_r[name]
        scale = max(1e-30, float(np.max(np.abs(b))))
        np.testing.assert_allclose(a, b, rtol=1e-8, atol=1e-10 * scale, err_msg=name)


CASES = [
    dict(seed=1, weights=LossWeights(), opts=RenderOptions()),
    dict(seed=2, weights=LossWeights(use_kl=True, kl_clip_norm=0.5), opts=RenderOptions()),
    dict(seed=3, weights=LossWeights(use_cos=False), opts=RenderOptions(early_exit=False)),
    dict(seed=4, weights=LossWeights(), opts=RenderOptions(), mapping=False),
    dict(seed=5, weights=LossWeights(mask_k=4), opts=RenderOptions(), semantic=False),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"seed{c['seed']}")
def test_backward_matches_reference(ctx, ref, case):
    cam = CameraModel(40, 30, 0, 0, 34.0, 34.0, 20.5, 14.5)
    pose = look_at([0.05, -0.02, -0.4], [0.0, 0.05, 2.5])
    gm = random_map(case["seed"], 220, cam, pose, k=4, num_classes=6, logit=(-1.5, 4.5))
    gm.colors[:] = np.clip(gm.colors, 0.05, 1.05)  # a few out-of-range colours
    fr = random_frame(case["seed"] + 100, cam, pose, 6)
    inc_m, inc_s = case.get("mapping", True), case.get("semantic", True)
    rep, g = sgm.backward(gm, cam, fr, case["weights"], inc_m, inc_s, case["opts"], ctx=ctx)
    rep_r, g_r = ref.backward(gm, cam, fr, case["weights"], inc_m, inc_s, case["opts"])
    compare(rep, g, rep_r, g_r)
    if inc_m:
        assert np.any(g.center != 0) and np.any(g.opacity_logit != 0)
    if inc_s:
        assert np.any(g.sem != 0)


def test_backward_cfg0_scene(ctx, ref):
    from paper_2506_00225_b200 import scenes
    gm = scenes.make_map(0, n=4000)
    cam = scenes.CONFIGS[0].camera()
    pose = scenes.render_poses(0, 1)[0]
    fr = random_frame(7, cam, pose, gm.num_classes())
    rep, g = sgm.backward(gm, cam, fr, ctx=ctx)
    rep_r, g_r = ref.backward(gm, cam, fr, sgm.LossWeights())
    compare(rep, g, rep_r, g_r)
