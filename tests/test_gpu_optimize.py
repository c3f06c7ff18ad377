"""optimize_map on the GPU (sgm_optimize_map: render(all(true)) -> losses ->
backward -> Adam step -> opacity pruning, map and moments resident in HBM) against the
reference's own optimize_map (proj/src/mapper.cpp:241-283) from the same map and frames.

One iteration from identical parameters is exact up to the gradient's fp64 atomic summation
order (~1e-15 relative, tests/test_gpu_backward.py); the snapshot activations use CUDA's
exp (<= 1 ulp from glibc). Both effects stay far below the tolerances asserted here over
tens of iterations, and the pruned set must be identical."""
import numpy as np
import pytest

from conftest import random_map
from test_gpu_backward import random_frame

import paper_2506_00225_b200 as sgm
from paper_2506_00225_b200._native import SgmError
from paper_2506_00225_b200.mapper import AdamParams, AdamState, MapperConfig, MapTrainer
from paper_2506_00225_b200.splatmap import CameraModel, look_at

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return sgm.Context(0)


def scene(seed, n=220):
    cam = CameraModel(40, 30, 0, 0, 34.0, 34.0, 20.5, 14.5)
    poses = [look_at([0.05, -0.02, -0.4], [0.0, 0.05, 2.5]),
             look_at([-0.06, 0.03, -0.35], [0.02, 0.0, 2.5])]
    gm = random_map(seed, n, cam, poses[0], k=4, num_classes=6, logit=(-1.5, 4.5))
    frames = [random_frame(seed + 50 + i, cam, p, 6) for i, p in enumerate(poses)]
    return cam, gm, frames


def compare_maps(gm, out, rtol):
    for name, ours in (("centers", gm.centers), ("log_radii", gm.log_radii),
                       ("opacity_logits", gm.opacity_logits), ("colors", gm.colors),
                       ("sem_probs", gm.sem_probs)):
        np.testing.assert_allclose(np.asarray(ours).reshape(-1), out[name], rtol=rtol,
                                   atol=rtol * 1e-3, err_msg=name)
    assert np.array_equal(np.asarray(gm.sem_indices).reshape(-1), out["sem_indices"])


@pytest.mark.parametrize("seed,iters,prune_every,thr", [(1, 16, 0, 0.005), (2, 12, 4, 0.35),
                                                        (3, 20, 5, 0.2)])
def test_optimize_matches_reference(ctx, ref, seed, iters, prune_every, thr):
    cam, gm, frames = scene(seed)
    cfg = MapperConfig(prune_every=prune_every, prune_opacity=thr)
    hist_r, out, err = ref.optimize_map(gm, frames, cam, cfg, iters)
    assert err is None
    st = AdamState()
    hist = sgm.optimize_map(gm, st, frames, cam, cfg, iters, ctx=ctx)
    assert len(hist) == len(hist_r) == iters
    for h, r in zip(hist, hist_r):
        np.testing.assert_allclose([h.photometric, h.depth, h.semantic], r[:3], rtol=1e-9)
        assert [h.photometric_px, h.depth_px, h.semantic_px, h.uncovered_px] == \
            [int(v) for v in r[3:]]
    assert gm.size() == len(out["log_radii"])
    compare_maps(gm, out, 1e-9)
    assert st.step_count() == iters
    if prune_every:
        assert gm.size() < 220  # the threshold removed some Gaussians


def test_resumed_state_equals_one_call(ctx):
    """Two calls through download/upload of the AdamState == one call of the sum."""
    cam, gm1, frames = scene(4)
    _, gm2, _ = scene(4)
    cfg = MapperConfig(prune_every=0)
    s1, s2 = AdamState(), AdamState()
    sgm.optimize_map(gm1, s1, frames, cam, cfg, 10, ctx=ctx)
    sgm.optimize_map(gm2, s2, frames, cam, cfg, 4, ctx=ctx)
    sgm.optimize_map(gm2, s2, frames, cam, cfg, 6, ctx=ctx)  # 4 % 2 == 0: same round-robin phase
    assert s1.step_count() == s2.step_count() == 10
    np.testing.assert_allclose(gm1.centers, gm2.centers, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(s1.v, s2.v, rtol=1e-9, atol=1e-30)


def test_loss_decreases_and_device_state(ctx):
    cam, gm, frames = scene(5)
    tr = MapTrainer(gm, ctx=ctx)
    dev = [sgm.DeviceFrame(f, ctx=ctx) for f in frames]
    hist = tr.optimize(dev, cam, MapperConfig(prune_every=0), 40)
    assert hist[-1].total() < hist[0].total()
    assert tr.step_count() == 40 and tr.size() == gm.size()


def test_errors_like_reference(ctx, ref):
    cam, gm, frames = scene(6)
    with pytest.raises(ValueError):
        sgm.optimize_map(gm, AdamState(), [], cam, MapperConfig(), 5, ctx=ctx)
    with pytest.raises(ValueError):
        sgm.optimize_map(gm, AdamState(), frames, cam, MapperConfig(), 0, ctx=ctx)
    # divergence: every iteration counts as diverged with factor 0 -> throw at the window
    cfg = MapperConfig(divergence_factor=0.0, divergence_window=3, prune_every=0)
    _, _, err = ref.optimize_map(gm, frames, cam, cfg, 10)
    assert err is not None and "diverged" in err
    tr = MapTrainer(gm, ctx=ctx)
    dev = [sgm.DeviceFrame(f, ctx=ctx) for f in frames]
    with pytest.raises(SgmError, match="diverged"):
        tr.optimize(dev, cam, cfg, 10)
    assert tr.step_count() == 3
