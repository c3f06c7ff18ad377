"""The score raster's tensor-memory accumulator (channel groups from SGM_TM_FIRST on held in
TMEM, `tcgen05.ld/st`): scores are bit-identical to the shared-memory accumulator for every
split, with distinct and repeated class ids, on plain and depth-prefix (dense) launches, and
match the oracle. By default only maps with k >= 24 use it (cfg4)."""
import numpy as np
import pytest

from conftest import random_map

import paper_2506_00225_b200 as sgm
from paper_2506_00225_b200 import scenes
from paper_2506_00225_b200.splatmap import CameraModel, RenderOptions

pytestmark = pytest.mark.gpu

ENT_RTOL = 1e-11


@pytest.fixture(scope="module")
def ctx():
    return sgm.Context(0)


def _scores(ctx, monkeypatch, gm, cam, poses, first, opts=None):
    monkeypatch.setenv("SGM_TM_FIRST", str(first))
    return sgm.score_poses(gm, cam, poses, options=opts, ctx=ctx)


@pytest.mark.parametrize("dup", [False, True])
@pytest.mark.parametrize("k", [3, 16, 32])
def test_tensor_memory_splits_bit_identical(ctx, orc, monkeypatch, k, dup):
    cam = CameraModel(96, 64, 0, 0, 80.0, 80.0, 48.0, 32.0)
    poses = [c.camera_pose() for c in scenes.make_candidates(0, 3)]
    pose = poses[0]
    gm = random_map(900 + k, 1500, cam, pose, k=k, num_classes=max(k, 60), rad_px=(1.0, 12.0), dup=dup)
    base = _scores(ctx, monkeypatch, gm, cam, [pose], 8)
    for first in (0, 3, 4, 7):
        nm, es = _scores(ctx, monkeypatch, gm, cam, [pose], first)
        assert np.array_equal(nm, base[0]) and np.array_equal(es, base[1]), first
    nm_o, es_o, _ = orc.score_views(gm, cam, [pose])
    assert base[0][0] == nm_o[0]
    np.testing.assert_allclose(base[1], es_o, rtol=ENT_RTOL, atol=1e-300)


def test_tensor_memory_on_dense_prefix_launches(ctx, monkeypatch):
    """cfg4's cube (k = 32: tensor memory by default) through depth-prefix binning with a small
    cap (many incomplete tiles redone): identical to the shared-memory accumulator."""
    gm = scenes.make_map(4, n=60_000)
    cam = CameraModel(240, 136, 0, 0, 120.0, 120.0, 119.5, 67.5)
    poses = [c.camera_pose() for c in scenes.make_candidates(4, 5)]
    monkeypatch.setenv("SGM_PREFIX_BINNING", "1")
    monkeypatch.setenv("SGM_PREFIX_CAP", "128")
    ref = _scores(ctx, monkeypatch, gm, cam, poses, 8)
    monkeypatch.delenv("SGM_TM_FIRST")
    nm, es = sgm.score_poses(gm, cam, poses, ctx=ctx)  # the default split (groups 4-7)
    assert np.array_equal(nm, ref[0]) and np.array_equal(es, ref[1])
    nm0, es0 = _scores(ctx, monkeypatch, gm, cam, poses, 0)
    assert np.array_equal(nm0, ref[0]) and np.array_equal(es0, ref[1])


def test_tensor_memory_column_limits(ctx, orc, monkeypatch):
    """Groups of more than 16 channels cannot share a lane quarter (groups 0-3 stay in shared
    memory), more than 32 do not fit 128 columns (no tensor memory): same scores."""
    cam = CameraModel(64, 48, 0, 0, 60.0, 60.0, 32.0, 24.0)
    pose = scenes.make_candidates(0, 1)[0].camera_pose()
    for nc in (150, 300):
        gm = random_map(77 + nc, 600, cam, pose, k=24, num_classes=nc, rad_px=(1.0, 8.0))
        base = _scores(ctx, monkeypatch, gm, cam, [pose], 8)
        nm, es = _scores(ctx, monkeypatch, gm, cam, [pose], 0)
        assert np.array_equal(nm, base[0]) and np.array_equal(es, base[1]), nc
        nm_o, es_o, _ = orc.score_views(gm, cam, [pose])
        assert nm[0] == nm_o[0]
        np.testing.assert_allclose(es, es_o, rtol=ENT_RTOL, atol=1e-300)
