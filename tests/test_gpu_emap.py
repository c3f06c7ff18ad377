"""SURVEY §8 f1 on the GPU: ExplorationMap / sample_candidates (sgm_emap, k_emap_rays)
against the reference's own explorer.cpp (oracle/_ref): bit-identical voxel states,
counts, changelog order and candidates."""
import numpy as np
import pytest

from emap_scenes import ROOM, camera, frames

import paper_2506_00225_b200 as sgm
from paper_2506_00225_b200._native import SgmError
from paper_2506_00225_b200.explore import Aabb, ExplorationMap, SamplingSchedule

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return sgm.Context(0)


def gpu_map(ctx, voxel, room=ROOM):
    return ExplorationMap(Aabb(np.array(room[0], float), np.array(room[1], float)), voxel, ctx=ctx)


def same(g, r):
    info = r.info()
    assert (g.free_count(), g.occupied_count(), g.changelog_size()) == \
        (info["free"], info["occupied"], info["changelog"])
    assert g.dims() == info["dims"]
    assert np.array_equal(g.grid(), r.grid())


@pytest.mark.parametrize("voxel,stride", [(0.05, 2), (0.1, 1), (0.13, 3)])
def test_integrate_matches_reference(ctx, ref, voxel, stride):
    cam = camera()
    g, r = gpu_map(ctx, voxel), ref.emap(*ROOM, voxel)
    for i, (pose, d) in enumerate(frames(ref, cam, seed=int(voxel * 100))):
        assert g.integrate_frame(d, cam, pose, stride) == r.integrate(cam, pose, d, stride)
        same(g, r)
        if i % 2:
            assert np.array_equal(g.take_changelog(), r.take_changelog())
    for sched in [SamplingSchedule.coarse(), SamplingSchedule.fine(),
                  SamplingSchedule(None, 0.37, 3, (0.05, 2.9))]:
        cands = sgm.sample_candidates(g, sched)
        pr, dr = r.sample_candidates(sched.v1, sched.v2, list(sched.heights))
        assert len(cands) == len(pr)
        if cands:
            assert np.array_equal(np.stack([c.position for c in cands]), pr)
            assert np.array_equal(np.stack([c.direction for c in cands]), dr)
        assert g.changelog_size() == 0
        g.reseed_changelog_with_free()
        r.reseed()
    same(g, r)


def test_device_depth_and_full_size(ctx, ref):
    """cfg1-sized frames (1200x680, fx=600) in an 8x6x3 m box at 5 cm, depth in HBM."""
    import torch
    from paper_2506_00225_b200.splatmap import CameraModel, look_at
    cam = CameraModel(1200, 680, 0, 0, 600.0, 600.0, 599.5, 339.5)
    room = ((0.0, 0.0, 0.0), (8.0, 3.0, 6.0))
    g, r = gpu_map(ctx, 0.05, room), ref.emap(*room, 0.05)
    for eye, tgt in [((4, 1.5, 3), (8, 1.2, 3)), ((1, 1.4, 1), (7, 0.5, 5)),
                     ((6, 2.0, 5), (0.5, 1.0, 0.5))]:
        pose = look_at(eye, tgt)
        d = ref.raycast_depth(*room, cam, pose, boxes=[(2, 0, 2, 3, 1, 3)],
                              spheres=[(6, 1, 1.5, 0.5)])
        nd = g.integrate_frame(torch.from_numpy(d).cuda(), cam, pose, 2)
        assert nd == r.integrate(cam, pose, d, 2)
        same(g, r)
    assert np.array_equal(g.take_changelog(), r.take_changelog())


def test_seed_reseed_and_outside_camera(ctx, ref):
    g, r = gpu_map(ctx, 0.1), ref.emap(*ROOM, 0.1)
    for box, occ in [(((0, 0, 0), (1, 1, 1)), False), (((0.5, 0.5, 0.5), (2, 2, 2)), True),
                     (((1.5, 0, 1.5), (4, 3, 4)), False)]:
        b = Aabb(np.array(box[0], float), np.array(box[1], float))
        (g.seed_occupied_region if occ else g.seed_free_region)(b)
        r.seed(*box, occupied=occ)
        same(g, r)
    assert np.array_equal(g.take_changelog(), r.take_changelog())
    g.reseed_changelog_with_free()
    r.reseed()
    assert np.array_equal(g.take_changelog(), r.take_changelog())
    from paper_2506_00225_b200.splatmap import look_at
    cam = camera(32, 24)
    rng = np.random.default_rng(3)
    for pose, d in [(look_at((-1.0, 1.5, 2.0), (4, 1.5, 2)), rng.uniform(0.5, 6, 32 * 24)),
                    (look_at((4.0, 3.0, 4.0), (0, 0, 0)), rng.uniform(0, 10, 32 * 24)),
                    (look_at((2, 1.5, 2), (3, 2.5, 3)), np.full(32 * 24, 1e-13))]:
        assert g.integrate_frame(d, cam, pose, 1) == r.integrate(cam, pose, d, 1)
        same(g, r)


def test_errors_and_empty(ctx):
    with pytest.raises(SgmError):
        gpu_map(ctx, 0.0)
    g = gpu_map(ctx, 0.05, ((0, 0, 0), (2, 2, 2)))
    assert sgm.sample_candidates(g, SamplingSchedule.coarse()) == []  # test_explorer.cpp:156-160
    with pytest.raises(SgmError):
        g.integrate_frame(np.zeros(16, np.float32), camera(4, 4), sgm.look_at((1, 1, 1), (2, 1, 1)), 0)
    assert g.voxel_at((0.01, 0.01, 0.01)) == 0 and g.voxel_at((-1, 0, 0)) == -1
