"""SURVEY §8 f1 on CPU: the C restatement of ExplorationMap / sample_candidates
(oracle/sgm_oracle.c) against the reference's own explorer.cpp (oracle/_ref), bit for
bit: voxel states, free/occupied counts, changelog order, sampled candidates. The
reference's own explorer tests (proj/tests/test_explorer.cpp:64-180, 335-357) run in
tests/test_oracle.py."""
import numpy as np
import pytest

from emap_scenes import ROOM, camera, frames


def same(a, b):
    assert a.info() == b.info()
    assert np.array_equal(a.grid(), b.grid())


@pytest.mark.parametrize("voxel,stride", [(0.05, 2), (0.1, 1), (0.13, 3)])
def test_integrate_matches_reference(orc, ref, voxel, stride):
    cam = camera()
    r, o = ref.emap(*ROOM, voxel), orc.emap(*ROOM, voxel)
    for i, (pose, d) in enumerate(frames(ref, cam, seed=int(voxel * 100))):
        assert r.integrate(cam, pose, d, stride) == o.integrate(cam, pose, d, stride)
        same(r, o)
        if i % 2:
            assert np.array_equal(r.take_changelog(), o.take_changelog())
    for sched in [(1.0, 5, [1.4]), (0.5, 15, [0.8, 1.4]), (0.37, 3, [0.05, 2.9])]:
        pr, dr = r.sample_candidates(*sched)
        po, do = o.sample_candidates(*sched)
        assert np.array_equal(pr, po) and np.array_equal(dr, do)
        r.reseed()
        o.reseed()
    same(r, o)


def test_seed_and_reseed_match_reference(orc, ref):
    r, o = ref.emap(*ROOM, 0.1), orc.emap(*ROOM, 0.1)
    for box, occ in [(((0, 0, 0), (1, 1, 1)), False), (((0.5, 0.5, 0.5), (2, 2, 2)), True),
                     (((1.5, 0, 1.5), (4, 3, 4)), False)]:
        r.seed(*box, occupied=occ)
        o.seed(*box, occupied=occ)
        same(r, o)
    assert np.array_equal(r.take_changelog(), o.take_changelog())
    r.reseed()
    o.reseed()
    assert np.array_equal(r.take_changelog(), o.take_changelog())


def test_camera_outside_grid_and_degenerate_frames(orc, ref):
    cam = camera(32, 24)
    from paper_2506_00225_b200.splatmap import look_at
    r, o = ref.emap(*ROOM, 0.07), orc.emap(*ROOM, 0.07)
    rng = np.random.default_rng(3)
    cases = [(look_at((-1.0, 1.5, 2.0), (4, 1.5, 2)), rng.uniform(0.5, 6, cam.width * cam.height)),
             (look_at((2, 1.5, 2), (2, 1.5, 4)), np.zeros(cam.width * cam.height)),
             (look_at((2, 1.5, 2), (3, 2.5, 3)), np.full(cam.width * cam.height, 1e-13)),
             (look_at((4.0, 3.0, 4.0), (0, 0, 0)), rng.uniform(0, 10, cam.width * cam.height))]
    for pose, d in cases:
        assert r.integrate(cam, pose, d, 1) == o.integrate(cam, pose, d, 1)
        same(r, o)


def test_fibonacci_and_schedule(orc, ref):
    for count in (1, 2, 5, 15, 40):
        for el in (45.0, 10.0, 89.0):
            assert np.array_equal(ref.fibonacci_directions(count, el),
                                  orc.fibonacci_directions(count, el))
    d = orc.fibonacci_directions(15)
    np.testing.assert_allclose(np.linalg.norm(d, axis=1), 1.0, rtol=1e-15)  # test_explorer.cpp:142-154
    assert np.all(np.abs(d[:, 1]) <= np.sin(np.deg2rad(45.0)) + 1e-12)


def test_empty_changelog_samples_nothing(orc, ref):
    for e in (ref.emap((0, 0, 0), (2, 2, 2), 0.05), orc.emap((0, 0, 0), (2, 2, 2), 0.05)):
        p, d = e.sample_candidates(1.0, 5, [1.4])  # test_explorer.cpp:156-160
        assert len(p) == 0


def test_bad_voxel_size(orc, ref):
    for mk in (ref.emap, orc.emap):
        with pytest.raises(ValueError):
            mk((0, 0, 0), (1, 1, 1), 0.0)
