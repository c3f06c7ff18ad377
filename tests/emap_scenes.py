"""Exploration-map test scenes shared by the CPU and GPU tests.

Frames are the reference simulator's own depth (raycast_frame, via oracle/_ref) of a
room with a box and a sphere, as in proj/tests/test_explorer.cpp:13-28, plus invalid
pixels, NaN depth and rays that end on the outer shell."""
import numpy as np

from paper_2506_00225_b200.splatmap import CameraModel, look_at

ROOM = ((0.0, 0.0, 0.0), (4.0, 3.0, 4.0))
BOXES = [(1.0, 0.0, 2.5, 1.6, 1.0, 3.2), (0.01, 0.01, 0.01, 0.05, 0.05, 0.05)]
SPHERES = [(3.0, 1.2, 1.0, 0.4)]
VIEWS = [((2, 1.5, 2), (4, 1.5, 2)), ((2, 1.5, 2), (2, 1.5, 4)), ((2, 1.5, 2), (0.3, 1.2, 0.3)),
         ((1.0, 1.0, 1.0), (3.0, 0.2, 3.5)), ((3.5, 2.5, 0.5), (0.5, 0.3, 3.5)),
         ((0.5, 1.4, 3.5), (3.5, 1.4, 0.5))]


def camera(w=64, h=48):
    return CameraModel(w, h, 0, 0, 0.8 * w, 0.8 * w, w / 2.0 - 0.5, h / 2.0 - 0.5)


def frames(ref, cam, seed=0, views=VIEWS, invalid=0.05):
    """(pose, depth) per view: raycast depth with a fraction of invalid / NaN pixels."""
    rng = np.random.default_rng(seed)
    out = []
    for eye, tgt in views:
        pose = look_at(eye, tgt)
        d = ref.raycast_depth(ROOM[0], ROOM[1], cam, pose, boxes=BOXES, spheres=SPHERES)
        d[rng.uniform(size=d.size) < invalid] = 0.0
        d[rng.integers(0, d.size, 3)] = np.nan
        d[rng.integers(0, d.size, 3)] = -1.0
        out.append((pose, d))
    return out
