"""Fisher-information extension: the CPU oracle pinned by central finite
differences of the oracle renderer (the reference has no Fisher term; its backward chain,
proj/src/losses.cpp:242-335, is what the oracle restates; parity is FD-pinned only).

Kink-free setup as the reference's own gradient harness: no early exit and a 12-sigma
truncation (proj/tests/grad_check.hpp:17-22), colours inside (0, 1), footprints below the
0.999999 cap."""
import numpy as np
import pytest

from conftest import random_map

from paper_2506_00225_b200.splatmap import CameraModel, Pose, RenderOptions, look_at

FD_OPTS = RenderOptions(early_exit=False, truncation_sigmas=12.0)


def _planes(orc, gm, cam, pose):
    o = orc.render(gm, cam, pose, 3, FD_OPTS)
    return np.concatenate([o["color"].reshape(-1, 3), o["depth"][:, None]], axis=1)


def _fd_fisher(orc, gm, cam, pose, eps=1e-6):
    """H_fd[i, theta] = sum_px sum_ch ((R(+eps) - R(-eps)) / 2 eps)^2."""
    n = gm.size()
    H = np.zeros((n, 8))
    slots = []
    for i in range(n):
        slots += [(gm.centers, (i, a)) for a in range(3)]
        slots += [(gm.log_radii, (i,)), (gm.opacity_logits, (i,))]
        slots += [(gm.colors, (i, a)) for a in range(3)]
    for s, (arr, ix) in enumerate(slots):
        saved = arr[ix]
        arr[ix] = saved + eps
        hi = _planes(orc, gm, cam, pose)
        arr[ix] = saved - eps
        lo = _planes(orc, gm, cam, pose)
        arr[ix] = saved
        J = (hi - lo) / (2 * eps)
        H[s // 8, s % 8] = float(np.sum(J * J))
    return H


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_fisher_diagonal_matches_finite_differences(orc, seed):
    cam = CameraModel(9, 7, 0, 0, 8.0, 8.5, 4.3, 3.6)
    pose = look_at([0.05 * seed, -0.02, -0.4], [0.0, 0.03, 2.0])
    gm = random_map(seed, 6, cam, pose, k=2, num_classes=3, rad_px=(1.0, 3.0), logit=(-1.5, 2.5),
                    depth=(0.8, 2.5), spread=0.7)
    gm.colors[:] = np.clip(gm.colors, 0.1, 0.9)  # away from the clamp kinks
    H = orc.fisher_accumulate(gm, cam, [pose], FD_OPTS)
    H_fd = _fd_fisher(orc, gm, cam, pose)
    assert np.all(H >= 0)
    np.testing.assert_allclose(H, H_fd, rtol=2e-4, atol=1e-9 * max(1.0, H_fd.max()))


def test_fisher_accumulates_over_poses_and_gain(orc):
    cam = CameraModel(16, 12, 0, 0, 14.0, 14.0, 8.0, 6.0)
    pose = look_at([0.0, 0.0, -0.4], [0.0, 0.0, 2.0])
    gm = random_map(5, 40, cam, pose, k=3, num_classes=5)
    poses = [look_at([0.03 * i, 0.0, -0.4], [0.0, 0.0, 2.0]) for i in range(3)]
    H = orc.fisher_accumulate(gm, cam, poses)
    H_sum = sum(orc.fisher_accumulate(gm, cam, [p]) for p in poses)
    np.testing.assert_allclose(H, H_sum, rtol=1e-12)
    lam = 1.0
    g = orc.fisher_gain(gm, cam, poses, H, lam)
    # linear in H_v: gain_v = sum H_v / (H_prior + lambda)
    for i, p in enumerate(poses):
        Hv = orc.fisher_accumulate(gm, cam, [p])
        assert g[i] == pytest.approx(float(np.sum(Hv / (H + lam))), rel=1e-10)
    # an unobserved view (facing away) carries no information
    away = look_at([0.0, 0.0, -0.4], [0.0, 0.0, -3.0])
    assert orc.fisher_gain(gm, cam, [away], H, lam)[0] == 0.0
