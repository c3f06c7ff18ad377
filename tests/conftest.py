import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "reference_scenes.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: large-size property checks")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build_oracle()
    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.build_ref():
        pytest.skip("reference build (oracle/_ref) unavailable")
    return oracle.RefLib()


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN, allow_pickle=False)


def golden_scene(g, name):
    """(map, camera, pose, options, channels, outputs-dict) of a golden scene."""
    from paper_2506_00225_b200.splatmap import CameraModel, GaussianMap, Pose, RenderOptions
    p = f"{name}/"
    k, m = (int(v) for v in g[p + "kc"])
    gm = GaussianMap.from_arrays(k, m, g[p + "centers"], g[p + "log_radii"],
                                 g[p + "opacity_logits"], g[p + "colors"], g[p + "sem_indices"],
                                 g[p + "sem_probs"])
    cv = g[p + "cam"]
    cam = CameraModel(int(cv[0]), int(cv[1]), 0.0, 0.0, cv[2], cv[3], cv[4], cv[5])
    pose = Pose(g[p + "R"], g[p + "t"])
    o = g[p + "opts"]
    opts = RenderOptions(bool(o[0]), float(o[1]), float(o[2]), float(o[3]), int(o[4]))
    outs = {key[len(p):]: g[key] for key in g.files if key.startswith(p)}
    return gm, cam, pose, opts, int(g[p + "channels"][0]), outs


def random_map(seed, n, cam, pose=None, k=4, num_classes=9, rad_px=(1.0, 6.0),
               logit=(-1.5, 2.5), depth=(0.6, 4.0), spread=1.1, dup=False):
    """A seeded splat cloud in the camera frustum (numpy; test-only generator)."""
    from paper_2506_00225_b200.splatmap import GaussianMap, Pose
    pose = pose if pose is not None else Pose()
    rng = np.random.default_rng(seed)
    z = rng.uniform(depth[0], depth[1], n)
    xn = (rng.uniform(0, 1, n) - 0.5) * spread * cam.width / cam.fx
    yn = (rng.uniform(0, 1, n) - 0.5) * spread * cam.height / cam.fy
    pc = np.stack([xn * z, yn * z, z], axis=1)
    centers = pc @ np.asarray(pose.R).T + np.asarray(pose.t)
    rp = rng.uniform(rad_px[0], rad_px[1], n)
    log_r = np.log(rp * z / cam.fy)
    logits = rng.uniform(logit[0], logit[1], n)
    colors = rng.uniform(-0.1, 1.1, (n, 3))
    C = num_classes + 1
    idx = np.stack([rng.choice(C, size=k, replace=False) for _ in range(n)]).astype(np.uint16)
    if dup and k >= 2:
        idx[::3, 1] = idx[::3, 0]
    pr = rng.gamma(0.5, 1.0, (n, k)) + 1e-3
    pr /= pr.sum(axis=1, keepdims=True)
    return GaussianMap.from_arrays(k, num_classes, centers, log_r, logits, colors, idx, pr)
