"""Seeded synthetic scenes for BASELINE.json configs 0-4.

The Replica / Matterport3D scenes the configs are "shaped" after are not in this
container and are not reproduced: these are Gaussian clouds with the stated
counts, boxes and parameter distributions, generated in fp64 from seed
1000 + cfg and rounded to fp32 (the SGMP v1 storage precision), so a map written
with GaussianMap.save and re-loaded is bit-identical to the generated one.

Interpretation decisions (recorded in every bench line):
  * world up = +Y; a box "W x D x H m" spans x in [0,W], z in [0,D], y in [0,H];
  * "k of C=101 classes" -> GaussianMap(k, num_classes=101) -> 102 channels;
  * isotropic parity mode: log_radius = mean of the three per-axis log-scale
    draws; the quaternion is still drawn so the RNG stream stays fixed;
  * candidate direction from yaw psi / pitch theta: (cos t cos p, sin t, cos t sin p).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

from .splatmap import CameraModel, CandidatePose, GaussianMap, look_at


@dataclass
class SceneConfig:
    cfg: int
    n: int
    box: Tuple[float, float, float]          # (W, D, H) metres -> x, z, y extents
    box_origin: Tuple[float, float, float]   # world-space min corner (x, y, z)
    log_scale_mu: float
    log_scale_sigma: float
    logit_mu: float
    k: int
    num_classes: int
    dirichlet: float
    width: int
    height: int
    f: float
    cx: float
    cy: float
    views: int
    name: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def seed(self) -> int:
        return 1000 + self.cfg

    def camera(self) -> CameraModel:
        return CameraModel(self.width, self.height, 0.0, 0.0, self.f, self.f, self.cx, self.cy)


CONFIGS = {
    0: SceneConfig(0, 20_000, (4.0, 4.0, 3.0), (0.0, 0.0, 0.0), -4.0, 0.5, 0.0, 16, 101, 0.3,
                   600, 340, 300.0, 300.0, 170.0, 8, "cpu-oracle-scene"),
    1: SceneConfig(1, 500_000, (8.0, 6.0, 3.0), (0.0, 0.0, 0.0), -4.0, 0.5, 0.0, 16, 101, 0.3,
                   1200, 680, 600.0, 599.5, 339.5, 64, "replica-shaped",
                   {"prior_poses": 32}),
    2: SceneConfig(2, 500_000, (8.0, 6.0, 3.0), (0.0, 0.0, 0.0), -4.0, 0.5, 0.0, 16, 101, 0.3,
                   1200, 680, 600.0, 599.5, 339.5, 1024, "candidate-sweep"),
    3: SceneConfig(3, 2_000_000, (20.0, 15.0, 3.0), (0.0, 0.0, 0.0), -3.5, 0.6, 0.0, 8, 41, 0.2,
                   1920, 1080, 960.0, 959.5, 539.5, 512, "matterport-shaped"),
    4: SceneConfig(4, 1_000_000, (1.0, 1.0, 1.0), (0.0, 0.0, 0.0), -2.5, 0.3, 1.0, 32, 101, 0.3,
                   1200, 680, 600.0, 599.5, 339.5, 256, "dense-overlap"),
}


def _f32(a: np.ndarray) -> np.ndarray:
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def make_map(cfg: int, n: int | None = None, aniso: bool = False) -> GaussianMap:
    """The config's Gaussian cloud (optionally its first-n-Gaussians prefix stream).

    aniso=True also attaches the drawn per-axis log-scales and quaternions (fp32-rounded),
    switching the map to the anisotropic EWA footprint."""
    sc = CONFIGS[cfg]
    n = sc.n if n is None else n
    rng = np.random.Generator(np.random.PCG64(sc.seed))
    W, D, H = sc.box
    ox, oy, oz = sc.box_origin
    centers = np.empty((n, 3))
    centers[:, 0] = ox + rng.uniform(0.0, W, n)
    centers[:, 2] = oz + rng.uniform(0.0, D, n)
    centers[:, 1] = oy + rng.uniform(0.0, H, n)
    log_scales = rng.normal(sc.log_scale_mu, sc.log_scale_sigma, (n, 3))
    quat = rng.normal(0.0, 1.0, (n, 4))
    quat /= np.linalg.norm(quat, axis=1, keepdims=True)  # drawn for stream stability (f4 mode)
    logits = rng.normal(sc.logit_mu, 1.0, n)
    colors = rng.uniform(0.0, 1.0, (n, 3))
    k, m = sc.k, sc.num_classes
    idx = np.empty((n, k), dtype=np.uint16)
    probs = np.empty((n, k))
    chunk = 65536
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        keys = rng.random((e - s, m), dtype=np.float32)
        idx[s:e] = np.argpartition(keys, k - 1, axis=1)[:, :k].astype(np.uint16)
        g = rng.gamma(sc.dirichlet, 1.0, (e - s, k))
        g = np.maximum(g, 1e-300)
        probs[s:e] = g / g.sum(axis=1, keepdims=True)
    gm = GaussianMap.from_arrays(k, m, _f32(centers), _f32(log_scales.mean(axis=1)), _f32(logits),
                                 _f32(colors), idx, _f32(probs))
    gm.quaternions = quat.astype(np.float32)  # unused by the isotropic path
    if aniso:
        gm.set_anisotropic(_f32(log_scales), _f32(quat))
    return gm


def _direction(yaw: float, pitch: float) -> np.ndarray:
    return np.array([math.cos(pitch) * math.cos(yaw), math.sin(pitch),
                     math.cos(pitch) * math.sin(yaw)])


def make_candidates(cfg: int, count: int | None = None, stream: int = 1) -> List[CandidatePose]:
    """Candidate poses of a config (stream 1 = candidates, stream 2 = prior poses)."""
    sc = CONFIGS[cfg]
    rng = np.random.Generator(np.random.PCG64([sc.seed, stream]))
    W, D, H = sc.box
    ox, oy, oz = sc.box_origin
    out: List[CandidatePose] = []
    if cfg == 0:
        c = np.array([ox + W / 2, oy + H / 2, oz + D / 2])
        count = sc.views if count is None else count
        for i in range(count):
            a = 2.0 * math.pi * i / count
            p = c + 1.5 * np.array([math.cos(a), 0.0, math.sin(a)])
            out.append(CandidatePose(position=p, direction=c - p))
    elif cfg == 2:
        # 16 x 8 lattice at 0.25 m, centred, y = 1.4 m, x 8 yaws = 1024 (Appendix A)
        cx0 = ox + W / 2 - 0.25 * 7.5
        cz0 = oz + D / 2 - 0.25 * 3.5
        for i in range(16):
            for j in range(8):
                p = np.array([cx0 + 0.25 * i, oy + 1.4, cz0 + 0.25 * j])
                for y in range(8):
                    out.append(CandidatePose(position=p.copy(),
                                             direction=_direction(2 * math.pi * y / 8, 0.0)))
        if count is not None:
            out = out[:count]
    elif cfg == 4:
        count = sc.views if count is None else count
        c = np.array([ox + W / 2, oy + H / 2, oz + D / 2])
        for _ in range(count):
            v = rng.normal(0.0, 1.0, 3)
            v /= np.linalg.norm(v)
            p = c + 1.2 * v
            out.append(CandidatePose(position=p, direction=c - p))
    else:
        count = sc.views if count is None else count
        if cfg == 1 and stream == 2:
            count = sc.extra["prior_poses"] if count is None else count
        m = 0.25
        for _ in range(count):
            p = np.array([ox + rng.uniform(m, W - m), oy + rng.uniform(m, H - m),
                          oz + rng.uniform(m, D - m)])
            yaw = rng.uniform(0.0, 2.0 * math.pi)
            pitch = math.radians(rng.uniform(-20.0, 20.0))
            out.append(CandidatePose(position=p, direction=_direction(yaw, pitch)))
    for i, cd in enumerate(out):
        cd.id = i
    return out


def make_decision_candidates(cfg: int, count: int = 16) -> List[CandidatePose]:
    """A candidate set whose views see the cloud only in part, so n_missing varies from view
    to view and combine_scores (explorer.cpp:225-248) has a non-trivial argmax. (Every view of
    make_candidates(1..3) lies inside the cloud and sees it everywhere: n_missing = 0, so
    i_geo = i_total = 0 and the reference reports the pool exhausted.)

    Positions lie outside the box, 0.6-1.6 box half-diagonals from its centre in the
    horizontal plane, at heights inside the box; each looks at the centre displaced by up to
    half the box extent, so part of every image is empty. Seeded (stream 3)."""
    sc = CONFIGS[cfg]
    rng = np.random.Generator(np.random.PCG64([sc.seed, 3]))
    W, D, H = sc.box
    ox, oy, oz = sc.box_origin
    c = np.array([ox + W / 2, oy + H / 2, oz + D / 2])
    half = 0.5 * math.hypot(W, D)
    out: List[CandidatePose] = []
    for i in range(count):
        phi = rng.uniform(0.0, 2.0 * math.pi)
        r = half * rng.uniform(0.6, 1.6)
        p = np.array([c[0] + r * math.cos(phi), oy + rng.uniform(0.2, 0.8) * H,
                      c[2] + r * math.sin(phi)])
        tgt = c + np.array([rng.uniform(-0.5, 0.5) * W, rng.uniform(-0.3, 0.3) * H,
                            rng.uniform(-0.5, 0.5) * D])
        out.append(CandidatePose(position=p, direction=tgt - p, id=i))
    return out


def render_poses(cfg: int, count: int | None = None):
    """Explicit render poses (cfg0: the 8 circle poses, look_at(p, centre))."""
    sc = CONFIGS[cfg]
    if cfg == 0:
        W, D, H = sc.box
        c = np.array([W / 2, H / 2, D / 2])
        count = sc.views if count is None else count
        return [look_at(c + 1.5 * np.array([math.cos(2 * math.pi * i / count), 0.0,
                                            math.sin(2 * math.pi * i / count)]), c)
                for i in range(count)]
    return [cd.camera_pose() for cd in make_candidates(cfg, count)]


def make_frame(cfg: int, pose, seed: int = 0, invalid: float = 0.1):
    """Synthetic posed RGB-D-semantic observation at the config's camera (Frame,
    frame.hpp:12-65): rgb in [0.1, 0.9], depth in [0.5, 3] m with `invalid` zeros, and a
    low-entropy semantic simplex (0.7 on one channel) per pixel. Seeded, float32."""
    from .splatmap import Frame
    c = CONFIGS[cfg]
    cam = c.camera()
    rng = np.random.default_rng(10_000 + 100 * cfg + seed)
    px = cam.width * cam.height
    C = c.num_classes + 1
    rgb = (0.1 + 0.8 * rng.uniform(0, 1, (px, 3))).astype(np.float32)
    depth = np.where(rng.uniform(0, 1, px) < invalid, 0.0,
                     0.5 + 2.5 * rng.uniform(0, 1, px)).astype(np.float32)
    p = 0.05 + rng.uniform(0, 1, (px, C))
    p /= p.sum(axis=1, keepdims=True)
    sem = 0.3 * p
    sem[np.arange(px), rng.integers(0, C, px)] += 0.7
    return Frame(cam.width, cam.height, c.num_classes, pose, rgb.reshape(-1), depth,
                 sem.astype(np.float32).reshape(-1))
