"""On-device map optimisation: optimize_map / AdamState on the GPU.

Mirrors proj/include/splatmap/optimizer.hpp:8-60 (AdamParams, AdamState),
proj/include/splatmap/mapper.hpp:18-80 (MapperConfig, optimize_map) and
proj/src/mapper.cpp:10-69, 241-283. Each iteration runs render(all(true)) -> mapping_loss
+ semantic_loss -> backward -> Adam step entirely in HBM (sgm_optimize_map); the map and
the Adam moments stay on the device for the whole call, so only the loss history
(56 B per iteration) crosses PCIe.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N
from .splatmap import (CameraModel, Context, Frame, GaussianMap, LossReport, LossWeights,
                       RenderOptions, _ctx)


@dataclass
class AdamParams:
    """optimizer.hpp:8-21."""

    lr_center: float = 1e-4
    lr_radius: float = 5e-3
    lr_opacity: float = 5e-2
    lr_color: float = 2.5e-3
    lr_sem: float = 1e-2
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    eps_sem: float = 1e-3

    def _c(self) -> N.sgm_adam_params:
        return N.sgm_adam_params(self.lr_center, self.lr_radius, self.lr_opacity, self.lr_color,
                                 self.lr_sem, self.beta1, self.beta2, self.eps, self.eps_sem)


@dataclass
class MapperConfig:
    """The fields of mapper.hpp:18-33 that optimize_map reads."""

    adam: AdamParams = field(default_factory=AdamParams)
    weights: LossWeights = field(default_factory=LossWeights)
    iters_per_step: int = 60
    prune_every: int = 100
    prune_opacity: float = 0.005
    divergence_factor: float = 10.0
    divergence_window: int = 100


class AdamState:
    """optimizer.hpp:24-60 on the host: moments in the layout
    center 3N | log_radius N | opacity_logit N | color 3N | sem kN, and the step count."""

    def __init__(self):
        self.m: Optional[np.ndarray] = None
        self.v: Optional[np.ndarray] = None
        self.t = 0

    def step_count(self) -> int:
        return self.t


def _weights(w: LossWeights) -> np.ndarray:
    return np.array([w.lambda_hd, w.lambda_cos, float(w.mask_k), float(w.use_hd),
                     float(w.use_cos), float(w.use_kl), w.kl_clip_norm])


class DeviceFrame:
    """A Frame uploaded once (sgm_frame)."""

    def __init__(self, frame: Frame, ctx: Optional[Context] = None):
        self._ctx = _ctx(ctx)
        h = C.c_void_p()
        pf = C.POINTER(C.c_float)
        rgb = np.ascontiguousarray(frame.rgb, dtype=np.float32).reshape(-1)
        dep = np.ascontiguousarray(frame.depth, dtype=np.float32).reshape(-1)
        sem = np.ascontiguousarray(frame.sem, dtype=np.float32).reshape(-1)
        px = frame.width * frame.height
        if rgb.size != 3 * px or dep.size != px or sem.size != px * (frame.num_classes + 1):
            raise ValueError("frame: plane sizes do not match width * height")
        pose = frame.pose._c()
        self._ctx.check(N.lib.sgm_frame_upload(self._ctx.handle, frame.width, frame.height,
                                               frame.num_classes, C.byref(pose),
                                               rgb.ctypes.data_as(pf), dep.ctypes.data_as(pf),
                                               sem.ctypes.data_as(pf), C.byref(h)))
        self.handle = h
        self.frame = frame

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            N.lib.sgm_frame_release(self._ctx.handle, h)
            self.handle = None


class MapTrainer:
    """A map plus its Adam state resident in HBM (sgm_trainer)."""

    def __init__(self, gmap: GaussianMap, adam: Optional[AdamState] = None,
                 ctx: Optional[Context] = None):
        if gmap.anisotropic():
            # the trainer optimises the reference's isotropic parameters (mapper.cpp:10-51):
            # log_radius, which an anisotropic footprint ignores, and no per-axis scales or
            # rotations, so an anisotropic map cannot be trained (nor re-indexed by pruning)
            raise ValueError("MapTrainer: anisotropic maps are not trainable (isotropic only); "
                             "call gmap.set_anisotropic(None, None) first")
        self.handle = None
        self._ctx = _ctx(ctx)
        self.k, self.num_classes = gmap.k(), gmap.num_classes()
        n = self._n0 = gmap.size()
        arrs = [np.ascontiguousarray(a, dtype=np.float64).reshape(-1) for a in
                (gmap.centers, gmap.log_radii, gmap.opacity_logits, gmap.colors, gmap.sem_probs)]
        idx = np.ascontiguousarray(gmap.sem_indices, dtype=np.uint16).reshape(-1)
        mv = None
        t = 0
        if adam is not None:
            t = adam.t
            if adam.m is not None:
                per = (8 + self.k) * n
                if adam.m.size != per or adam.v.size != per:
                    raise ValueError("AdamState moments do not match the map size")
                mv = np.ascontiguousarray(np.concatenate([adam.m, adam.v]), dtype=np.float64)
        h = C.c_void_p()
        self._ctx.check(N.lib.sgm_trainer_create(
            self._ctx.handle, n, self.k, self.num_classes, N.dptr(arrs[0]), N.dptr(arrs[1]),
            N.dptr(arrs[2]), N.dptr(arrs[3]), idx.ctypes.data_as(C.POINTER(C.c_uint16)),
            N.dptr(arrs[4]), N.dptr(mv), int(t), C.byref(h)))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            N.lib.sgm_trainer_destroy(self._ctx.handle, h)
            self.handle = None

    def size(self) -> int:
        n = C.c_uint64()
        self._ctx.check(N.lib.sgm_trainer_size(self._ctx.handle, self.handle, C.byref(n), None))
        return int(n.value)

    def step_count(self) -> int:
        t = C.c_int64()
        self._ctx.check(N.lib.sgm_trainer_size(self._ctx.handle, self.handle, None, C.byref(t)))
        return int(t.value)

    def optimize(self, frames: Sequence[DeviceFrame], camera: CameraModel,
                 cfg: Optional[MapperConfig] = None, iters: Optional[int] = None,
                 options: Optional[RenderOptions] = None) -> List[LossReport]:
        """optimize_map (mapper.cpp:241-283) on the resident state."""
        cfg = cfg if cfg is not None else MapperConfig()
        iters = cfg.iters_per_step if iters is None else int(iters)
        fh = (C.c_void_p * max(len(frames), 1))(*[f.handle.value for f in frames])
        hist = np.zeros((max(iters, 1), 7))
        done = C.c_int32()
        cam = camera._c()
        adam = cfg.adam._c()
        cfg_c = N.sgm_optimize_config(int(cfg.prune_every), float(cfg.prune_opacity),
                                      float(cfg.divergence_factor), int(cfg.divergence_window))
        opt = (options if options is not None else RenderOptions())._c()
        w = _weights(cfg.weights)
        code = N.lib.sgm_optimize_map(self._ctx.handle, self.handle, C.byref(cam), len(frames),
                                      fh if frames else None, C.byref(opt), C.byref(adam),
                                      N.dptr(w), C.byref(cfg_c), iters, N.dptr(hist),
                                      C.byref(done))
        self._ctx.check(code)
        return [LossReport(float(r[0]), float(r[1]), float(r[2]), int(r[3]), int(r[4]),
                           int(r[5]), int(r[6])) for r in hist[: int(done.value)]]

    def download(self, gmap: GaussianMap, adam: Optional[AdamState] = None) -> None:
        """Writes the resident parameters (and moments) back into `gmap` / `adam`."""
        n, k = self.size(), self.k
        centers, logr, logit = np.zeros(3 * n), np.zeros(n), np.zeros(n)
        colors, idx, probs = np.zeros(3 * n), np.zeros(k * n, np.uint16), np.zeros(k * n)
        mv = np.zeros(2 * (8 + k) * n) if adam is not None else None
        self._ctx.check(N.lib.sgm_trainer_download(
            self._ctx.handle, self.handle, N.dptr(centers), N.dptr(logr), N.dptr(logit),
            N.dptr(colors), idx.ctypes.data_as(C.POINTER(C.c_uint16)), N.dptr(probs),
            N.dptr(mv)))
        rows = np.zeros(n, np.uint32)
        self._ctx.check(N.lib.sgm_trainer_rows(self._ctx.handle, self.handle,
                                               rows.ctypes.data_as(C.POINTER(C.c_uint32))))
        src = np.asarray(gmap.source_frames, dtype=np.uint32)
        gmap.source_frames = src[rows] if src.size == self._n0 else np.zeros(n, np.uint32)
        gmap.centers = centers.reshape(n, 3)
        gmap.log_radii = logr
        gmap.opacity_logits = logit
        gmap.colors = colors.reshape(n, 3)
        gmap.sem_indices = idx.reshape(n, k)
        gmap.sem_probs = probs.reshape(n, k)
        gmap.touch()
        if adam is not None:
            half = (8 + k) * n
            adam.m, adam.v = mv[:half].copy(), mv[half:].copy()
            adam.t = self.step_count()


def optimize_map(gmap: GaussianMap, adam: AdamState, frames: Sequence[Frame],
                 camera: CameraModel, cfg: Optional[MapperConfig] = None, iters: int = 60,
                 ctx: Optional[Context] = None) -> List[LossReport]:
    """optimize_map (mapper.hpp:76-80): round-robin keyframe optimisation on the GPU.
    Updates `gmap` and `adam` in place and returns the per-iteration loss history; raises
    like the reference on no frames, iters < 1, divergence or a non-finite gradient."""
    if not frames:
        raise ValueError("optimize_map: no frames")
    if iters < 1:
        raise ValueError("optimize_map: iters must be >= 1")
    c = _ctx(ctx)
    tr = MapTrainer(gmap, adam, ctx=c)
    dev = [DeviceFrame(f, ctx=c) for f in frames]
    try:
        hist = tr.optimize(dev, camera, cfg, iters)
    except Exception:
        # the reference updates the map and AdamState in place up to the iteration that
        # throws (mapper.cpp:262-272): hand back the same partial progress, then re-raise
        try:
            tr.download(gmap, adam)
        except Exception:
            pass
        raise
    tr.download(gmap, adam)
    return hist
