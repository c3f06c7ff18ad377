"""Host-side mirror of the reference's renderer / scoring API over the C ABI.

Same names, argument meaning and error behaviour as
  proj/include/splatmap/{camera,geometry,gaussian_map,splat_render,explorer}.hpp
so code (and tests) written against the reference read the same here:

  render(map, camera, pose, channels, options)      splat_render.hpp:78-80
  render_reference(map, camera, pose, channels)     splat_render.hpp:82-86
  clipped_entropy(probs) / render_entropy(...)      splat_render.hpp:88-95
  refresh_candidate_scores(candidates, map, cam)    explorer.hpp:114-115
  combine_scores(candidates, current_position)      explorer.hpp:117-121
  score_candidates / prune_pool / CandidatePool     explorer.hpp:123-148

Every compute call goes to the sm_100a library (libsgm_b200.so); there is no
CPU fallback. Host-side pieces the reference also keeps scalar (combine_scores,
look_at, clipped_entropy of one pixel) run in the library's host code.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import struct
import threading
import weakref
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N

# --------------------------------------------------------------------------- math / camera


def deg_to_rad(d: float) -> float:
    return d * math.pi / 180.0  # geometry.hpp:86


def sigmoid(x: float) -> float:
    return 1.0 / (1.0 + math.exp(-x))  # geometry.hpp:84


def _lround(x: float) -> int:
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


@dataclass
class CameraModel:
    """Pinhole camera, camera.hpp:11-50. Pixel (x, y) looks along
    ((x+0.5-cx)/fx, (y+0.5-cy)/fy, 1); depth is camera-space Z."""

    width: int = 0
    height: int = 0
    vfov_deg: float = 0.0
    hfov_deg: float = 0.0
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0

    @staticmethod
    def from_fov(width: int, height: int, vfov_deg: float, hfov_deg: float) -> "CameraModel":
        if width <= 0 or height <= 0:
            raise ValueError("camera: resolution must be positive")
        if vfov_deg <= 0 or vfov_deg >= 180 or hfov_deg <= 0 or hfov_deg >= 180:
            raise ValueError("camera: FOV must be in (0, 180) degrees")
        c = CameraModel(width, height, vfov_deg, hfov_deg)
        c.fy = (height / 2.0) / math.tan(deg_to_rad(vfov_deg) / 2.0)
        c.fx = (width / 2.0) / math.tan(deg_to_rad(hfov_deg) / 2.0)
        c.cx = width / 2.0
        c.cy = height / 2.0
        return c

    @staticmethod
    def desk_default() -> "CameraModel":
        return CameraModel.from_fov(160, 120, 60.0, 90.0)

    def scaled(self, scale: float) -> "CameraModel":
        w = max(1, _lround(self.width * scale))
        h = max(1, _lround(self.height * scale))
        return CameraModel.from_fov(w, h, self.vfov_deg, self.hfov_deg)

    def pixel_ray(self, x: int, y: int) -> np.ndarray:
        return np.array([(x + 0.5 - self.cx) / self.fx, (y + 0.5 - self.cy) / self.fy, 1.0])

    def pixel_count(self) -> int:
        return self.width * self.height

    def _c(self) -> N.sgm_camera:
        return N.sgm_camera(int(self.width), int(self.height), float(self.fx), float(self.fy),
                            float(self.cx), float(self.cy))


@dataclass
class Pose:
    """Rigid camera-to-world transform x_world = R x_cam + t (geometry.hpp:18-41)."""

    R: np.ndarray = field(default_factory=lambda: np.eye(3))
    t: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def to_world(self, p_cam) -> np.ndarray:
        p = np.asarray(p_cam, dtype=np.float64)
        # Eigen lazy product row = x0 + (x1 + x2), then + t
        return np.array([_dot3(self.R[i], p) + self.t[i] for i in range(3)])

    def to_camera(self, p_world) -> np.ndarray:
        d = np.asarray(p_world, dtype=np.float64) - self.t
        return np.array([_dot3(self.R[:, i], d) for i in range(3)])

    def _c(self) -> N.sgm_pose:
        p = N.sgm_pose()
        R = np.ascontiguousarray(self.R, dtype=np.float64).reshape(9)
        for i in range(9):
            p.R[i] = float(R[i])
        for i in range(3):
            p.t[i] = float(self.t[i])
        return p

    @staticmethod
    def _from_c(p: N.sgm_pose) -> "Pose":
        return Pose(np.array(p.R[:], dtype=np.float64).reshape(3, 3),
                    np.array(p.t[:], dtype=np.float64))


def _dot3(a, b) -> float:
    a0, a1, a2 = (float(v) for v in a)
    b0, b1, b2 = (float(v) for v in b)
    return a0 * b0 + (a1 * b1 + a2 * b2)


def look_at(position, target, up=(0.0, 1.0, 0.0)) -> Pose:
    """geometry.hpp:44-56 (camera +Z forward, +Y image-down, world up +Y)."""
    if tuple(float(u) for u in up) == (0.0, 1.0, 0.0):
        out = N.sgm_pose()
        pos = np.ascontiguousarray(position, dtype=np.float64)
        tgt = np.ascontiguousarray(target, dtype=np.float64)
        N.lib.sgm_look_at(N.dptr(pos), N.dptr(tgt), C.byref(out))
        return Pose._from_c(out)
    # general `up`: the same Eigen-order arithmetic in Python floats
    z = [float(target[i]) - float(position[i]) for i in range(3)]
    z = _normalized(z)
    x = _cross(z, [float(u) for u in up])
    if math.sqrt(_sqnorm(x)) < 1e-9:
        x = _cross(z, [1.0, 0.0, 0.0])
    x = _normalized(x)
    y = _cross(z, x)
    R = np.array([[x[i], y[i], z[i]] for i in range(3)], dtype=np.float64)
    return Pose(R, np.array([float(p) for p in position]))


def _sqnorm(v) -> float:
    return v[0] * v[0] + (v[1] * v[1] + v[2] * v[2])


def _normalized(v):
    s = _sqnorm(v)
    if s > 0.0:
        r = math.sqrt(s)
        return [v[0] / r, v[1] / r, v[2] / r]
    return list(v)


def _cross(a, b):
    return [a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]]


# --------------------------------------------------------------------------- map

@dataclass
class SemanticGaussian:
    """Isotropic splat (gaussian_map.hpp:28-38)."""

    center: np.ndarray = field(default_factory=lambda: np.zeros(3))
    log_radius: float = 0.0
    opacity_logit: float = 0.0
    color: np.ndarray = field(default_factory=lambda: np.zeros(3))
    sem_indices: Sequence[int] = ()
    sem_probs: Sequence[float] = ()
    source_frame: int = 0

    def radius(self) -> float:
        return math.exp(self.log_radius)

    def opacity(self) -> float:
        return sigmoid(self.opacity_logit)


_SGMP_MAGIC = 0x53474D50
_SGMP_VERSION = 1


_MAP_ARRAYS = frozenset({"centers", "log_radii", "opacity_logits", "colors", "sem_indices",
                         "sem_probs", "log_scales", "quats"})


class GaussianMap:
    """Structure-of-arrays splat storage (gaussian_map.hpp:61-114).

    A Context caches one device snapshot per map *version* (the reference reads live spans on
    every call; re-uploading 112 MB per call would dominate scoring). Reassigning an array
    attribute (`gmap.colors = ...`) bumps the version by itself; after editing an array IN
    PLACE (`gmap.colors[i] = ...`) call `touch()`, or the next call renders the snapshot
    taken before the edit."""

    def __setattr__(self, name, value):
        object.__setattr__(self, name, value)
        if name in _MAP_ARRAYS and "_version" in self.__dict__:
            self.__dict__["_version"] += 1

    def __init__(self, k: int, num_classes: int):
        if k < 1 or k > num_classes + 1:
            raise ValueError("map: k must be in [1, num_classes+1]")
        self._k = int(k)
        self._num_classes = int(num_classes)
        self.centers = np.zeros((0, 3))
        self.log_radii = np.zeros(0)
        self.opacity_logits = np.zeros(0)
        self.colors = np.zeros((0, 3))
        self.sem_indices = np.zeros((0, self._k), dtype=np.uint16)
        self.sem_probs = np.zeros((0, self._k))
        self.source_frames = np.zeros(0, dtype=np.uint32)
        # Anisotropic splat mode (no reference counterpart): optional
        # per-axis log-scales (N x 3) and rotation quaternions (w, x, y, z) (N x 4).
        # When both are set, render / score use EWA footprints instead of log_radii.
        self.log_scales: Optional[np.ndarray] = None
        self.quats: Optional[np.ndarray] = None
        self._version = 0

    @classmethod
    def from_arrays(cls, k, num_classes, centers, log_radii, opacity_logits, colors,
                    sem_indices, sem_probs, source_frames=None, log_scales=None,
                    quats=None) -> "GaussianMap":
        m = cls(k, num_classes)
        n = len(log_radii)
        m.centers = np.ascontiguousarray(np.asarray(centers, dtype=np.float64).reshape(n, 3))
        m.log_radii = np.ascontiguousarray(log_radii, dtype=np.float64).reshape(n)
        m.opacity_logits = np.ascontiguousarray(opacity_logits, dtype=np.float64).reshape(n)
        m.colors = np.ascontiguousarray(np.asarray(colors, dtype=np.float64).reshape(n, 3))
        m.sem_indices = np.ascontiguousarray(np.asarray(sem_indices).reshape(n, k), dtype=np.uint16)
        m.sem_probs = np.ascontiguousarray(np.asarray(sem_probs, dtype=np.float64).reshape(n, k))
        m.source_frames = (np.zeros(n, dtype=np.uint32) if source_frames is None
                           else np.ascontiguousarray(source_frames, dtype=np.uint32))
        if log_scales is not None or quats is not None:
            m.set_anisotropic(log_scales, quats)
        return m

    def set_anisotropic(self, log_scales, quats) -> None:
        """Per-Gaussian anisotropic footprints (f4 extension); (None, None) reverts to the
        reference's isotropic log_radius footprint."""
        if log_scales is None and quats is None:
            self.log_scales = self.quats = None
        else:
            n = self.size()
            self.log_scales = np.ascontiguousarray(np.asarray(log_scales, dtype=np.float64).reshape(n, 3))
            self.quats = np.ascontiguousarray(np.asarray(quats, dtype=np.float64).reshape(n, 4))
        self.touch()

    def anisotropic(self) -> bool:
        return self.log_scales is not None and self.quats is not None

    def k(self) -> int:
        return self._k

    def num_classes(self) -> int:
        return self._num_classes

    def channels(self) -> int:
        return self._num_classes + 1

    def size(self) -> int:
        return int(self.log_radii.shape[0])

    def empty(self) -> bool:
        return self.size() == 0

    def touch(self) -> None:
        """Marks the map modified so the device snapshot is re-uploaded."""
        self._version += 1

    def add(self, g: SemanticGaussian) -> None:
        if len(g.sem_indices) != self._k:
            raise ValueError("map: sparse vector k mismatch")
        self.centers = np.vstack([self.centers, np.asarray(g.center, dtype=np.float64)[None]])
        self.log_radii = np.append(self.log_radii, float(g.log_radius))
        self.opacity_logits = np.append(self.opacity_logits, float(g.opacity_logit))
        self.colors = np.vstack([self.colors, np.asarray(g.color, dtype=np.float64)[None]])
        self.sem_indices = np.vstack([self.sem_indices,
                                      np.asarray(g.sem_indices, dtype=np.uint16)[None]])
        self.sem_probs = np.vstack([self.sem_probs, np.asarray(g.sem_probs, dtype=np.float64)[None]])
        if self.anisotropic():  # a plain SemanticGaussian joins as a sphere of its radius
            self.log_scales = np.vstack([self.log_scales, np.full((1, 3), float(g.log_radius))])
            self.quats = np.vstack([self.quats, np.array([[1.0, 0.0, 0.0, 0.0]])])
        self.source_frames = np.append(self.source_frames, np.uint32(g.source_frame))
        self.touch()

    def get(self, i: int) -> SemanticGaussian:
        return SemanticGaussian(self.centers[i].copy(), float(self.log_radii[i]),
                                float(self.opacity_logits[i]), self.colors[i].copy(),
                                [int(v) for v in self.sem_indices[i]],
                                [float(v) for v in self.sem_probs[i]], int(self.source_frames[i]))

    def center(self, i: int) -> np.ndarray:
        return self.centers[i].copy()

    # SGMP v1 (gaussian_map.cpp:126-189): 24-byte header, then per record
    # 8 f32 (center, log_r, logit, color), u32 source frame, k u16 ids, k f32 probs.
    def _record_dtype(self):
        return np.dtype([("f", "<f4", (8,)), ("src", "<u4"), ("idx", "<u2", (self._k,)),
                         ("prob", "<f4", (self._k,))])

    def save(self, path: str) -> None:
        rec = np.zeros(self.size(), dtype=self._record_dtype())
        rec["f"][:, 0:3] = self.centers
        rec["f"][:, 3] = self.log_radii
        rec["f"][:, 4] = self.opacity_logits
        rec["f"][:, 5:8] = self.colors
        rec["src"] = self.source_frames
        rec["idx"] = self.sem_indices
        rec["prob"] = self.sem_probs
        with open(path, "wb") as f:
            f.write(struct.pack("<IIQII", _SGMP_MAGIC, _SGMP_VERSION, self.size(), self._k,
                                self._num_classes))
            f.write(rec.tobytes())

    @classmethod
    def load(cls, path: str) -> "GaussianMap":
        with open(path, "rb") as f:
            head = f.read(24)
            if len(head) < 24:
                raise RuntimeError("map: truncated file")
            magic, version, n, k, m = struct.unpack("<IIQII", head)
            if magic != _SGMP_MAGIC:
                raise RuntimeError("map: bad magic")
            if version != _SGMP_VERSION:
                raise RuntimeError("map: bad version")
            out = cls(k, m)
            rec = np.frombuffer(f.read(), dtype=out._record_dtype())
        if rec.shape[0] < n:
            raise RuntimeError("map: truncated file")
        rec = rec[:n]
        f8 = rec["f"].astype(np.float64)  # widen exactly, as GaussianMap::load does
        return cls.from_arrays(k, m, f8[:, 0:3], f8[:, 3], f8[:, 4], f8[:, 5:8], rec["idx"],
                               rec["prob"].astype(np.float64), rec["src"])


# --------------------------------------------------------------------------- render types

@dataclass
class RenderChannels:
    color: bool = True
    depth: bool = True
    semantics: bool = True
    retain_contributors: bool = False

    @staticmethod
    def all(retain: bool = False) -> "RenderChannels":
        return RenderChannels(True, True, True, retain)

    @staticmethod
    def scoring() -> "RenderChannels":
        return RenderChannels(False, False, True, False)

    def flags(self) -> int:
        return ((N.SGM_COLOR if self.color else 0) | (N.SGM_DEPTH if self.depth else 0)
                | (N.SGM_SEMANTICS if self.semantics else 0)
                | (N.SGM_RETAIN_CONTRIBUTORS if self.retain_contributors else 0))


@dataclass
class RenderOptions:
    early_exit: bool = True
    transmittance_eps: float = 1e-4
    z_near: float = 0.01
    truncation_sigmas: float = 3.0
    tile_size: int = 8

    def _c(self) -> N.sgm_options:
        return N.sgm_options(1 if self.early_exit else 0, float(self.transmittance_eps),
                             float(self.z_near), float(self.truncation_sigmas),
                             int(self.tile_size))


K_MAX_FOOTPRINT = 0.999999  # splat_render.hpp:41

PROJECTION_DTYPE = np.dtype([("mx", "<f8"), ("my", "<f8"), ("rad_px", "<f8"), ("z", "<f8"),
                             ("alpha", "<f8"), ("index", "<u4"), ("reserved", "<u4")])


@dataclass
class RenderOutput:
    """splat_render.hpp:45-65. Planes are flat fp64 arrays in the reference layout."""

    width: int = 0
    height: int = 0
    channels: int = 0
    proj_fx: float = 0.0
    proj_fy: float = 0.0
    proj_cx: float = 0.0
    proj_cy: float = 0.0
    color: np.ndarray = field(default_factory=lambda: np.zeros(0))
    depth: np.ndarray = field(default_factory=lambda: np.zeros(0))
    silhouette: np.ndarray = field(default_factory=lambda: np.zeros(0))
    sem: np.ndarray = field(default_factory=lambda: np.zeros(0))
    projections: np.ndarray = field(default_factory=lambda: np.zeros(0, PROJECTION_DTYPE))
    contrib: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    contrib_offset: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))

    def pixel_count(self) -> int:
        return self.width * self.height

    def silhouette_at(self, x: int, y: int) -> float:
        return float(self.silhouette[y * self.width + x])

    def depth_at(self, x: int, y: int) -> float:
        return float(self.depth[y * self.width + x])

    def color_at(self, x: int, y: int) -> np.ndarray:
        i = (y * self.width + x) * 3
        return self.color[i:i + 3]

    def sem_at(self, x: int, y: int) -> np.ndarray:
        i = (y * self.width + x) * self.channels
        return self.sem[i:i + self.channels]


# --------------------------------------------------------------------------- device context

class Context:
    """One per GPU (sgm_ctx). Caches the device snapshot of each live map."""

    _defaults: dict = {}
    _lock = threading.Lock()

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        code = N.lib.sgm_ctx_create(int(device), C.byref(h))
        N.check(code, None)
        self.handle = h
        self.device = device
        self._maps: dict = {}

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        with cls._lock:
            ctx = cls._defaults.get(device)
            if ctx is None:
                ctx = cls._defaults[device] = Context(device)
            return ctx

    def close(self) -> None:
        if self.handle:
            for _, ent in list(self._maps.items()):
                N.lib.sgm_map_release(self.handle, ent[2])
            self._maps.clear()
            N.lib.sgm_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, code: int) -> None:
        N.check(code, self.handle)

    @property
    def stream(self) -> int:
        return N.lib.sgm_ctx_stream(self.handle) or 0

    def synchronize(self) -> None:
        self.check(N.lib.sgm_ctx_synchronize(self.handle))

    def set_profiling(self, on: bool) -> None:
        self.check(N.lib.sgm_ctx_set_profiling(self.handle, 1 if on else 0))

    def stats(self) -> dict:
        s = N.sgm_stats()
        self.check(N.lib.sgm_ctx_get_stats(self.handle, C.byref(s)))
        return {name: getattr(s, name) for name, _ in N.sgm_stats._fields_}

    def reset_stats(self) -> None:
        self.check(N.lib.sgm_ctx_reset_stats(self.handle))

    def upload(self, gmap: GaussianMap) -> C.c_void_p:
        """Device snapshot of `gmap`, re-uploaded when the map's version changes (a
        DeviceMap already is one)."""
        if isinstance(gmap, DeviceMap):
            if gmap.ctx is not self:
                raise ValueError("DeviceMap belongs to another Context")
            return gmap.handle
        key = id(gmap)
        hit = self._maps.get(key)
        if hit is not None:
            ref, ver, handle = hit[:3]
            if ref() is gmap and ver == gmap._version:
                return handle
            N.lib.sgm_map_release(self.handle, handle)
            del self._maps[key]
        handle, keep = self._upload_async(gmap)
        self._maps[key] = (weakref.ref(gmap, lambda _r, k=key: self._forget(k)), gmap._version,
                           handle, keep)
        return handle

    def _forget(self, key) -> None:
        try:
            hit = self._maps.pop(key, None)
            if hit is not None and self.handle:
                N.lib.sgm_map_release(self.handle, hit[2])
        except Exception:  # interpreter exit: module globals and builtins already torn down
            pass

    def _upload_async(self, gmap: GaussianMap):
        """sgm_map_upload_async: returns (handle, arrays the staging thread still reads). The
        compute call that follows in the same API function waits for the staging."""
        n = gmap.size()
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
                (gmap.centers, gmap.log_radii, gmap.opacity_logits, gmap.colors)]
        idx = np.ascontiguousarray(gmap.sem_indices, dtype=np.uint16)
        probs = np.ascontiguousarray(gmap.sem_probs, dtype=np.float64)
        h = C.c_void_p()
        upload = getattr(N.lib, "sgm_map_upload_async", None) or N.lib.sgm_map_upload
        self.check(upload(
            self.handle, n, gmap.k(), gmap.num_classes(), N.dptr(arrs[0]), N.dptr(arrs[1]),
            N.dptr(arrs[2]), N.dptr(arrs[3]), idx.ctypes.data_as(C.POINTER(C.c_uint16)),
            N.dptr(probs), C.byref(h)))
        if gmap.anisotropic():
            ls = np.ascontiguousarray(gmap.log_scales, dtype=np.float64)
            qs = np.ascontiguousarray(gmap.quats, dtype=np.float64)
            try:
                self.check(N.lib.sgm_map_set_anisotropic(self.handle, h, N.dptr(ls), N.dptr(qs)))
            except Exception:
                N.lib.sgm_map_release(self.handle, h)
                raise
        return h, (arrs, idx, probs)

    def upload_arrays(self, gmap: GaussianMap) -> C.c_void_p:
        n = gmap.size()
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
                (gmap.centers, gmap.log_radii, gmap.opacity_logits, gmap.colors)]
        idx = np.ascontiguousarray(gmap.sem_indices, dtype=np.uint16)
        probs = np.ascontiguousarray(gmap.sem_probs, dtype=np.float64)
        h = C.c_void_p()
        self.check(N.lib.sgm_map_upload(
            self.handle, n, gmap.k(), gmap.num_classes(), N.dptr(arrs[0]), N.dptr(arrs[1]),
            N.dptr(arrs[2]), N.dptr(arrs[3]), idx.ctypes.data_as(C.POINTER(C.c_uint16)),
            N.dptr(probs), C.byref(h)))
        if gmap.anisotropic():
            ls = np.ascontiguousarray(gmap.log_scales, dtype=np.float64)
            qs = np.ascontiguousarray(gmap.quats, dtype=np.float64)
            try:
                self.check(N.lib.sgm_map_set_anisotropic(self.handle, h, N.dptr(ls), N.dptr(qs)))
            except Exception:
                N.lib.sgm_map_release(self.handle, h)
                raise
        return h

    def release(self, handle) -> None:
        N.lib.sgm_map_release(self.handle, handle)

    # ---- device snapshot interchange (the map broadcast)
    def export_bytes(self, gmap) -> int:
        b = C.c_uint64()
        self.check(N.lib.sgm_map_export_bytes(self.handle, self.upload(gmap), C.byref(b)))
        return b.value

    def export_map(self, gmap, d_blob: int, capacity: int) -> None:
        """Packs `gmap`'s device snapshot into device memory at d_blob (this ctx's device)."""
        self.check(N.lib.sgm_map_export(self.handle, self.upload(gmap), C.c_void_p(d_blob),
                                        int(capacity)))

    def import_map(self, d_blob: int, nbytes: int) -> "DeviceMap":
        """A map from a snapshot blob in device memory (e.g. received by ncclBroadcast)."""
        h = C.c_void_p()
        self.check(N.lib.sgm_map_import(self.handle, C.c_void_p(d_blob), int(nbytes), C.byref(h)))
        return DeviceMap(self, h)


class DeviceMap:
    """A map that exists only as a device snapshot on one Context (sgm_map_import): accepted
    wherever a GaussianMap is (render, score_poses, fisher_prior, ...). Released with it."""

    def __init__(self, ctx: Context, handle: C.c_void_p):
        self.ctx, self.handle = ctx, handle
        n, k, m, a = C.c_uint64(), C.c_int32(), C.c_int32(), C.c_int32()
        ctx.check(N.lib.sgm_map_info(ctx.handle, handle, C.byref(n), C.byref(k), C.byref(m),
                                     C.byref(a)))
        self._n, self._k, self._num_classes, self._aniso = n.value, k.value, m.value, bool(a.value)

    def size(self) -> int:
        return self._n

    def k(self) -> int:
        return self._k

    def num_classes(self) -> int:
        return self._num_classes

    def channels(self) -> int:
        return self._num_classes + 1

    def anisotropic(self) -> bool:
        return self._aniso

    def empty(self) -> bool:
        return self._n == 0

    def __del__(self):
        try:
            if self.handle and self.ctx.handle:
                N.lib.sgm_map_release(self.ctx.handle, self.handle)
        except Exception:
            pass
        self.handle = None


class MultiContext:
    """Several GPUs driven from one process (sgm_multi): one Context per device,
    the map uploaded once and replicated device to device, candidate views sharded over the
    devices. score_poses / refresh_candidate_scores accept it as `ctx`; per-view results are
    bit-identical to a single Context. devices=None: every visible device."""

    def __init__(self, devices: Optional[Sequence[int]] = None):
        h = C.c_void_p()
        if devices is None:
            code = N.lib.sgm_multi_create(0, None, C.byref(h))
        else:
            arr = (C.c_int32 * len(devices))(*[int(d) for d in devices])
            code = N.lib.sgm_multi_create(len(devices), arr, C.byref(h))
        N.check(code, None)
        self.handle = h
        self._maps: dict = {}

    def device_count(self) -> int:
        return int(N.lib.sgm_multi_device_count(self.handle))

    def check(self, code: int) -> None:
        if code != N.SGM_OK:
            msg = N.lib.sgm_multi_last_error(self.handle)
            raise N.SgmError(code, msg.decode() if msg else "")

    def upload(self, gmap: GaussianMap):
        key = id(gmap)
        hit = self._maps.get(key)
        if hit is not None:
            ref, ver, handle = hit
            if ref() is gmap and ver == gmap._version:
                return handle
            N.lib.sgm_multi_map_release(self.handle, handle)
            del self._maps[key]
        if gmap.anisotropic():
            raise ValueError("MultiContext: anisotropic maps are scored per Context")
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
                (gmap.centers, gmap.log_radii, gmap.opacity_logits, gmap.colors)]
        idx = np.ascontiguousarray(gmap.sem_indices, dtype=np.uint16)
        probs = np.ascontiguousarray(gmap.sem_probs, dtype=np.float64)
        h = C.c_void_p()
        self.check(N.lib.sgm_multi_map_upload(
            self.handle, gmap.size(), gmap.k(), gmap.num_classes(), N.dptr(arrs[0]),
            N.dptr(arrs[1]), N.dptr(arrs[2]), N.dptr(arrs[3]),
            idx.ctypes.data_as(C.POINTER(C.c_uint16)), N.dptr(probs), C.byref(h)))
        self._maps[key] = (weakref.ref(gmap), gmap._version, h)
        return h

    def close(self) -> None:
        if self.handle:
            for _, (_, _, m) in list(self._maps.items()):
                N.lib.sgm_multi_map_release(self.handle, m)
            self._maps.clear()
            N.lib.sgm_multi_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _ctx(ctx: Optional[Context]) -> Context:
    return ctx if ctx is not None else Context.default()


# --------------------------------------------------------------------------- render API

def render(gmap: GaussianMap, camera: CameraModel, pose: Pose,
           channels: Optional[RenderChannels] = None, options: Optional[RenderOptions] = None,
           ctx: Optional[Context] = None) -> RenderOutput:
    """Tiled front-to-back compositor (splat_render.hpp:78-80) on the GPU."""
    return _render(gmap, camera, pose, channels, options, ctx, reference_form=False)


def _render(gmap, camera, pose, channels, options, ctx, reference_form: bool) -> RenderOutput:
    ch = channels if channels is not None else RenderChannels()
    opt = options if options is not None else RenderOptions()
    c = _ctx(ctx)
    handle = c.upload(gmap)
    px = camera.pixel_count()
    Cn = gmap.channels()
    out = RenderOutput(camera.width, camera.height, Cn if ch.semantics else 0, camera.fx,
                       camera.fy, camera.cx, camera.cy)
    out.silhouette = np.empty(px)
    out.color = np.empty(px * 3) if ch.color else np.zeros(0)
    out.depth = np.empty(px) if ch.depth else np.zeros(0)
    out.sem = np.empty(px * Cn) if ch.semantics else np.zeros(0)
    nproj = C.c_uint64()
    cam_c, pose_c, opt_c = camera._c(), pose._c(), opt._c()
    planes = (N.dptr(out.color) if ch.color else None, N.dptr(out.depth) if ch.depth else None,
              N.dptr(out.silhouette), N.dptr(out.sem) if ch.semantics else None, C.byref(nproj))
    if reference_form:
        c.check(N.lib.sgm_render_reference(c.handle, handle, C.byref(cam_c), C.byref(pose_c),
                                           ch.flags(), *planes))
    else:
        c.check(N.lib.sgm_render(c.handle, handle, C.byref(cam_c), C.byref(pose_c), ch.flags(),
                                 C.byref(opt_c), *planes))
    proj = np.zeros(nproj.value, dtype=PROJECTION_DTYPE)
    if nproj.value:
        c.check(N.lib.sgm_last_projections(
            c.handle, proj.ctypes.data_as(C.POINTER(N.sgm_projection)), nproj.value))
    out.projections = proj
    if ch.retain_contributors:  # RenderOutput.contrib / contrib_offset (:125-137)
        ncon = C.c_uint64()
        c.check(N.lib.sgm_last_contributors(c.handle, None, None, 0, C.byref(ncon)))
        out.contrib_offset = np.zeros(px + 1, dtype=np.uint32)
        con = np.zeros(max(ncon.value, 1), dtype=np.uint32)
        c.check(N.lib.sgm_last_contributors(
            c.handle, out.contrib_offset.ctypes.data_as(C.POINTER(C.c_uint32)),
            con.ctypes.data_as(C.POINTER(C.c_uint32)), ncon.value, C.byref(ncon)))
        out.contrib = con[:ncon.value]
    return out


def render_device(gmap: GaussianMap, camera: CameraModel, pose: Pose, channels: RenderChannels,
                  options: Optional[RenderOptions] = None, ctx: Optional[Context] = None, *,
                  color_ptr: int = 0, depth_ptr: int = 0, sil_ptr: int = 0,
                  sem_ptr: int = 0) -> int:
    """render() into caller-owned DEVICE planes (reference layout, fp64), on the ctx stream
    (sgm_render_device). Returns the number of projections."""
    c = _ctx(ctx)
    handle = c.upload(gmap)
    nproj = C.c_uint64()
    opt = (options if options is not None else RenderOptions())._c()
    cam_c, pose_c = camera._c(), pose._c()
    c.check(N.lib.sgm_render_device(c.handle, handle, C.byref(cam_c), C.byref(pose_c),
                                    channels.flags(), C.byref(opt), color_ptr or None,
                                    depth_ptr or None, sil_ptr or None, sem_ptr or None,
                                    C.byref(nproj)))
    return nproj.value


def bins_of_last_render(tiles: int, ctx: Optional[Context] = None):
    """The tile bins the last render() on `ctx` built at RenderOptions::tile_size
    (bit-exactness hook; splat_render.cpp:188-213 keeps them local):
    (tile_offsets[tiles+1], ids[P] projection ids in bin order, probe3[P,3] f32)."""
    c = _ctx(ctx)
    npairs = C.c_uint64()
    c.check(N.lib.sgm_last_bins(c.handle, None, None, None, 0, C.byref(npairs)))
    P = npairs.value
    offsets = np.zeros(tiles + 1, dtype=np.uint32)
    ids = np.zeros(max(P, 1), dtype=np.uint32)
    probe = np.zeros((max(P, 1), 3), dtype=np.float32)
    c.check(N.lib.sgm_last_bins(c.handle, offsets.ctypes.data_as(C.POINTER(C.c_uint32)),
                                ids.ctypes.data_as(C.POINTER(C.c_uint32)),
                                probe.ctypes.data_as(C.POINTER(C.c_float)), P, C.byref(npairs)))
    return offsets, ids[:P], probe[:P]


def render_reference(gmap: GaussianMap, camera: CameraModel, pose: Pose,
                     channels: Optional[RenderChannels] = None,
                     ctx: Optional[Context] = None) -> RenderOutput:
    """splat_render.hpp:82-86 / splat_render.cpp:330-358: every projection composited in depth
    order with no early exit, with composite_pixel's footprint form (:86-92):
    f = min(alpha exp(-d2 / (2 r^2)), kMaxFootprint), f <= 0 skipped (so alpha == 0 splats
    are not listed as contributors). On the GPU: the tiled compositor with that footprint
    (sgm_render_reference); each pixel's depth-ordered candidate set is the same, since the
    tile rectangles and the float probe (:276-278) only drop splats the exact test rejects."""
    return _render(gmap, camera, pose, channels, RenderOptions(early_exit=False), ctx,
                   reference_form=True)


def clipped_entropy(probs) -> float:
    """splat_render.cpp:360-369 (host, one pixel)."""
    p = np.ascontiguousarray(probs, dtype=np.float64)
    return float(N.lib.sgm_clipped_entropy(N.dptr(p), p.size))


def render_entropy(gmap: GaussianMap, camera: CameraModel, pose: Pose,
                   options: Optional[RenderOptions] = None,
                   ctx: Optional[Context] = None) -> np.ndarray:
    """splat_render.cpp:378-390: per-pixel clipped entropy of the sem render."""
    c = _ctx(ctx)
    handle = c.upload(gmap)
    out = np.empty(camera.pixel_count())
    opt = (options if options is not None else RenderOptions())._c()
    cam_c, pose_c = camera._c(), pose._c()
    c.check(N.lib.sgm_render_entropy(c.handle, handle, C.byref(cam_c), C.byref(pose_c),
                                     C.byref(opt), N.dptr(out)))
    return out


# --------------------------------------------------------------------------- scoring API

class CandidateState(enum.Enum):
    Active = 0
    Pruned = 1
    Visited = 2


@dataclass
class CandidatePose:
    """explorer.hpp:93-106."""

    position: np.ndarray = field(default_factory=lambda: np.zeros(3))
    direction: np.ndarray = field(default_factory=lambda: np.array([1.0, 0.0, 0.0]))
    state: CandidateState = CandidateState.Active
    n_missing: float = 0.0
    entropy_sum: float = 0.0
    i_geo: float = 0.0
    i_sem: float = 0.0
    i_total: float = 0.0
    id: int = -1
    # Fisher extension (not in the reference): the view's FisherRF gain, the
    # combined scalar gain (fisher_gain + w_sem * entropy_sum) and its ranking criterion
    fisher_gain: float = 0.0
    gain: float = 0.0
    i_gain: float = 0.0

    State = CandidateState

    def camera_pose(self) -> Pose:
        out = N.sgm_pose()
        p = np.ascontiguousarray(self.position, dtype=np.float64)
        d = np.ascontiguousarray(self.direction, dtype=np.float64)
        N.lib.sgm_candidate_pose(N.dptr(p), N.dptr(d), C.byref(out))
        return Pose._from_c(out)


def score_poses(gmap: GaussianMap, camera: CameraModel, poses: Sequence[Pose],
                options: Optional[RenderOptions] = None, ctx: Optional[Context] = None):
    """Batched GPU scoring of explicit poses: (n_missing[n], entropy_sum[n]). With a
    MultiContext the views are sharded over its devices."""
    c = _ctx(ctx)
    handle = c.upload(gmap)
    n = len(poses)
    nm = np.zeros(n)
    es = np.zeros(n)
    if n == 0:
        return nm, es
    arr = (N.sgm_pose * n)(*[p._c() for p in poses])
    opt = (options if options is not None else RenderOptions())._c()
    cam_c = camera._c()
    fn = N.lib.sgm_multi_score_views if isinstance(c, MultiContext) else N.lib.sgm_score_views
    c.check(fn(c.handle, handle, C.byref(cam_c), n, arr, C.byref(opt), N.dptr(nm), N.dptr(es)))
    return nm, es


# --------------------------------------------------------------------------- mapping step

@dataclass
class Frame:
    """Posed RGB-D-semantic observation (frame.hpp:12-65): rgb (H*W*3), depth (H*W, 0 =
    invalid), sem (H*W*(num_classes+1)), all float32."""

    width: int
    height: int
    num_classes: int
    pose: Pose
    rgb: np.ndarray
    depth: np.ndarray
    sem: np.ndarray

    def channels(self) -> int:
        return self.num_classes + 1


@dataclass
class LossWeights:
    """losses.hpp:9-17."""

    lambda_hd: float = 0.8
    lambda_cos: float = 0.2
    mask_k: int = 16
    use_hd: bool = True
    use_cos: bool = True
    use_kl: bool = False
    kl_clip_norm: float = 1.0


@dataclass
class LossReport:
    """losses.hpp:19-31."""

    photometric: float = 0.0
    depth: float = 0.0
    semantic: float = 0.0
    photometric_px: int = 0
    depth_px: int = 0
    semantic_px: int = 0
    uncovered_px: int = 0

    def mapping_total(self) -> float:
        return self.depth + 0.5 * self.photometric

    def total(self) -> float:
        return self.mapping_total() + self.semantic


@dataclass
class ParamGradients:
    """losses.hpp:47-63 (arrays parallel to GaussianMap storage)."""

    center: np.ndarray
    log_radius: np.ndarray
    opacity_logit: np.ndarray
    color: np.ndarray
    sem: np.ndarray


def backward(gmap: GaussianMap, camera: CameraModel, frame: Frame,
             weights: Optional[LossWeights] = None, include_mapping: bool = True,
             include_semantic: bool = True, options: Optional[RenderOptions] = None,
             ctx: Optional[Context] = None):
    """One mapping step on the GPU: render(map, camera, frame.pose, all(true)), mapping_loss +
    semantic_loss, and the analytic backward (losses.cpp:40-362). Returns (LossReport,
    ParamGradients); raises like the reference on a non-finite gradient."""
    w = weights if weights is not None else LossWeights()
    c = _ctx(ctx)
    handle = c.upload(gmap)
    n, k = gmap.size(), gmap.k()
    wv = np.array([w.lambda_hd, w.lambda_cos, float(w.mask_k), float(w.use_hd),
                   float(w.use_cos), float(w.use_kl), w.kl_clip_norm])
    rep = np.zeros(7)
    g = ParamGradients(np.zeros(3 * n), np.zeros(n), np.zeros(n), np.zeros(3 * n), np.zeros(k * n))
    rgb = np.ascontiguousarray(frame.rgb, dtype=np.float32)
    dep = np.ascontiguousarray(frame.depth, dtype=np.float32)
    sem = np.ascontiguousarray(frame.sem, dtype=np.float32)
    pf = C.POINTER(C.c_float)
    opt = (options if options is not None else RenderOptions())._c()
    cam_c, pose_c = camera._c(), frame.pose._c()
    c.check(N.lib.sgm_backward(c.handle, handle, C.byref(cam_c), C.byref(pose_c), C.byref(opt),
                               rgb.ctypes.data_as(pf), dep.ctypes.data_as(pf),
                               sem.ctypes.data_as(pf), N.dptr(wv), int(include_mapping),
                               int(include_semantic), N.dptr(rep), N.dptr(g.center),
                               N.dptr(g.log_radius), N.dptr(g.opacity_logit), N.dptr(g.color),
                               N.dptr(g.sem)))
    report = LossReport(float(rep[0]), float(rep[1]), float(rep[2]), int(rep[3]), int(rep[4]),
                        int(rep[5]), int(rep[6]))
    return report, g


def fisher_prior(gmap: GaussianMap, camera: CameraModel, poses: Sequence[Pose],
                 lam: float = 1.0, options: Optional[RenderOptions] = None,
                 ctx: Optional[Context] = None) -> np.ndarray:
    """Fisher-information prior (extension): the diagonal Fisher information of
    the rendered colour and depth w.r.t. each Gaussian's (mu xyz, log_radius, opacity_logit,
    rgb), summed over `poses` (e.g. past keyframes). Kept with the map's device snapshot for
    score_poses_fisher; returns H as an (N, 8) array."""
    c = _ctx(ctx)
    handle = c.upload(gmap)
    n = len(poses)
    H = np.zeros((max(gmap.size(), 1), 8))
    arr = (N.sgm_pose * max(n, 1))(*[p._c() for p in poses])
    opt = (options if options is not None else RenderOptions())._c()
    cam_c = camera._c()
    c.check(N.lib.sgm_fisher_prior(c.handle, handle, C.byref(cam_c), n, arr, C.byref(opt),
                                   float(lam), N.dptr(H)))
    return H[:gmap.size()]


def fisher_set_prior(gmap: GaussianMap, H: np.ndarray, lam: float = 1.0,
                     ctx: Optional[Context] = None) -> None:
    """Installs a Fisher prior given as an (N, 8) array (e.g. the all-reduced sum of per-rank
    fisher_prior results over sharded past poses, dist.fisher_prior_sharded)."""
    c = _ctx(ctx)
    handle = c.upload(gmap)
    Hc = np.ascontiguousarray(np.asarray(H, dtype=np.float64).reshape(gmap.size(), 8))
    c.check(N.lib.sgm_fisher_set_prior(c.handle, handle, N.dptr(Hc), float(lam)))


def score_poses_fisher(gmap: GaussianMap, camera: CameraModel, poses: Sequence[Pose],
                       options: Optional[RenderOptions] = None, ctx: Optional[Context] = None):
    """Per view (n_missing, entropy_sum, fisher_gain) with the FisherRF-style gain
    sum_{i,theta} H_view / (H_prior + lambda) against the map's fisher_prior."""
    c = _ctx(ctx)
    handle = c.upload(gmap)
    n = len(poses)
    nm, es, fg = np.zeros(n), np.zeros(n), np.zeros(n)
    if n == 0:
        return nm, es, fg
    arr = (N.sgm_pose * n)(*[p._c() for p in poses])
    opt = (options if options is not None else RenderOptions())._c()
    cam_c = camera._c()
    c.check(N.lib.sgm_score_views_fisher(c.handle, handle, C.byref(cam_c), n, arr, C.byref(opt),
                                         N.dptr(nm), N.dptr(es), N.dptr(fg)))
    return nm, es, fg


def refresh_candidate_scores(candidates: List[CandidatePose], gmap: GaussianMap,
                             scoring_camera: CameraModel, ctx: Optional[Context] = None) -> None:
    """explorer.cpp:186-205: caches n_missing and entropy_sum on every Active
    candidate; all active candidates are scored in one batched GPU call."""
    active = [cd for cd in candidates if cd.state == CandidateState.Active]
    if not active:
        return
    c = _ctx(ctx)
    handle = c.upload(gmap)
    n = len(active)
    arr = (N.sgm_candidate * n)()
    for i, cd in enumerate(active):
        for a in range(3):
            arr[i].position[a] = float(cd.position[a])
            arr[i].direction[a] = float(cd.direction[a])
    nm = np.zeros(n)
    es = np.zeros(n)
    opt = RenderOptions()._c()
    cam_c = scoring_camera._c()
    fn = (N.lib.sgm_multi_score_candidates if isinstance(c, MultiContext)
          else N.lib.sgm_score_candidates)
    c.check(fn(c.handle, handle, C.byref(cam_c), n, arr, C.byref(opt), N.dptr(nm), N.dptr(es)))
    for i, cd in enumerate(active):
        cd.n_missing = float(nm[i])
        cd.entropy_sum = float(es[i])


def combine_scores(candidates: List[CandidatePose], current_position) -> bool:
    """explorer.cpp:225-248 (host fp64, bit-identical restatement)."""
    n = len(candidates)
    if n == 0:
        return False
    nm = np.array([cd.n_missing for cd in candidates], dtype=np.float64)
    es = np.array([cd.entropy_sum for cd in candidates], dtype=np.float64)
    pos = np.ascontiguousarray([np.asarray(cd.position, dtype=np.float64) for cd in candidates])
    cur = np.ascontiguousarray(current_position, dtype=np.float64)
    geo, sem, tot = np.zeros(n), np.zeros(n), np.zeros(n)
    rc = N.lib.sgm_combine_scores(n, N.dptr(nm), N.dptr(es), N.dptr(pos), N.dptr(cur),
                                  N.dptr(geo), N.dptr(sem), N.dptr(tot))
    if rc < 0:
        raise ValueError("combine_scores: invalid arguments")
    for i, cd in enumerate(candidates):
        cd.i_geo, cd.i_sem, cd.i_total = float(geo[i]), float(sem[i]), float(tot[i])
    return rc == 1


def refresh_candidate_scores_fisher(candidates: List[CandidatePose], gmap: GaussianMap,
                                    scoring_camera: CameraModel,
                                    ctx: Optional[Context] = None) -> None:
    """refresh_candidate_scores plus the Fisher extension: caches n_missing, entropy_sum and
    fisher_gain (against the map's fisher_prior) on every Active candidate, in one batched
    GPU call (sgm_score_views_fisher)."""
    active = [cd for cd in candidates if cd.state == CandidateState.Active]
    if not active:
        return
    nm, es, fg = score_poses_fisher(gmap, scoring_camera, [cd.camera_pose() for cd in active],
                                    ctx=ctx)
    for i, cd in enumerate(active):
        cd.n_missing, cd.entropy_sum, cd.fisher_gain = float(nm[i]), float(es[i]), float(fg[i])


def combine_scores_fisher(candidates: List[CandidatePose], current_position,
                          w_sem: float = 1.0) -> bool:
    """The Fisher extension's scalar gain and ranking criterion (sgm_combine_scores_fisher):
    gain = fisher_gain + w_sem * entropy_sum; i_gain = (1 - softmax(distance)) *
    softmax(ln gain), the slot of combine_scores (explorer.cpp:225-248). Returns whether any
    i_gain > 0."""
    n = len(candidates)
    if n == 0:
        return False
    fg = np.array([cd.fisher_gain for cd in candidates], dtype=np.float64)
    es = np.array([cd.entropy_sum for cd in candidates], dtype=np.float64)
    pos = np.ascontiguousarray([np.asarray(cd.position, dtype=np.float64) for cd in candidates])
    cur = np.ascontiguousarray(current_position, dtype=np.float64)
    gain, tot = np.zeros(n), np.zeros(n)
    rc = N.lib.sgm_combine_scores_fisher(n, N.dptr(fg), N.dptr(es), N.dptr(pos), N.dptr(cur),
                                         float(w_sem), N.dptr(gain), N.dptr(tot))
    if rc < 0:
        raise ValueError("combine_scores_fisher: invalid arguments")
    for i, cd in enumerate(candidates):
        cd.gain, cd.i_gain = float(gain[i]), float(tot[i])
    return rc == 1


def score_candidates_fisher(candidates: List[CandidatePose], gmap: GaussianMap,
                            scoring_camera: CameraModel, current_position, w_sem: float = 1.0,
                            ctx: Optional[Context] = None) -> bool:
    """score_candidates (explorer.cpp:250-259) with the Fisher extension's gain: refresh,
    combine_scores_fisher, then sort by i_gain descending, id ascending."""
    refresh_candidate_scores_fisher(candidates, gmap, scoring_camera, ctx)
    any_pos = combine_scores_fisher(candidates, current_position, w_sem)
    candidates.sort(key=lambda cd: (-cd.i_gain, cd.id))
    return any_pos


def score_candidates(candidates: List[CandidatePose], gmap: GaussianMap,
                     scoring_camera: CameraModel, current_position,
                     ctx: Optional[Context] = None) -> bool:
    """explorer.cpp:250-259: refresh + combine + sort by i_total desc, id asc."""
    refresh_candidate_scores(candidates, gmap, scoring_camera, ctx)
    any_pos = combine_scores(candidates, current_position)
    candidates.sort(key=lambda cd: (-cd.i_total, cd.id))
    return any_pos


def prune_pool(candidates: List[CandidatePose], scoring_camera: CameraModel) -> List[CandidatePose]:
    """explorer.cpp:261-272."""
    threshold = 0.005 * scoring_camera.width * scoring_camera.height
    return [cd for cd in candidates
            if cd.state != CandidateState.Visited and not (cd.n_missing < threshold)]


class CandidatePool:
    """explorer.hpp:134-148 / explorer.cpp:274-292."""

    def __init__(self):
        self._active: List[CandidatePose] = []
        self._visited: set = set()
        self._next_id = 0

    def absorb(self, fresh: List[CandidatePose]) -> None:
        for cd in fresh:
            cd.id = self._next_id
            self._next_id += 1
            cd.state = CandidateState.Active
            self._active.append(cd)

    def active(self) -> List[CandidatePose]:
        return self._active

    def mark_visited(self, cid: int) -> None:
        self._visited.add(cid)
        for cd in self._active:
            if cd.id == cid:
                cd.state = CandidateState.Visited

    def prune(self, scoring_camera: CameraModel) -> int:
        before = len(self._active)
        self._active = prune_pool(self._active, scoring_camera)
        return before - len(self._active)

    def ever_visited(self, cid: int) -> bool:
        return cid in self._visited

    def visited_count(self) -> int:
        return len(self._visited)
