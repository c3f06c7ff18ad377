"""Exploration map and candidate sampling on the GPU.

Mirrors proj/include/splatmap/explorer.hpp:11-112 and proj/src/explorer.cpp:11-184:
`ExplorationMap` (integrate_frame, changelog, seeding), `fibonacci_directions`,
`SamplingSchedule` and `sample_candidates`. The voxel grid and changelog live in HBM
(`sgm_emap`); the depth walk is the kernel `k_emap_rays` (sgm_emap.cu). Results are
bit-identical to the reference: voxel states, counts and changelog order.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N
from .splatmap import CameraModel, CandidatePose, Context, Pose, _ctx


class VoxelState(enum.IntEnum):
    """explorer.hpp:11."""

    Unknown = 0
    Free = 1
    Occupied = 2


@dataclass
class Aabb:
    """geometry.hpp:58-67."""

    min: np.ndarray = field(default_factory=lambda: np.zeros(3))
    max: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def extent(self) -> np.ndarray:
        return np.asarray(self.max, dtype=np.float64) - np.asarray(self.min, dtype=np.float64)

    def contains(self, p) -> bool:
        p = np.asarray(p, dtype=np.float64)
        return bool(np.all(p >= self.min) and np.all(p <= self.max))

    def _c(self) -> N.sgm_aabb:
        b = N.sgm_aabb()
        for a in range(3):
            b.min[a] = float(self.min[a])
            b.max[a] = float(self.max[a])
        return b


class ExplorationMap:
    """Dense occupancy grid over the scene envelope (explorer.hpp:14-83), device-resident."""

    def __init__(self, bounds: Aabb, voxel_size: float = 0.05, ctx: Optional[Context] = None):
        self._ctx = _ctx(ctx)
        h = C.c_void_p()
        b = bounds._c()
        self._ctx.check(N.lib.sgm_emap_create(self._ctx.handle, C.byref(b), float(voxel_size),
                                              C.byref(h)))
        self.handle = h
        origin = np.zeros(3)
        vox = C.c_double()
        dims = np.zeros(3, np.int32)
        self._ctx.check(N.lib.sgm_emap_info(self._ctx.handle, h, N.dptr(origin), C.byref(vox),
                                            dims.ctypes.data_as(N._pi32), None, None, None))
        self._origin, self._voxel, self._dims = origin, float(vox.value), tuple(int(d) for d in dims)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            N.lib.sgm_emap_destroy(self._ctx.handle, h)
            self.handle = None

    # geometry (explorer.hpp:18-40)
    def voxel_size(self) -> float:
        return self._voxel

    def origin(self) -> np.ndarray:
        return self._origin.copy()

    def dims(self) -> tuple:
        return self._dims

    def voxel_count(self) -> int:
        return self._dims[0] * self._dims[1] * self._dims[2]

    def linear_index(self, ix: int, iy: int, iz: int) -> int:
        return (iz * self._dims[1] + iy) * self._dims[0] + ix

    def voxel_at(self, p) -> int:
        """explorer.cpp:22-29 (host arithmetic, same fp64 ops)."""
        idx = [int(np.floor((float(p[a]) - self._origin[a]) / self._voxel)) for a in range(3)]
        if not all(0 <= idx[a] < self._dims[a] for a in range(3)):
            return -1
        return self.linear_index(*idx)

    def voxel_center(self, i: int) -> np.ndarray:
        """explorer.cpp:31-36."""
        d = self._dims
        ijk = (i % d[0], (i // d[0]) % d[1], i // (d[0] * d[1]))
        return np.array([self._origin[a] + self._voxel * (ijk[a] + 0.5) for a in range(3)])

    def _info(self):
        f, o, n = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self._ctx.check(N.lib.sgm_emap_info(self._ctx.handle, self.handle, None, None, None,
                                            C.byref(f), C.byref(o), C.byref(n)))
        return int(f.value), int(o.value), int(n.value)

    def free_count(self) -> int:
        return self._info()[0]

    def occupied_count(self) -> int:
        return self._info()[1]

    def changelog_size(self) -> int:
        return self._info()[2]

    def grid(self) -> np.ndarray:
        """States as uint8 (VoxelState values), linear id order."""
        out = np.zeros(self.voxel_count(), np.uint8)
        self._ctx.check(N.lib.sgm_emap_grid(self._ctx.handle, self.handle,
                                            out.ctypes.data_as(N._pu8), out.size))
        return out

    def state(self, i: int) -> VoxelState:
        return VoxelState(int(self.grid()[i]))

    def state_at(self, p) -> VoxelState:
        """explorer.hpp:36-39: outside the grid reads as occupied."""
        i = self.voxel_at(p)
        return VoxelState.Occupied if i < 0 else self.state(i)

    def integrate_frame(self, depth, camera: CameraModel, pose: Pose, stride: int = 2) -> int:
        """integrate_frame (explorer.cpp:53-110). `depth` is the frame's H*W float plane
        (numpy on the host, or a CUDA torch tensor already in HBM). Returns the number of
        newly freed voxels."""
        cam, p = camera._c(), pose._c()
        n = C.c_uint64()
        if hasattr(depth, "data_ptr") and getattr(depth, "is_cuda", False):
            if depth.numel() < camera.width * camera.height:
                raise ValueError("depth plane smaller than the camera")
            self._ctx.check(N.lib.sgm_emap_integrate_device(
                self._ctx.handle, self.handle, C.byref(cam), C.byref(p),
                C.c_void_p(depth.data_ptr()), int(stride), C.byref(n)))
        else:
            d = np.ascontiguousarray(depth, dtype=np.float32).reshape(-1)
            if d.size < camera.width * camera.height:
                raise ValueError("depth plane smaller than the camera")
            self._ctx.check(N.lib.sgm_emap_integrate(
                self._ctx.handle, self.handle, C.byref(cam), C.byref(p),
                d.ctypes.data_as(N._pf), int(stride), C.byref(n)))
        return int(n.value)

    def take_changelog(self) -> np.ndarray:
        """explorer.cpp:112-116."""
        n = self.changelog_size()
        out = np.zeros(max(n, 1), np.int32)
        got = C.c_uint64()
        self._ctx.check(N.lib.sgm_emap_take_changelog(self._ctx.handle, self.handle,
                                                      out.ctypes.data_as(N._pi32), out.size,
                                                      C.byref(got)))
        return out[: int(got.value)].copy()

    def reseed_changelog_with_free(self) -> None:
        self._ctx.check(N.lib.sgm_emap_reseed_changelog_with_free(self._ctx.handle, self.handle))

    def seed_free_region(self, box: Aabb) -> None:
        b = box._c()
        self._ctx.check(N.lib.sgm_emap_seed_region(self._ctx.handle, self.handle, C.byref(b), 0))

    def seed_occupied_region(self, box: Aabb) -> None:
        b = box._c()
        self._ctx.check(N.lib.sgm_emap_seed_region(self._ctx.handle, self.handle, C.byref(b), 1))


def fibonacci_directions(count: int, max_elevation_deg: float = 45.0) -> np.ndarray:
    """explorer.cpp:142-155: (count, 3) unit directions, Y up."""
    out = np.zeros((max(int(count), 0), 3))
    if count > 0:
        N.lib.sgm_fibonacci_directions(int(count), float(max_elevation_deg), N.dptr(out))
    return out


@dataclass
class SamplingSchedule:
    """explorer.hpp:85-93."""

    class Stage(enum.Enum):
        Coarse = 0
        Fine = 1

    stage: "SamplingSchedule.Stage" = None  # type: ignore[assignment]
    v1: float = 1.0
    v2: int = 5
    heights: Sequence[float] = (1.4,)

    def __post_init__(self):
        if self.stage is None:
            self.stage = SamplingSchedule.Stage.Coarse

    @staticmethod
    def coarse() -> "SamplingSchedule":
        return SamplingSchedule(SamplingSchedule.Stage.Coarse, 1.0, 5, (1.4,))

    @staticmethod
    def fine() -> "SamplingSchedule":
        return SamplingSchedule(SamplingSchedule.Stage.Fine, 0.5, 15, (0.8, 1.4))


def sample_candidates_arrays(emap: ExplorationMap, schedule: SamplingSchedule):
    """sample_candidates as (positions (n,3), directions (n,3)); consumes the changelog."""
    h = np.ascontiguousarray(schedule.heights, dtype=np.float64)
    c = emap._ctx
    need = C.c_uint64()
    hp = N.dptr(h) if h.size else None
    code = N.lib.sgm_sample_candidates(c.handle, emap.handle, float(schedule.v1),
                                       int(schedule.v2), hp, int(h.size), None, 0,
                                       C.byref(need))
    if code == N.SGM_OK:  # nothing sampled (changelog consumed) or nothing logged
        return np.zeros((0, 3)), np.zeros((0, 3))
    n = int(need.value)
    if n == 0:
        c.check(code)
    out = (N.sgm_candidate * max(n, 1))()
    got = C.c_uint64()
    c.check(N.lib.sgm_sample_candidates(c.handle, emap.handle, float(schedule.v1),
                                        int(schedule.v2), hp, int(h.size), out, n, C.byref(got)))
    arr = np.ctypeslib.as_array(C.cast(out, C.POINTER(C.c_double)), shape=(max(n, 1), 6))
    arr = arr[: int(got.value)].copy()
    return arr[:, :3].copy(), arr[:, 3:].copy()


def sample_candidates(emap: ExplorationMap, schedule: SamplingSchedule) -> List[CandidatePose]:
    """explorer.cpp:157-184: lattice positions inside freshly freed voxels at the schedule
    heights, each fanned into v2 fibonacci directions. Consumes the changelog."""
    pos, dirs = sample_candidates_arrays(emap, schedule)
    return [CandidatePose(position=pos[i].copy(), direction=dirs[i].copy())
            for i in range(len(pos))]
