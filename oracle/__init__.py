"""ctypes bindings for the CPU checkers. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
import this package. Two libraries:

  Oracle  -> oracle/_build/libsgm_oracle.so : the C restatement (sgm_oracle.c),
             always buildable (gcc).
  RefLib  -> oracle/_ref/libsgm_ref.so      : the reference's own TUs compiled
             unmodified from /root/reference with from-scratch shims
             (oracle/Makefile). Built here; the prebuilt .so travels to the GPU box.

Both take maps duck-typed like paper_2506_00225_b200.GaussianMap (centers,
log_radii, opacity_logits, colors, sem_indices, sem_probs arrays; k(),
num_classes()). Cameras/poses/options likewise (fields width, height, fx, fy,
cx, cy; R, t; early_exit, transmittance_eps, z_near, truncation_sigmas,
tile_size).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "libsgm_oracle.so"
REF_SO = HERE / "_ref" / "libsgm_ref.so"

_pd = C.POINTER(C.c_double)
_pu16 = C.POINTER(C.c_uint16)
_pu32 = C.POINTER(C.c_uint32)
_pu64 = C.POINTER(C.c_uint64)
_pf = C.POINTER(C.c_float)
_pi32 = C.POINTER(C.c_int32)


def _dp(a):
    return None if a is None else a.ctypes.data_as(_pd)


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def build_ref() -> bool:
    """Builds oracle/_ref from /root/reference when it is present (this container)."""
    if not Path("/root/reference/proj/src/splat_render.cpp").exists():
        return REF_SO.exists()
    subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)
    return True


class orc_camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_double),
                ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double)]


class orc_pose(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("t", C.c_double * 3)]


class orc_options(C.Structure):
    _fields_ = [("early_exit", C.c_int32), ("transmittance_eps", C.c_double),
                ("z_near", C.c_double), ("truncation_sigmas", C.c_double),
                ("tile_size", C.c_int32)]


class orc_map(C.Structure):
    _fields_ = [("n", C.c_uint64), ("k", C.c_int32), ("num_classes", C.c_int32),
                ("centers", _pd), ("log_radii", _pd), ("opacity_logits", _pd),
                ("colors", _pd), ("sem_idx", _pu16), ("sem_probs", _pd),
                ("log_scales", _pd), ("quats", _pd)]


class orc_proj(C.Structure):
    _fields_ = [("mx", C.c_double), ("my", C.c_double), ("rad_px", C.c_double),
                ("z", C.c_double), ("alpha", C.c_double), ("index", C.c_uint32),
                ("rx", C.c_double), ("ry", C.c_double), ("qa", C.c_double), ("qb", C.c_double),
                ("qc", C.c_double)]


class orc_stats(C.Structure):
    _fields_ = [("visible", C.c_uint64), ("pairs", C.c_uint64), ("probe_tests", C.c_uint64),
                ("exact_tests", C.c_uint64), ("contributors", C.c_uint64)]


class orc_emap(C.Structure):
    _fields_ = [("origin", C.c_double * 3), ("voxel", C.c_double), ("dims", C.c_int32 * 3),
                ("nvox", C.c_uint64), ("grid", C.POINTER(C.c_uint8)), ("log", C.POINTER(C.c_int32)),
                ("log_n", C.c_uint64), ("free_count", C.c_uint64), ("occupied_count", C.c_uint64)]


PROJ_DTYPE = np.dtype([("mx", "<f8"), ("my", "<f8"), ("rad_px", "<f8"), ("z", "<f8"),
                       ("alpha", "<f8"), ("index", "<u4"), ("pad", "<u4"), ("rx", "<f8"),
                       ("ry", "<f8"), ("qa", "<f8"), ("qb", "<f8"), ("qc", "<f8")])


def _cam(cam) -> orc_camera:
    return orc_camera(int(cam.width), int(cam.height), float(cam.fx), float(cam.fy),
                      float(cam.cx), float(cam.cy))


def _pose(p) -> orc_pose:
    out = orc_pose()
    R = np.asarray(p.R, dtype=np.float64).reshape(9)
    for i in range(9):
        out.R[i] = float(R[i])
    for i in range(3):
        out.t[i] = float(p.t[i])
    return out


def _opts(o) -> orc_options:
    if o is None:
        return orc_options(1, 1e-4, 0.01, 3.0, 8)
    return orc_options(1 if o.early_exit else 0, float(o.transmittance_eps), float(o.z_near),
                       float(o.truncation_sigmas), int(o.tile_size))


class _MapArrays:
    """Keeps contiguous copies alive while a C call uses them."""

    def __init__(self, m):
        self.k = int(m.k())
        self.num_classes = int(m.num_classes())
        self.n = int(m.size())
        self.centers = np.ascontiguousarray(m.centers, dtype=np.float64)
        self.log_radii = np.ascontiguousarray(m.log_radii, dtype=np.float64)
        self.logits = np.ascontiguousarray(m.opacity_logits, dtype=np.float64)
        self.colors = np.ascontiguousarray(m.colors, dtype=np.float64)
        self.idx = np.ascontiguousarray(m.sem_indices, dtype=np.uint16)
        self.probs = np.ascontiguousarray(m.sem_probs, dtype=np.float64)
        # anisotropic mode: optional per-axis log-scales and quaternions
        ls, qs = getattr(m, "log_scales", None), getattr(m, "quats", None)
        self.log_scales = None if ls is None else np.ascontiguousarray(ls, dtype=np.float64)
        self.quats = None if qs is None else np.ascontiguousarray(qs, dtype=np.float64)

    def c(self) -> orc_map:
        return orc_map(self.n, self.k, self.num_classes, _dp(self.centers), _dp(self.log_radii),
                       _dp(self.logits), _dp(self.colors), self.idx.ctypes.data_as(_pu16),
                       _dp(self.probs), _dp(self.log_scales), _dp(self.quats))


class Oracle:
    """The C restatement (oracle/sgm_oracle.c)."""

    def __init__(self, path: Path = ORACLE_SO):
        if not Path(path).exists():
            build_oracle()
        L = self.lib = C.CDLL(str(path))
        L.orc_project.restype = C.c_uint64
        L.orc_project.argtypes = [C.POINTER(orc_map), C.POINTER(orc_camera), C.POINTER(orc_pose),
                                  C.POINTER(orc_options), C.POINTER(orc_proj)]
        L.orc_bins.restype = C.c_uint64
        L.orc_bins.argtypes = [C.POINTER(orc_proj), C.c_uint64, C.POINTER(orc_camera),
                               C.POINTER(orc_options), _pu32, _pu32, _pf, C.c_uint64]
        L.orc_render.restype = C.c_int
        L.orc_render.argtypes = [C.POINTER(orc_map), C.POINTER(orc_camera), C.POINTER(orc_pose),
                                 C.c_uint32, C.POINTER(orc_options), _pd, _pd, _pd, _pd,
                                 C.POINTER(orc_stats)]
        L.orc_clipped_entropy.restype = C.c_double
        L.orc_clipped_entropy.argtypes = [_pd, C.c_int]
        L.orc_score_views.restype = C.c_int
        L.orc_score_views.argtypes = [C.POINTER(orc_map), C.POINTER(orc_camera), C.c_uint64,
                                      C.POINTER(orc_pose), C.POINTER(orc_options), C.c_int, _pd,
                                      _pd, C.POINTER(orc_stats)]
        L.orc_render_entropy.restype = C.c_int
        L.orc_render_entropy.argtypes = [C.POINTER(orc_map), C.POINTER(orc_camera),
                                         C.POINTER(orc_pose), C.POINTER(orc_options), _pd]
        L.orc_combine_scores.restype = C.c_int
        L.orc_combine_scores.argtypes = [C.c_uint64, _pd, _pd, _pd, _pd, _pd, _pd, _pd]
        L.orc_candidate_pose.restype = None
        L.orc_candidate_pose.argtypes = [_pd, _pd, C.POINTER(orc_pose)]
        L.orc_look_at.restype = None
        L.orc_look_at.argtypes = [_pd, _pd, C.POINTER(orc_pose)]
        L.orc_fisher_accumulate.restype = C.c_int
        L.orc_fisher_accumulate.argtypes = [C.POINTER(orc_map), C.POINTER(orc_camera), C.c_uint64,
                                            C.POINTER(orc_pose), C.POINTER(orc_options), _pd]
        L.orc_fisher_gain.restype = C.c_int
        L.orc_fisher_gain.argtypes = [C.POINTER(orc_map), C.POINTER(orc_camera), C.c_uint64,
                                      C.POINTER(orc_pose), C.POINTER(orc_options), _pd,
                                      C.c_double, _pd]
        L.orc_emap_init.restype = C.c_int
        L.orc_emap_init.argtypes = [C.POINTER(orc_emap), _pd, _pd, C.c_double]
        L.orc_emap_free.argtypes = [C.POINTER(orc_emap)]
        L.orc_emap_integrate.restype = C.c_uint64
        L.orc_emap_integrate.argtypes = [C.POINTER(orc_emap), C.POINTER(orc_camera),
                                         C.POINTER(orc_pose), _pf, C.c_int]
        L.orc_emap_seed.argtypes = [C.POINTER(orc_emap), _pd, _pd, C.c_int]
        L.orc_emap_reseed.argtypes = [C.POINTER(orc_emap)]
        L.orc_fibonacci_directions.argtypes = [C.c_int, C.c_double, _pd]
        L.orc_sample_candidates.restype = C.c_uint64
        L.orc_sample_candidates.argtypes = [C.POINTER(orc_emap), C.c_double, C.c_int, _pd, C.c_int,
                                            _pd, C.c_uint64]

    def emap(self, bmin, bmax, voxel) -> "OracleEmap":
        return OracleEmap(self, bmin, bmax, voxel)

    def fibonacci_directions(self, count, max_elev=45.0) -> np.ndarray:
        out = np.zeros((max(count, 0), 3))
        if count > 0:
            self.lib.orc_fibonacci_directions(count, max_elev, _dp(out))
        return out

    def fisher_accumulate(self, m, cam, poses, opt=None) -> np.ndarray:
        """Fisher diagonal summed over `poses`: (N, 8) = (mu xyz, log_r, logit, rgb)."""
        ma = _MapArrays(m)
        H = np.zeros((max(ma.n, 1), 8))
        arr = (orc_pose * max(len(poses), 1))(*[_pose(p) for p in poses])
        cm, cc, co = ma.c(), _cam(cam), _opts(opt)
        assert self.lib.orc_fisher_accumulate(C.byref(cm), C.byref(cc), len(poses), arr,
                                              C.byref(co), _dp(H)) == 0
        return H[:ma.n]

    def fisher_gain(self, m, cam, poses, H_prior, lam, opt=None) -> np.ndarray:
        ma = _MapArrays(m)
        Hp = np.ascontiguousarray(H_prior, dtype=np.float64)
        g = np.zeros(len(poses))
        arr = (orc_pose * max(len(poses), 1))(*[_pose(p) for p in poses])
        cm, cc, co = ma.c(), _cam(cam), _opts(opt)
        assert self.lib.orc_fisher_gain(C.byref(cm), C.byref(cc), len(poses), arr, C.byref(co),
                                        _dp(Hp), float(lam), _dp(g)) == 0
        return g

    def project(self, m, cam, pose, opt=None) -> np.ndarray:
        ma = _MapArrays(m)
        buf = (orc_proj * max(ma.n, 1))()
        cm, cc, cp, co = ma.c(), _cam(cam), _pose(pose), _opts(opt)
        v = self.lib.orc_project(C.byref(cm), C.byref(cc), C.byref(cp), C.byref(co), buf)
        return np.frombuffer(buf, dtype=PROJ_DTYPE, count=v).copy()

    def bins(self, proj: np.ndarray, cam, opt=None):
        co = _opts(opt)
        ts = co.tile_size
        tiles = ((cam.width + ts - 1) // ts) * ((cam.height + ts - 1) // ts)
        pr = np.ascontiguousarray(proj, dtype=PROJ_DTYPE)
        pp = pr.ctypes.data_as(C.POINTER(orc_proj))
        offsets = np.zeros(tiles + 1, dtype=np.uint32)
        cc = _cam(cam)
        P = self.lib.orc_bins(pp, len(pr), C.byref(cc), C.byref(co),
                              offsets.ctypes.data_as(_pu32), None, None, 0)
        ids = np.zeros(max(P, 1), dtype=np.uint32)
        probe = np.zeros((max(P, 1), 3), dtype=np.float32)
        self.lib.orc_bins(pp, len(pr), C.byref(cc), C.byref(co), offsets.ctypes.data_as(_pu32),
                          ids.ctypes.data_as(_pu32), probe.ctypes.data_as(_pf), P)
        return offsets, ids[:P], probe[:P]

    def render(self, m, cam, pose, channels=7, opt=None):
        """Returns dict(color, depth, silhouette, sem, stats) in the reference layout."""
        ma = _MapArrays(m)
        px = cam.width * cam.height
        C_ = ma.num_classes + 1
        out = {"silhouette": np.zeros(px),
               "color": np.zeros(px * 3) if channels & 1 else None,
               "depth": np.zeros(px) if channels & 2 else None,
               "sem": np.zeros(px * C_) if channels & 4 else None}
        st = orc_stats()
        cm, cc, cp, co = ma.c(), _cam(cam), _pose(pose), _opts(opt)
        rc = self.lib.orc_render(C.byref(cm), C.byref(cc), C.byref(cp), channels, C.byref(co),
                                 _dp(out["color"]), _dp(out["depth"]), _dp(out["silhouette"]),
                                 _dp(out["sem"]), C.byref(st))
        assert rc == 0
        out["stats"] = {f: getattr(st, f) for f, _ in orc_stats._fields_}
        return out

    def score_views(self, m, cam, poses, opt=None, threads=1):
        ma = _MapArrays(m)
        n = len(poses)
        arr = (orc_pose * max(n, 1))(*[_pose(p) for p in poses])
        nm, es = np.zeros(n), np.zeros(n)
        st = orc_stats()
        cm, cc, co = ma.c(), _cam(cam), _opts(opt)
        rc = self.lib.orc_score_views(C.byref(cm), C.byref(cc), n, arr, C.byref(co), int(threads),
                                      _dp(nm), _dp(es), C.byref(st))
        assert rc == 0
        return nm, es, {f: getattr(st, f) for f, _ in orc_stats._fields_}

    def render_entropy(self, m, cam, pose, opt=None) -> np.ndarray:
        ma = _MapArrays(m)
        out = np.zeros(cam.width * cam.height)
        cm, cc, cp, co = ma.c(), _cam(cam), _pose(pose), _opts(opt)
        assert self.lib.orc_render_entropy(C.byref(cm), C.byref(cc), C.byref(cp), C.byref(co),
                                           _dp(out)) == 0
        return out

    def clipped_entropy(self, p) -> float:
        a = np.ascontiguousarray(p, dtype=np.float64)
        return float(self.lib.orc_clipped_entropy(_dp(a), a.size))

    def combine_scores(self, n_missing, entropy_sum, positions, current):
        nm = np.ascontiguousarray(n_missing, dtype=np.float64)
        es = np.ascontiguousarray(entropy_sum, dtype=np.float64)
        pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
        cur = np.ascontiguousarray(current, dtype=np.float64)
        n = nm.size
        g, s, t = np.zeros(n), np.zeros(n), np.zeros(n)
        any_ = self.lib.orc_combine_scores(n, _dp(nm), _dp(es), _dp(pos), _dp(cur), _dp(g), _dp(s),
                                           _dp(t))
        return bool(any_), g, s, t

    def candidate_pose(self, pos, direction):
        p = np.ascontiguousarray(pos, dtype=np.float64)
        d = np.ascontiguousarray(direction, dtype=np.float64)
        out = orc_pose()
        self.lib.orc_candidate_pose(_dp(p), _dp(d), C.byref(out))
        return np.array(out.R[:]).reshape(3, 3), np.array(out.t[:])

    def look_at(self, pos, target):
        p = np.ascontiguousarray(pos, dtype=np.float64)
        t = np.ascontiguousarray(target, dtype=np.float64)
        out = orc_pose()
        self.lib.orc_look_at(_dp(p), _dp(t), C.byref(out))
        return np.array(out.R[:]).reshape(3, 3), np.array(out.t[:])


def _frames_blob(frames):
    """(poses (n*12 f64: R row-major, t), planes (per frame rgb | depth | sem, f32))."""
    poses = np.concatenate([np.concatenate([np.asarray(f.pose.R, np.float64).reshape(9),
                                            np.asarray(f.pose.t, np.float64)]) for f in frames])
    planes = np.concatenate([np.concatenate([np.asarray(f.rgb, np.float32).reshape(-1),
                                             np.asarray(f.depth, np.float32).reshape(-1),
                                             np.asarray(f.sem, np.float32).reshape(-1)])
                             for f in frames]).astype(np.float32)
    return np.ascontiguousarray(poses), np.ascontiguousarray(planes)


def _v3(v):
    return np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(3))


def _depth(depth):
    return np.ascontiguousarray(depth, dtype=np.float32).reshape(-1)


class OracleEmap:
    """ExplorationMap restated in C (orc_emap_*). Same interface as RefEmap."""

    def __init__(self, orc, bmin, bmax, voxel):
        self.o = orc
        self.e = orc_emap()
        if orc.lib.orc_emap_init(C.byref(self.e), _dp(_v3(bmin)), _dp(_v3(bmax)), float(voxel)):
            raise ValueError("emap: voxel size must be > 0")

    def __del__(self):
        if getattr(self, "e", None) is not None:
            self.o.lib.orc_emap_free(C.byref(self.e))

    def integrate(self, cam, pose, depth, stride=2) -> int:
        c, p, d = _cam(cam), _pose(pose), _depth(depth)
        return int(self.o.lib.orc_emap_integrate(C.byref(self.e), C.byref(c), C.byref(p),
                                                   d.ctypes.data_as(_pf), int(stride)))

    def grid(self) -> np.ndarray:
        return np.ctypeslib.as_array(self.e.grid, shape=(self.e.nvox,)).copy()

    def info(self) -> dict:
        return {"free": int(self.e.free_count), "occupied": int(self.e.occupied_count),
                "changelog": int(self.e.log_n), "dims": tuple(self.e.dims),
                "origin": tuple(self.e.origin), "voxels": int(self.e.nvox)}

    def take_changelog(self) -> np.ndarray:
        n = int(self.e.log_n)
        out = (np.ctypeslib.as_array(self.e.log, shape=(n,)).copy() if n
               else np.zeros(0, np.int32))
        self.e.log_n = 0
        return out

    def reseed(self) -> None:
        self.o.lib.orc_emap_reseed(C.byref(self.e))

    def seed(self, bmin, bmax, occupied=False) -> None:
        self.o.lib.orc_emap_seed(C.byref(self.e), _dp(_v3(bmin)), _dp(_v3(bmax)), int(occupied))

    def sample_candidates(self, v1, v2, heights):
        h = np.ascontiguousarray(heights, dtype=np.float64)
        e2 = orc_emap.from_buffer_copy(self.e)  # count first, without consuming
        n = int(self.o.lib.orc_sample_candidates(C.byref(e2), float(v1), int(v2), _dp(h), len(h),
                                                  None, 0))
        out = np.zeros((max(n, 1), 6))
        self.o.lib.orc_sample_candidates(C.byref(self.e), float(v1), int(v2), _dp(h), len(h),
                                         _dp(out), n)
        return out[:n, :3].copy(), out[:n, 3:].copy()


class RefEmap:
    """The reference's own ExplorationMap (explorer.cpp:11-184) via ref_emap_*."""

    def __init__(self, ref, bmin, bmax, voxel):
        self.r = ref
        self.voxel = float(voxel)
        self.h = ref.lib.ref_emap_create(_dp(_v3(bmin)), _dp(_v3(bmax)), float(voxel))
        if not self.h:
            raise ValueError("emap: voxel size must be > 0")

    def __del__(self):
        if getattr(self, "h", None):
            self.r.lib.ref_emap_destroy(self.h)
            self.h = None

    def integrate(self, cam, pose, depth, stride=2) -> int:
        wh, intr = RefLib._cam(cam)
        R, t = RefLib._pose(pose)
        d = _depth(depth)
        return int(self.r.lib.ref_emap_integrate(self.h, wh.ctypes.data_as(_pi32), _dp(intr),
                                                 _dp(R), _dp(t), d.ctypes.data_as(_pf),
                                                 int(stride)))

    def info(self) -> dict:
        info = np.zeros(4, np.uint64)
        dims = np.zeros(3, np.int32)
        origin = np.zeros(3)
        self.r.lib.ref_emap_info(self.h, info.ctypes.data_as(_pu64), dims.ctypes.data_as(_pi32),
                                 _dp(origin))
        return {"free": int(info[0]), "occupied": int(info[1]), "changelog": int(info[2]),
                "dims": tuple(int(v) for v in dims), "origin": tuple(float(v) for v in origin),
                "voxels": int(info[3])}

    def grid(self) -> np.ndarray:
        out = np.zeros(self.info()["voxels"], np.uint8)
        self.r.lib.ref_emap_grid(self.h, out.ctypes.data_as(C.POINTER(C.c_uint8)))
        return out

    def take_changelog(self) -> np.ndarray:
        out = np.zeros(max(self.info()["changelog"], 1), np.int32)
        n = int(self.r.lib.ref_emap_take_changelog(self.h, out.ctypes.data_as(_pi32)))
        return out[:n].copy()

    def reseed(self) -> None:
        self.r.lib.ref_emap_reseed(self.h)

    def seed(self, bmin, bmax, occupied=False) -> None:
        self.r.lib.ref_emap_seed(self.h, _dp(_v3(bmin)), _dp(_v3(bmax)), int(occupied))

    def sample_candidates(self, v1, v2, heights):
        h = np.ascontiguousarray(heights, dtype=np.float64)
        # upper bound: every lattice point free and fresh
        info = self.info()
        nx = int(info["dims"][0] * self.voxel / v1) + 2
        nz = int(info["dims"][2] * self.voxel / v1) + 2
        cap = max(1, len(h) * nx * nz * int(v2))
        out = np.zeros((cap, 6))
        n = int(self.r.lib.ref_sample_candidates(self.h, float(v1), int(v2), _dp(h), len(h),
                                                 _dp(out), cap))
        assert n <= cap
        return out[:n, :3].copy(), out[:n, 3:].copy()


class RefLib:
    """The reference's own code (oracle/_ref/libsgm_ref.so)."""

    def __init__(self, path: Path = REF_SO):
        if not Path(path).exists():
            raise FileNotFoundError(f"{path} missing (make -C oracle ref)")
        L = self.lib = C.CDLL(str(path))
        L.ref_map_create.restype = C.c_void_p
        L.ref_map_create.argtypes = [C.c_uint64, C.c_int, C.c_int, _pd, _pd, _pd, _pd, _pu16, _pd]
        L.ref_map_destroy.argtypes = [C.c_void_p]
        L.ref_map_load.restype = C.c_void_p
        L.ref_map_load.argtypes = [C.c_char_p]
        L.ref_map_size.restype = C.c_uint64
        L.ref_map_size.argtypes = [C.c_void_p]
        L.ref_render.restype = C.c_int
        L.ref_render.argtypes = [C.c_void_p, C.c_int, _pi32, _pd, _pd, _pd, C.c_uint32, _pd, _pd,
                                 _pd, _pd, _pd, _pd, _pu64, _pu32, _pu32, C.c_uint64, _pu64]
        L.ref_render_entropy.argtypes = [C.c_void_p, _pi32, _pd, _pd, _pd, _pd, _pd]
        L.ref_clipped_entropy.restype = C.c_double
        L.ref_clipped_entropy.argtypes = [_pd, C.c_uint64]
        L.ref_refresh_scores.argtypes = [C.c_void_p, _pi32, _pd, C.c_uint64, _pd, _pd, C.c_int,
                                         _pd, _pd]
        L.ref_combine_scores.restype = C.c_int
        L.ref_combine_scores.argtypes = [C.c_uint64, _pd, _pd, _pd, _pd, _pd, _pd, _pd]
        L.ref_candidate_pose.argtypes = [_pd, _pd, _pd, _pd]
        L.ref_look_at.argtypes = [_pd, _pd, _pd, _pd]
        L.ref_random_splat_map.argtypes = [C.c_uint64, _pi32, _pd, _pd, _pd, _pd, _pd, _pd, _pd,
                                           _pd, _pu16, _pd, _pi32]
        L.ref_camera_from_fov.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, _pd]
        L.ref_emap_create.restype = C.c_void_p
        L.ref_emap_create.argtypes = [_pd, _pd, C.c_double]
        L.ref_emap_destroy.argtypes = [C.c_void_p]
        L.ref_emap_info.argtypes = [C.c_void_p, _pu64, _pi32, _pd]
        L.ref_emap_integrate.restype = C.c_uint64
        L.ref_emap_integrate.argtypes = [C.c_void_p, _pi32, _pd, _pd, _pd, _pf, C.c_int]
        L.ref_emap_grid.argtypes = [C.c_void_p, C.POINTER(C.c_uint8)]
        L.ref_emap_take_changelog.restype = C.c_uint64
        L.ref_emap_take_changelog.argtypes = [C.c_void_p, _pi32]
        L.ref_emap_reseed.argtypes = [C.c_void_p]
        L.ref_emap_seed.argtypes = [C.c_void_p, _pd, _pd, C.c_int]
        L.ref_sample_candidates.restype = C.c_uint64
        L.ref_sample_candidates.argtypes = [C.c_void_p, C.c_double, C.c_int, _pd, C.c_int, _pd,
                                            C.c_uint64]
        L.ref_fibonacci_directions.argtypes = [C.c_int, C.c_double, _pd]
        L.ref_raycast_depth.restype = C.c_int
        L.ref_raycast_depth.argtypes = [_pd, _pd, C.c_int, _pd, C.c_int, _pd, _pi32, _pd, _pd,
                                        _pd, _pf]
        L.ref_optimize_map.restype = C.c_int64
        L.ref_optimize_map.argtypes = [C.c_uint64, C.c_int, C.c_int, _pd, _pd, _pd, _pd, _pu16,
                                       _pd, _pi32, _pd, C.c_int, _pd, _pf, _pd, _pd, _pd, C.c_int,
                                       _pd, _pi32, C.c_char_p, C.c_int]
        L.ref_eval.restype = C.c_int
        L.ref_eval.argtypes = [C.c_void_p, _pi32, _pd, C.c_int, C.c_int, _pd, _pf, _pd, _pd, _pd,
                               _pd, _pu64, C.c_char_p, C.c_int]
        L.ref_backward.restype = C.c_int
        L.ref_backward.argtypes = [C.c_void_p, _pi32, _pd, _pd, _pd, _pd, C.c_int, _pf, _pf, _pf,
                                   _pd, C.c_int, C.c_int, _pd, _pd, _pd, _pd, _pd, _pd,
                                   C.c_char_p, C.c_int]

    def emap(self, bmin, bmax, voxel) -> RefEmap:
        return RefEmap(self, bmin, bmax, voxel)

    def fibonacci_directions(self, count, max_elev=45.0) -> np.ndarray:
        out = np.zeros((max(count, 0), 3))
        if count > 0:
            self.lib.ref_fibonacci_directions(count, max_elev, _dp(out))
        return out

    def raycast_depth(self, bmin, bmax, cam, pose, boxes=(), spheres=()) -> np.ndarray:
        """Depth plane of raycast_frame (scene_sim.hpp:31) for a room with boxes / spheres."""
        b = np.ascontiguousarray(np.asarray(boxes, dtype=np.float64).reshape(-1, 6))
        sp = np.ascontiguousarray(np.asarray(spheres, dtype=np.float64).reshape(-1, 4))
        wh, intr = self._cam(cam)
        R, t = self._pose(pose)
        out = np.zeros(cam.width * cam.height, np.float32)
        rc = self.lib.ref_raycast_depth(_dp(_v3(bmin)), _dp(_v3(bmax)), len(b), _dp(b), len(sp),
                                        _dp(sp), wh.ctypes.data_as(_pi32), _dp(intr), _dp(R),
                                        _dp(t), out.ctypes.data_as(_pf))
        if rc:
            raise ValueError("raycast_depth: invalid scene")
        return out

    def evaluate(self, m, cam, frames):
        """The reference's semantic_metrics + photometric_metrics over its own render of `m`
        at each frame's pose. Returns (summary[7], per_view_miou, per_view_psnr,
        per_class (rows of 5))."""
        h = self.map_create(m)
        wh, intr = self._cam(cam)
        poses, planes = _frames_blob(frames)
        nf = len(frames)
        summary = np.zeros(7)
        pvm, pvp = np.zeros(max(nf, 1)), np.zeros(max(nf, 1))
        pc = np.zeros((max(m.num_classes(), 1), 5))
        npc = C.c_uint64(0)
        err = C.create_string_buffer(512)
        rc = self.lib.ref_eval(h, wh.ctypes.data_as(_pi32), _dp(intr), m.num_classes(), nf,
                               _dp(poses), planes.ctypes.data_as(_pf), _dp(summary), _dp(pvm),
                               _dp(pvp), _dp(pc), C.byref(npc), err, 512)
        self.map_destroy(h)
        if rc:
            raise ValueError(err.value.decode())
        return summary, pvm[:nf], pvp[:nf], pc[: npc.value]

    def optimize_map(self, m, frames, cam, cfg, iters):
        """The reference's optimize_map (mapper.cpp:241-283) from a zero AdamState.
        Returns (history (n_done, 7), arrays dict of the final map, error or None)."""
        n, k = m.size(), m.k()
        arr = {"centers": np.ascontiguousarray(m.centers, dtype=np.float64).reshape(-1).copy(),
               "log_radii": np.ascontiguousarray(m.log_radii, dtype=np.float64).copy(),
               "opacity_logits": np.ascontiguousarray(m.opacity_logits, dtype=np.float64).copy(),
               "colors": np.ascontiguousarray(m.colors, dtype=np.float64).reshape(-1).copy(),
               "sem_indices": np.ascontiguousarray(m.sem_indices, dtype=np.uint16).reshape(-1).copy(),
               "sem_probs": np.ascontiguousarray(m.sem_probs, dtype=np.float64).reshape(-1).copy()}
        wh, intr = self._cam(cam)
        poses, planes = _frames_blob(frames)
        a = cfg.adam
        adam = np.array([a.lr_center, a.lr_radius, a.lr_opacity, a.lr_color, a.lr_sem, a.beta1,
                         a.beta2, a.eps, a.eps_sem])
        c = np.array([float(cfg.prune_every), cfg.prune_opacity, cfg.divergence_factor,
                      float(cfg.divergence_window)])
        w = cfg.weights
        wv = np.array([w.lambda_hd, w.lambda_cos, float(w.mask_k), float(w.use_hd),
                       float(w.use_cos), float(w.use_kl), w.kl_clip_norm])
        hist = np.zeros((max(iters, 1), 7))
        nh = C.c_int(0)
        err = C.create_string_buffer(512)
        pf = C.POINTER(C.c_float)
        m_final = self.lib.ref_optimize_map(
            n, k, m.num_classes(), _dp(arr["centers"]), _dp(arr["log_radii"]),
            _dp(arr["opacity_logits"]), _dp(arr["colors"]), arr["sem_indices"].ctypes.data_as(_pu16),
            _dp(arr["sem_probs"]), wh.ctypes.data_as(_pi32), _dp(intr), len(frames), _dp(poses),
            planes.ctypes.data_as(pf), _dp(adam), _dp(c), _dp(wv), int(iters), _dp(hist),
            C.byref(nh), err, 512)
        if m_final < 0:
            return hist[:0], None, err.value.decode()
        mf = int(m_final)
        out = {"centers": arr["centers"][:3 * mf], "log_radii": arr["log_radii"][:mf],
               "opacity_logits": arr["opacity_logits"][:mf], "colors": arr["colors"][:3 * mf],
               "sem_indices": arr["sem_indices"][:k * mf], "sem_probs": arr["sem_probs"][:k * mf]}
        return hist[: nh.value], out, None

    def backward(self, m, cam, frame, weights, include_mapping=True, include_semantic=True,
                 opt=None):
        """The reference's render(all(true)) + mapping_loss + semantic_loss + backward."""
        h = self.map_create(m)
        wh, intr = self._cam(cam)
        R, t = self._pose(frame.pose)
        o = self._opts(opt)
        n, k = m.size(), m.k()
        wv = np.array([weights.lambda_hd, weights.lambda_cos, float(weights.mask_k),
                       float(weights.use_hd), float(weights.use_cos), float(weights.use_kl),
                       weights.kl_clip_norm])
        rep = np.zeros(7)
        out = {"center": np.zeros(3 * n), "log_radius": np.zeros(n),
               "opacity_logit": np.zeros(n), "color": np.zeros(3 * n), "sem": np.zeros(k * n)}
        err = C.create_string_buffer(512)
        pf = C.POINTER(C.c_float)
        rgb = np.ascontiguousarray(frame.rgb, dtype=np.float32)
        dep = np.ascontiguousarray(frame.depth, dtype=np.float32)
        sem = np.ascontiguousarray(frame.sem, dtype=np.float32)
        rc = self.lib.ref_backward(h, wh.ctypes.data_as(_pi32), _dp(intr), _dp(R), _dp(t), _dp(o),
                                   frame.num_classes, rgb.ctypes.data_as(pf), dep.ctypes.data_as(pf),
                                   sem.ctypes.data_as(pf), _dp(wv), int(include_mapping),
                                   int(include_semantic), _dp(rep), _dp(out["center"]),
                                   _dp(out["log_radius"]), _dp(out["opacity_logit"]),
                                   _dp(out["color"]), _dp(out["sem"]), err, 512)
        self.map_destroy(h)
        if rc != 0:
            raise RuntimeError(err.value.decode())
        return rep, out

    # --- maps
    def map_create(self, m):
        ma = _MapArrays(m)
        return self.lib.ref_map_create(ma.n, ma.k, ma.num_classes, _dp(ma.centers),
                                       _dp(ma.log_radii), _dp(ma.logits), _dp(ma.colors),
                                       ma.idx.ctypes.data_as(_pu16), _dp(ma.probs))

    def map_destroy(self, h) -> None:
        self.lib.ref_map_destroy(h)

    @staticmethod
    def _cam(cam):
        wh = np.array([cam.width, cam.height], dtype=np.int32)
        intr = np.array([cam.fx, cam.fy, cam.cx, cam.cy], dtype=np.float64)
        return wh, intr

    @staticmethod
    def _pose(p):
        return (np.ascontiguousarray(np.asarray(p.R, dtype=np.float64).reshape(9)),
                np.ascontiguousarray(p.t, dtype=np.float64))

    @staticmethod
    def _opts(o):
        if o is None:
            return np.array([1.0, 1e-4, 0.01, 3.0, 8.0])
        return np.array([1.0 if o.early_exit else 0.0, o.transmittance_eps, o.z_near,
                         o.truncation_sigmas, float(o.tile_size)])

    def render(self, m, cam, pose, channels=7, opt=None, which=0, handle=None, n_map=None):
        own = handle is None
        h = self.map_create(m) if own else handle
        n = m.size() if n_map is None else n_map
        C_ = m.num_classes() + 1
        px = cam.width * cam.height
        wh, intr = self._cam(cam)
        R, t = self._pose(pose)
        o = self._opts(opt)
        out = {"silhouette": np.zeros(px),
               "color": np.zeros(px * 3) if channels & 1 else None,
               "depth": np.zeros(px) if channels & 2 else None,
               "sem": np.zeros(px * C_) if channels & 4 else None}
        proj = np.zeros((max(n, 1), 6))
        nproj = C.c_uint64()
        ncon = C.c_uint64()
        off = np.zeros(px + 1, dtype=np.uint32) if channels & 8 else None
        cap = px * max(n, 1) if channels & 8 else 0
        con = np.zeros(max(cap, 1), dtype=np.uint32) if channels & 8 else None
        self.lib.ref_render(h, which, wh.ctypes.data_as(_pi32), _dp(intr), _dp(R), _dp(t),
                            channels, _dp(o), _dp(out["color"]), _dp(out["depth"]),
                            _dp(out["silhouette"]), _dp(out["sem"]), _dp(proj), C.byref(nproj),
                            None if off is None else off.ctypes.data_as(_pu32),
                            None if con is None else con.ctypes.data_as(_pu32), cap,
                            C.byref(ncon))
        if channels & 8:
            out["contrib_offset"] = off
            out["contrib"] = con[:ncon.value].copy()
        p6 = proj[:nproj.value]
        arr = np.zeros(nproj.value, dtype=PROJ_DTYPE)
        for i, f in enumerate(["mx", "my", "rad_px", "z", "alpha"]):
            arr[f] = p6[:, i]
        arr["index"] = p6[:, 5].astype(np.uint32)
        out["projections"] = arr
        if own:
            self.map_destroy(h)
        return out

    def render_entropy(self, m, cam, pose, opt=None):
        h = self.map_create(m)
        wh, intr = self._cam(cam)
        R, t = self._pose(pose)
        o = self._opts(opt)
        out = np.zeros(cam.width * cam.height)
        self.lib.ref_render_entropy(h, wh.ctypes.data_as(_pi32), _dp(intr), _dp(R), _dp(t), _dp(o),
                                    _dp(out))
        self.map_destroy(h)
        return out

    def refresh_scores(self, m, cam, positions, directions, threads=1, handle=None):
        own = handle is None
        h = self.map_create(m) if own else handle
        pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
        dirs = np.ascontiguousarray(directions, dtype=np.float64).reshape(-1, 3)
        n = pos.shape[0]
        wh, intr = self._cam(cam)
        nm, es = np.zeros(n), np.zeros(n)
        self.lib.ref_refresh_scores(h, wh.ctypes.data_as(_pi32), _dp(intr), n, _dp(pos), _dp(dirs),
                                    int(threads), _dp(nm), _dp(es))
        if own:
            self.map_destroy(h)
        return nm, es

    def clipped_entropy(self, p) -> float:
        a = np.ascontiguousarray(p, dtype=np.float64)
        return float(self.lib.ref_clipped_entropy(_dp(a), a.size))

    def combine_scores(self, n_missing, entropy_sum, positions, current):
        nm = np.ascontiguousarray(n_missing, dtype=np.float64)
        es = np.ascontiguousarray(entropy_sum, dtype=np.float64)
        pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
        cur = np.ascontiguousarray(current, dtype=np.float64)
        n = nm.size
        g, s, t = np.zeros(n), np.zeros(n), np.zeros(n)
        any_ = self.lib.ref_combine_scores(n, _dp(nm), _dp(es), _dp(pos), _dp(cur), _dp(g), _dp(s),
                                           _dp(t))
        return bool(any_), g, s, t

    def candidate_pose(self, pos, direction):
        p = np.ascontiguousarray(pos, dtype=np.float64)
        d = np.ascontiguousarray(direction, dtype=np.float64)
        R, t = np.zeros(9), np.zeros(3)
        self.lib.ref_candidate_pose(_dp(p), _dp(d), _dp(R), _dp(t))
        return R.reshape(3, 3), t

    def look_at(self, pos, target):
        p = np.ascontiguousarray(pos, dtype=np.float64)
        tg = np.ascontiguousarray(target, dtype=np.float64)
        R, t = np.zeros(9), np.zeros(3)
        self.lib.ref_look_at(_dp(p), _dp(tg), _dp(R), _dp(t))
        return R.reshape(3, 3), t

    def random_splat_map(self, seed, cam, pose, num_splats=8, num_classes=5, k=0, min_prob=0.02,
                         alpha_logit_min=-1.5, alpha_logit_max=2.5, rad_px_min=1.0,
                         rad_px_max=4.0):
        """testutil::random_splat_map (proj/tests/test_helpers.hpp:46-67) -> arrays dict."""
        wh, intr = self._cam(cam)
        R, t = self._pose(pose)
        prm = np.array([num_splats, num_classes, k, min_prob, alpha_logit_min, alpha_logit_max,
                        rad_px_min, rad_px_max], dtype=np.float64)
        kk = k if k > 0 else num_classes + 1
        out = {"centers": np.zeros((num_splats, 3)), "log_radii": np.zeros(num_splats),
               "opacity_logits": np.zeros(num_splats), "colors": np.zeros((num_splats, 3)),
               "sem_indices": np.zeros((num_splats, kk), dtype=np.uint16),
               "sem_probs": np.zeros((num_splats, kk))}
        kout = C.c_int32()
        self.lib.ref_random_splat_map(seed, wh.ctypes.data_as(_pi32), _dp(intr), _dp(R), _dp(t),
                                      _dp(prm), _dp(out["centers"]), _dp(out["log_radii"]),
                                      _dp(out["opacity_logits"]), _dp(out["colors"]),
                                      out["sem_indices"].ctypes.data_as(_pu16),
                                      _dp(out["sem_probs"]), C.byref(kout))
        out["k"] = int(kout.value)
        out["num_classes"] = num_classes
        return out

    def camera_from_fov(self, w, h, vfov, hfov):
        out = np.zeros(6)
        self.lib.ref_camera_from_fov(w, h, vfov, hfov, _dp(out))
        return out


def ref_available() -> bool:
    return REF_SO.exists()


def cpu_count() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
