"""ctypes bindings for the C ABI in include/sgm.h (libsgm_b200.so, built in-tree).

The library is the only compute path: there is no CPU fallback. If the shared
object is missing this module raises ImportError on import, and creating a
context without a CUDA device raises RuntimeError.

The library is mapped on the first use of `lib` (any compute or host-math call), not
at import: code that only builds scenes or candidate geometry (e.g. bench.py's
reference arm, which must run the reference alone) never maps it.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("SGM_B200_LIB", _HERE / "_lib" / "libsgm_b200.so"))

if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is missing: build the sm_100a extension first "
        "(python -c 'import __graft_entry__ as g; g.build()' or make -C "
        "paper_2506_00225_b200/csrc). There is no CPU fallback."
    )

_lib = None
_lib_lock = __import__("threading").Lock()

SGM_ABI_VERSION = 1
SGM_OK = 0
SGM_ERR_INVALID = 1
SGM_ERR_CUDA = 2
SGM_ERR_OOM = 3
SGM_ERR_UNSUPPORTED = 4
SGM_COLOR, SGM_DEPTH, SGM_SEMANTICS, SGM_RETAIN_CONTRIBUTORS = 1, 2, 4, 8


class sgm_camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_double),
                ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double)]


class sgm_pose(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("t", C.c_double * 3)]


class sgm_options(C.Structure):
    _fields_ = [("early_exit", C.c_int32), ("transmittance_eps", C.c_double),
                ("z_near", C.c_double), ("truncation_sigmas", C.c_double),
                ("tile_size", C.c_int32)]


class sgm_projection(C.Structure):
    _fields_ = [("mx", C.c_double), ("my", C.c_double), ("rad_px", C.c_double),
                ("z", C.c_double), ("alpha", C.c_double), ("index", C.c_uint32),
                ("reserved", C.c_uint32)]


class sgm_candidate(C.Structure):
    _fields_ = [("position", C.c_double * 3), ("direction", C.c_double * 3)]


class sgm_aabb(C.Structure):
    _fields_ = [("min", C.c_double * 3), ("max", C.c_double * 3)]


class sgm_adam_params(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("lr_center", "lr_radius", "lr_opacity", "lr_color",
                                          "lr_sem", "beta1", "beta2", "eps", "eps_sem")]


class sgm_optimize_config(C.Structure):
    _fields_ = [("prune_every", C.c_int32), ("prune_opacity", C.c_double),
                ("divergence_factor", C.c_double), ("divergence_window", C.c_int32)]


class sgm_stats(C.Structure):
    _fields_ = [("kernel_launches", C.c_uint64), ("views", C.c_uint64),
                ("visible", C.c_uint64), ("pairs", C.c_uint64),
                ("contributors", C.c_uint64), ("raster_launches", C.c_uint64),
                ("raster_ms", C.c_double), ("binning_ms", C.c_double)]


_vp = C.c_void_p
_pd = C.POINTER(C.c_double)
_pu16 = C.POINTER(C.c_uint16)
_pu32 = C.POINTER(C.c_uint32)
_pu64 = C.POINTER(C.c_uint64)
_pf = C.POINTER(C.c_float)

# Every symbol include/sgm.h declares, with its ctypes signature.
_pi32 = C.POINTER(C.c_int32)
_pu8 = C.POINTER(C.c_uint8)

SIGNATURES = {
    "sgm_eval_create": (C.c_int, [_vp, C.c_int32, C.POINTER(_vp)]),
    "sgm_eval_destroy": (None, [_vp, _vp]),
    "sgm_eval_add_view": (C.c_int, [_vp, _vp, _vp, C.POINTER(sgm_camera), C.POINTER(sgm_options),
                                    _vp]),
    "sgm_eval_report": (C.c_int, [_vp, _vp, _pd, _pd, _pd, _pd, _pu64]),
    "sgm_frame_upload": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, C.POINTER(sgm_pose),
                                   _pf, _pf, _pf, C.POINTER(_vp)]),
    "sgm_frame_release": (None, [_vp, _vp]),
    "sgm_trainer_create": (C.c_int, [_vp, C.c_uint64, C.c_int32, C.c_int32, _pd, _pd, _pd, _pd,
                                     _pu16, _pd, _pd, C.c_int64, C.POINTER(_vp)]),
    "sgm_trainer_destroy": (None, [_vp, _vp]),
    "sgm_trainer_size": (C.c_int, [_vp, _vp, _pu64, C.POINTER(C.c_int64)]),
    "sgm_trainer_rows": (C.c_int, [_vp, _vp, _pu32]),
    "sgm_trainer_download": (C.c_int, [_vp, _vp, _pd, _pd, _pd, _pd, _pu16, _pd, _pd]),
    "sgm_optimize_map": (C.c_int, [_vp, _vp, C.POINTER(sgm_camera), C.c_uint64, C.POINTER(_vp),
                                   C.POINTER(sgm_options), C.POINTER(sgm_adam_params), _pd,
                                   C.POINTER(sgm_optimize_config), C.c_int32, _pd,
                                   C.POINTER(C.c_int32)]),
    "sgm_emap_create": (C.c_int, [_vp, C.POINTER(sgm_aabb), C.c_double, C.POINTER(_vp)]),
    "sgm_emap_destroy": (None, [_vp, _vp]),
    "sgm_emap_info": (C.c_int, [_vp, _vp, _pd, _pd, _pi32, _pu64, _pu64, _pu64]),
    "sgm_emap_integrate": (C.c_int, [_vp, _vp, C.POINTER(sgm_camera), C.POINTER(sgm_pose), _pf,
                                     C.c_int32, _pu64]),
    "sgm_emap_integrate_device": (C.c_int, [_vp, _vp, C.POINTER(sgm_camera),
                                            C.POINTER(sgm_pose), _vp, C.c_int32, _pu64]),
    "sgm_emap_take_changelog": (C.c_int, [_vp, _vp, _pi32, C.c_uint64, _pu64]),
    "sgm_emap_reseed_changelog_with_free": (C.c_int, [_vp, _vp]),
    "sgm_emap_seed_region": (C.c_int, [_vp, _vp, C.POINTER(sgm_aabb), C.c_int]),
    "sgm_emap_grid": (C.c_int, [_vp, _vp, _pu8, C.c_uint64]),
    "sgm_sample_candidates": (C.c_int, [_vp, _vp, C.c_double, C.c_int32, _pd, C.c_int32,
                                        C.POINTER(sgm_candidate), C.c_uint64, _pu64]),
    "sgm_fibonacci_directions": (None, [C.c_int32, C.c_double, _pd]),
    "sgm_abi_version": (C.c_int, []),
    "sgm_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "sgm_ctx_destroy": (None, [_vp]),
    "sgm_last_error": (C.c_char_p, [_vp]),
    "sgm_ctx_stream": (_vp, [_vp]),
    "sgm_ctx_synchronize": (C.c_int, [_vp]),
    "sgm_ctx_set_profiling": (C.c_int, [_vp, C.c_int]),
    "sgm_ctx_get_stats": (C.c_int, [_vp, C.POINTER(sgm_stats)]),
    "sgm_ctx_reset_stats": (C.c_int, [_vp]),
    "sgm_map_upload": (C.c_int, [_vp, C.c_uint64, C.c_int32, C.c_int32, _pd, _pd, _pd, _pd,
                                 _pu16, _pd, C.POINTER(_vp)]),
    "sgm_map_upload_async": (C.c_int, [_vp, C.c_uint64, C.c_int32, C.c_int32, _pd, _pd, _pd, _pd,
                                       _pu16, _pd, C.POINTER(_vp)]),
    "sgm_map_wait": (C.c_int, [_vp, _vp]),
    "sgm_map_release": (None, [_vp, _vp]),
    "sgm_map_set_anisotropic": (C.c_int, [_vp, _vp, _pd, _pd]),
    "sgm_map_info": (C.c_int, [_vp, _vp, _pu64, _pi32, _pi32, _pi32]),
    "sgm_map_export_bytes": (C.c_int, [_vp, _vp, _pu64]),
    "sgm_map_export": (C.c_int, [_vp, _vp, _vp, C.c_uint64]),
    "sgm_map_import": (C.c_int, [_vp, _vp, C.c_uint64, C.POINTER(_vp)]),
    "sgm_multi_create": (C.c_int, [C.c_int32, _pi32, C.POINTER(_vp)]),
    "sgm_multi_destroy": (None, [_vp]),
    "sgm_multi_last_error": (C.c_char_p, [_vp]),
    "sgm_multi_device_count": (C.c_int32, [_vp]),
    "sgm_multi_ctx": (_vp, [_vp, C.c_int32]),
    "sgm_multi_map_upload": (C.c_int, [_vp, C.c_uint64, C.c_int32, C.c_int32, _pd, _pd, _pd, _pd,
                                       _pu16, _pd, C.POINTER(_vp)]),
    "sgm_multi_map_release": (None, [_vp, _vp]),
    "sgm_multi_score_views": (C.c_int, [_vp, _vp, C.POINTER(sgm_camera), C.c_uint64,
                                        C.POINTER(sgm_pose), C.POINTER(sgm_options), _pd, _pd]),
    "sgm_multi_score_candidates": (C.c_int, [_vp, _vp, C.POINTER(sgm_camera), C.c_uint64,
                                             C.POINTER(sgm_candidate), C.POINTER(sgm_options),
                                             _pd, _pd]),
    "sgm_render": (C.c_int, [_vp, _vp, C.POINTER(sgm_camera), C.POINTER(sgm_pose), C.c_uint32,
                             C.POINTER(sgm_options), _pd, _pd, _pd, _pd, _pu64]),
    "sgm_render_reference": (C.c_int, [_vp, _vp, C.POINTER(sgm_camera), C.POINTER(sgm_pose),
                                       C.c_uint32, _pd, _pd, _pd, _pd, _pu64]),
    "sgm_render_device": (C.c_int, [_vp, _vp, C.POINTER(sgm_camera), C.POINTER(sgm_pose),
                                    C.c_uint32, C.POINTER(sgm_options), _vp, _vp, _vp, _vp,
                                    _pu64]),
    "sgm_last_projections": (C.c_int, [_vp, C.POINTER(sgm_projection), C.c_uint64]),
    "sgm_last_bins": (C.c_int, [_vp, _pu32, _pu32, _pf, C.c_uint64, _pu64]),
    "sgm_last_contributors": (C.c_int, [_vp, _pu32, _pu32, C.c_uint64, _pu64]),
    "sgm_clipped_entropy": (C.c_double, [_pd, C.c_uint64]),
    "sgm_render_entropy": (C.c_int, [_vp, _vp, C.POINTER(sgm_camera), C.POINTER(sgm_pose),
                                     C.POINTER(sgm_options), _pd]),
    "sgm_score_views": (C.c_int, [_vp, _vp, C.POINTER(sgm_camera), C.c_uint64,
                                  C.POINTER(sgm_pose), C.POINTER(sgm_options), _pd, _pd]),
    "sgm_score_candidates": (C.c_int, [_vp, _vp, C.POINTER(sgm_camera), C.c_uint64,
                                       C.POINTER(sgm_candidate), C.POINTER(sgm_options), _pd,
                                       _pd]),
    "sgm_fisher_prior": (C.c_int, [_vp, _vp, C.POINTER(sgm_camera), C.c_uint64,
                                   C.POINTER(sgm_pose), C.POINTER(sgm_options), C.c_double, _pd]),
    "sgm_fisher_set_prior": (C.c_int, [_vp, _vp, _pd, C.c_double]),
    "sgm_score_views_fisher": (C.c_int, [_vp, _vp, C.POINTER(sgm_camera), C.c_uint64,
                                         C.POINTER(sgm_pose), C.POINTER(sgm_options), _pd, _pd,
                                         _pd]),
    "sgm_backward": (C.c_int, [_vp, _vp, C.POINTER(sgm_camera), C.POINTER(sgm_pose),
                               C.POINTER(sgm_options), _pf, _pf, _pf, _pd, C.c_int, C.c_int, _pd,
                               _pd, _pd, _pd, _pd, _pd]),
    "sgm_combine_scores_fisher": (C.c_int, [C.c_uint64, _pd, _pd, _pd, _pd, C.c_double, _pd, _pd]),
    "sgm_combine_scores": (C.c_int, [C.c_uint64, _pd, _pd, _pd, _pd, _pd, _pd, _pd]),
    "sgm_candidate_pose": (None, [_pd, _pd, C.POINTER(sgm_pose)]),
    "sgm_look_at": (None, [_pd, _pd, C.POINTER(sgm_pose)]),
}



def _load():
    global _lib
    with _lib_lock:
        if _lib is None:
            h = C.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                try:
                    fn = getattr(h, name)
                except AttributeError:  # an older build (A/B runs): that entry point unusable
                    continue
                fn.restype = res
                fn.argtypes = args
            if h.sgm_abi_version() != SGM_ABI_VERSION:
                raise ImportError(f"{LIB_PATH}: unexpected ABI version {h.sgm_abi_version()}")
            _lib = h
    return _lib


def __getattr__(name):  # module attribute `lib`: the library, mapped on first use
    if name == "lib":
        return _load()
    raise AttributeError(name)


def loaded() -> bool:
    """Whether this process has mapped libsgm_b200.so."""
    return _lib is not None


class SgmError(RuntimeError):
    """Raised for a non-zero status; carries the library's last-error text."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[sgm status {code}] {msg}")
        self.code = code


def check(code: int, ctx=None) -> None:
    if code != SGM_OK:
        msg = _load().sgm_last_error(ctx)
        raise SgmError(code, msg.decode() if msg else "")


def dptr(a):
    return a.ctypes.data_as(_pd) if a is not None else None
