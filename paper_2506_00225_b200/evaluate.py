"""Evaluation metrics on device-resident render planes.

Mirrors proj/include/splatmap/evaluator.hpp:12-60 (PerClassMetric, MetricReport,
semantic_metrics, photometric_metrics) and proj/src/evaluator.cpp:93-297. The reference
takes already-rendered RenderOutputs; here the evaluator renders the map at each frame's
pose into HBM (RenderChannels::all()) and consumes the px*(5+C) fp64 planes on the device
(sgm_eval_*), so nothing of the size of a plane crosses PCIe.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N
from .mapper import DeviceFrame
from .splatmap import CameraModel, Context, Frame, GaussianMap, RenderOptions, _ctx


@dataclass
class PerClassMetric:
    """evaluator.hpp:12-18."""

    class_id: int = 0
    iou_pct: float = 0.0
    ap_pct: float = 0.0
    f1_pct: float = 0.0
    gt_pixels: int = 0


@dataclass
class MetricReport:
    """The semantic and photometric fields of evaluator.hpp:20-42."""

    miou_pct: float = 0.0
    top1_pct: float = 0.0
    top3_pct: float = 0.0
    map_pct: float = 0.0
    f1_pct: float = 0.0
    psnr_db: float = 0.0
    depth_l1_cm: float = 0.0
    per_view_miou: List[float] = field(default_factory=list)
    per_view_psnr: List[float] = field(default_factory=list)
    per_class: List[PerClassMetric] = field(default_factory=list)


class Evaluator:
    """Streaming semantic_metrics + photometric_metrics (sgm_evaluator)."""

    def __init__(self, num_classes: int, ctx: Optional[Context] = None):
        self._ctx = _ctx(ctx)
        self.num_classes = int(num_classes)
        h = C.c_void_p()
        self._ctx.check(N.lib.sgm_eval_create(self._ctx.handle, self.num_classes, C.byref(h)))
        self.handle = h
        self.views = 0

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            N.lib.sgm_eval_destroy(self._ctx.handle, h)
            self.handle = None

    def add_view(self, gmap: GaussianMap, camera: CameraModel, frame, options=None) -> None:
        """Renders `gmap` at the frame's pose on the GPU and accumulates its statistics.
        `frame` is a Frame or an already uploaded DeviceFrame."""
        df = frame if isinstance(frame, DeviceFrame) else DeviceFrame(frame, ctx=self._ctx)
        handle = self._ctx.upload(gmap)
        cam = camera._c()
        opt = (options if options is not None else RenderOptions())._c()
        self._ctx.check(N.lib.sgm_eval_add_view(self._ctx.handle, self.handle, handle,
                                                C.byref(cam), C.byref(opt), df.handle))
        self.views += 1

    def report(self) -> MetricReport:
        summary = np.zeros(7)
        nv = max(self.views, 1)
        pvm, pvp = np.zeros(nv), np.zeros(nv)
        pc = np.zeros((max(self.num_classes, 1), 5))
        npc = C.c_uint64()
        self._ctx.check(N.lib.sgm_eval_report(self._ctx.handle, self.handle, N.dptr(summary),
                                              N.dptr(pvm), N.dptr(pvp), N.dptr(pc),
                                              C.byref(npc)))
        return MetricReport(
            *[float(v) for v in summary], per_view_miou=[float(v) for v in pvm[: self.views]],
            per_view_psnr=[float(v) for v in pvp[: self.views]],
            per_class=[PerClassMetric(int(r[0]), float(r[1]), float(r[2]), float(r[3]),
                                      int(r[4])) for r in pc[: npc.value]])


def evaluate(gmap: GaussianMap, camera: CameraModel, frames: Sequence[Frame],
             options: Optional[RenderOptions] = None,
             ctx: Optional[Context] = None) -> MetricReport:
    """semantic_metrics + photometric_metrics of `gmap` rendered at every frame's pose.
    Raises like the reference on no frames ("view count mismatch") or a frame whose size
    does not match the camera ("resolution mismatch")."""
    ev = Evaluator(gmap.num_classes(), ctx=ctx)
    for f in frames:
        ev.add_view(gmap, camera, f, options)
    return ev.report()


def semantic_metrics(gmap: GaussianMap, camera: CameraModel, frames: Sequence[Frame],
                     ctx: Optional[Context] = None) -> MetricReport:
    """evaluator.hpp semantic_metrics; the photometric fields are left at their defaults."""
    r = evaluate(gmap, camera, frames, ctx=ctx)
    return MetricReport(r.miou_pct, r.top1_pct, r.top3_pct, r.map_pct, r.f1_pct,
                        per_view_miou=r.per_view_miou, per_class=r.per_class)


def photometric_metrics(gmap: GaussianMap, camera: CameraModel, frames: Sequence[Frame],
                        ctx: Optional[Context] = None) -> MetricReport:
    """evaluator.hpp photometric_metrics (psnr_db, depth_l1_cm, per_view_psnr)."""
    r = evaluate(gmap, camera, frames, ctx=ctx)
    return MetricReport(psnr_db=r.psnr_db, depth_l1_cm=r.depth_l1_cm,
                        per_view_psnr=r.per_view_psnr)
