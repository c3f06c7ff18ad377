"""Candidate-view scoring benchmark (BASELINE.json metric: candidate views scored/sec).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 1]

A step = scoring one batch of candidate views of the config-1 scene (500k
Gaussians, 1200x680, k=16 of 101 classes): per view the exact-zero silhouette
count and the summed clipped entropy (refresh_candidate_scores, explorer.cpp:186-205),
64 views per GPU per step (weak scaling over ranks), followed by the all-gather
of per-view scores and combine_scores on every rank.

value : views/s with the map resident in HBM (device timeline, CUDA events on the
        library's stream, max over ranks, L2 flushed between steps).
e2e   : the same through the public API with host inputs: every step re-uploads the
        map from host memory (map version bump) and returns per-view scores to host.
--impl reference: the reference's own CPU code (oracle/_ref, compiled unmodified from
        the reference sources) on all usable host cores, same config and metric.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

VIEWS_PER_GPU = 64
METRIC = "candidate views scored/sec"
UNIT = "views/s"
DATA = "synthetic (seeded, BASELINE cfg%d)"
CURRENT_POSITION = np.array([4.0, 1.5, 3.0])  # combine_scores' current position (box centre)


def _mem_available_gb() -> float:
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable"):
                return int(line.split()[1]) / 1e6
    except OSError:
        pass
    return 16.0


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self._t:
            self._t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(smax)) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


REF_SAMPLE_MAX = 16  # views per reference step: a bounded sample (about 2.5 s per view per core)


def reference_threads() -> int:
    """Host threads for the reference: all usable cores, bounded by RAM (one 0.7 GB
    RenderOutput per concurrent cfg1 view) and by the sample size."""
    import oracle
    return max(1, min(oracle.cpu_count(), int(_mem_available_gb() // 1.5), REF_SAMPLE_MAX))


def assert_reference_alone() -> None:
    """The reference arm must not map the product library (libsgm_b200.so)."""
    try:
        maps = open("/proc/self/maps").read()
    except OSError:
        return
    if "libsgm_b200" in maps:
        raise RuntimeError("reference arm: libsgm_b200.so is mapped in this process")


def cpu_reference_run(gm, cam, cands, threads: int, steps: int = 1, warmup: int = 0, ref=None,
                      handle=None):
    """The reference's refresh_candidate_scores (oracle/_ref, compiled unmodified) over
    `cands`, the views split into disjoint spans over `threads` host threads.
    Returns (views/s, mean s per call, n_missing, entropy_sum)."""
    import oracle
    ref = ref or oracle.RefLib()
    h = handle or ref.map_create(gm)
    pos = np.array([c.position for c in cands])
    dirs = np.array([c.direction for c in cands])
    times = []
    nm = es = None
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        nm, es = ref.refresh_scores(gm, cam, pos, dirs, threads=threads, handle=h)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    if handle is None:
        ref.map_destroy(h)
    return len(cands) / float(np.mean(times)), float(np.mean(times)), nm, es


def reference_one_thread(gm, cam, cand, ref, handle) -> dict:
    """The reference as shipped: one thread (its candidate loop is serial,
    explorer.cpp:188), one cfg view."""
    v, sec, _, _ = cpu_reference_run(gm, cam, [cand], 1, 1, 0, ref=ref, handle=handle)
    return {"value": v, "unit": UNIT, "cores": 1, "sample": f"candidate view {cand.id}, "
            f"{sec:.2f} s"}


def compare_scores(nm_a, es_a, nm_b, es_b, positions, current, ref) -> dict:
    """Per-view parity of two score sets (a = ours, b = the reference) and of the
    combine_scores decision on them (the reference's own combine_scores for both)."""
    nm_a, es_a = np.asarray(nm_a, float), np.asarray(es_a, float)
    nm_b, es_b = np.asarray(nm_b, float), np.asarray(es_b, float)
    any_a, _, _, ta = ref.combine_scores(nm_a, es_a, positions, current)
    any_b, _, _, tb = ref.combine_scores(nm_b, es_b, positions, current)
    both_tiny = (np.abs(ta) < 1e-300) & (np.abs(tb) < 1e-300)  # SURVEY 8d parity rule
    rel_t = np.where(both_tiny, 0.0, np.abs(ta - tb) / np.maximum(np.abs(tb), 1e-300))
    order = lambda t: sorted(range(len(t)), key=lambda i: (-t[i], i))  # episode.cpp:410-414
    oa, ob = order(ta), order(tb)
    err = float(np.max(np.abs(es_a - es_b))) if len(es_a) else 0.0
    srt = np.sort(es_b)[::-1]
    return {"views": int(len(nm_a)),
            "n_missing_equal": bool(np.array_equal(nm_a, nm_b)),
            "entropy_max_rel": float(np.max(np.abs(es_a - es_b) / np.abs(es_b))) if len(es_b) else 0.0,
            "entropy_max_abs_nats": err,
            "i_total_max_rel": float(np.max(rel_t)) if len(rel_t) else 0.0,
            "argmax_equal": bool(oa[0] == ob[0]), "argmax": int(ob[0]),
            "order_equal": bool(oa == ob),
            "pool_exhausted": {"ours": not any_a, "reference": not any_b},
            "n_missing_min_max": [float(nm_b.min()), float(nm_b.max())],
            "top2_entropy_gap_nats": float(srt[0] - srt[1]) if len(srt) > 1 else None,
            "top2_i_total": [float(tb[ob[0]]), float(tb[ob[1]])] if len(tb) > 1 else None}


def run_reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    import oracle
    from paper_2506_00225_b200 import scenes  # scene / candidate geometry only: no product library
    threads = reference_threads()
    cfg = args.config
    gm = scenes.make_map(cfg)
    cam = scenes.CONFIGS[cfg].camera()
    # the first `threads` candidate views of the list the GPU arm scores (one per thread)
    cands = scenes.make_candidates(cfg, VIEWS_PER_GPU * args.gpus)[:threads]
    ref = oracle.RefLib()
    h = ref.map_create(gm)
    value, sec, nm, es = cpu_reference_run(gm, cam, cands, threads, args.steps, args.warmup,
                                           ref=ref, handle=h)
    one = reference_one_thread(gm, cam, cands[0], ref, h)
    dec = scenes.make_decision_candidates(cfg)
    dpos = np.array([c.position for c in dec])
    _, _, dnm, des = cpu_reference_run(gm, cam, dec, threads, 1, 0, ref=ref, handle=h)
    _, _, _, dt = ref.combine_scores(dnm, des, dpos, CURRENT_POSITION)
    ref.map_destroy(h)
    assert_reference_alone()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": DATA % cfg,
        "config": workload_config(cfg, args.gpus),
        "views_per_step": len(cands),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"candidate views 0..{len(cands) - 1} of the GPU arm's list, "
                                   f"one per thread, {_cpu_model()}",
                         "one_thread": one},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "product_library_mapped": False,
        "scores": {"ids": [c.id for c in cands], "n_missing": nm.tolist(),
                   "entropy_sum": es.tolist()},
        "decision": {"set": "make_decision_candidates(%d): 16 views seeing the cloud in part" % cfg,
                     "n_missing": dnm.tolist(), "entropy_sum": des.tolist(),
                     "argmax": int(min(range(len(dt)), key=lambda i: (-dt[i], i)))},
    }
    print(json.dumps(line), flush=True)


def measure_render(ctx, stream, flush, args) -> dict:
    """Full render (colour + depth + silhouette + 102-channel semantics, reference layout,
    fp64) of one frame: device-resident planes and through the host API (D2H included),
    for cfg0 (340x600, the paper's resolution) and cfg1 (680x1200); the reference's own
    render() on one host core beside each (the paper publishes 3.1 ms/frame at
    340x600x102 on an RTX A6000)."""
    import torch
    from paper_2506_00225_b200 import scenes
    from paper_2506_00225_b200.splatmap import RenderChannels, render, render_device
    out = {}
    for cfg in (0, 1):
        gm = scenes.make_map(cfg)
        cam = scenes.CONFIGS[cfg].camera()
        pose = scenes.render_poses(cfg, 1)[0]
        px = cam.pixel_count()
        C = gm.channels()
        planes = torch.empty(px * (5 + C), dtype=torch.float64, device="cuda")
        base = planes.data_ptr()
        ptrs = dict(sil_ptr=base, color_ptr=base + 8 * px, depth_ptr=base + 32 * px,
                    sem_ptr=base + 40 * px)
        ch = RenderChannels.all()
        for _ in range(3):
            render_device(gm, cam, pose, ch, ctx=ctx, **ptrs)
        ms = []
        for _ in range(max(3, args.steps)):
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            render_device(gm, cam, pose, ch, ctx=ctx, **ptrs)
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        render(gm, cam, pose, ch, ctx=ctx)
        t0 = time.perf_counter()
        reps = 2
        for _ in range(reps):
            render(gm, cam, pose, ch, ctx=ctx)
        host_ms = (time.perf_counter() - t0) * 1e3 / reps
        entry = {"device_ms": float(np.median(ms)), "e2e_host_ms": host_ms,
                 "planes_bytes": int(8 * px * (5 + C)),
                 "resolution": f"{cam.width}x{cam.height}x{C}"}
        if True:  # the reference's own render() on one host core (cfg1: a few seconds)
            try:
                import oracle
                ref = oracle.RefLib()
                h = ref.map_create(gm)
                ref.render(gm, cam, pose, 7, handle=h, n_map=gm.size())
                t0 = time.perf_counter()
                ref.render(gm, cam, pose, 7, handle=h, n_map=gm.size())
                entry["reference_cpu_1core_ms"] = (time.perf_counter() - t0) * 1e3
                ref.map_destroy(h)
            except Exception as exc:
                entry["reference_cpu_1core_ms"] = repr(exc)
        out[f"cfg{cfg}"] = entry
        del planes
    return out


def measure_mapping(ctx, args) -> dict:
    """The mapping caller of render: optimize_map iterations (render all(true) ->
    losses -> backward -> Adam) on the cfg1 map against two resident synthetic keyframes,
    timed with CUDA events on the library stream; the reference's own optimize_map on one
    host core beside it (one iteration)."""
    import torch
    from paper_2506_00225_b200 import scenes
    from paper_2506_00225_b200.mapper import DeviceFrame, MapperConfig, MapTrainer
    cfg = 1
    gm = scenes.make_map(cfg)
    cam = scenes.CONFIGS[cfg].camera()
    poses = scenes.render_poses(cfg, 2)
    frames = [scenes.make_frame(cfg, p, seed=i) for i, p in enumerate(poses)]
    dev = [DeviceFrame(f, ctx=ctx) for f in frames]
    mc = MapperConfig(prune_every=0)
    tr = MapTrainer(gm, ctx=ctx)
    tr.optimize(dev, cam, mc, 2)
    stream = torch.cuda.ExternalStream(ctx.stream)
    iters = 60  # MapperConfig::iters_per_step (mapper.hpp:23)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    hist = tr.optimize(dev, cam, mc, iters)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    out = {"ms_per_iter": ms / iters, "iters": iters, "frames": 2,
           "workload": "cfg1 map (500k Gaussians), 1200x680x102 keyframes, render all(true) + "
                       "mapping_loss + semantic_loss + backward + Adam per iteration",
           "loss_first_last": [hist[0].total(), hist[-1].total()]}
    try:
        import oracle
        ref = oracle.RefLib()
        t0 = time.perf_counter()
        ref.optimize_map(gm, frames, cam, mc, 1)
        out["reference_cpu_1core_ms_per_iter"] = (time.perf_counter() - t0) * 1e3
    except Exception as exc:
        out["reference_cpu_1core_ms_per_iter"] = repr(exc)
    return out


def workload_config(cfg: int, n_gpus: int) -> dict:
    """The workload both arms report (identical dicts, so the driver's same_config holds)."""
    from paper_2506_00225_b200 import scenes
    sc = scenes.CONFIGS[cfg]
    return {"workload": f"cfg{cfg} {sc.name}: {sc.n} Gaussians, {sc.width}x{sc.height} px, "
                        f"k={sc.k} of {sc.num_classes} classes, candidate views",
            "seed": sc.seed, "box_m": list(sc.box),
            "candidates": f"make_candidates({cfg}): {VIEWS_PER_GPU} views per GPU per step on the "
                          f"GPU arm; the reference arm times the first views of the same list",
            "l2": "flushed (256 MiB write) between timed steps",
            "isotropic": "log_radius = mean of 3 per-axis log-scale draws (SURVEY App. A)",
            "gain": "reference Eq.6-8 (n_missing, clipped-entropy sum, combine_scores)",
            "parallelism": f"dp{n_gpus}: candidate views sharded over ranks (GPU arm) or host "
                           f"threads (reference arm); map replicated"}


def measure_aniso(ctx, stream, flush, args, cfg, cam, poses) -> dict:
    """The same candidate views scored with anisotropic EWA footprints (no
    reference counterpart): the config's drawn per-axis log-scales and quaternions."""
    import torch

    from paper_2506_00225_b200 import scenes
    from paper_2506_00225_b200.splatmap import score_poses

    gma = scenes.make_map(cfg, aniso=True)
    for _ in range(max(1, args.warmup)):
        score_poses(gma, cam, poses, ctx=ctx)
    ctx.reset_stats()
    ms = []
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        score_poses(gma, cam, poses, ctx=ctx)
        ev1.record(stream)
        ev1.synchronize()
        ms.append(ev0.elapsed_time(ev1))
    st = ctx.stats()
    views = max(1, st["views"])
    return {"views_per_s": len(poses) * args.steps / (float(np.sum(ms)) / 1e3),
            "ms_per_step": float(np.mean(ms)),
            "visible_per_view": st["visible"] / views, "pairs_per_view": st["pairs"] / views,
            "contributors_per_view": st["contributors"] / views,
            "footprint": "EWA: Sigma2D = J R_cw Sigma R_cw^T J^T, alpha exp(-q/2), q <= trunc^2; "
                         "Sigma from the config's per-axis log-scales and quaternions"}


def measure_dense(ctx, stream, flush) -> dict:
    """cfg4 (dense overlap: 1M Gaussians in a 1 m cube, k = 32 of 102, 1.19 G tile pairs per
    view) on 32 of its candidate views: the depth-prefix binning and tensor-memory path."""
    import torch
    from paper_2506_00225_b200 import scenes
    from paper_2506_00225_b200.splatmap import score_poses
    gm4 = scenes.make_map(4)
    cam4 = scenes.CONFIGS[4].camera()
    poses4 = [c.camera_pose() for c in scenes.make_candidates(4, 32)]
    ctx.upload(gm4)
    score_poses(gm4, cam4, poses4, ctx=ctx)  # warm-up (scratch sized)
    ms = []
    for _ in range(2):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)  # evict L2 (outside the events)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        nm, es = score_poses(gm4, cam4, poses4, ctx=ctx)
        ev1.record(stream)
        ev1.synchronize()
        ms.append(ev0.elapsed_time(ev1))
    ctx.reset_stats()
    score_poses(gm4, cam4, poses4, ctx=ctx)
    st = ctx.stats()
    t = float(np.mean(ms))
    return {"config": "cfg4 dense overlap: 1M Gaussians in a 1 m cube, 1200x680, k = 32 of 102, "
                      "32 candidate views 1.2 m from the centre",
            "views": len(poses4), "views_per_s": len(poses4) / (t / 1e3), "ms_per_pass": t,
            "pairs_per_view": st["pairs"] / len(poses4),
            "contributors_per_view": st["contributors"] / len(poses4),
            "n_missing_sum": float(np.sum(nm)), "entropy_sum_total": float(np.sum(es))}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--force-dist", action="store_true",
                    help="use the torch.distributed path (NCCL broadcast / all-gather) even at N=1")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch
    import torch.distributed as tdist

    from paper_2506_00225_b200 import dist as sd
    from paper_2506_00225_b200 import scenes
    from paper_2506_00225_b200.splatmap import (Context, combine_scores,
                                                refresh_candidate_scores, score_poses)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    dist_on = world > 1 or args.force_dist
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if dist_on:
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))

    cfg = args.config
    sc = scenes.CONFIGS[cfg]
    cam = sc.camera()
    n_total = VIEWS_PER_GPU * world
    cands = scenes.make_candidates(cfg, n_total)
    s, e = sd.shard_range(n_total, rank, world)
    mine = cands[s:e]
    poses = [c.camera_pose() for c in mine]

    ctx = Context(local)
    gm_host = scenes.make_map(cfg) if rank == 0 else None  # the host map lives on rank 0
    if dist_on:
        # C1: rank 0 uploads once; its device snapshot goes device to device over NCCL;
        # the other ranks score a DeviceMap
        gm = sd.broadcast_map(gm_host, ctx)
    else:
        gm = gm_host
        ctx.upload(gm)
    stream = torch.cuda.ExternalStream(ctx.stream)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def barrier():
        if dist_on:
            tdist.barrier()
        torch.cuda.synchronize()

    def step_resident():
        nm, es = score_poses(gm, cam, poses, ctx=ctx)
        if dist_on:
            nm, es = sd.gather_scores(n_total, nm, es)
        return nm, es

    for _ in range(args.warmup):
        step_resident()
    ctx.reset_stats()
    ctx.set_profiling(True)
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    step_ms = []
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)  # evict L2 between timed steps (outside the events)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        nm_all, es_all = step_resident()
        ev1.record(stream)
        ev1.synchronize()
        step_ms.append(ev0.elapsed_time(ev1))
    barrier()
    clk = clocks.stop()
    st = ctx.stats()
    ctx.set_profiling(False)
    total_ms = float(np.sum(step_ms))
    if dist_on:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = n_total * args.steps / (total_ms / 1e3)

    # all ranks agree on the argmax (combine_scores on the gathered records)
    for c, a, b in zip(cands, nm_all, es_all):
        c.n_missing, c.entropy_sum = float(a), float(b)
    combine_scores(cands, CURRENT_POSITION)
    best = max(range(n_total), key=lambda i: (cands[i].i_total, -i))

    # ---- cfg1 with the Fisher-information gain: prior from 32 past poses,
    #      then the same candidates scored with n_missing + entropy + Fisher gain ----
    fisher = None
    try:
        from paper_2506_00225_b200.splatmap import fisher_prior, score_poses_fisher
        prior_poses = [c.camera_pose() for c in scenes.make_candidates(cfg, 32, stream=2)]
        prior_times = []
        for _ in range(2):  # the first call allocates the prior buffers: time the second
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            if dist_on:  # past poses sharded over the ranks, H all-reduced
                sd.fisher_prior_sharded(gm, cam, prior_poses, lam=1.0, ctx=ctx)
            else:
                fisher_prior(gm, cam, prior_poses, lam=1.0, ctx=ctx)
            ev1.record(stream)
            ev1.synchronize()
            prior_times.append(ev0.elapsed_time(ev1))
        prior_ms = prior_times[-1]
        for _ in range(max(1, args.warmup)):
            score_poses_fisher(gm, cam, poses, ctx=ctx)
        f_ms = []
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            _, _, gains = score_poses_fisher(gm, cam, poses, ctx=ctx)
            ev1.record(stream)
            ev1.synchronize()
            f_ms.append(ev0.elapsed_time(ev1))
        # the combined scalar gain (fisher + entropy) and the ranking that uses it (a14)
        from paper_2506_00225_b200.splatmap import CandidatePose, combine_scores_fisher
        _, esf, _ = score_poses_fisher(gm, cam, poses, ctx=ctx)
        fc = [CandidatePose(position=c.position, direction=c.direction, entropy_sum=float(esf[i]),
                            fisher_gain=float(gains[i]), id=c.id) for i, c in enumerate(mine)]
        combine_scores_fisher(fc, CURRENT_POSITION, w_sem=1.0)
        ranked = sorted(fc, key=lambda c: (-c.i_gain, c.id))
        fisher = {"views_per_s": len(poses) * args.steps / (float(np.sum(f_ms)) / 1e3),
                  "argmax_view_combined_gain": int(ranked[0].id),
                  "top2_i_gain": [ranked[0].i_gain, ranked[1].i_gain] if len(ranked) > 1 else None,
                  "combined_gain": "gain = fisher_gain + 1.0 * entropy_sum; i_gain = (1 - "
                                   "softmax(|pos - current|)) * softmax(ln gain); rank i_gain desc, "
                                   "id asc (sgm_combine_scores_fisher)",
                  "ms_per_step": float(np.mean(f_ms)), "prior_poses": len(prior_poses),
                  "prior_ms": prior_ms, "lambda": 1.0,
                  "gain": "sum_{i,theta} H_view / (H_prior + lambda), theta = mu xyz, log_r, "
                          "logit, rgb; channels R,G,B,depth"}
    except Exception as exc:  # reported, not fatal
        fisher = {"error": repr(exc)}

    # ---- secondary metric: semantic render ms/frame (device-resident and e2e) ----
    render_info = None
    mapping_info = None
    aniso_info = None
    if rank == 0:
        try:
            aniso_info = measure_aniso(ctx, stream, flush, args, cfg, cam, poses)
        except Exception as exc:  # reported, not fatal
            aniso_info = {"error": repr(exc)}
        try:
            render_info = measure_render(ctx, stream, flush, args)
        except Exception as exc:  # reported, not fatal
            render_info = {"error": repr(exc)}
        try:
            mapping_info = measure_mapping(ctx, args)
        except Exception as exc:  # reported, not fatal
            mapping_info = {"error": repr(exc)}

    # ---- cfg2: the candidate sweep, the cfg1 map from 1024 lattice poses sharded over the
    #      ranks (strong scaling: the same 1024 views at every N) ----
    sweep = None
    if cfg == 1:
        sw = scenes.make_candidates(2)
        ss, se = sd.shard_range(len(sw), rank, world)
        sw_poses = [c.camera_pose() for c in sw[ss:se]]
        score_poses(gm, cam, sw_poses, ctx=ctx)  # warm-up (scratch sized for the sweep)
        sw_ms = []
        for _ in range(2):
            barrier()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            snm, ses = score_poses(gm, cam, sw_poses, ctx=ctx)
            if dist_on:
                snm, ses = sd.gather_scores(len(sw), snm, ses)
            ev1.record(stream)
            ev1.synchronize()
            sw_ms.append(ev0.elapsed_time(ev1))
        t_sw = float(np.mean(sw_ms))
        if dist_on:
            t = torch.tensor([t_sw], dtype=torch.float64, device="cuda")
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            t_sw = float(t.item())
        for c, a, b in zip(sw, snm, ses):
            c.n_missing, c.entropy_sum = float(a), float(b)
        combine_scores(sw, CURRENT_POSITION)
        sweep = {"config": "cfg2 candidate sweep: the cfg1 map, 16 x 8 lattice at 0.25 m "
                           "(y = 1.4 m) x 8 yaws = 1024 views, sharded over the ranks",
                 "scaling": "strong", "views": len(sw), "views_per_s": len(sw) / (t_sw / 1e3),
                 "ms_per_pass": t_sw, "n_gpus": world,
                 "argmax_view": int(max(range(len(sw)), key=lambda i: (sw[i].i_total, -i))),
                 "n_missing_all_zero": bool(np.all(np.asarray(snm) == 0))}

    # ---- cfg4: dense views (rank 0; a secondary leg) ----
    dense_info = None
    if rank == 0 and cfg == 1:
        try:
            dense_info = measure_dense(ctx, stream, flush)
        except Exception as exc:  # reported, not fatal
            dense_info = {"error": repr(exc)}

    # ---- e2e through the public API (host inputs, map re-upload every step; at N > 1 rank 0
    #      uploads and broadcasts the device snapshot, the others import it) ----
    h2d = (int(gm_host.centers.nbytes + gm_host.log_radii.nbytes + gm_host.opacity_logits.nbytes +
               gm_host.colors.nbytes + gm_host.sem_indices.nbytes + gm_host.sem_probs.nbytes)
           if gm_host is not None else 0) + 96 * len(mine)
    d2h = 16 * len(mine)
    e2e_ms = []
    for i in range(args.warmup + args.steps):
        if gm_host is not None:
            gm_host.touch()
        fresh = [type(c)(position=c.position, direction=c.direction, id=c.id) for c in mine]
        barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        gm_e = sd.broadcast_map(gm_host, ctx) if dist_on else gm_host
        refresh_candidate_scores(fresh, gm_e, cam, ctx=ctx)
        if dist_on:
            sd.gather_scores(n_total, np.array([c.n_missing for c in fresh]),
                             np.array([c.entropy_sum for c in fresh]))
        ev1.record(stream)
        ev1.synchronize()
        if i >= args.warmup:
            e2e_ms.append(ev0.elapsed_time(ev1))
    e2e_total = float(np.sum(e2e_ms))
    if dist_on:
        t = torch.tensor([e2e_total], dtype=torch.float64, device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = n_total * args.steps / (e2e_total / 1e3)

    # ---- roofline of the dominant kernel (raster-score) ----
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except (OSError, ValueError):
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    raster_launches = max(1, st["raster_launches"])
    raster_ms = st["raster_ms"] / raster_launches
    views_timed = st["views"]
    per_launch_views = views_timed / raster_launches
    vis_per_view = st["visible"] / max(1, views_timed)
    N = gm.size()
    k = gm.k()
    alg_bytes = per_launch_views * (20.0 * N + 6.0 * k * vis_per_view + 16.0)
    achieved = alg_bytes / (raster_ms * 1e-3) / 1e9
    traffic = None
    prof_json = ROOT / "profiles" / "raster_traffic.json"
    if prof_json.exists():
        try:
            traffic = json.loads(prof_json.read_text()).get("dram_bytes_per_launch")
        except ValueError:
            traffic = None
    clock_ghz = (clk.get("sm_mhz") or 1965.0) / 1e3
    smem_peak = 148 * 128 * clock_ghz  # GB/s, LDS/STS crossbar
    K_per_launch = st["contributors"] / raster_launches
    smem_bytes = K_per_launch * 2 * k * 8  # fp64 read+write per sparse scatter
    # ncu counters of one raster launch (profiles/, newest round): the pipes that bound it
    ncu, ncu_src = {}, None
    for cand in sorted(ROOT.glob("profiles/r*_raster_summary.json"), reverse=True):
        try:
            ncu, ncu_src = json.loads(cand.read_text()), str(cand.relative_to(ROOT))
            break
        except ValueError:
            continue
    K_view = st["contributors"] / max(1, views_timed)
    # the fp64 accumulator floor: one 8-byte read + one 8-byte write of shared memory per
    # (pixel, class) update, k updates per contributor, at the crossbar rate
    floor_ms_view = 16.0 * k * K_view / (smem_peak * 1e9) * 1e3
    roofline = {"bound": "lsu", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic,
                "kernel": "k_raster<score> (K5)", "raster_ms_per_launch": raster_ms,
                "views_per_launch": per_launch_views,
                "algorithmic_bytes_per_view": "20*N + 6*k*V + 16 (SURVEY 8d)",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)",
                "binding_pipe": "LSU data pipe: shared-memory wavefronts of the fp64 semantic "
                                "accumulator, the staged weights and rows (not HBM: achieved/peak "
                                "above is the HBM fraction the contract asks for)",
                "lsu_data_pipe_frac": (ncu.get("lsu_data_pipe_pct") or 0.0) / 100.0 or None,
                "lsu_shared_pipe_frac": (ncu.get("smem_pipe_pct") or 0.0) / 100.0 or None,
                "issue_active_frac": (ncu.get("issue_active_pct") or 0.0) / 100.0 or None,
                "fp64_pipe_frac": (ncu.get("fp64_pipe_pct") or 0.0) / 100.0 or None,
                "ncu_source": ncu_src,
                "fp64_accumulator_floor_ms_per_view": floor_ms_view,
                "fp64_accumulator_floor_views_per_s": 1e3 / floor_ms_view if floor_ms_view else None,
                "floor_note": "16 B x k x K per view at 148 SMs x 128 B/clk (LDS/STS crossbar) "
                              "at the sampled SM clock; K = contributors per view"}
    roofline_aux = {"smem_rmw_GBps": smem_bytes / (raster_ms * 1e-3) / 1e9,
                    "smem_peak_GBps": smem_peak,
                    "smem_rmw_frac": (smem_bytes / (raster_ms * 1e-3) / 1e9) / smem_peak,
                    "contributors_per_view": K_view,
                    "visible_per_view": vis_per_view,
                    "pairs_per_view": st["pairs"] / max(1, views_timed),
                    "batch_span_ms_per_raster_launch": st["binning_ms"] / raster_launches}

    # ---- the decision on a candidate set with varying n_missing (every cfg1 headline view
    #      has n_missing = 0, so its i_total is 0 and combine_scores reports exhaustion) ----
    dec = scenes.make_decision_candidates(cfg)
    dec_poses = [c.camera_pose() for c in dec]
    dnm, des = score_poses(gm, cam, dec_poses, ctx=ctx)
    for c, a_, b_ in zip(dec, dnm, des):
        c.n_missing, c.entropy_sum = float(a_), float(b_)
    combine_scores(dec, CURRENT_POSITION)
    dec_total = [c.i_total for c in dec]

    cpu_baseline = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle
            ref = oracle.RefLib()
            threads = reference_threads()
            sample = cands[:threads]
            h = ref.map_create(gm)
            v, sec, rnm, res = cpu_reference_run(gm, cam, sample, threads, 1, 0, ref=ref, handle=h)
            one = reference_one_thread(gm, cam, sample[0], ref, h)
            _, _, rdnm, rdes = cpu_reference_run(gm, cam, dec, threads, 1, 0, ref=ref, handle=h)
            ref.map_destroy(h)
            cpu_baseline = {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                            "sample": f"candidate views 0..{threads - 1} of this run's list, one "
                                      f"per thread, {sec:.1f} s, {_cpu_model()}",
                            "one_thread": one}
            pos = np.array([c.position for c in sample])
            dpos = np.array([c.position for c in dec])
            parity = {
                "reference": "oracle/_ref: the reference's refresh_candidate_scores and "
                             "combine_scores compiled unmodified, on the same views",
                "headline_views": dict(compare_scores(nm_all[:threads], es_all[:threads], rnm,
                                                      res, pos, CURRENT_POSITION, ref),
                                       note="every cfg1 headline view sees the cloud at every "
                                            "pixel: n_missing = 0, so i_geo = i_total = 0 and "
                                            "combine_scores returns false (pool exhausted); "
                                            "the argmax is the id tie-break"),
                "decision_views": dict(compare_scores(dnm, des, rdnm, rdes, dpos,
                                                      CURRENT_POSITION, ref),
                                       set="make_decision_candidates(%d): 16 views seeing the "
                                           "cloud in part (n_missing varies)" % cfg)}
            hv, dv = parity["headline_views"], parity["decision_views"]
            parity["all_equal"] = bool(hv["n_missing_equal"] and dv["n_missing_equal"] and
                                       hv["argmax_equal"] and dv["argmax_equal"] and
                                       max(hv["entropy_max_rel"], dv["entropy_max_rel"]) < 1e-9 and
                                       max(hv["i_total_max_rel"], dv["i_total_max_rel"]) < 1e-3)
        except Exception as exc:  # reported, not fatal
            cpu_baseline = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                            "sample": f"failed: {exc!r}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": DATA % cfg,
            "config": workload_config(cfg, world),
            "views_per_step": n_total,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": int(st["kernel_launches"]),
            "roofline": roofline, "roofline_aux": roofline_aux,
            "cpu_baseline": cpu_baseline, "clocks": clk,
            "parity": parity,
            "headline_n_missing_all_zero": bool(np.all(np.asarray(nm_all) == 0)),
            "argmax_view": int(best),
            "decision_argmax_view": int(max(range(len(dec)), key=lambda i: (dec_total[i], -i))),
            "with_fisher_gain": fisher,
            "render_ms_per_frame": render_info,
            "mapping_optimize": mapping_info,
            "anisotropic_ewa": aniso_info,
            "cfg2_sweep": sweep,
            "cfg4_dense": dense_info,
        }
        print(json.dumps(line), flush=True)
    if dist_on:
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
