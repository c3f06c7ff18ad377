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


def cpu_reference_run(cfg: int, views: int, threads: int, steps: int = 1, warmup: int = 0):
    """The reference's refresh_candidate_scores (oracle/_ref) on host cores."""
    import oracle
    from paper_2506_00225_b200 import scenes
    ref = oracle.RefLib()
    gm = scenes.make_map(cfg)
    cam = scenes.CONFIGS[cfg].camera()
    cands = scenes.make_candidates(cfg, views)
    h = ref.map_create(gm)
    pos = np.array([c.position for c in cands])
    dirs = np.array([c.direction for c in cands])
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        ref.refresh_scores(gm, cam, pos, dirs, threads=threads, handle=h)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    ref.map_destroy(h)
    return views / float(np.mean(times)), float(np.mean(times))


def run_reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    import oracle
    cores = oracle.cpu_count()
    # one 0.7 GB RenderOutput per concurrent view in the reference: bound by RAM
    threads = max(1, min(cores, int(_mem_available_gb() // 1.5), 64))
    views = threads  # one view per thread per step: a bounded sample of the workload
    value, sec = cpu_reference_run(args.config, views, threads, args.steps, args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.config),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{views} cfg{args.config} candidate views per step "
                                   f"(one per thread), {_cpu_model()}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
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


def workload_config(cfg: int) -> dict:
    from paper_2506_00225_b200 import scenes
    sc = scenes.CONFIGS[cfg]
    return {"workload": f"cfg{cfg} {sc.name}: {sc.n} Gaussians in {sc.box[0]:g}x{sc.box[1]:g}x"
                        f"{sc.box[2]:g} m, {sc.width}x{sc.height} px, k={sc.k} of "
                        f"{sc.num_classes} classes ({sc.num_classes + 1} channels), "
                        f"{VIEWS_PER_GPU} candidate views per GPU per step",
            "seed": sc.seed, "views_per_gpu_per_step": VIEWS_PER_GPU,
            "l2": "flushed (256 MiB write) between timed steps",
            "isotropic": "log_radius = mean of 3 per-axis log-scale draws (SURVEY App. A)",
            "gain": "reference Eq.6-8 (n_missing, clipped-entropy sum, combine_scores)"}


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
    gm = scenes.make_map(cfg) if rank == 0 else None
    if dist_on:
        gm = sd.broadcast_map(gm)  # C1 over NCCL
    n_total = VIEWS_PER_GPU * world
    cands = scenes.make_candidates(cfg, n_total)
    s, e = sd.shard_range(n_total, rank, world)
    mine = cands[s:e]
    poses = [c.camera_pose() for c in mine]

    ctx = Context(local)
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
    combine_scores(cands, np.array([4.0, 1.5, 3.0]))
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
        fisher = {"views_per_s": len(poses) * args.steps / (float(np.sum(f_ms)) / 1e3),
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

    # ---- e2e through the public API (host inputs, map re-upload every step) ----
    h2d = int(gm.centers.nbytes + gm.log_radii.nbytes + gm.opacity_logits.nbytes +
              gm.colors.nbytes + gm.sem_indices.nbytes + gm.sem_probs.nbytes) + 96 * len(mine)
    d2h = 16 * len(mine)
    e2e_ms = []
    for i in range(args.warmup + args.steps):
        gm.touch()
        fresh = [type(c)(position=c.position, direction=c.direction, id=c.id) for c in mine]
        barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        refresh_candidate_scores(fresh, gm, cam, ctx=ctx)
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
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic,
                "kernel": "k_raster<score> (K5)", "raster_ms_per_launch": raster_ms,
                "views_per_launch": per_launch_views,
                "algorithmic_bytes_per_view": "20*N + 6*k*V + 16 (SURVEY 8d)",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)"}
    ncu = {}
    prof_sum = ROOT / "profiles" / "r01_raster_summary.json"
    if prof_sum.exists():
        try:
            ncu = json.loads(prof_sum.read_text())
        except ValueError:
            ncu = {}
    roofline_aux = {"ncu_lsu_shared_pipe_frac": (ncu.get("smem_pipe_pct") or 0.0) / 100.0 or None,
                    "ncu_lsu_data_pipe_frac": (ncu.get("lsu_data_pipe_pct") or 0.0) / 100.0 or None,
                    "ncu_issue_active_frac": (ncu.get("issue_active_pct") or 0.0) / 100.0 or None,
                    "ncu_source": "profiles/r01_raster_summary.json (ncu --set full, one raster "
                                  "launch of 8 cfg1 views): the pipes that bound this kernel",
                    "smem_rmw_GBps": smem_bytes / (raster_ms * 1e-3) / 1e9,
                    "smem_peak_GBps": smem_peak,
                    "smem_frac": (smem_bytes / (raster_ms * 1e-3) / 1e9) / smem_peak,
                    "contributors_per_view": st["contributors"] / max(1, views_timed),
                    "visible_per_view": vis_per_view,
                    "pairs_per_view": st["pairs"] / max(1, views_timed),
                    "batch_span_ms_per_raster_launch": st["binning_ms"] / raster_launches}

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle
            cores = oracle.cpu_count()
            threads = max(1, min(cores, int(_mem_available_gb() // 1.5), 64))
            v, sec = cpu_reference_run(cfg, threads, threads, 1, 0)
            cpu_baseline = {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                            "sample": f"{threads} cfg{cfg} candidate views, one per thread, "
                                      f"{sec:.1f} s, {_cpu_model()}"}
        except Exception as exc:  # reported, not fatal
            cpu_baseline = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                            "sample": f"failed: {exc!r}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE cfg%d)" % cfg,
            "config": dict(workload_config(cfg),
                           parallelism=f"dp{world}: candidate views sharded over the ranks, map "
                                       f"replicated (NCCL broadcast), per-view scores all-gathered"),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": int(st["kernel_launches"]),
            "roofline": roofline, "roofline_aux": roofline_aux,
            "cpu_baseline": cpu_baseline, "clocks": clk,
            "argmax_view": int(best), "views_total_per_step": n_total,
            "with_fisher_gain": fisher,
            "render_ms_per_frame": render_info,
            "mapping_optimize": mapping_info,
            "anisotropic_ewa": aniso_info,
        }
        print(json.dumps(line), flush=True)
    if dist_on:
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
