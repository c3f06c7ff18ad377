"""Candidate views scored/s for every BASELINE config on one B200, next to the reference's
own refresh_candidate_scores (oracle/_ref, compiled unmodified) on the host cores.

  python scripts/config_table.py [--cfgs 1,2,3,4] [--cpu-views 16] [--out profiles/x.json]

GPU: the config's full candidate set (cfg2: 1024, cfg3: 512, cfg4: 256, cfg1: 64 views), map
resident, CUDA events around score_poses, L2 flushed before the timed call, best of 3.
CPU: a bounded sample of the same candidates, one view per thread (RAM-bounded thread count).
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2506_00225_b200 import scenes  # noqa: E402
from paper_2506_00225_b200.splatmap import Context, score_poses  # noqa: E402


def mem_available_gb() -> float:
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemAvailable:"):
                return int(ln.split()[1]) / 1e6
    except OSError:
        pass
    return 16.0


def gpu_leg(ctx, cfg, flush, stream):
    import torch
    sc = scenes.CONFIGS[cfg]
    gm = scenes.make_map(cfg)
    cam = sc.camera()
    poses = [c.camera_pose() for c in scenes.make_candidates(cfg, sc.views)]
    score_poses(gm, cam, poses[: min(16, len(poses))], ctx=ctx)  # warm-up (upload, buffers)
    best = None
    for _ in range(3):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        ctx.reset_stats()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        nm, es = score_poses(gm, cam, poses, ctx=ctx)
        ev1.record(stream)
        ev1.synchronize()
        ms = ev0.elapsed_time(ev1)
        if best is None or ms < best[0]:
            best = (ms, ctx.stats(), nm, es)
    ms, st, nm, es = best
    v = len(poses)
    return gm, cam, {"views": v, "ms": ms, "views_per_s": v / (ms / 1e3),
                     "visible_per_view": st["visible"] / v, "pairs_per_view": st["pairs"] / v,
                     "contributors_per_view": st["contributors"] / v,
                     "argmax_entropy_view": int(np.argmax(es))}


def cpu_leg(gm, cam, cfg, views, pairs_per_view):
    import oracle
    ref = oracle.RefLib()
    px = cam.width * cam.height
    # the reference's RenderOutput plus its per-tile Probe bins (16 B per pair) per thread
    per_view_gb = px * (5 + gm.channels()) * 8 / 1e9 + 16 * pairs_per_view / 1e9 + 0.2
    threads = max(1, min(oracle.cpu_count(), views, int(mem_available_gb() * 0.7 // per_view_gb)))
    cands = scenes.make_candidates(cfg, threads)
    h = ref.map_create(gm)
    pos = np.array([c.position for c in cands])
    dirs = np.array([c.direction for c in cands])
    t0 = time.perf_counter()
    ref.refresh_scores(gm, cam, pos, dirs, threads=threads, handle=h)
    sec = time.perf_counter() - t0
    ref.map_destroy(h)
    return {"views": threads, "threads": threads, "seconds": sec, "views_per_s": threads / sec,
            "sec_per_view_per_core": sec}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfgs", default="1,2,3,4")
    ap.add_argument("--cpu-views", type=int, default=16)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    ctx = Context(0)
    ctx.set_profiling(True)
    stream = torch.cuda.ExternalStream(ctx.stream)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    rows = []
    for cfg in [int(c) for c in a.cfgs.split(",")]:
        gm, cam, g = gpu_leg(ctx, cfg, flush, stream)
        c = None if a.no_cpu else cpu_leg(gm, cam, cfg, a.cpu_views, g["pairs_per_view"])
        sc = scenes.CONFIGS[cfg]
        row = {"cfg": cfg, "name": sc.name, "N": gm.size(), "k": gm.k(), "C": gm.channels(),
               "resolution": f"{cam.width}x{cam.height}", "gpu": g, "cpu_reference": c,
               "ratio_vs_all_cores": None if c is None else g["views_per_s"] / c["views_per_s"],
               "ratio_vs_one_core": None if c is None else g["views_per_s"] * c["sec_per_view_per_core"]}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del gm
    if a.out:
        Path(a.out).write_text(json.dumps({"device": torch.cuda.get_device_name(0),
                                           "host_cores": os.cpu_count(), "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
