"""Kernel timeline of one scoring call (CUPTI activity records through torch.profiler: every
kernel of the process, ours included), reduced to where the step's time goes: raster busy,
other kernels running while no raster runs (exposed binning), and idle gaps.
  python scripts/timeline.py --config 1 --views 64"""
import argparse
import sys
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2506_00225_b200 import scenes  # noqa: E402
from paper_2506_00225_b200.splatmap import Context, score_poses  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--views", type=int, default=64)
ap.add_argument("--top", type=int, default=14)
ap.add_argument("--fisher", action="store_true", help="the Fisher-gain scoring (prior from 32 poses)")
a = ap.parse_args()
torch.cuda.init()
ctx = Context(0)
gm = scenes.make_map(a.config)
cam = scenes.CONFIGS[a.config].camera()
poses = [c.camera_pose() for c in scenes.make_candidates(a.config, a.views)]
ctx.upload(gm)
if a.fisher:
    from paper_2506_00225_b200.splatmap import fisher_prior, score_poses_fisher
    fisher_prior(gm, cam, [c.camera_pose() for c in scenes.make_candidates(a.config, 32, stream=2)], ctx=ctx)
    run = lambda: score_poses_fisher(gm, cam, poses, ctx=ctx)  # noqa: E731
else:
    run = lambda: score_poses(gm, cam, poses, ctx=ctx)  # noqa: E731
for _ in range(2):
    run()
ctx.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run()
    ctx.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ks = []
for e in ev:
    t0 = e.time_range.start
    t1 = e.time_range.end
    if t1 > t0:
        ks.append((t0, t1, e.name))
ks.sort()
T0, T1 = min(k[0] for k in ks), max(k[1] for k in ks)


def union(iv):
    iv = sorted(iv)
    tot, cs, ce = 0.0, None, None
    out = []
    for s, e in iv:
        if cs is None or s > ce:
            if cs is not None:
                out.append((cs, ce))
            cs, ce = s, e
        else:
            ce = max(ce, e)
    if cs is not None:
        out.append((cs, ce))
    return out


def length(iv):
    return sum(e - s for s, e in iv)


ras = union([(s, e) for s, e, n in ks if "k_raster" in n or "k_fisher" in n])
alls = union([(s, e) for s, e, n in ks])
span = T1 - T0
print(f"cfg{a.config} {a.views} views: span {span / 1e3:.2f} ms, raster busy {length(ras) / 1e3:.2f} ms, "
      f"any kernel busy {length(alls) / 1e3:.2f} ms, idle {(span - length(alls)) / 1e3:.2f} ms, "
      f"non-raster only {(length(alls) - length(ras)) / 1e3:.2f} ms, kernels {len(ks)}")
# per kernel family: time running while no raster runs (exposed)
import collections
import re
exp = collections.Counter()
tot = collections.Counter()
j = 0
for s, e, n in ks:
    m = re.search(r"(k_\w+)", n)
    key = m.group(1) if m else n[:40]
    tot[key] += e - s
    if "k_raster" in n:
        continue
    # overlap of [s, e) with the raster union
    ov = 0.0
    for rs, re_ in ras:
        if re_ <= s:
            continue
        if rs >= e:
            break
        ov += min(e, re_) - max(s, rs)
    exp[key] += (e - s) - ov
print("busy per family: " + ", ".join(f"{k} {v / 1e3:.2f} ms" for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:4]))
print("| kernel | total ms | exposed (no raster running) ms |\n|---|---|---|")
for k, v in sorted(tot.items(), key=lambda kv: -exp[kv[0]])[: a.top]:
    print(f"| {k} | {v / 1e3:.3f} | {exp[k] / 1e3:.3f} |")
# the first raster's start and gaps between consecutive rasters
print(f"first raster starts {(ras[0][0] - T0) / 1e3:.2f} ms after the first kernel; raster gaps "
      f"{[round((ras[i + 1][0] - ras[i][1]) / 1e3, 3) for i in range(len(ras) - 1)][:12]}")
