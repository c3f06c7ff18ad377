"""Times the Fisher-gain leg of bench.py on cfg1 (prior from 32 poses, then 64 views scored
with the gain) for A/B comparisons of k_fisher variants.
  python scripts/time_fisher.py [--views 64] [--repeat 3]"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2506_00225_b200 import scenes  # noqa: E402
from paper_2506_00225_b200.splatmap import Context, fisher_prior, score_poses_fisher  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, default=64)
    ap.add_argument("--repeat", type=int, default=3)
    a = ap.parse_args()
    import torch
    gm = scenes.make_map(1)
    cam = scenes.CONFIGS[1].camera()
    ctx = Context(0)
    ctx.upload(gm)
    prior = [c.camera_pose() for c in scenes.make_candidates(1, 32, stream=2)]
    poses = [c.camera_pose() for c in scenes.make_candidates(1, a.views)]
    times, gt = [], []
    for i in range(a.repeat + 1):  # (the calls return results to the host: synchronous)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fisher_prior(gm, cam, prior, lam=1.0, ctx=ctx)
        t1 = time.perf_counter()
        if i:
            times.append(1e3 * (t1 - t0))
    for i in range(a.repeat + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, _, gains = score_poses_fisher(gm, cam, poses, ctx=ctx)
        t1 = time.perf_counter()
        if i:
            gt.append(1e3 * (t1 - t0))
    g = np.asarray(gains, dtype=np.float64)
    print(f"fisher prior (32 poses): {np.mean(times):.2f} ms; gain {a.views} views: {np.mean(gt):.2f} ms "
          f"{a.views / (np.mean(gt) / 1e3):.1f} views/s  sum(gain)={g.sum():.12e}")


if __name__ == "__main__":
    main()
