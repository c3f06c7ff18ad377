"""Times candidate-view scoring (score_poses) on a config with the map resident and
prints per-view results for A/B comparisons between kernel variants.

  python scripts/time_score.py --config 1 --views 64 --repeat 5 [--dump out.npz]
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2506_00225_b200 import scenes  # noqa: E402
from paper_2506_00225_b200.splatmap import Context, score_poses  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--views", type=int, default=64)
    ap.add_argument("--repeat", type=int, default=5)
    ap.add_argument("--dump", default="")
    a = ap.parse_args()
    import torch
    gm = scenes.make_map(a.config)
    cam = scenes.CONFIGS[a.config].camera()
    cands = scenes.make_candidates(a.config, a.views)
    poses = [c.camera_pose() for c in cands]
    ctx = Context(0)
    ctx.upload(gm)
    nm, es = score_poses(gm, cam, poses, ctx=ctx)  # warm-up
    times = []
    for _ in range(a.repeat):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        nm, es = score_poses(gm, cam, poses, ctx=ctx)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.median(times))
    print(f"cfg{a.config} {a.views} views: {ms:.2f} ms/step  {a.views / ms * 1e3:.1f} views/s  "
          f"sum(entropy)={float(np.sum(es)):.12e} sum(missing)={float(np.sum(nm)):.0f}", flush=True)
    print(ctx.stats())
    if a.dump:
        np.savez(a.dump, n_missing=nm, entropy_sum=es)


if __name__ == "__main__":
    main()
