"""Small driver for ncu: scores `--views` cfg views once (one raster launch).

  python scripts/profile_raster.py --config 1 --views 8
"""
import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2506_00225_b200 import scenes  # noqa: E402
from paper_2506_00225_b200.splatmap import Context, score_poses  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--views", type=int, default=8)
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--fisher", action="store_true", help="profile the Fisher-gain path")
    a = ap.parse_args()
    gm = scenes.make_map(a.config)
    cam = scenes.CONFIGS[a.config].camera()
    poses = scenes.render_poses(a.config, a.views)
    ctx = Context(0)
    ctx.upload(gm)
    ctx.set_profiling(True)
    if a.fisher:
        from paper_2506_00225_b200.splatmap import fisher_prior, score_poses_fisher
        fisher_prior(gm, cam, poses[:2], ctx=ctx)
    for _ in range(a.repeat):
        t0 = time.perf_counter()
        if a.fisher:
            score_poses_fisher(gm, cam, poses, ctx=ctx)
        else:
            nm, es = score_poses(gm, cam, poses, ctx=ctx)
        print(f"{a.views} views in {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    print(ctx.stats())


if __name__ == "__main__":
    main()
