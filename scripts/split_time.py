"""Raster vs binning time of score_poses on a config (profiling counters of the library).
  python scripts/split_time.py --config 3 --views 32"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2506_00225_b200 import scenes  # noqa: E402
from paper_2506_00225_b200.splatmap import Context, score_poses  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--views", type=int, default=32)
a = ap.parse_args()
ctx = Context(0)
gm = scenes.make_map(a.config)
cam = scenes.CONFIGS[a.config].camera()
poses = [c.camera_pose() for c in scenes.make_candidates(a.config, a.views)]
score_poses(gm, cam, poses, ctx=ctx)  # warm-up: buffers at steady-state size
ctx.set_profiling(True)
ctx.reset_stats()
ctx.synchronize()
t = time.perf_counter()
score_poses(gm, cam, poses, ctx=ctx)
ctx.synchronize()
st = ctx.stats()
print(f"cfg{a.config} {a.views} views: wall {1e3 * (time.perf_counter() - t):.1f} ms, raster "
      f"{st['raster_ms']:.1f} ms, binning span {st['binning_ms']:.1f} ms, pairs/view "
      f"{st['pairs'] / a.views:.3g}", flush=True)
