"""Wall time of render() through the host API (planes copied to numpy) for a config.
  python scripts/time_render.py --config 1"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2506_00225_b200 import scenes  # noqa: E402
from paper_2506_00225_b200.splatmap import Context, RenderChannels, render  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
a = ap.parse_args()
ctx = Context(0)
gm = scenes.make_map(a.config)
cam = scenes.CONFIGS[a.config].camera()
pose = scenes.render_poses(a.config, 1)[0]
render(gm, cam, pose, RenderChannels.all(), ctx=ctx)
ts = []
for _ in range(4):
    t = time.perf_counter()
    out = render(gm, cam, pose, RenderChannels.all(), ctx=ctx)
    ts.append(1e3 * (time.perf_counter() - t))
print(f"cfg{a.config} render e2e: " + " ".join(f"{v:.1f}" for v in ts) + f" ms ({out.sem.nbytes / 1e6:.0f} MB sem)")
