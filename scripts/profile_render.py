"""One device-resident render (all planes) of a config's first pose, for ncu launch lists.
  python scripts/profile_render.py --config 1 --repeat 3"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2506_00225_b200 import scenes  # noqa: E402
from paper_2506_00225_b200.splatmap import Context, RenderChannels, render_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--repeat", type=int, default=3)
a = ap.parse_args()
import torch  # noqa: E402
ctx = Context(0)
gm = scenes.make_map(a.config)
cam = scenes.CONFIGS[a.config].camera()
pose = scenes.render_poses(a.config, 1)[0]
px, C = cam.pixel_count(), gm.channels()
planes = torch.empty(px * (5 + C), dtype=torch.float64, device="cuda")
b = planes.data_ptr()
for _ in range(a.repeat):
    render_device(gm, cam, pose, RenderChannels.all(), ctx=ctx, sil_ptr=b, color_ptr=b + 8 * px,
                  depth_ptr=b + 32 * px, sem_ptr=b + 40 * px)
ctx.synchronize()
print("ok")
