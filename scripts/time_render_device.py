"""Device-resident render time (all planes, reference layout) for a config.
  python scripts/time_render_device.py --config 1"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2506_00225_b200 import scenes  # noqa: E402
from paper_2506_00225_b200.splatmap import Context, RenderChannels, render_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
a = ap.parse_args()
import torch  # noqa: E402
ctx = Context(0)
gm = scenes.make_map(a.config)
cam = scenes.CONFIGS[a.config].camera()
pose = scenes.render_poses(a.config, 1)[0]
px, C = cam.pixel_count(), gm.channels()
planes = torch.empty(px * (5 + C), dtype=torch.float64, device="cuda")
b = planes.data_ptr()
ptrs = dict(sil_ptr=b, color_ptr=b + 8 * px, depth_ptr=b + 32 * px, sem_ptr=b + 40 * px)
stream = torch.cuda.ExternalStream(ctx.stream)
for _ in range(3):
    render_device(gm, cam, pose, RenderChannels.all(), ctx=ctx, **ptrs)
ms = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    render_device(gm, cam, pose, RenderChannels.all(), ctx=ctx, **ptrs)
    e1.record(stream)
    e1.synchronize()
    ms.append(e0.elapsed_time(e1))
print(f"cfg{a.config} render device: {np.median(ms):.3f} ms")
ctx.set_profiling(True)
ctx.reset_stats()
render_device(gm, cam, pose, RenderChannels.all(), ctx=ctx, **ptrs)
ctx.synchronize()
st = ctx.stats()
print(f"  raster {st['raster_ms']:.3f} ms of a {st['binning_ms']:.3f} ms call span (profiled run)")
