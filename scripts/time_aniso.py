"""Anisotropic-mode scoring time on cfg1 (64 views, map resident).
  python scripts/time_aniso.py"""
import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_2506_00225_b200 import scenes
from paper_2506_00225_b200.splatmap import Context, score_poses
import torch
ctx = Context(0)
gm = scenes.make_map(1, aniso=True)
cam = scenes.CONFIGS[1].camera()
poses = [c.camera_pose() for c in scenes.make_candidates(1, 64)]
ctx.upload(gm)
score_poses(gm, cam, poses, ctx=ctx)
ts = []
for _ in range(5):
    torch.cuda.synchronize(); t = time.perf_counter()
    nm, es = score_poses(gm, cam, poses, ctx=ctx)
    torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
ms = 1e3 * float(np.median(ts))
print(f"aniso cfg1 64 views: {ms:.2f} ms  {64 / ms * 1e3:.1f} views/s  sum(entropy)={float(np.sum(es)):.12e} sum(missing)={float(np.sum(nm)):.0f}")
