"""Render through the host API (cfg1): fresh output arrays (as render() returns them) vs
arrays already touched, to separate the first-touch page faults from the copy.
  python scripts/time_render_host.py"""
import time, ctypes as C, numpy as np, sys
sys.path.insert(0, '.')
from paper_2506_00225_b200 import scenes, _native as N
from paper_2506_00225_b200.splatmap import Context, render, RenderChannels, RenderOptions
ctx = Context(0)
gm = scenes.make_map(1); cam = scenes.CONFIGS[1].camera(); pose = scenes.render_poses(1, 1)[0]
ch = RenderChannels.all()
render(gm, cam, pose, ch, ctx=ctx)
t = time.perf_counter(); 
for _ in range(3): render(gm, cam, pose, ch, ctx=ctx)
print("render() fresh arrays: %.1f ms" % ((time.perf_counter() - t) * 1e3 / 3))
px = cam.pixel_count(); Cn = gm.channels()
t = time.perf_counter(); a = np.empty(px * Cn); a.fill(0.0); print("np.empty+fill sem plane (1 thread): %.1f ms" % ((time.perf_counter() - t) * 1e3))
sil = np.zeros(px); col = np.zeros(px * 3); dep = np.zeros(px); sem = np.zeros(px * Cn)
handle = ctx.upload(gm)
cam_c, pose_c, opt_c = cam._c(), pose._c(), RenderOptions()._c()
nproj = C.c_uint64()
for i in range(4):
    t = time.perf_counter()
    ctx.check(N.lib.sgm_render(ctx.handle, handle, C.byref(cam_c), C.byref(pose_c), ch.flags(), C.byref(opt_c), N.dptr(col), N.dptr(dep), N.dptr(sil), N.dptr(sem), C.byref(nproj)))
    if i: print("sgm_render into touched arrays: %.1f ms" % ((time.perf_counter() - t) * 1e3))
