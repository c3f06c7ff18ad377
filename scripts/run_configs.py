"""Runs every BASELINE config on the GPU at full map size (a few views each) and checks
size-independent properties: scores finite and bounded, n_missing in [0, px], planes of one
render mass-conserving (sum_c sem = S up to the f32 prob rounding). Prints one line per config."""
import math
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2506_00225_b200 import scenes  # noqa: E402
from paper_2506_00225_b200.splatmap import (Context, RenderChannels, render,  # noqa: E402
                                            score_poses)

ctx = Context(0)
ctx.set_profiling(True)
for cfg in (0, 1, 2, 3, 4):
    t0 = time.perf_counter()
    gm = scenes.make_map(cfg)
    cam = scenes.CONFIGS[cfg].camera()
    views = 8 if cfg != 4 else 4
    poses = scenes.render_poses(cfg, views)
    ctx.reset_stats()
    t1 = time.perf_counter()
    nm, es = score_poses(gm, cam, poses, ctx=ctx)
    t2 = time.perf_counter()
    st = ctx.stats()
    px = cam.pixel_count()
    C = gm.channels()
    assert np.all((nm >= 0) & (nm <= px)), nm
    assert np.all(np.isfinite(es)) and np.all(es > 0) and np.all(es <= px * math.log(C) + 1e-6), es
    out = render(gm, cam, poses[0], RenderChannels.scoring(), ctx=ctx)
    s = out.sem.reshape(-1, C).sum(axis=1)
    mass = float(np.max(np.abs(s - out.silhouette)))
    assert mass < 1e-5, mass
    print(f"cfg{cfg}: N={gm.size()} {cam.width}x{cam.height} k={gm.k()} C={C} views={views} "
          f"score {1e3 * (t2 - t1) / views:.2f} ms/view (gen {t1 - t0:.1f} s) "
          f"V/view={st['visible'] / views:.0f} P/view={st['pairs'] / views:.0f} "
          f"K/view={st['contributors'] / views:.0f} raster_ms={st['raster_ms']:.1f} "
          f"n_missing={nm.astype(int).tolist()} max|sum sem - S|={mass:.1e}", flush=True)
