"""Where the e2e step's time goes (cfg1, 64 views): map upload alone, scoring with the map
resident, and the e2e step (map touched + refresh_candidate_scores), wall clock with syncs.
  python scripts/time_e2e.py"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2506_00225_b200 import scenes  # noqa: E402
from paper_2506_00225_b200.splatmap import (CandidatePose, Context,  # noqa: E402
                                            refresh_candidate_scores, score_poses)

ctx = Context(0)
gm = scenes.make_map(1)
cam = scenes.CONFIGS[1].camera()
cands = scenes.make_candidates(1, 64)
poses = [c.camera_pose() for c in cands]
score_poses(gm, cam, poses, ctx=ctx)


def t(fn, rep=5):
    out = []
    for _ in range(rep):
        ctx.synchronize()
        t0 = time.perf_counter()
        fn()
        ctx.synchronize()
        out.append(1e3 * (time.perf_counter() - t0))
    return float(np.median(out))


def up():
    gm.touch()
    ctx.upload(gm)


def e2e():
    gm.touch()
    fresh = [CandidatePose(position=c.position, direction=c.direction, id=c.id) for c in cands]
    refresh_candidate_scores(fresh, gm, cam, ctx=ctx)


print(f"upload {t(up):.2f} ms  score-resident {t(lambda: score_poses(gm, cam, poses, ctx=ctx)):.2f} ms  "
      f"e2e {t(e2e):.2f} ms", flush=True)

# the two upload phases: the async call returns after phase A (geometry); sgm_map_wait covers
# phase B (colours + rows staging, their copies and the row sort)
import ctypes as C  # noqa: E402
from paper_2506_00225_b200 import _native as N  # noqa: E402
ta, tb = [], []
for _ in range(5):
    gm.touch()
    ctx.synchronize()
    t0 = time.perf_counter()
    h, keep = ctx._upload_async(gm)
    t1 = time.perf_counter()
    N.lib.sgm_map_wait(ctx.handle, h)
    t2 = time.perf_counter()
    N.lib.sgm_map_release(ctx.handle, h)
    ta.append(1e3 * (t1 - t0))
    tb.append(1e3 * (t2 - t1))
print(f"upload phase A {np.median(ta):.2f} ms, phase B + copies {np.median(tb):.2f} ms", flush=True)
