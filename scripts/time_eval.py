"""Time evaluate() (render + semantic/photometric metrics on device planes) vs the
reference's render + semantic_metrics + photometric_metrics.
python scripts/time_eval.py --config 1 --views 4"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2506_00225_b200 as sgm  # noqa: E402
from paper_2506_00225_b200 import scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=0)
    ap.add_argument("--views", type=int, default=4)
    ap.add_argument("--no-ref", action="store_true")
    a = ap.parse_args()
    gm = scenes.make_map(a.config)
    cam = scenes.CONFIGS[a.config].camera()
    poses = scenes.render_poses(a.config, a.views)
    frames = [scenes.make_frame(a.config, p, seed=i) for i, p in enumerate(poses)]
    ctx = sgm.Context(0)
    dev = [sgm.DeviceFrame(f, ctx=ctx) for f in frames]
    sgm.evaluate(gm, cam, dev[:1], ctx=ctx)  # warm-up
    t0 = time.perf_counter()
    ev = sgm.Evaluator(gm.num_classes(), ctx=ctx)
    for f in dev:
        ev.add_view(gm, cam, f)
    t1 = time.perf_counter()
    rep = ev.report()
    t2 = time.perf_counter()
    print(f"cfg{a.config} gpu evaluate {a.views} views: add_view {1e3 * (t1 - t0) / a.views:.2f} ms/view, "
          f"report {1e3 * (t2 - t1):.1f} ms; miou {rep.miou_pct:.4f} top1 {rep.top1_pct:.4f} "
          f"mAP {rep.map_pct:.4f} psnr {rep.psnr_db:.4f}", flush=True)
    if a.no_ref:
        return
    from oracle import RefLib
    ref = RefLib()
    t0 = time.perf_counter()
    summary, *_ = ref.evaluate(gm, cam, frames)
    dt = time.perf_counter() - t0
    print(f"cfg{a.config} reference render + metrics (1 core): {dt:.2f} s "
          f"({1e3 * dt / a.views:.0f} ms/view); mAP {summary[3]:.4f}")
    np.testing.assert_allclose(rep.map_pct, summary[3], rtol=1e-9)


if __name__ == "__main__":
    main()
