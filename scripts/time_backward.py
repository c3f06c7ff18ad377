"""Time the GPU mapping step (render + losses + backward) vs the reference's, and check parity
at full config size. python scripts/time_backward.py --config 1"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2506_00225_b200 as sgm  # noqa: E402
from paper_2506_00225_b200 import scenes  # noqa: E402
from test_gpu_backward import random_frame  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=0)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-ref", action="store_true")
    ap.add_argument("--optimize", type=int, default=0,
                    help="time N optimize_map iterations on 2 resident frames instead")
    a = ap.parse_args()
    if a.optimize:
        return time_optimize(a)
    gm = scenes.make_map(a.config)
    cam = scenes.CONFIGS[a.config].camera()
    pose = scenes.render_poses(a.config, 1)[0]
    fr = random_frame(11, cam, pose, gm.num_classes())
    ctx = sgm.Context(0)
    rep, g = sgm.backward(gm, cam, fr, ctx=ctx)
    ts = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        rep, g = sgm.backward(gm, cam, fr, ctx=ctx)
        ts.append(time.perf_counter() - t0)
    print(f"cfg{a.config} gpu backward (API, host frame in/grads out): median "
          f"{1e3 * np.median(ts):.2f} ms  report={rep}", flush=True)
    if a.no_ref:
        return
    from oracle import RefLib
    ref = RefLib()
    t0 = time.perf_counter()
    rep_r, g_r = ref.backward(gm, cam, fr, sgm.LossWeights())
    print(f"cfg{a.config} reference backward (1 core): {1e3 * (time.perf_counter() - t0):.1f} ms")
    np.testing.assert_allclose([rep.photometric, rep.depth, rep.semantic], rep_r[:3], rtol=1e-10)
    for name in ("center", "log_radius", "opacity_logit", "color", "sem"):
        x, y = getattr(g, name), g_r[name]
        scale = max(1e-30, float(np.max(np.abs(y))))
        err = float(np.max(np.abs(x - y))) / scale
        print(f"  {name}: max|diff|/max|ref| = {err:.3e}")
        assert err < 1e-9, name
    print("PARITY OK")


def time_optimize(a):
    import torch
    from paper_2506_00225_b200.mapper import DeviceFrame, MapperConfig, MapTrainer
    gm = scenes.make_map(a.config)
    cam = scenes.CONFIGS[a.config].camera()
    poses = scenes.render_poses(a.config, 2)
    frames = [random_frame(11 + i, cam, p, gm.num_classes()) for i, p in enumerate(poses)]
    ctx = sgm.Context(0)
    dev = [DeviceFrame(f, ctx=ctx) for f in frames]
    cfg = MapperConfig(prune_every=0)
    tr = MapTrainer(gm, ctx=ctx)
    tr.optimize(dev, cam, cfg, 2)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hist = tr.optimize(dev, cam, cfg, a.optimize)
    dt = time.perf_counter() - t0
    print(f"cfg{a.config} gpu optimize_map: {a.optimize} iters in {dt * 1e3:.1f} ms = "
          f"{dt * 1e3 / a.optimize:.2f} ms/iter; loss {hist[0].total():.5f} -> {hist[-1].total():.5f}",
          flush=True)
    if a.no_ref:
        return
    from oracle import RefLib
    ref = RefLib()
    t0 = time.perf_counter()
    hr, _, err = ref.optimize_map(gm, frames, cam, cfg, 2)
    dt = time.perf_counter() - t0
    print(f"cfg{a.config} reference optimize_map (1 core): 2 iters in {dt * 1e3:.0f} ms = "
          f"{dt * 1e3 / 2:.0f} ms/iter")


if __name__ == "__main__":
    main()
