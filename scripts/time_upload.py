"""Wall time of one map upload (host activations + pinned staging + H2D + row sort) for a
config, the e2e step's only per-step cost besides scoring.
  python scripts/time_upload.py --config 1"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2506_00225_b200 import scenes  # noqa: E402
from paper_2506_00225_b200.splatmap import Context  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--repeat", type=int, default=5)
a = ap.parse_args()
ctx = Context(0)
gm = scenes.make_map(a.config)
ctx.upload(gm)
ts = []
for _ in range(a.repeat):
    gm.touch()
    ctx.synchronize()
    t = time.perf_counter()
    ctx.upload(gm)
    ctx.synchronize()
    ts.append(1e3 * (time.perf_counter() - t))
print(f"cfg{a.config} upload: " + " ".join(f"{v:.2f}" for v in ts) + " ms", flush=True)
