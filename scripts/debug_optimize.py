"""Debug: per-iteration comparison of GPU optimize_map vs the reference."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2506_00225_b200 as sgm  # noqa: E402
from oracle import RefLib  # noqa: E402
from test_gpu_optimize import scene  # noqa: E402
from paper_2506_00225_b200.mapper import AdamState, MapperConfig  # noqa: E402

ref = RefLib()
ctx = sgm.Context(0)
for iters in (1, 2, 3):
    cam, gm, frames = scene(1)
    cfg = MapperConfig(prune_every=0)
    hr, out, err = ref.optimize_map(gm, frames, cam, cfg, iters)
    h = sgm.optimize_map(gm, AdamState(), frames, cam, cfg, iters, ctx=ctx)
    print("iters", iters, "sem loss gpu", [x.semantic for x in h], "ref", list(hr[:, 2]))
    for name in ("centers", "log_radii", "opacity_logits", "colors", "sem_probs"):
        a = np.asarray(getattr(gm, name)).reshape(-1)
        b = out[name]
        d = np.abs(a - b)
        i = int(np.argmax(d))
        print(f"  {name}: max diff {d.max():.3e} at {i} ({a[i]!r} vs {b[i]!r})")
    if iters == 1:
        a = np.asarray(gm.sem_probs).reshape(-1, 4)
        b = out["sem_probs"].reshape(-1, 4)
        bad = np.where(np.abs(a - b).max(axis=1) > 1e-12)[0]
        print("  bad rows", bad[:10], len(bad))
        for r in bad[:3]:
            print("   ", r, a[r], b[r], np.asarray(gm.sem_indices)[r])
