"""Generates tests/golden/reference_scenes.npz from the REFERENCE's own code.

Run in the build container (needs /root/reference to build oracle/_ref):
    python tests/golden/make_golden.py

Scenes are the ones the reference's hot-path tests use:
  proj/tests/test_splat_render.cpp:24-265 and proj/tests/test_explorer.cpp:360-378,
built with the reference's own fixture code (testutil::random_splat_map,
proj/tests/test_helpers.hpp:46-67) and rendered/scored with the reference's own
render / render_reference / render_entropy / refresh_candidate_scores /
combine_scores (compiled unmodified into oracle/_ref/libsgm_ref.so). The GPU
tests compare against these outputs with no access to /root/reference.
"""
from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_2506_00225_b200.splatmap import (  # noqa: E402
    CameraModel, GaussianMap, Pose, RenderOptions, look_at)

OUT = Path(__file__).resolve().parent / "reference_scenes.npz"


def cam_from_fov(ref, w, h, vf, hf) -> CameraModel:
    v = ref.camera_from_fov(w, h, vf, hf)
    c = CameraModel(int(v[0]), int(v[1]), vf, hf, v[2], v[3], v[4], v[5])
    py = CameraModel.from_fov(w, h, vf, hf)
    assert (py.fx, py.fy, py.cx, py.cy) == (c.fx, c.fy, c.cx, c.cy), "from_fov mismatch"
    return c


def ref_look_at(ref, p, t) -> Pose:
    R, tt = ref.look_at(p, t)
    return Pose(R, tt)


def splat_at_pixel(cam, px, py, z, rad_px, logit):
    # proj/tests/test_splat_render.cpp:13-20
    center = [(px + 0.5 - cam.cx) * z / cam.fx, (py + 0.5 - cam.cy) * z / cam.fy, z]
    return center, math.log(rad_px * z / cam.fy), logit


def map_from(d) -> GaussianMap:
    return GaussianMap.from_arrays(d["k"], d["num_classes"], d["centers"], d["log_radii"],
                                   d["opacity_logits"], d["colors"], d["sem_indices"],
                                   d["sem_probs"])


def main() -> None:
    oracle.build_ref()
    ref = oracle.RefLib()
    store = {}
    scenes = []

    def add_scene(name, gmap, cam, pose, opts: RenderOptions, channels=15):
        out = ref.render(gmap, cam, pose, channels=channels, opt=opts)
        pre = f"{name}/"
        store[pre + "centers"] = gmap.centers
        store[pre + "log_radii"] = gmap.log_radii
        store[pre + "opacity_logits"] = gmap.opacity_logits
        store[pre + "colors"] = gmap.colors
        store[pre + "sem_indices"] = gmap.sem_indices
        store[pre + "sem_probs"] = gmap.sem_probs
        store[pre + "kc"] = np.array([gmap.k(), gmap.num_classes()])
        store[pre + "cam"] = np.array([cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy])
        store[pre + "R"] = np.asarray(pose.R)
        store[pre + "t"] = np.asarray(pose.t)
        store[pre + "opts"] = np.array([1.0 if opts.early_exit else 0.0, opts.transmittance_eps,
                                        opts.z_near, opts.truncation_sigmas, opts.tile_size])
        store[pre + "channels"] = np.array([channels])
        for key in ("silhouette", "color", "depth", "sem", "contrib", "contrib_offset"):
            if out.get(key) is not None:
                store[pre + key] = out[key]
        store[pre + "projections"] = out["projections"]
        store[pre + "entropy"] = ref.render_entropy(gmap, cam, pose, opts)
        scenes.append(name)

    # --- known-answer scenes (test_splat_render.cpp:24-74) ---
    cam16 = cam_from_fov(ref, 16, 12, 60, 70)
    c, lr, lg = splat_at_pixel(cam16, 8, 6, 1.5, 3.0, 40.0)
    add_scene("saturated", GaussianMap.from_arrays(1, 3, [c], [lr], [lg], [[0.2, 0.6, 0.9]], [[2]],
                                                   [[1.0]]), cam16, Pose(), RenderOptions())
    a = splat_at_pixel(cam16, 8, 6, 1.0, 4.0, 0.0)
    b = splat_at_pixel(cam16, 8, 6, 2.0, 4.0, 0.0)
    add_scene("two_half", GaussianMap.from_arrays(1, 3, [b[0], a[0]], [b[1], a[1]], [b[2], a[2]],
                                                  [[0, 0, 0], [0, 0, 0]], [[0], [0]],
                                                  [[1.0], [1.0]]), cam16, Pose(), RenderOptions())
    c, lr, lg = splat_at_pixel(cam16, 8, 6, 1.2, 3.0, 40.0)
    add_scene("sparse_scatter", GaussianMap.from_arrays(2, 9, [c], [lr], [lg], [[0, 0, 0]],
                                                        [[3, 7]], [[0.9, 0.1]]), cam16, Pose(),
              RenderOptions())

    # --- random_splat_map scenes ---
    cam32 = cam_from_fov(ref, 32, 24, 60, 80)
    pose_a = ref_look_at(ref, [0.3, -0.2, -0.5], [0.2, 0.1, 2.0])
    for seed in (11, 22, 33):  # k = M vs dense oracle, no early exit (:76-98)
        d = ref.random_splat_map(seed, cam32, pose_a, num_splats=50, num_classes=7)
        add_scene(f"kM_{seed}", map_from(d), cam32, pose_a, RenderOptions(early_exit=False))
    pose_b = ref_look_at(ref, [0, 0, -0.3], [0, 0, 2])
    for seed in (5, 6, 7, 8):  # mass conservation, k = 3 (:100-117)
        d = ref.random_splat_map(seed, cam32, pose_b, num_splats=40, num_classes=6, k=3)
        add_scene(f"mass_{seed}", map_from(d), cam32, pose_b, RenderOptions())
    cam24 = cam_from_fov(ref, 24, 18, 60, 80)
    pose_c = ref_look_at(ref, [0.1, 0, -0.4], [0, 0.05, 2])
    d = ref.random_splat_map(19, cam24, pose_c, num_splats=30, num_classes=5, k=2)
    add_scene("perm_19", map_from(d), cam24, pose_c, RenderOptions())
    cam40 = cam_from_fov(ref, 40, 30, 60, 80)
    pose_d = ref_look_at(ref, [0, 0.1, -0.2], [0.1, 0, 2])
    d = ref.random_splat_map(91, cam40, pose_d, num_splats=60, num_classes=4)
    add_scene("tiled_91", map_from(d), cam40, pose_d, RenderOptions(early_exit=False))
    pose_e = ref_look_at(ref, [0, 0, -0.5], [0, 0, 2])
    d = ref.random_splat_map(55, cam24, pose_e, num_splats=80, num_classes=5, alpha_logit_max=4.0)
    add_scene("early_55", map_from(d), cam24, pose_e, RenderOptions())
    add_scene("noearly_55", map_from(d), cam24, pose_e, RenderOptions(early_exit=False))

    # --- scoring caches (test_explorer.cpp:360-378) ---
    view = ref_look_at(ref, [0, 0, -1], [0, 0, 1])
    d = ref.random_splat_map(8, cam32, view, num_splats=40, num_classes=5)
    gm = map_from(d)
    add_scene("score_8", gm, cam32, view, RenderOptions())
    pos = np.array([[0, 0, -1], [0, 0, -1]], dtype=np.float64)
    dirs = np.array([[0, 0, 1], [0, 0, -1]], dtype=np.float64)
    nm, es = ref.refresh_scores(gm, cam32, pos, dirs)
    store["score_8/cand_pos"] = pos
    store["score_8/cand_dir"] = dirs
    store["score_8/n_missing"] = nm
    store["score_8/entropy_sum"] = es

    # --- a larger mixed scene for the scorer: 400 splats, many views ---
    cam64 = cam_from_fov(ref, 64, 48, 60, 80)
    d = ref.random_splat_map(2024, cam64, view, num_splats=400, num_classes=20, k=6,
                             alpha_logit_max=3.0, rad_px_max=9.0)
    gm = map_from(d)
    add_scene("multi_2024", gm, cam64, view, RenderOptions())
    rng = np.random.default_rng(7)
    pos = np.tile([0.0, 0.0, -1.0], (12, 1)) + rng.normal(0, 0.05, (12, 3))
    dirs = np.tile([0.0, 0.0, 1.0], (12, 1)) + rng.normal(0, 0.15, (12, 3))
    dirs[5] = [0, 0, -1]  # faces away
    nm, es = ref.refresh_scores(gm, cam64, pos, dirs)
    store["multi_2024/cand_pos"] = pos
    store["multi_2024/cand_dir"] = dirs
    store["multi_2024/n_missing"] = nm
    store["multi_2024/entropy_sum"] = es
    cur = np.array([0.02, 0.0, -1.0])
    any_, g, s, t = ref.combine_scores(nm, es, pos, cur)
    store["multi_2024/current"] = cur
    store["multi_2024/i_geo"] = g
    store["multi_2024/i_sem"] = s
    store["multi_2024/i_total"] = t

    store["scenes"] = np.array(scenes)
    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1024:.1f} KiB, {len(scenes)} scenes)")


if __name__ == "__main__":
    main()
