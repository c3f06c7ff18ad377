"""The C-ABI library (CPU-side checks: no kernels are launched here)."""
import math
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, has_gpu

import paper_2506_00225_b200 as sgm
from paper_2506_00225_b200 import _native as N


def declared_symbols():
    text = (ROOT / "include" / "sgm.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sgm_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(N.lib, s), f"{s} not exported by {N.LIB_PATH}"
        assert s in N.SIGNATURES, f"{s} has no ctypes signature"
    assert N.lib.sgm_abi_version() == 1


def test_library_is_sm100a_build():
    import subprocess
    r = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True,
                       text=True)
    assert "sm_100a" in r.stdout, r.stdout[-2000:]


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU error path")
def test_ctx_create_fails_loudly_without_gpu():
    with pytest.raises(RuntimeError, match="no CUDA device"):
        sgm.Context(0)


def test_host_combine_scores_matches_reference(ref, orc):
    rng = np.random.default_rng(2)
    for n in (1, 2, 5, 33):
        nm = np.floor(rng.uniform(0, 300, n))
        nm[n // 2] = 0
        es = rng.uniform(50, 900, n)
        pos = rng.normal(0, 2, (n, 3))
        cur = rng.normal(0, 1, 3)
        cands = [sgm.CandidatePose(position=pos[i], n_missing=nm[i], entropy_sum=es[i], id=i)
                 for i in range(n)]
        any_ = sgm.combine_scores(cands, cur)
        r = ref.combine_scores(nm, es, pos, cur)
        assert any_ == r[0]
        np.testing.assert_array_equal([c.i_total for c in cands], r[3])
        np.testing.assert_array_equal([c.i_geo for c in cands], r[1])
        np.testing.assert_array_equal([c.i_sem for c in cands], r[2])
    assert sgm.combine_scores([], [0, 0, 0]) is False


def test_combine_scores_reference_kats():
    # test_explorer.cpp:183-220
    c = [sgm.CandidatePose(position=np.array([float(i), 0, 0]), id=i) for i in range(3)]
    c[0].n_missing, c[1].n_missing, c[2].n_missing = math.exp(2.0), math.exp(3.0), 0.0
    for x in c:
        x.entropy_sum = 5.0
    assert sgm.combine_scores(c, [1, 0, 0])
    assert sum(x.i_geo for x in c) == pytest.approx(1.0, rel=1e-9)
    assert c[2].i_geo == 0.0
    two = [sgm.CandidatePose(position=np.zeros(3), n_missing=math.exp(2.0), entropy_sum=5.0),
           sgm.CandidatePose(position=np.zeros(3), n_missing=math.exp(3.0), entropy_sum=5.0)]
    sgm.combine_scores(two, [0, 0, 0])
    assert two[0].i_geo == pytest.approx(0.2689, rel=1e-3)
    assert two[1].i_geo == pytest.approx(0.7311, rel=1e-3)
    one = [sgm.CandidatePose(position=np.array([5.0, 0, 0]), n_missing=50, entropy_sum=10)]
    sgm.combine_scores(one, [0, 0, 0])
    assert one[0].i_total == pytest.approx(1.0)


def test_look_at_and_candidate_pose_match_reference(ref):
    rng = np.random.default_rng(4)
    for _ in range(40):
        p, d = rng.normal(0, 2, 3), rng.normal(0, 1, 3)
        pose = sgm.CandidatePose(position=p, direction=d).camera_pose()
        R, t = ref.candidate_pose(p, d)
        np.testing.assert_array_equal(pose.R, R)
        np.testing.assert_array_equal(pose.t, t)
        tg = rng.normal(0, 2, 3)
        np.testing.assert_array_equal(sgm.look_at(p, tg).R, ref.look_at(p, tg)[0])
        # Python fallback path (non-default up given as +Y explicitly in another form)
        a = sgm.splatmap.look_at(p, tg, up=(0.0, 1.0 + 0.0, 0.0))
        np.testing.assert_array_equal(a.R, ref.look_at(p, tg)[0])


def test_clipped_entropy_host(ref):
    rng = np.random.default_rng(1)
    for n in (2, 7, 102):
        p = rng.dirichlet(np.full(n, 0.3))
        assert sgm.clipped_entropy(p) == ref.clipped_entropy(p)
    assert sgm.clipped_entropy(np.zeros(10)) == pytest.approx(math.log(10.0), rel=1e-12)


def test_camera_from_fov_matches_reference(ref):
    for args in ((16, 12, 60, 70), (32, 24, 60, 80), (160, 120, 60.0, 90.0), (7, 3, 33.3, 101.0)):
        c = sgm.CameraModel.from_fov(*args)
        v = ref.camera_from_fov(*args)
        assert (c.width, c.height, c.fx, c.fy, c.cx, c.cy) == tuple(v)
    with pytest.raises(ValueError):
        sgm.CameraModel.from_fov(0, 10, 60, 60)
    with pytest.raises(ValueError):
        sgm.CameraModel.from_fov(10, 10, 180, 60)
    s = sgm.CameraModel.from_fov(160, 120, 60.0, 90.0).scaled(0.25)
    assert (s.width, s.height) == (40, 30)


def test_gaussian_map_invariants_and_sgmp_roundtrip(tmp_path):
    with pytest.raises(ValueError):
        sgm.GaussianMap(0, 5)
    with pytest.raises(ValueError):
        sgm.GaussianMap(7, 5)
    m = sgm.GaussianMap(2, 5)
    m.add(sgm.SemanticGaussian(np.array([0.5, 0.25, 2.0]), -3.0, 1.5, np.array([0.1, 0.2, 0.3]),
                               [1, 4], [0.75, 0.25], 7))
    with pytest.raises(ValueError):
        m.add(sgm.SemanticGaussian(sem_indices=[1], sem_probs=[1.0]))
    path = tmp_path / "m.sgmp"
    m.save(str(path))
    back = sgm.GaussianMap.load(str(path))
    assert back.size() == 1 and back.k() == 2 and back.num_classes() == 5
    np.testing.assert_array_equal(back.centers, m.centers)  # all values exact in f32
    np.testing.assert_array_equal(back.sem_indices, m.sem_indices)
    assert int(back.source_frames[0]) == 7
    (tmp_path / "bad").write_bytes(b"XXXX" + bytes(20))
    with pytest.raises(RuntimeError, match="bad magic"):
        sgm.GaussianMap.load(str(tmp_path / "bad"))


def test_sgmp_loads_in_reference(tmp_path, ref):
    from paper_2506_00225_b200 import scenes
    m = scenes.make_map(0, n=300)
    path = tmp_path / "cfg0.sgmp"
    m.save(str(path))
    h = ref.lib.ref_map_load(str(path).encode())
    assert ref.lib.ref_map_size(h) == 300
    cam = scenes.CONFIGS[0].camera()
    pose = scenes.render_poses(0, 1)[0]
    a = ref.render(m, cam, pose, 7)
    b = ref.render(m, cam, pose, 7, handle=h, n_map=300)
    for key in ("silhouette", "color", "depth", "sem"):
        np.testing.assert_array_equal(a[key], b[key])
    ref.map_destroy(h)


def test_prune_pool_and_candidate_pool():
    # test_explorer.cpp:299-313 and :315-334
    scoring = sgm.CameraModel.from_fov(160, 120, 60, 90)
    cs = [sgm.CandidatePose(n_missing=v, id=i) for i, v in enumerate([95, 0, 160 * 120, 400])]
    cs[3].state = sgm.CandidateState.Visited
    out = sgm.prune_pool(cs, scoring)
    assert [c.id for c in out] == [2]
    pool = sgm.CandidatePool()
    pool.absorb([sgm.CandidatePose(n_missing=500) for _ in range(6)])
    pool.mark_visited(2)
    assert pool.prune(sgm.CameraModel.from_fov(40, 30, 60, 90)) == 1
    assert all(c.id != 2 for c in pool.active()) and pool.ever_visited(2)
    pool.absorb([sgm.CandidatePose(n_missing=500) for _ in range(3)])
    assert sorted(c.id for c in pool.active()) == [0, 1, 3, 4, 5, 6, 7, 8]


def _softmax(v):
    v = np.asarray(v, dtype=np.float64)
    fin = np.isfinite(v)
    out = np.zeros_like(v)
    if not fin.any():
        return out
    e = np.where(fin, np.exp(np.where(fin, v, 0.0) - v[fin].max()), 0.0)
    return e / e.sum()


def test_combine_scores_fisher_matches_its_definition():
    """The Fisher extension's scalar gain: gain = fisher_gain + w_sem *
    entropy_sum, i_gain = (1 - softmax(dist)) * softmax(ln gain), ranked i_gain desc, id asc."""
    rng = np.random.default_rng(5)
    for n, w in ((1, 1.0), (2, 0.0), (7, 1.0), (40, 0.25)):
        fg = rng.uniform(0.0, 3e4, n)
        es = rng.uniform(1e5, 3e5, n)
        fg[n // 2] = 0.0
        pos = rng.normal(0, 2, (n, 3))
        cur = rng.normal(0, 1, 3)
        cands = [sgm.CandidatePose(position=pos[i], entropy_sum=es[i], fisher_gain=fg[i], id=i)
                 for i in range(n)]
        any_ = sgm.combine_scores_fisher(cands, cur, w_sem=w)
        gain = fg + w * es
        with np.errstate(divide="ignore"):
            share = _softmax(np.where(gain > 0, np.log(np.where(gain > 0, gain, 1.0)), -np.inf))
        dist = np.sqrt(((pos - cur) ** 2).sum(axis=1))
        tot = (1.0 if n == 1 else 1.0 - _softmax(dist)) * share
        np.testing.assert_allclose([c.gain for c in cands], gain, rtol=1e-15)
        np.testing.assert_allclose([c.i_gain for c in cands], tot, rtol=1e-12, atol=1e-300)
        assert any_ == bool((tot > 0).any())
    zero = [sgm.CandidatePose(position=np.zeros(3), id=i) for i in range(3)]
    assert sgm.combine_scores_fisher(zero, [0, 0, 0]) is False  # no gain anywhere: exhausted
    with pytest.raises(ValueError):
        sgm.combine_scores_fisher(zero, [0, 0, 0], w_sem=-1.0)


def test_trainer_rejects_anisotropic_maps():
    """optimize_map trains the reference's isotropic parameters only (mapper.cpp:10-51)."""
    from paper_2506_00225_b200.mapper import MapTrainer
    gm = sgm.GaussianMap.from_arrays(1, 3, [[0, 0, 1.0]], [-2.0], [0.0], [[0, 0, 0]], [[2]], [[1.0]],
                                     log_scales=[[-2.0, -2.1, -1.9]], quats=[[1.0, 0, 0, 0]])
    with pytest.raises(ValueError, match="anisotropic"):
        MapTrainer(gm)


def test_map_version_bumps_on_array_reassignment():
    gm = sgm.GaussianMap.from_arrays(1, 3, [[0, 0, 1.0]], [-2.0], [0.0], [[0, 0, 0]], [[2]], [[1.0]])
    v = gm._version
    gm.colors = np.array([[0.5, 0.5, 0.5]])
    assert gm._version > v
    v = gm._version
    gm.touch()
    assert gm._version == v + 1
