"""The multi-GPU paths with the real GPU scorer, on the one GPU this pool provides.

* the device snapshot interchange (sgm_map_export / sgm_map_import, collective C1's payload):
  an imported map renders and scores bit-identically to the uploaded one;
* MultiContext (sgm_multi, the C++ drop-in's refresh_candidate_scores) with two contexts on
  the same device: views sharded 2 ways, results bit-identical to one Context;
* two processes (gloo, world size 2) sharing GPU 0: rank 0 uploads and broadcasts the device
  snapshot, each rank scores its shard with its own Context, scores are all-gathered, and
  every rank agrees on combine_scores' argmax; per-view results bit-identical to N = 1.
The ranks' kernels never wait on one another (the collectives are host-side gloo ops).
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2506_00225_b200 as sgm
from paper_2506_00225_b200 import scenes

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("aniso", [False, True])
def test_snapshot_export_import_is_bit_identical(aniso):
    import torch
    ctx = sgm.Context(0)
    gm = scenes.make_map(0, n=5000, aniso=aniso)
    cam = scenes.CONFIGS[0].camera()
    poses = scenes.render_poses(0, 3)
    nbytes = ctx.export_bytes(gm)
    blob = torch.empty(nbytes, dtype=torch.uint8, device="cuda:0")
    ctx.export_map(gm, blob.data_ptr(), nbytes)
    dm = ctx.import_map(blob.data_ptr(), nbytes)
    assert (dm.size(), dm.k(), dm.num_classes(), dm.anisotropic()) == \
        (gm.size(), gm.k(), gm.num_classes(), aniso)
    del blob  # the import owns its own buffers
    a = sgm.render(gm, cam, poses[0], ctx=ctx)
    b = sgm.render(dm, cam, poses[0], ctx=ctx)
    for key in ("silhouette", "color", "depth", "sem"):
        assert np.array_equal(getattr(a, key), getattr(b, key)), key
    assert np.array_equal(a.projections, b.projections)
    nm, es = sgm.score_poses(gm, cam, poses, ctx=ctx)
    nm2, es2 = sgm.score_poses(dm, cam, poses, ctx=ctx)
    assert np.array_equal(nm, nm2) and np.array_equal(es, es2)
    with pytest.raises(RuntimeError, match="null|truncated|header"):
        ctx.import_map(0, 16)


def test_multi_context_shards_bit_identically():
    ctx = sgm.Context(0)
    gm = scenes.make_map(0, n=8000)
    cam = scenes.CONFIGS[0].camera()
    cands = scenes.make_decision_candidates(0, 13)
    one = [sgm.CandidatePose(position=c.position, direction=c.direction, id=c.id) for c in cands]
    sgm.refresh_candidate_scores(one, gm, cam, ctx=ctx)
    mg = sgm.MultiContext([0, 0])  # two contexts on one device: a 7 + 6 split
    assert mg.device_count() == 2
    two = [sgm.CandidatePose(position=c.position, direction=c.direction, id=c.id) for c in cands]
    sgm.refresh_candidate_scores(two, gm, cam, ctx=mg)
    assert [c.n_missing for c in one] == [c.n_missing for c in two]
    assert [c.entropy_sum for c in one] == [c.entropy_sum for c in two]
    poses = [c.camera_pose() for c in cands]
    nm, es = sgm.score_poses(gm, cam, poses, ctx=mg)
    assert nm.tolist() == [c.n_missing for c in one] and es.tolist() == [c.entropy_sum for c in one]
    mg.close()


def _rank(rank, world, port, out):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch
    import torch.distributed as dist
    import paper_2506_00225_b200 as sgm
    from paper_2506_00225_b200 import dist as sd
    from paper_2506_00225_b200 import scenes

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = sgm.Context(0)
    gm = sd.broadcast_map(scenes.make_map(0, n=6000) if rank == 0 else None, ctx)
    assert isinstance(gm, sgm.GaussianMap if rank == 0 else sgm.DeviceMap)
    cam = scenes.CONFIGS[0].camera()
    cands = scenes.make_decision_candidates(0, 9)
    s, e = sd.shard_range(len(cands), rank, world)
    nm, es = sgm.score_poses(gm, cam, [c.camera_pose() for c in cands[s:e]], ctx=ctx)
    nm_all, es_all = sd.gather_scores(len(cands), nm, es)
    for c, a, b in zip(cands, nm_all, es_all):
        c.n_missing, c.entropy_sum = float(a), float(b)
    sgm.combine_scores(cands, np.array([2.0, 1.5, 2.0]))
    best = max(range(len(cands)), key=lambda i: (cands[i].i_total, -i))
    out[rank] = (nm_all.tobytes(), es_all.tobytes(), best)
    dist.destroy_process_group()


def test_two_ranks_share_gpu0_broadcast_score_gather():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_rank, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out[0] == out[1]  # identical gathered scores and argmax on both ranks
    ctx = sgm.Context(0)
    gm = scenes.make_map(0, n=6000)
    cam = scenes.CONFIGS[0].camera()
    cands = scenes.make_decision_candidates(0, 9)
    nm, es = sgm.score_poses(gm, cam, [c.camera_pose() for c in cands], ctx=ctx)
    assert out[0][0] == nm.tobytes() and out[0][1] == es.tobytes()  # == N = 1, bit for bit
    assert len(set(nm.tolist())) > 2
