"""Multi-rank host logic on CPU with gloo (world_size 2): map broadcast, view
sharding, score all-gather and the rank-identical argmax. The per-view scoring
itself is replaced by the oracle here (no GPU on this box)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2506_00225_b200.dist import shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 64, 1024, 1025):
        for w in (1, 2, 3, 4, 8):
            cover = []
            for r in range(w):
                s, e = shard_range(n, r, w)
                assert 0 <= s <= e <= n
                cover.extend(range(s, e))
            assert cover == list(range(n))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out, aniso=False):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist
    import oracle
    from paper_2506_00225_b200 import dist as sd
    from paper_2506_00225_b200 import scenes
    from paper_2506_00225_b200.splatmap import CameraModel, Pose

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gm = scenes.make_map(0, n=600, aniso=aniso) if rank == 0 else None
    gm = sd.broadcast_map_arrays(gm)
    cam = CameraModel(48, 30, 0, 0, 30.0, 30.0, 24.0, 15.0)
    cands = scenes.make_candidates(0, 7)
    s, e = sd.shard_range(len(cands), rank, world)
    orc = oracle.Oracle()
    nm, es, _ = orc.score_views(gm, cam, [c.camera_pose() for c in cands[s:e]])
    nm_all, es_all = sd.gather_scores(len(cands), nm, es)
    _, _, _, tot = orc.combine_scores(nm_all, es_all, [c.position for c in cands], [2.0, 1.5, 2.0])
    out[rank] = (gm.centers.tobytes(), gm.sem_indices.tobytes(), nm_all.tobytes(),
                 es_all.tobytes(), int(np.argmax(tot)),
                 None if gm.log_scales is None else (gm.log_scales.tobytes() + gm.quats.tobytes()))
    dist.destroy_process_group()


@pytest.mark.parametrize("aniso", [False, True])
def test_two_rank_gloo_broadcast_shard_gather(orc, aniso):
    from paper_2506_00225_b200 import scenes
    from paper_2506_00225_b200.splatmap import CameraModel
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out, aniso), nprocs=2, join=True)
    a, b = out[0], out[1]
    assert a == b  # identical map, identical gathered scores, identical argmax on every rank
    gm = scenes.make_map(0, n=600, aniso=aniso)
    assert (a[5] is not None) == aniso
    assert a[0] == gm.centers.tobytes()
    cam = CameraModel(48, 30, 0, 0, 30.0, 30.0, 24.0, 15.0)
    cands = scenes.make_candidates(0, 7)
    nm, es, _ = orc.score_views(gm, cam, [c.camera_pose() for c in cands])
    assert a[2] == nm.tobytes() and a[3] == es.tobytes()  # sharding-invariant


def _prior_worker(rank, world, port, out):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist
    import oracle
    from paper_2506_00225_b200 import dist as sd
    from paper_2506_00225_b200 import scenes
    from paper_2506_00225_b200.splatmap import CameraModel

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gm = sd.broadcast_map_arrays(scenes.make_map(0, n=300) if rank == 0 else None)
    cam = CameraModel(40, 26, 0, 0, 30.0, 30.0, 20.0, 13.0)
    poses = [c.camera_pose() for c in scenes.make_candidates(0, 5, stream=2)]
    s, e = sd.shard_range(len(poses), rank, world)
    H = oracle.Oracle().fisher_accumulate(gm, cam, poses[s:e]) if e > s else np.zeros((gm.size(), 8))
    out[rank] = sd.all_reduce_prior(H).tobytes()
    dist.destroy_process_group()


def test_two_rank_gloo_fisher_prior_all_reduce(orc):
    """C2: the prior over sharded past poses, all-reduced, equals the prior over all poses
    (to reassociation) on every rank."""
    from paper_2506_00225_b200 import scenes
    from paper_2506_00225_b200.splatmap import CameraModel
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_prior_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out[0] == out[1]
    gm = scenes.make_map(0, n=300)
    cam = CameraModel(40, 26, 0, 0, 30.0, 30.0, 20.0, 13.0)
    poses = [c.camera_pose() for c in scenes.make_candidates(0, 5, stream=2)]
    want = orc.fisher_accumulate(gm, cam, poses)
    got = np.frombuffer(out[0], dtype=np.float64).reshape(want.shape)
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-300)
    assert np.any(want > 0)
