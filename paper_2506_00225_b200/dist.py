"""Candidate views sharded across ranks (one process per GPU, torch.distributed).

Views are independent (explorer.cpp:188-204), so the data path has
no collective. The only exchanges are the ones the planning step really has:
  C1 broadcast_map   - the map's DEVICE snapshot from rank 0, once per map version: rank 0
                       uploads (host activations + H2D, once), exports the snapshot blob into
                       a device tensor, ncclBroadcast sends it over NVLink, every other rank
                       imports it (sgm_map_export / sgm_map_import); no rank re-derives it
                       from host arrays. broadcast_map_arrays is the host-array variant for
                       processes without a device (the gloo CPU tests).
  C2 all_reduce_prior - the Fisher prior H (N x 8) summed over ranks, each rank having
                       accumulated its shard of the past poses (fisher_prior_sharded)
  C3 gather_scores   - every rank's (n_missing, entropy_sum) records, so every
                       rank can run the reference-identical combine_scores and
                       agree on the argmax.
Per-view results are bit-identical for any world size (each view's reduction
is deterministic and local to its GPU).
"""
from __future__ import annotations

from typing import Optional, Tuple

import numpy as np
import torch
import torch.distributed as dist

from .splatmap import GaussianMap


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block of view indices owned by `rank` (sizes differ by <= 1)."""
    base, rem = divmod(n, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def _device() -> torch.device:
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def broadcast_map(gmap: Optional[GaussianMap], ctx, src: int = 0):
    """C1: rank `src`'s map snapshot to every rank, device to device. Returns `gmap` on src and
    a DeviceMap (bit-identical snapshot on `ctx`'s device) on every other rank. With NCCL the
    blob goes device to device; with gloo (no device transport) it is staged through host
    memory, the same bytes."""
    rank = dist.get_rank()
    cuda = torch.device("cuda", ctx.device)
    if rank == src:
        nbytes = ctx.export_bytes(gmap)
        blob = torch.empty(nbytes, dtype=torch.uint8, device=cuda)
        ctx.export_map(gmap, blob.data_ptr(), nbytes)  # synchronous on the ctx stream
    size = torch.tensor([nbytes if rank == src else 0], dtype=torch.int64, device=_device())
    dist.broadcast(size, src)
    nbytes = int(size.item())
    if rank != src:
        blob = torch.empty(nbytes, dtype=torch.uint8, device=cuda)
    if dist.get_backend() == "nccl":
        dist.broadcast(blob, src)
    else:
        host = blob.cpu() if rank == src else torch.empty(nbytes, dtype=torch.uint8)
        dist.broadcast(host, src)
        if rank != src:
            blob.copy_(host)
    torch.cuda.current_stream(cuda).synchronize()  # the blob is complete before the import
    if rank == src:
        return gmap
    return ctx.import_map(blob.data_ptr(), nbytes)


def broadcast_map_arrays(gmap: Optional[GaussianMap], src: int = 0) -> GaussianMap:
    """C1 for processes without a device: every rank receives rank `src`'s host arrays
    (fp64 SoA + u16 ids), bit-identical."""
    dev = _device()
    rank = dist.get_rank()
    if rank == src:
        head = torch.tensor([gmap.size(), gmap.k(), gmap.num_classes(),
                             1 if gmap.anisotropic() else 0], dtype=torch.int64)
    else:
        head = torch.zeros(4, dtype=torch.int64)
    head = head.to(dev)
    dist.broadcast(head, src)
    n, k, m, aniso = (int(v) for v in head.cpu())
    extra = 7 * n if aniso else 0  # f4: per-axis log-scales (3N) and quaternions (4N)
    if rank == src:
        parts = [gmap.centers.reshape(-1), gmap.log_radii, gmap.opacity_logits,
                 gmap.colors.reshape(-1), gmap.sem_probs.reshape(-1)]
        if aniso:
            parts += [gmap.log_scales.reshape(-1), gmap.quats.reshape(-1)]
        buf = torch.from_numpy(np.ascontiguousarray(np.concatenate(parts))).to(dev)
        ids = torch.from_numpy(gmap.sem_indices.astype(np.int32).reshape(-1)).to(dev)
    else:
        buf = torch.empty(n * (8 + k) + extra, dtype=torch.float64, device=dev)
        ids = torch.empty(n * k, dtype=torch.int32, device=dev)
    dist.broadcast(buf, src)
    dist.broadcast(ids, src)
    if rank == src:
        return gmap
    a = buf.cpu().numpy()
    o = 0

    def take(cnt):
        nonlocal o
        out = a[o:o + cnt]
        o += cnt
        return out

    centers = take(3 * n).reshape(n, 3)
    log_r = take(n)
    logits = take(n)
    colors = take(3 * n).reshape(n, 3)
    probs = take(k * n).reshape(n, k)
    idx = ids.cpu().numpy().astype(np.uint16).reshape(n, k)
    ls = take(3 * n).reshape(n, 3) if aniso else None
    qs = take(4 * n).reshape(n, 4) if aniso else None
    return GaussianMap.from_arrays(k, m, centers, log_r, logits, colors, idx, probs,
                                   log_scales=ls, quats=qs)


def all_reduce_prior(H_local: np.ndarray) -> np.ndarray:
    """C2: element-wise sum of every rank's (N, 8) Fisher prior share (fp64)."""
    t = torch.from_numpy(np.ascontiguousarray(H_local, dtype=np.float64)).to(_device())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.cpu().numpy()


def fisher_prior_sharded(gmap: GaussianMap, camera, poses, lam: float = 1.0, options=None,
                         ctx=None) -> np.ndarray:
    """The Fisher prior over `poses` with the poses sharded across ranks: each rank
    accumulates its contiguous block (fisher_prior), the shares are all-reduced (C2) and the
    sum is installed on every rank's map (fisher_set_prior). Returns the summed H."""
    from .splatmap import fisher_prior, fisher_set_prior
    s, e = shard_range(len(poses), dist.get_rank(), dist.get_world_size())
    H = fisher_prior(gmap, camera, list(poses[s:e]), lam=lam, options=options, ctx=ctx)
    H = all_reduce_prior(H)
    fisher_set_prior(gmap, H, lam=lam, ctx=ctx)
    return H


def gather_scores(n_total: int, n_missing: np.ndarray, entropy_sum: np.ndarray
                  ) -> Tuple[np.ndarray, np.ndarray]:
    """C3: all-gather every rank's contiguous shard into full (n_missing, entropy_sum)."""
    dev = _device()
    world = dist.get_world_size()
    per = max(shard_range(n_total, r, world)[1] - shard_range(n_total, r, world)[0]
              for r in range(world))
    local = torch.zeros(2, per, dtype=torch.float64)
    local[0, :len(n_missing)] = torch.from_numpy(np.asarray(n_missing, dtype=np.float64))
    local[1, :len(entropy_sum)] = torch.from_numpy(np.asarray(entropy_sum, dtype=np.float64))
    local = local.to(dev)
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local)
    nm = np.zeros(n_total)
    es = np.zeros(n_total)
    for r, p in enumerate(parts):
        s, e = shard_range(n_total, r, world)
        pc = p.cpu().numpy()
        nm[s:e] = pc[0, :e - s]
        es[s:e] = pc[1, :e - s]
    return nm, es
