"""Multi-GPU image sharding.

Images are independent, so a batch partitions across ranks with NO collective
on the data path: rank k of G extracts images [k*B/G, (k+1)*B/G) on its own
GPU (one process per GPU, one dsift_ctx per process).  The reference's
analogue is worker-count invariance (io.hpp:17-18): output bytes do not
depend on G.  A consumer that needs every descriptor on one device calls
``gather_to_rank0`` — per-image counts are exchanged first (all_gather of
int64), then the variable-size keypoint/descriptor blocks move once, padded
to the largest shard (NCCL over NVLink on GPUs, gloo on CPU).
"""
from __future__ import annotations

import numpy as np


def shard_range(n_images: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block of rank `rank`: [floor(k*B/G), floor((k+1)*B/G))."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return (rank * n_images) // world, ((rank + 1) * n_images) // world


def assign_mixed(pixel_counts: list[int], world: int) -> list[list[int]]:
    """Deterministic greedy assignment of mixed-size images (C5 sweep):
    images in index order go to the rank with the fewest assigned pixels
    (ties -> lowest rank).  A pure function of (sizes, world)."""
    load = [0] * world
    out: list[list[int]] = [[] for _ in range(world)]
    for i, px in enumerate(pixel_counts):
        r = min(range(world), key=lambda k: (load[k], k))
        out[r].append(i)
        load[r] += int(px)
    return out


def gather_to_rank0(keypoints: np.ndarray, descriptors: np.ndarray, counts: np.ndarray, device=None):
    """Gather this rank's result blocks to rank 0 (torch.distributed must be
    initialised).  keypoints: structured [n] (28 B each), descriptors [n, 128]
    float32, counts: per-image keypoint counts of this rank's images.
    Returns (keypoints, descriptors, counts) concatenated in rank order on
    rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size()
    rank = dist.get_rank()
    dev = device if device is not None else torch.device("cpu")
    n_local = torch.tensor([len(keypoints), len(counts)], dtype=torch.int64, device=dev)
    sizes = [torch.zeros(2, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, n_local)
    sizes = [tuple(int(v) for v in s.tolist()) for s in sizes]
    max_k = max(s[0] for s in sizes)
    max_i = max(s[1] for s in sizes)
    row = 28 + 512
    blob = np.zeros((max_k, row), np.uint8)
    if len(keypoints):
        blob[: len(keypoints), :28] = np.frombuffer(keypoints.tobytes(), np.uint8).reshape(-1, 28)
        blob[: len(keypoints), 28:] = np.ascontiguousarray(descriptors, np.float32).view(np.uint8).reshape(-1, 512)
    cnt = np.zeros(max_i, np.int64)
    cnt[: len(counts)] = counts
    t_blob = torch.from_numpy(blob).to(dev)
    t_cnt = torch.from_numpy(cnt).to(dev)
    blobs = [torch.zeros_like(t_blob) for _ in range(world)]
    cnts = [torch.zeros_like(t_cnt) for _ in range(world)]
    dist.all_gather(blobs, t_blob)
    dist.all_gather(cnts, t_cnt)
    if rank != 0:
        return None
    from . import KEYPOINT_DTYPE
    kp_parts, d_parts, c_parts = [], [], []
    for r, (nk, ni) in enumerate(sizes):
        b = blobs[r][:nk].cpu().numpy()
        kp_parts.append(np.frombuffer(np.ascontiguousarray(b[:, :28]).tobytes(), KEYPOINT_DTYPE))
        d_parts.append(np.ascontiguousarray(b[:, 28:]).view(np.float32).reshape(nk, 128))
        c_parts.append(cnts[r][:ni].cpu().numpy())
    return np.concatenate(kp_parts), np.concatenate(d_parts), np.concatenate(c_parts)
