"""Multi-GPU image sharding.

Images are independent, so a batch partitions across ranks with NO collective
on the data path: rank k of G extracts images [k*B/G, (k+1)*B/G) on its own
GPU (one process per GPU, one dsift_ctx per process).  The reference's
analogue is worker-count invariance (io.hpp:17-18): output bytes do not
depend on G.  A consumer that needs every descriptor on one device calls
``gather_to_rank0`` on the exported device buffers: the per-rank sizes are
all-gathered (16 bytes per rank), then every rank sends its blocks once,
straight into its slice of rank 0's output (ncclSend / ncclRecv over NVLink
on GPUs, gloo on CPU) — no padding, no host staging.
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


def gather_to_rank0(keypoints, descriptors, counts):
    """Gather every rank's result to rank 0 without padding or host staging
    (torch.distributed must be initialised).

    keypoints: [n, 7] float32 (the 28-byte reference keypoint, e.g.
    Extractor.export_torch(0)), descriptors: [n, 128] float32
    (export_torch(1)), counts: [m] int64 keypoints per image of this rank's
    shard — torch tensors on this rank's device (NCCL) or CPU (gloo); numpy
    arrays are accepted and moved to the process group's device.

    1. all_gather of the (n, m) pairs — 16 bytes per rank;
    2. one send per block from every rank r > 0 straight into its slice of
       rank 0's exactly-sized output (ncclSend / ncclRecv over NVLink on GPUs),
       issued together with batch_isend_irecv.
    Returns (keypoints, descriptors, counts) concatenated in rank order on
    rank 0 (device tensors), None elsewhere.  The bytes do not depend on the
    rank count (worker invariance, io.hpp:17-18)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size()
    rank = dist.get_rank()
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")

    def as_tensor(x, dtype, cols):
        if not isinstance(x, torch.Tensor):
            arr = np.ascontiguousarray(x)
            if arr.dtype.fields is not None:   # structured keypoints -> [n, 7] float32 view
                arr = arr.view(np.float32).reshape(-1, 7)
            x = torch.from_numpy(np.ascontiguousarray(arr, dtype))
        x = x.to(dev).contiguous()
        return x.view(-1, cols) if cols else x.view(-1)

    kp = as_tensor(keypoints, np.float32, 7)
    de = as_tensor(descriptors, np.float32, 128)
    ct = as_tensor(counts, np.int64, 0)
    if kp.dtype != torch.float32 or de.dtype != torch.float32 or ct.dtype != torch.int64 or len(kp) != len(de):
        raise ValueError("gather_to_rank0: keypoints [n, 7] f32, descriptors [n, 128] f32, counts int64")
    n_local = torch.tensor([kp.shape[0], ct.shape[0]], dtype=torch.int64, device=dev)
    sizes = [torch.zeros(2, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, n_local)
    sizes = [(int(s[0]), int(s[1])) for s in sizes]
    ops = []
    if rank != 0:
        for t in (kp, de, ct):
            if t.numel():
                ops.append(dist.P2POp(dist.isend, t, 0))
        for w in dist.batch_isend_irecv(ops) if ops else []:
            w.wait()
        return None
    nk = sum(s[0] for s in sizes)
    ni = sum(s[1] for s in sizes)
    out_k = torch.empty((nk, 7), dtype=torch.float32, device=dev)
    out_d = torch.empty((nk, 128), dtype=torch.float32, device=dev)
    out_c = torch.empty(ni, dtype=torch.int64, device=dev)
    ok, oi = sizes[0]
    out_k[:ok].copy_(kp)
    out_d[:ok].copy_(de)
    out_c[:oi].copy_(ct)
    for r in range(1, world):
        k_r, i_r = sizes[r]
        for buf in (out_k[ok:ok + k_r], out_d[ok:ok + k_r], out_c[oi:oi + i_r]):
            if buf.numel():
                ops.append(dist.P2POp(dist.irecv, buf, r))
        ok += k_r
        oi += i_r
    for w in dist.batch_isend_irecv(ops) if ops else []:
        w.wait()
    return out_k, out_d, out_c


def nvlink_bytes_per_image(keypoints_per_image: float) -> float:
    """Bytes one image's result moves in gather_to_rank0: 28 + 512 per keypoint
    (+ 8 for its count)."""
    return keypoints_per_image * (28 + 512) + 8
