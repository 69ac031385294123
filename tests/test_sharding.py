"""CPU, world_size 2 over gloo: the multi-GPU host logic.  Each rank extracts
its contiguous shard (here with the CPU oracle standing in for the device, as
the checker), results are gathered to rank 0, and the gathered bytes equal the
single-process result — output does not depend on the rank count
(io.hpp:17-18 worker invariance)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2605_17869_b200.shard import assign_mixed, shard_range

N_IMAGES = 5
W, H = 64, 48


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _images():
    from oracle.oracle import Oracle
    port = Oracle("port")
    return [port.value_noise(W, H, 0x5EED0000 + i, 5, 6) for i in range(N_IMAGES)]


def _run_rank(rank, world, port_no, out_q):
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_2605_17869_b200.shard import gather_to_rank0

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    port = Oracle("port")
    imgs = _images()
    lo, hi = shard_range(N_IMAGES, world, rank)
    kps, descs, counts = [], [], []
    for i in range(lo, hi):
        k, d = port.extract(imgs[i])
        kps.append(k)
        descs.append(d)
        counts.append(len(k))
    from oracle.oracle import KEYPOINT_DTYPE
    k = np.concatenate(kps) if kps else np.zeros(0, KEYPOINT_DTYPE)
    d = np.concatenate(descs) if descs else np.zeros((0, 128), np.float32)
    res = gather_to_rank0(k, d, np.array(counts, np.int64))
    if rank == 0:
        gk = res[0].numpy().view(KEYPOINT_DTYPE).reshape(-1)
        out_q.put((gk.tobytes(), res[1].numpy().tobytes(), res[2].tolist()))
    else:
        assert res is None
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_partitions():
    for n in [0, 1, 5, 8, 256, 257]:
        for g in [1, 2, 3, 4, 8]:
            parts = [shard_range(n, g, r) for r in range(g)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(g - 1))
            assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1


def test_assign_mixed_deterministic():
    px = [640 * 480, 3840 * 2160, 1600 * 1200, 800 * 600, 1920 * 1080, 2560 * 1440] * 5
    a = assign_mixed(px, 4)
    assert a == assign_mixed(px, 4)
    assert sorted(i for part in a for i in part) == list(range(len(px)))
    loads = [sum(px[i] for i in part) for part in a]
    assert max(loads) / min(loads) < 1.6


@pytest.mark.parametrize("world", [1, 2, 4])
def test_gloo_gather_matches_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_run_rank, args=(r, world, port_no, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from oracle.oracle import Oracle
    port = Oracle("port")
    ref_k, ref_d, ref_c = [], [], []
    for img in _images():
        k, d = port.extract(img)
        ref_k.append(k)
        ref_d.append(d)
        ref_c.append(len(k))
    assert got[0] == np.concatenate(ref_k).tobytes()
    assert got[1] == np.concatenate(ref_d).tobytes()
    assert got[2] == ref_c
