"""CPU: bench.py's multi-rank control flow (the `--gpus N` torchrun path) as a
dry run on gloo — sharding by contiguous image blocks, barriers, max-over-ranks
timing and the gather to rank 0 — at world sizes 1, 2 and 4; the gathered
bytes must not depend on the rank count."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, batch):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", str(world),
           "--steps", "1", "--warmup", "0", "--batch", str(batch), "--width", "64", "--height", "48", "--dry-run"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env={**os.environ, "OMP_NUM_THREADS": "1"})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_dry_run_rank_count_invariance():
    # the same 4 images at world sizes 1, 2, 4 (batch 4 / 2 / 1 per rank)
    one = _run(1, 4)
    assert one["dry_run"] and one["n_gpus"] == 1 and one["images_per_step"] == 4
    for world in (2, 4):
        got = _run(world, 4 // world)
        assert got["n_gpus"] == world and got["images_per_step"] == 4
        assert got["gathered_counts"] == one["gathered_counts"]
        assert got["gathered_sha"] == one["gathered_sha"]
