"""Workload for tests/test_gpu_controls.py: gather_to_rank0 over NCCL on the
exported device buffers (world size 1 on the one GPU — the device-tensor path,
all_gather of the sizes and the rank-0 assembly), compared with the host copy."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2605_17869_b200 as ds  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
from paper_2605_17869_b200.shard import gather_to_rank0  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
port = Oracle("port")
imgs = np.stack([port.value_noise(320, 240, 0x5EED0000 + i, 5, 16) for i in range(3)])
with ds.Extractor(device=0) as ex:
    ex.submit(imgs)
    ex.sync()
    host = ex.results(with_u8=False)
    kp = ex.export_torch(0)
    de = ex.export_torch(1)
    counts = torch.tensor([len(f) for f in host], dtype=torch.int64, device="cuda")
    gk, gd, gc = gather_to_rank0(kp, de, counts)
    assert gk.is_cuda and gd.is_cuda
    ref_k = np.concatenate([f.keypoints for f in host])
    ref_d = np.concatenate([f.descriptors for f in host])
    assert gk.cpu().numpy().tobytes() == ref_k.tobytes()
    assert gd.cpu().numpy().tobytes() == ref_d.tobytes()
    assert gc.cpu().tolist() == [len(f) for f in host]
dist.destroy_process_group()
print("nccl gather ok", int(gk.shape[0]))
