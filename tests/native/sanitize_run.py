"""Workload for tests/test_gpu_controls.py's compute-sanitizer runs: a batch of
two 320x240 value-noise images (plus a ragged 160x120 one) through every
extraction kernel via the C ABI, checked against the CPU oracle so a
sanitizer-clean run is also a correct one."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2605_17869_b200 as ds  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402

port = Oracle("port")
imgs = np.stack([port.value_noise(320, 240, 0x5EED0000 + i, 5, 16) for i in range(2)])
small = port.value_noise(160, 120, 0x5EED0002, 5, 8)
with ds.Extractor(device=0) as ex:
    ex.submit(imgs)
    ex.sync()
    shas = [ex.sha256(i) for i in range(2)]
    fs = ex.extract_images([imgs[0], small])
for i in range(2):
    kps, desc = port.extract(imgs[i])
    assert shas[i] == port.hash_features(kps, desc), i
kps, desc = port.extract(small)
assert fs[1].keypoints.tobytes() == kps.tobytes()
print("sanitize workload ok")
