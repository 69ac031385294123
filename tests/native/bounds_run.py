"""Workload for tests/test_gpu_controls.py::test_bounds_build_clean: extraction
cases that reach every indexed path of K1 (bridge, strip, decimate, small
octaves), K2, K4 and K5 (interior and border descriptor lattices, the exact
fallback, FORCE_EXACT) through the library named by argv[1].  Prints one JSON
line: the per-image digests and, for the bounds-check build, the device
counters of failed index conditions (tests/native/libdsift_bounds.so,
DSIFT_BOUND in csrc/dsift_common.cuh)."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_17869_b200 as ds  # noqa: E402

lib = ds.load_library(sys.argv[1])
out = {}
if hasattr(lib, "dsift_test_bounds_selftest"):   # the counters see a deliberate failure, then reset
    buf = (C.c_ulonglong * 2)()
    assert lib.dsift_test_bounds_selftest() == 0
    assert lib.dsift_test_bounds_describe(buf, 1) == 0
    out["selftest"] = [int(buf[0]), int(buf[1])]
SEED0 = 0x5EED0000
# (w, h, n, cells, force_exact): C3 (upsampled, 8 octaves), a not-upsampled
# 2301x1799 with a TMA-incompatible pitch, odd and tiny sizes (border lattices,
# small-octave kernel), and the exact descriptor kernel for everything
cases = [(1600, 1200, 2, 80, 0), (2301, 1799, 1, 96, 0), (257, 199, 3, 12, 0), (37, 29, 2, 4, 0),
         (320, 240, 2, 16, 1)]
out["digests"] = {}
for (w, h, n, cells, exact) in cases:
    with ds.Extractor(device=0) as ex:
        if exact:
            ex.set_force_exact(True)
        imgs = torch.empty((n, h, w), dtype=torch.float32, device="cuda")
        ex.synth_value_noise(imgs.data_ptr(), n, w, h, SEED0, 5, cells)
        torch.cuda.synchronize()
        ex.submit(None, n=n, w=w, h=h, device_ptr=imgs.data_ptr())
        nk = ex.sync()
        out["digests"][f"{w}x{h}x{n}{'e' if exact else ''}"] = [nk] + [ex.sha256(i) for i in range(n)]
    torch.cuda.synchronize()
# a ragged batch in one call (mixed sizes, one size group each)
with ds.Extractor(device=0) as ex:
    a = torch.empty((1, 240, 320), dtype=torch.float32, device="cuda")
    b = torch.empty((1, 199, 257), dtype=torch.float32, device="cuda")
    ex.synth_value_noise(a.data_ptr(), 1, 320, 240, SEED0 + 7, 5, 16)
    ex.synth_value_noise(b.data_ptr(), 1, 257, 199, SEED0 + 8, 5, 12)
    torch.cuda.synchronize()
    ex.submit_images([(a.data_ptr(), 320, 240), (b.data_ptr(), 257, 199)], device=True)
    nk = ex.sync()
    out["digests"]["ragged"] = [nk] + [ex.sha256(i) for i in range(2)]
torch.cuda.synchronize()
counters = {}
for unit in ("pyramid", "detect", "orient", "describe"):
    fn = getattr(lib, f"dsift_test_bounds_{unit}", None)
    if fn is None:
        continue
    buf = (C.c_ulonglong * 2)()
    assert fn(buf, 0) == 0, unit
    counters[unit] = [int(buf[0]), int(buf[1])]
out["bounds"] = counters
print(json.dumps(out))
