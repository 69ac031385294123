"""Generate tests/golden/ fixtures from the UNMODIFIED reference.

Runs the reference's own detsift::extract (oracle/_ref/libdetsift_ref.so,
compiled in place from /root/reference by oracle/Makefile) on a fixed set of
synthetic inputs and records, per case: the input recipe, keypoint count,
octave plan, SHA-256 of the DSF1 serialization (detsum.cpp:129-132) and the
first keypoints' bit patterns.  Small cases also store the full input image,
keypoints and descriptors (golden_*.npz).

Run here (where /root/reference exists):   python tests/golden/make_golden.py
The fixtures are committed; /root/reference is never read at test time.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, make_config  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# (name, input recipe, config overrides, store_full)
CASES = [
    ("vn96x64", {"kind": "value_noise", "w": 96, "h": 64, "seed": 3, "octaves": 5, "cells": 6}, {}, True),
    ("vn160x120", {"kind": "value_noise", "w": 160, "h": 120, "seed": 7, "octaves": 5, "cells": 8}, {}, True),
    ("vn200x150", {"kind": "value_noise", "w": 200, "h": 150, "seed": 0x5EED0000, "octaves": 5, "cells": 10}, {},
     False),
    ("vn320x240", {"kind": "value_noise", "w": 320, "h": 240, "seed": 11, "octaves": 5, "cells": 16}, {}, False),
    ("c1_640x480", {"kind": "value_noise", "w": 640, "h": 480, "seed": 0x5EED0000, "octaves": 5, "cells": 32}, {},
     False),
    ("noup320x240", {"kind": "value_noise", "w": 320, "h": 240, "seed": 5, "octaves": 5, "cells": 16},
     {"upsample_pixel_limit": 0}, False),
    ("s2_160x120", {"kind": "value_noise", "w": 160, "h": 120, "seed": 21, "octaves": 5, "cells": 8},
     {"intervals": 2}, False),
    ("s4_160x120", {"kind": "value_noise", "w": 160, "h": 120, "seed": 22, "octaves": 5, "cells": 8},
     {"intervals": 4}, False),
    ("dsp1_160x120", {"kind": "value_noise", "w": 160, "h": 120, "seed": 23, "octaves": 5, "cells": 8},
     {"dsp_scales": (1.0,)}, False),
    ("bins18_160x120", {"kind": "value_noise", "w": 160, "h": 120, "seed": 24, "octaves": 5, "cells": 8},
     {"orientation_bins": 18, "orientation_peak_ratio": 0.7}, False),
    ("oct3_160x120", {"kind": "value_noise", "w": 160, "h": 120, "seed": 25, "octaves": 5, "cells": 8},
     {"num_octaves": 3}, False),
    ("blobs128", {"kind": "blob_field", "w": 128, "h": 128, "seed": 9, "count": 25}, {}, True),
    ("constant64", {"kind": "constant", "w": 64, "h": 64, "value": 0.5}, {}, True),
    ("single_blob128", {"kind": "single_blob", "w": 128, "h": 128}, {}, True),
    ("odd_97x53", {"kind": "value_noise", "w": 97, "h": 53, "seed": 77, "octaves": 4, "cells": 7}, {}, True),
]


def make_input(ref: Oracle, r: dict) -> np.ndarray:
    if r["kind"] == "value_noise":
        return ref.value_noise(r["w"], r["h"], r["seed"], r["octaves"], r["cells"])
    if r["kind"] == "blob_field":
        out = np.empty((r["h"], r["w"]), np.float32)
        ref.lib.oref_blob_field(r["w"], r["h"], r["seed"], r["count"], out.ctypes.data)
        return out
    if r["kind"] == "constant":
        return np.full((r["h"], r["w"]), r["value"], np.float32)
    if r["kind"] == "single_blob":   # test_io.cpp:99-108
        img = np.full((r["h"], r["w"]), 0.2, np.float32)
        ref.lib.oref_add_blob(img.ctypes.data, r["w"], r["h"], 64.0, 64.0, 4.0, 0.6)
        return img
    raise ValueError(r)


def main():
    ref = Oracle("reference")
    out = []
    for name, recipe, over, full in CASES:
        img = make_input(ref, recipe)
        cfg = make_config(**over)
        kps, desc = ref.extract(img, cfg)
        ss = ref.scale_space(img, cfg)
        entry = {
            "name": name, "input": recipe, "config": {k: (list(v) if isinstance(v, tuple) else v)
                                                       for k, v in over.items()},
            "n_keypoints": int(len(kps)), "sha256": ref.hash_features(kps, desc),
            "n_octaves": ss.n_oct, "upsampled": ss.upsampled, "dims": ss.dims,
            "first_keypoints_u32": [k.tobytes().hex() for k in kps[:3]],
            "image_sha256_f32": __import__("hashlib").sha256(img.tobytes()).hexdigest(),
        }
        out.append(entry)
        if full:
            np.savez_compressed(os.path.join(HERE, f"golden_{name}.npz"), image=img, keypoints=kps,
                                descriptors=desc)
        print(name, entry["n_keypoints"], entry["sha256"][:16])
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py (reference: oracle/_ref/libdetsift_ref.so)",
                   "cases": out}, f, indent=1)


if __name__ == "__main__":
    main()
