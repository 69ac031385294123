import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference (oracle/_ref); skipped where it was not built."""
    from oracle.oracle import Oracle, available
    if not available("reference"):
        pytest.skip("oracle/_ref/libdetsift_ref.so not built")
    return Oracle("reference")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)["cases"]


def golden_input(port, case):
    """Regenerate a golden case's input (value noise via the pinned port, else stored)."""
    r = case["input"]
    if r["kind"] == "value_noise":
        return port.value_noise(r["w"], r["h"], r["seed"], r["octaves"], r["cells"])
    if r["kind"] == "constant":
        return np.full((r["h"], r["w"]), r["value"], np.float32)
    return np.load(os.path.join(GOLDEN, f"golden_{case['name']}.npz"))["image"]


def golden_config(case, kind="oracle"):
    over = dict(case["config"])
    if "dsp_scales" in over:
        over["dsp_scales"] = tuple(over["dsp_scales"])
    if kind == "oracle":
        from oracle.oracle import make_config
        return make_config(**over)
    import paper_2605_17869_b200 as ds
    mapping = {"intervals": "intervals_per_octave"}
    return ds.SiftConfig(**{mapping.get(k, k): v for k, v in over.items()})


@pytest.fixture(scope="session")
def gpu_extractor():
    import paper_2605_17869_b200 as ds
    ex = ds.Extractor(device=0)
    yield ex
    ex.close()
