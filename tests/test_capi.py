"""CPU: the C-ABI boundary (include/dsift.h) — the library loads without a
GPU, exports every declared symbol, validates configs with the reference's
messages, and fails loudly (no CPU fallback) when no device exists."""
import ctypes as C
import os
import re

import pytest

import paper_2605_17869_b200 as ds
from oracle.oracle import make_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "dsift.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dsift_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ds.load_library()
    names = declared_functions()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_no_fallback_symbols_or_cpu_paths():
    # the product library links no oracle / reference code
    out = os.popen(f"nm -D --defined-only {ds.library_path()}").read()
    assert "dor_" not in out and "oref_" not in out and "detsift" not in out


def test_abi_version_and_strerror():
    lib = ds.load_library()
    assert lib.dsift_abi_version() == 2
    assert lib.dsift_strerror(2) == b"device capacity exceeded"


def test_config_default_matches_reference_defaults():
    lib = ds.load_library()
    c = ds._Config()
    lib.dsift_config_default(C.byref(c))
    assert (c.sigma0, c.intervals, c.assumed_blur, c.contrast_threshold, c.edge_ratio) == \
        (pytest.approx(1.6), 3, 0.5, pytest.approx(0.04), 10.0)
    assert c.upsample_pixel_limit == 4_000_000 and c.n_dsp_scales == 5
    assert [c.dsp_scales[i] for i in range(5)] == [0.5, 1.0 / 1.4142135623730951, 1.0, 1.4142135623730951, 2.0]
    assert (c.orientation_bins, c.num_octaves) == (36, 0)


def test_config_validation_messages_match_reference(ref):
    bad = [dict(sigma0=0.0), dict(intervals=0), dict(contrast_threshold=0.0), dict(edge_ratio=1.0),
           dict(max_refine_iters=0), dict(upsample_pixel_limit=-1), dict(dsp_scales=()),
           dict(dsp_scales=(1.0, 0.5)), dict(descriptor_clip=0.0), dict(orientation_bins=1),
           dict(orientation_peak_ratio=0.0), dict(num_octaves=-1), dict(assumed_blur=2.0)]
    lib = ds.load_library()
    for over in bad:
        oc = make_config(**over)
        rc = lib.dsift_config_validate(C.byref(oc))   # same struct layout (dsift_config)
        assert rc == ds.DSIFT_EINVAL
        assert lib.dsift_last_error().decode() == ref.config_validate(oc), over
    assert lib.dsift_config_validate(C.byref(make_config())) == 0


def test_python_config_validate_raises_invalid_argument():
    with pytest.raises(ds.InvalidArgument, match="edge_ratio must be > 1"):
        ds.SiftConfig(edge_ratio=0.5).validate()


def test_create_without_gpu_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(ds.DsiftError) as e:
        ds.Extractor()
    assert e.value.code == ds.DSIFT_ECUDA


def test_keypoint_layout():
    assert ds.KEYPOINT_DTYPE.itemsize == 28 == C.sizeof(C.c_float) * 5 + C.sizeof(C.c_int32) * 2
