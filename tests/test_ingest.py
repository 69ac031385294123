"""§8(f1) image ingest: load_image (reference io.cpp:49-81).

CPU: the product's PNM parser (dsift_load_image, C ABI) and the oracle's
restatement agree with the unmodified reference on payload, dimensions and
every error message; the oracle's float conversion is bit-exact.
GPU (marked): the device uint8 -> float conversion equals the reference's
GrayImage bit for bit, and extract over 8-bit input equals
extract(load_image(path)) of the reference."""
import os

import numpy as np
import pytest

import paper_2605_17869_b200 as ds
from oracle.oracle import Oracle, OracleError, available


def _write(path, header: bytes, payload: bytes):
    with open(path, "wb") as f:
        f.write(header + payload)
    return str(path)


@pytest.fixture(scope="module")
def images(tmp_path_factory):
    d = tmp_path_factory.mktemp("pnm")
    rng = np.random.default_rng(11)
    g = rng.integers(0, 256, (37, 53), dtype=np.uint8)
    c = rng.integers(0, 256, (29, 41, 3), dtype=np.uint8)
    return {
        "gray": (_write(d / "g.pgm", b"P5\n# a comment\n53 37\n255\n", g.tobytes()), g),
        "color": (_write(d / "c.ppm", b"P6 41\t29 #x\n255 ", c.tobytes()), c),
        "bad_magic": (_write(d / "m.pgm", b"P3\n1 1\n255\n", b"0"), None),
        "bad_maxval": (_write(d / "v.pgm", b"P5\n2 2\n65535\n", b"0000"), None),
        "truncated": (_write(d / "t.pgm", b"P5\n4 4\n255\n", b"12"), None),
        "bad_width": (_write(d / "w.pgm", b"P5\n-3 2\n255\n", b""), None),
        "bad_height": (_write(d / "h.pgm", b"P5\n3 x\n255\n", b""), None),
        "stoi_prefix": (_write(d / "s.pgm", b"P5\n12abc 1\n255\n", b"y" * 12), None),
        "missing": (str(d / "nope.pgm"), None),
    }


def _ref_or_skip():
    if not available("reference"):
        pytest.skip("oracle/_ref not built")
    return Oracle("reference")


def test_load_image_payload_matches_reference(images):
    ref, port = _ref_or_skip(), Oracle("port")
    for key in ("gray", "color", "stoi_prefix"):
        path, pix = images[key]
        a = ref.load_image(path)
        b = port.load_image(path)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), key
        u = ds.load_image(path)
        assert u.shape[:2] == a.shape
        if pix is not None:
            assert np.array_equal(u, pix)


def test_load_image_errors_match_reference(images):
    ref, port = _ref_or_skip(), Oracle("port")
    for key in ("bad_magic", "bad_maxval", "truncated", "bad_width", "bad_height", "missing"):
        path = images[key][0]
        with pytest.raises(OracleError) as e_ref:
            ref.load_image(path)
        with pytest.raises(OracleError) as e_port:
            port.load_image(path)
        with pytest.raises(ds.ImageIOError) as e_ds:
            ds.load_image(path)
        assert str(e_ref.value) == str(e_port.value), key
        assert str(e_ds.value).endswith(str(e_ref.value)), (key, str(e_ds.value))


@pytest.mark.gpu
def test_device_ingest_bit_exact(images):
    ref = _ref_or_skip()
    with ds.Extractor() as ex:
        for key in ("gray", "color"):
            path, pix = images[key]
            got = ex.ingest_u8(pix)
            want = ref.load_image(path)
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), key


@pytest.mark.gpu
def test_extract_u8_matches_reference_pipeline(tmp_path):
    ref = _ref_or_skip()
    port = Oracle("port")
    base = port.value_noise(160, 120, 0x5EED0007, 5, 8)
    rgb = np.stack([np.clip(np.rint(base * 255 * s), 0, 255) for s in (1.0, 0.8, 0.6)], -1).astype(np.uint8)
    path = _write(tmp_path / "x.ppm", b"P6\n160 120\n255\n", rgb.tobytes())
    img = ref.load_image(path)
    k, d = ref.extract(img, None, os.cpu_count() or 1)
    with ds.Extractor() as ex:
        fs = ex.extract_u8(ds.load_image(path)[None])[0]
        assert ex.sha256(0) == ref.hash_features(k, d)
    assert fs.keypoints.tobytes() == k.tobytes()
