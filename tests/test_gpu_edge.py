"""GPU parity at the edges of the input domain the reference accepts.

The reference checks only the image size (>= 8x8, scalespace.cpp:148-151) and
the config; pixel values are taken as they come (io.cpp:111-142).  So every
float image of any shape >= 8x8 must give the reference's bytes -- or the
reference's exception -- here too:

* shapes: the 8x8 minimum, one-octave slivers (8 x N, N x 9), a prime-sized
  image, a 2x-upsampled base with a 1-pixel-wide last octave;
* values: denormal-only pixels (the positive-normal flags that let K1 widen
  on the integer pipe must be off), magnitudes where the gradients leave the
  fast atan2f domain [2^-39, 2^20) (the warp-uniform general path),
  negative images, all-zero and constant images (no keypoints), a NaN / Inf
  pixel (the reference throws std::out_of_range from the histogram bin);
* batches: n = 0 (rejected; the context stays usable), and a ragged batch
  mixing the shapes above.
"""
import os

import numpy as np
import pytest

import paper_2605_17869_b200 as ds

pytestmark = pytest.mark.gpu

SEED0 = 0x5EED0000


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def ref_outcome(ref, img):
    """(keypoints, descriptors, sha) from the reference, or ("error", message)."""
    from oracle.oracle import OracleError
    try:
        kps, desc = ref.extract(img, None, os.cpu_count() or 1)
    except OracleError as e:
        return ("error", str(e))
    return (np.ascontiguousarray(kps).tobytes(), bits(desc).tobytes(), ref.hash_features(kps, desc))


def gpu_outcome(ex, img):
    try:
        fs = ex.extract(img)
    except (ds.OutOfRange, ds.InvalidArgument) as e:
        return ("error", str(e))
    return (fs.keypoints.tobytes(), bits(fs.descriptors).tobytes(), ex.sha256(0))


def assert_same(ref, img):
    want = ref_outcome(ref, img)
    with ds.Extractor() as ex:
        got = gpu_outcome(ex, img)
    if want[0] == "error" or got[0] == "error":
        assert got == want   # the same exception text, or both returned features
    else:
        assert got[0] == want[0]
        assert got[1] == want[1]
        assert got[2] == want[2]
    return want


def noise(ref, w, h, seed):
    return ref.value_noise(w, h, SEED0 + seed, 5, max(8, w // 20))


@pytest.mark.parametrize("size", [(8, 8), (9, 8), (8, 600), (700, 9), (16, 16), (211, 97), (2003, 11)])
def test_extreme_shapes(ref, size):
    w, h = size
    assert_same(ref, noise(ref, w, h, w * 7 + h))


@pytest.mark.parametrize("size,fails", [((7, 8), False), ((4, 4), True), ((3, 100), True), ((1, 1), True)])
def test_minimum_size_is_checked_after_upsampling(ref, size, fails):
    # 7x8 is upsampled to 14x16 and runs; 4x4 (an 8x8 base), 3x100 and 1x1
    # raise the reference's error, with the reference's text
    w, h = size
    want = assert_same(ref, noise(ref, w, h, 15) if min(w, h) >= 4 else np.zeros((h, w), np.float32))
    assert (want[0] == "error") == fails


@pytest.mark.parametrize("scale", [1e-40, 1e-30, 3e4, 2e7, -1.0])
def test_value_ranges(ref, scale):
    # 1e-40: every pixel denormal; 1e-30: blur outputs and gradients near the
    # fast atan2f domain's lower edge; 2e7: gradients above 2^20; -1: negative
    img = (noise(ref, 320, 240, 11) * np.float32(scale)).astype(np.float32)
    assert_same(ref, img)


def test_offset_and_mixed_sign(ref):
    img = noise(ref, 300, 200, 12) - np.float32(0.5)
    assert_same(ref, img)


@pytest.mark.parametrize("fill", [0.0, -0.0, 0.25, 1e-42])
def test_flat_images_have_no_keypoints(ref, fill):
    img = np.full((120, 160), fill, np.float32)
    want = assert_same(ref, img)
    assert want[0] == b""


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_non_finite_pixel(ref, bad):
    img = noise(ref, 160, 120, 13)
    img[60, 80] = bad
    assert_same(ref, img)


def test_empty_batches_are_rejected_and_leave_the_context_usable(ref):
    img = noise(ref, 64, 64, 14)
    with ds.Extractor() as ex:
        with pytest.raises(ds.InvalidArgument):
            ex.extract_batch(np.zeros((0, 64, 64), np.float32))
        with pytest.raises(ds.InvalidArgument):
            ex.extract_images([])
        got = gpu_outcome(ex, img)
    assert got == ref_outcome(ref, img)


def test_ragged_batch_of_edge_shapes(ref):
    sizes = [(8, 8), (8, 600), (700, 9), (211, 97), (2003, 11), (16, 16)]
    imgs = [noise(ref, w, h, 100 + i) for i, (w, h) in enumerate(sizes)]
    with ds.Extractor() as ex:
        res = ex.extract_images(imgs)
        shas = [ex.sha256(i) for i in range(len(imgs))]
    for i, img in enumerate(imgs):
        want = ref_outcome(ref, img)
        assert res[i].keypoints.tobytes() == want[0]
        assert bits(res[i].descriptors).tobytes() == want[1]
        assert shas[i] == want[2]


@pytest.mark.parametrize("size,scale", [((640, 480), 1.0), ((211, 97), 1.0), ((320, 240), 1e-40)])
def test_texture_and_load_gathers_agree(ref, size, scale):
    # K5 reads the bilinear footprints with tld4 texture gathers; the plain-load
    # path (taken when a level stack exceeds the texture limits) must give the
    # same bytes, and both the reference's
    w, h = size
    img = (noise(ref, w, h, 16) * np.float32(scale)).astype(np.float32)
    want = ref_outcome(ref, img)
    outs = []
    for tex in (True, False):
        with ds.Extractor() as ex:
            ex.set_texture_gathers(tex)
            outs.append(gpu_outcome(ex, img))
    assert outs[0] == outs[1] == want
