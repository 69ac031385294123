"""CPU: the product's restatements of the host libm calls on the path
(paper_2605_17869_b200/csrc/dsift_math.cuh, compiled here as host code with
no FP contraction) reproduce this host's glibc bit-for-bit.  The GPU test
test_gpu_parity.py::test_device_libm_matches_host closes the loop device ->
host twin; together: device == glibc, the function the reference calls."""
import ctypes as C
import os

import pytest

LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "native", "liblibmcheck.so")


@pytest.fixture(scope="module")
def lc():
    if not os.path.exists(LIB):
        pytest.skip("tests/native/liblibmcheck.so not built (run __graft_entry__.build())")
    lib = C.CDLL(LIB)
    lib.lc_atan2f_mismatch.restype = C.c_int64
    lib.lc_atan2f_mismatch.argtypes = [C.c_uint64, C.c_int64, C.c_int, C.c_void_p]
    lib.lc_exp_mismatch.restype = C.c_int64
    lib.lc_exp_mismatch.argtypes = [C.c_uint64, C.c_int64, C.c_double, C.c_double, C.c_int, C.c_void_p]
    lib.lc_sincos_mismatch.restype = C.c_int64
    lib.lc_sincos_mismatch.argtypes = [C.c_uint64, C.c_int64, C.c_void_p]
    return lib


@pytest.mark.parametrize("mode,n", [(0, 4_000_000), (1, 8_000_000), (2, 20_000)])
def test_atan2f_bit_exact(lc, mode, n):
    first = (C.c_float * 3)()
    bad = lc.lc_atan2f_mismatch(12345 + mode, n, mode, first)
    assert bad == 0, f"{bad} mismatches, first (y, x, got) = {list(first)}"


@pytest.mark.parametrize("lo,hi,mode", [(-10.0, 0.0, 0), (-1.6, 0.0, 1), (-745.2, 709.8, 0),
                                        (-1e-12, 1e-12, 0), (-1e-15, 1e-15, 0), (-760.0, -700.0, 0),
                                        (-511.9, 511.9, 0)])
def test_exp_bit_exact(lc, lo, hi, mode):
    first = (C.c_double * 2)()
    bad = lc.lc_exp_mismatch(777, 4_000_000, lo, hi, mode, first)
    assert bad == 0, f"{bad} mismatches, first (x, got) = {list(first)}"


def test_sincos_bit_exact(lc):
    # cos/sin feed the double sample coordinates (describe.cpp:51-52): the
    # restatement of glibc's __sin_fma/__cos_fma must equal the live libm
    fb = C.c_int64()
    bad = lc.lc_sincos_mismatch(99, 4_000_000, C.byref(fb))
    assert bad == 0 and fb.value == 0


def test_sincos_exhaustive_float_angles(lc):
    lc.lc_sincos_exhaustive.restype = C.c_int64
    lc.lc_sincos_exhaustive.argtypes = [C.c_int]
    assert lc.lc_sincos_exhaustive(os.cpu_count() or 4) == 0


def test_div_2pi_exhaustive(lc):
    # the orientation-bin quotient (orient.cpp:52, describe.cpp:92) for every
    # float numerator up to 64 bins * 2pi
    lc.lc_div2pi_mismatch.restype = C.c_int64
    lc.lc_div2pi_mismatch.argtypes = [C.c_float]
    assert lc.lc_div2pi_mismatch(512.0) == 0


@pytest.mark.parametrize("mode,n", [(0, 2_000_000), (1, 1_000_000), (2, 196)])
def test_hypot_bit_exact(lc, mode, n):
    # Hartley normalization's std::hypot (geom.cpp:83-84) restated from glibc
    lc.lc_hypot_mismatch.restype = C.c_int64
    lc.lc_hypot_mismatch.argtypes = [C.c_uint64, C.c_int64, C.c_int, C.c_void_p]
    first = (C.c_double * 3)()
    bad = lc.lc_hypot_mismatch(4242 + mode, n, mode, first)
    assert bad == 0, f"{bad} mismatches, first (x, y, got) = {list(first)}"


def test_atan2f_x_equal_one(lc):
    # fdlibm routes x == 1 to atanf(y); the restatement takes its generic fast
    # path there (y / 1 == y, atanf odd bit for bit) -- check against glibc
    libm = C.CDLL("libm.so.6")
    libm.atan2f.restype = C.c_float
    libm.atan2f.argtypes = [C.c_float, C.c_float]
    lc.lc_atan2f_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
    import numpy as np
    rng = np.random.default_rng(11)
    bits = rng.integers(0, 2**32, 200_000, dtype=np.uint64).astype(np.uint32)
    y = bits.view(np.float32)
    y = y[np.isfinite(y)]
    y = np.concatenate([y, rng.uniform(-4, 4, 50_000).astype(np.float32), np.float32([0.0, -0.0, 1e-30, -3e38])])
    x = np.ones_like(y)
    out = np.empty_like(y)
    lc.lc_atan2f_batch(y.ctypes.data, x.ctypes.data, len(y), out.ctypes.data)
    ref = np.array([libm.atan2f(float(v), 1.0) for v in y], np.float32)
    assert out.view(np.uint32).tolist() == ref.view(np.uint32).tolist()
