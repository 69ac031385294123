"""MAGSAC-lite homography estimation (geom.cpp:104-333).

The inputs are the reference's own test fixtures (tests/test_geom.cpp:130-216,
acceptance.cpp:255-281), regenerated here with the same SplitMix64 stream and
the same double arithmetic, plus larger random sets.  The device result
(success, best iteration, score, H, inlier mask) must equal the reference's
bit for bit (oracle/_ref: the unmodified reference compiled in place).
"""
import numpy as np
import pytest

import paper_2605_17869_b200 as ds

from oracle import oracle as orc

gpu = pytest.mark.gpu


class SplitMix64:
    """geom.hpp:32-41."""

    def __init__(self, seed):
        self.s = seed & 0xFFFFFFFFFFFFFFFF

    def next(self):
        M = 0xFFFFFFFFFFFFFFFF
        self.s = (self.s + 0x9E3779B97F4A7C15) & M
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)

    def uniform(self, lo, hi):
        return lo + (hi - lo) * float(self.next() >> 11) / 9007199254740992.0


def apply_h(h, x, y):
    """Homography::apply (geom.cpp:15-20), same operation order."""
    w = h[6] * x + h[7] * y + h[8]
    return (h[0] * x + h[1] * y + h[2]) / w, (h[3] * x + h[4] * y + h[5]) / w


def inliers_outliers(h, seed, n_in, n_out, lo=10.0, hi_x=630.0, hi_y=470.0, seed_mult=1):
    rng = SplitMix64(seed * seed_mult)
    pts = []
    for _ in range(n_in):
        x = rng.uniform(lo, hi_x)
        y = rng.uniform(lo, hi_y)
        px, py = apply_h(h, x, y)
        pts.append((x, y, px, py))
    for _ in range(n_out):
        a = rng.uniform(0, 640)
        b = rng.uniform(0, 480)
        c = rng.uniform(0, 640)
        d = rng.uniform(0, 480)
        pts.append((a, b, c, d))
    return np.array(pts, np.float64)


def exact_inliers():
    """test_geom.cpp:130-144."""
    t = [1.05, -0.02, 8.0, 0.03, 0.98, -5.0, 1e-5, -1e-5, 1.0]
    rng = SplitMix64(17)
    pts = []
    for _ in range(40):
        x = 20 + float(rng.next() % 600)
        y = 20 + float(rng.next() % 440)
        px, py = apply_h(t, x, y)
        pts.append((x, y, px, py))
    return np.array(pts, np.float64)


H_6040 = [1.08, 0.04, -12.0, -0.05, 0.95, 9.0, 2e-5, -1e-5, 1.0]
H_DET = [1.0, 0.01, 3.0, -0.01, 1.0, -2.0, 0, 0, 1.0]
H_ACC = [1.07, 0.03, -10.0, -0.04, 0.96, 8.0, 2e-5, -1e-5, 1.0]


def cases():
    """(name, matches, iterations, tau, seed)"""
    out = [("exact_inliers", exact_inliers(), 200, 3.0, 7),
           ("inl60_out40", inliers_outliers(H_6040, 99, 60, 40), 1500, 3.0, 5)]
    det = inliers_outliers(H_DET, 55, 50, 30, lo=5.0, hi_x=635.0, hi_y=475.0)
    out += [("determinism_s42", det, 300, 3.0, 42), ("determinism_s43", det, 300, 3.0, 43)]
    rng = SplitMix64(3)
    allout = np.array([(rng.uniform(0, 640), rng.uniform(0, 480), rng.uniform(0, 640), rng.uniform(0, 480))
                       for _ in range(5)], np.float64)
    out.append(("all_outliers", allout, 10, 1e-6, 2))
    for seed in (1, 4, 10):   # acceptance.cpp:255-281 (criterion 8)
        out.append((f"acceptance_seed{seed}", inliers_outliers(H_ACC, seed, 60, 40, seed_mult=1234567), 1500, 3.0,
                    seed))
    big = inliers_outliers([0.97, 0.05, 14.0, -0.03, 1.02, -6.0, 3e-5, 2e-5, 1.0], 7, 1200, 800)
    out.append(("n2000_40pct_outliers", big, 400, 2.0, 11))
    return out


def _ref():
    if not orc.available("reference"):
        pytest.skip("oracle/_ref not built")
    return orc.Oracle("reference")


# ---------------------------------------------------------------- CPU tests
def test_fixture_generator_matches_reference_stream():
    # SplitMix64 restated in Python == the reference's (via its shim)
    import ctypes as C
    ref = _ref()
    r = SplitMix64(12345)
    state = C.c_uint64(12345)
    ref.lib.oref_splitmix_next.restype = C.c_uint64
    ref.lib.oref_splitmix_next.argtypes = [C.POINTER(C.c_uint64)]
    for _ in range(8):
        assert ref.lib.oref_splitmix_next(C.byref(state)) == r.next()


def test_corner_error_matches_reference():
    ref = _ref()
    rng = np.random.default_rng(3)
    for _ in range(200):
        he = np.eye(3).ravel() + rng.normal(0, 1e-3, 9) * [1, 1, 50, 1, 1, 50, 1e-3, 1e-3, 0]
        hg = np.eye(3).ravel() + rng.normal(0, 1e-3, 9) * [1, 1, 50, 1, 1, 50, 1e-3, 1e-3, 0]
        a = ds.corner_error(he, hg, 640, 480)
        b = ref.corner_error(he, hg, 640, 480)
        assert a == b
    # test_geom.cpp:91-104: a 3-4-5 translation moves every corner by exactly 5
    t = np.array([1, 0, 3, 0, 1, 4, 0, 0, 1], np.float64)
    assert ds.corner_error(t, np.eye(3), 640, 480) == 5.0


def test_corner_error_infinity_raises():
    bad = np.array([1, 0, 0, 0, 1, 0, -1.0 / 640.0, 0, 1])
    with pytest.raises(ds.GeometryError):
        ds.corner_error(bad, np.eye(3), 640, 480)


def test_reference_fixtures_reproduce_reference_test_expectations():
    # the regenerated fixtures behave as the reference's own tests expect
    ref = _ref()
    ok, best, score, h, mask = ref.magsac_lite(exact_inliers(), 200, 3.0, 7)
    assert ok and abs(score - 40.0) < 40.0 * 1e-6 and mask.sum() == 40
    m = inliers_outliers(H_6040, 99, 60, 40)
    ok, best, score, h, mask = ref.magsac_lite(m, 1500, 3.0, 5)
    assert ok and ref.corner_error(h, np.array(H_6040), 640, 480) < 1.0


# ---------------------------------------------------------------- GPU tests
@pytest.fixture(scope="module")
def ex():
    e = ds.Extractor()
    yield e
    e.close()


@gpu
@pytest.mark.parametrize("name,matches,iters,tau,seed", cases(), ids=[c[0] for c in cases()])
def test_magsac_bit_exact(ex, name, matches, iters, tau, seed):
    ref = _ref()
    ok, best, score, h, mask = ref.magsac_lite(matches, iters, tau, seed, workers=4)
    r = ex.magsac_lite(matches, iters, tau, seed)
    assert r.success == ok
    if not ok:
        return
    assert r.best_iteration == best
    assert np.float64(r.score).tobytes() == np.float64(score).tobytes()
    assert r.h.ravel().tobytes() == h.tobytes()
    assert np.array_equal(r.inlier_mask, mask)


@gpu
def test_magsac_recovers_acceptance_homography(ex):
    # acceptance criterion 8 (acceptance.cpp:255-281): corner error < 1 px for >= 9/10 seeds
    good = 0
    for seed in range(1, 11):
        m = inliers_outliers(H_ACC, seed, 60, 40, seed_mult=1234567)
        r = ex.magsac_lite(m, 1500, 3.0, seed)
        good += r.success and ds.corner_error(r.h, np.array(H_ACC), 640, 480) < 1.0
    assert good >= 9


@gpu
def test_magsac_preconditions(ex):
    m = np.array([[0, 0, 0, 0], [1, 1, 1, 1], [2, 0, 2, 0]], np.float64)
    with pytest.raises(ds.InvalidArgument):
        ex.magsac_lite(m, 100, 3.0, 1)
    m4 = exact_inliers()
    with pytest.raises(ds.InvalidArgument):
        ex.magsac_lite(m4, 100, 0.0, 1)
    with pytest.raises(ds.InvalidArgument):
        ex.magsac_lite(m4, 0, 3.0, 1)


def _dlt_cases():
    quad = [(10.0, 20.0), (200.0, 35.0), (180.0, 210.0), (25.0, 190.0)]
    ident = [1, 0, 0, 0, 1, 0, 0, 0, 1]
    trans = [1, 0, 5.5, 0, 1, -3.25, 0, 0, 1]
    proj = [1.1, 0.05, -7.0, -0.04, 0.92, 12.0, 1e-4, -5e-5, 1.0]
    out = []
    for name, h in (("identity", ident), ("translation", trans)):
        out.append((name, np.array([(x, y, *apply_h(h, x, y)) for x, y in quad]), None))
    rng = SplitMix64(8)
    pts = [(rng.uniform(0, 640), rng.uniform(0, 480)) for _ in range(25)]
    out.append(("projective_25", np.array([(x, y, *apply_h(proj, x, y)) for x, y in pts]), None))
    noisy = np.array([(x, y, apply_h(proj, x, y)[0] + rng.uniform(-1, 1), apply_h(proj, x, y)[1]
                       + rng.uniform(-1, 1)) for x, y in pts])
    w = np.array([rng.uniform(0.05, 1.0) for _ in pts])
    out.append(("weighted_noisy_25", noisy, w))
    return out


@gpu
@pytest.mark.parametrize("name,m,w", _dlt_cases(), ids=[c[0] for c in _dlt_cases()])
def test_dlt_bit_exact(ex, name, m, w):
    ref = _ref()
    assert ex.dlt_homography(m, w).ravel().tobytes() == ref.dlt_homography(m, w).tobytes()


@gpu
def test_dlt_degenerate_raises(ex):
    # test_geom.cpp:56-63: three collinear source points
    m = np.array([[0, 0, 0, 0], [1, 1, 2, 3], [2, 2, 5, 1], [7, 3, 1, 9]], np.float64)
    with pytest.raises(ds.GeometryError):
        ex.dlt_homography(m)
    with pytest.raises(ds.InvalidArgument):
        ex.dlt_homography(m[:3])
