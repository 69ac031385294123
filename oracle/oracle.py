"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY (the CPU parity checker).

ctypes front-end for the two CPU implementations of the reference extraction
path (``detsift::extract``, /root/reference/proj/src/io.cpp:111-142):

* ``Oracle("port")``      -> oracle/liboracle.so, the plain-C restatement
                              (oracle/dsift_oracle.c);
* ``Oracle("reference")`` -> oracle/_ref/libdetsift_ref.so, the unmodified
                              reference compiled in place by oracle/Makefile.

Both expose the same stage-level surface (scale space, extrema, refinement,
orientation, descriptors, canonical sort, DSF1/SHA-256) so tests can diff them
against each other and against the CUDA product.  Only tests/,
``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may import this.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "port": os.path.join(HERE, "liboracle.so"),
    "reference": os.path.join(HERE, "_ref", "libdetsift_ref.so"),
}
PREFIX = {"port": "dor_", "reference": "oref_"}

KEYPOINT_DTYPE = np.dtype(
    [("x", "<f4"), ("y", "<f4"), ("sigma", "<f4"), ("angle", "<f4"),
     ("response", "<f4"), ("octave", "<i4"), ("interval", "<i4")])
DESC_DIM = 128


class Config(C.Structure):
    """Mirror of detsift::SiftConfig (core.hpp:30-47) / dsift_config."""
    _fields_ = [
        ("sigma0", C.c_float), ("intervals", C.c_int32), ("assumed_blur", C.c_float),
        ("contrast_threshold", C.c_float), ("edge_ratio", C.c_float),
        ("max_refine_iters", C.c_int32), ("upsample_pixel_limit", C.c_int64),
        ("dsp_scales", C.POINTER(C.c_double)), ("n_dsp_scales", C.c_int32),
        ("descriptor_clip", C.c_float), ("orientation_bins", C.c_int32),
        ("orientation_peak_ratio", C.c_float), ("num_octaves", C.c_int32),
    ]


DEFAULT_DSP = (0.5, 1.0 / 1.4142135623730951, 1.0, 1.4142135623730951, 2.0)


def make_config(**kw) -> Config:
    """SiftConfig defaults (core.hpp:30-47) with keyword overrides."""
    scales = tuple(kw.pop("dsp_scales", DEFAULT_DSP))
    c = Config(sigma0=1.6, intervals=3, assumed_blur=0.5, contrast_threshold=0.04,
               edge_ratio=10.0, max_refine_iters=5, upsample_pixel_limit=4_000_000,
               descriptor_clip=0.2, orientation_bins=36, orientation_peak_ratio=0.8,
               num_octaves=0)
    for k, v in kw.items():
        setattr(c, k, v)
    arr = (C.c_double * max(1, len(scales)))(*scales)
    c._scales = arr  # keep alive
    c.dsp_scales = C.cast(arr, C.POINTER(C.c_double))
    c.n_dsp_scales = len(scales)
    return c


class OracleError(ValueError):
    pass


def _fp(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


@dataclass
class ScaleSpace:
    lib: "Oracle"
    handle: int
    n_oct: int
    upsampled: bool
    dims: list
    s: int

    def level(self, o: int, kind: str, i: int) -> np.ndarray:
        w, h = self.dims[o]
        out = np.empty((h, w), np.float32)
        self.lib._f("ss_level")(C.c_void_p(self.handle), o, 0 if kind == "gauss" else 1, i, _fp(out))
        return out

    def __del__(self):
        try:
            self.lib._f("ss_free")(C.c_void_p(self.handle))
        except Exception:
            pass


class Oracle:
    def __init__(self, kind: str = "port"):
        path = LIBS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run make -C oracle)")
        self.kind = kind
        self.lib = C.CDLL(path)
        self.p = PREFIX[kind]
        self._setup()

    def _f(self, name):
        return getattr(self.lib, self.p + name)

    def _setup(self):
        f = self._f
        f("last_error").restype = C.c_char_p
        f("extract").argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(Config)] + (
            [C.c_int, C.POINTER(C.c_void_p)] if self.kind == "reference"
            else [C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_int64)])
        f("tree_sum").restype = C.c_float
        if self.kind != "reference":
            self.lib.dor_free.argtypes = [C.c_void_p]
            self.lib.dor_build_scale_space.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(Config),
                                                       C.POINTER(C.c_void_p)]
        f("tree_sum_f64").restype = C.c_double
        f("hash_features").argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_char_p]
        f("serialize").restype = C.c_int64
        f("serialize").argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64]
        f("find_extrema").restype = C.c_int64
        f("detect").restype = C.c_int64
        f("nearest_gauss_level").argtypes = [C.c_void_p, C.c_double]
        f("value_noise").argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_void_p]
        f("gaussian_kernel").argtypes = [C.c_double, C.c_void_p, C.c_int]
        f("raw_descriptor").argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.POINTER(Config), C.c_void_p]
        f("ss_from_levels").restype = C.c_void_p
        f("ss_from_levels").argtypes = [C.c_int, C.c_int, C.c_float, C.c_int, C.c_void_p,
                                        C.c_void_p, C.c_void_p]
        if self.kind == "reference":
            self.lib.oref_fs_size.restype = C.c_int64
            self.lib.oref_fs_size.argtypes = [C.c_void_p]
            self.lib.oref_fs_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
            self.lib.oref_fs_free.argtypes = [C.c_void_p]
            self.lib.oref_ss_build.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(Config), C.c_int,
                                               C.POINTER(C.c_void_p)]
            self.lib.oref_splitmix_next.restype = C.c_uint64
            self.lib.oref_blob_field.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_void_p]
            self.lib.oref_add_blob.argtypes = [C.c_void_p, C.c_int, C.c_int] + [C.c_double] * 4
            self.lib.oref_photometric.argtypes = [C.c_void_p, C.c_int, C.c_int] + [C.c_double] * 3 + [C.c_void_p]
            self.lib.oref_warp_similarity.argtypes = ([C.c_void_p, C.c_int, C.c_int] + [C.c_double] * 4
                                                      + [C.c_int, C.c_int, C.c_void_p])
            self.lib.oref_brute_force_detect.restype = C.c_int64

    def error(self) -> str:
        return self._f("last_error")().decode()

    # ---- synthetic input -------------------------------------------------
    def value_noise(self, w, h, seed, octaves=4, cells=8) -> np.ndarray:
        out = np.empty((h, w), np.float32)
        self._f("value_noise")(w, h, C.c_uint64(seed), octaves, cells, out.ctypes.data)
        return out

    # ---- matching (match.cpp:71-119), reference only ----------------------
    def ratio_match(self, da: np.ndarray, db: np.ndarray, ratio: float = 0.8, workers: int = 1):
        """MatchSet ratio_match(a, b, ratio): (pairs [k, 3] int32 with the distance
        bits in column 2, putative_a, putative_b)."""
        if self.kind != "reference":
            raise OracleError("ratio_match: the reference library only")
        da = np.ascontiguousarray(da, np.float32)
        db = np.ascontiguousarray(db, np.float32)
        fn = self.lib.oref_ratio_match
        fn.restype = C.c_int64
        fn.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int, C.c_float, C.c_int,
                       C.c_void_p, C.c_int64, C.c_void_p]
        cap = max(1, min(len(da), len(db)))
        out = np.zeros((cap, 3), np.int32)
        put = np.zeros(2, np.int64)
        n = fn(da.ctypes.data, len(da), db.ctypes.data, len(db), da.shape[1] if da.ndim == 2 else 128,
               C.c_float(ratio), workers, out.ctypes.data, cap, put.ctypes.data)
        if n < 0:
            raise OracleError(self.error())
        return out[:n], int(put[0]), int(put[1])

    # ---- geometry (geom.cpp:108-333), reference only ----------------------
    def _geom_rc(self, rc):
        if rc == 1:
            raise ValueError(self.error())
        if rc == 2:
            raise RuntimeError(self.error())

    def magsac_lite(self, matches, iterations: int, tau: float, seed: int, workers: int = 1):
        """(success, best_iteration, score, h [9], inlier_mask [n]) of
        detsift::magsac_lite."""
        if self.kind != "reference":
            raise OracleError("magsac_lite: the reference library only")
        m = np.ascontiguousarray(matches, np.float64).reshape(-1, 4)
        fn = self.lib.oref_magsac_lite
        fn.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_void_p,
                       C.c_void_p, C.c_void_p]
        sb = np.zeros(2, np.int32)
        sh = np.zeros(10, np.float64)
        mask = np.zeros(len(m), np.uint8)
        self._geom_rc(fn(m.ctypes.data, len(m), int(iterations), C.c_double(tau), C.c_uint64(seed), workers,
                         sb.ctypes.data, sh.ctypes.data, mask.ctypes.data))
        return bool(sb[0]), int(sb[1]), float(sh[0]), sh[1:].copy(), mask

    def dlt_homography(self, matches, weights=None) -> np.ndarray:
        if self.kind != "reference":
            raise OracleError("dlt_homography: the reference library only")
        m = np.ascontiguousarray(matches, np.float64).reshape(-1, 4)
        fn = self.lib.oref_dlt_homography
        fn.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
        w = None if weights is None else np.ascontiguousarray(weights, np.float64)
        out = np.zeros(9, np.float64)
        self._geom_rc(fn(m.ctypes.data, len(m), None if w is None else w.ctypes.data, out.ctypes.data))
        return out

    def corner_error(self, h_est, h_gt, width: float, height: float) -> float:
        fn = self.lib.oref_corner_error
        fn.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_void_p]
        a = np.ascontiguousarray(h_est, np.float64).reshape(9)
        b = np.ascontiguousarray(h_gt, np.float64).reshape(9)
        out = C.c_double()
        self._geom_rc(fn(a.ctypes.data, b.ctypes.data, float(width), float(height), C.byref(out)))
        return out.value

    def descriptor_distance(self, a: np.ndarray, b: np.ndarray) -> float:
        fn = self.lib.oref_descriptor_distance
        fn.restype = C.c_float
        fn.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return fn(a.ctypes.data, b.ctypes.data, len(a))

    # ---- image ingest (io.cpp:49-81) -------------------------------------
    def load_image(self, path: str) -> np.ndarray:
        w, h = C.c_int(), C.c_int()
        fn = self._f("load_image")
        fn.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p]
        if fn(os.fsencode(path), C.byref(w), C.byref(h), None):
            raise OracleError(self.error())
        out = np.empty((h.value, w.value), np.float32)
        if fn(os.fsencode(path), C.byref(w), C.byref(h), out.ctypes.data):
            raise OracleError(self.error())
        return out

    # ---- full pipeline -----------------------------------------------------
    def extract(self, img: np.ndarray, cfg: Config | None = None, workers: int = 1):
        img = np.ascontiguousarray(img, np.float32)
        cfg = cfg or make_config()
        h, w = img.shape
        if self.kind == "reference":
            fs = C.c_void_p()
            rc = self.lib.oref_extract(img.ctypes.data, w, h, C.byref(cfg), workers, C.byref(fs))
            if rc:
                raise OracleError(self.error())
            n = self.lib.oref_fs_size(fs)
            kps = np.empty(n, KEYPOINT_DTYPE)
            desc = np.empty((n, DESC_DIM), np.float32)
            self.lib.oref_fs_copy(fs, kps.ctypes.data, desc.ctypes.data)
            self.lib.oref_fs_free(fs)
            return kps, desc
        kp_p, d_p, n = C.c_void_p(), C.c_void_p(), C.c_int64()
        rc = self.lib.dor_extract(img.ctypes.data, w, h, C.byref(cfg), C.byref(kp_p), C.byref(d_p),
                                  C.byref(n))
        if rc:
            raise OracleError(self.error())
        kps = np.empty(n.value, KEYPOINT_DTYPE)
        desc = np.empty((n.value, DESC_DIM), np.float32)
        C.memmove(kps.ctypes.data, kp_p, kps.nbytes)
        C.memmove(desc.ctypes.data, d_p, desc.nbytes)
        self.lib.dor_free(kp_p)
        self.lib.dor_free(d_p)
        return kps, desc

    def hash_features(self, kps, desc) -> str:
        buf = C.create_string_buffer(65)
        self._f("hash_features")(kps.ctypes.data, desc.ctypes.data, len(kps), buf)
        return buf.value.decode()

    def serialize(self, kps, desc) -> bytes:
        n = self._f("serialize")(kps.ctypes.data, desc.ctypes.data, len(kps), None, 0)
        out = np.empty(n, np.uint8)
        self._f("serialize")(kps.ctypes.data, desc.ctypes.data, len(kps), out.ctypes.data, n)
        return out.tobytes()

    def canonical_sort(self, kps, desc):
        kps = kps.copy()
        desc = np.ascontiguousarray(desc, np.float32).copy()
        self._f("canonical_sort")(kps.ctypes.data, desc.ctypes.data, C.c_int64(len(kps)))
        return kps, desc

    # ---- stages ---------------------------------------------------------------
    def scale_space(self, img: np.ndarray, cfg: Config | None = None) -> ScaleSpace:
        img = np.ascontiguousarray(img, np.float32)
        cfg = cfg or make_config()
        h, w = img.shape
        hnd = C.c_void_p()
        if self.kind == "reference":
            rc = self.lib.oref_ss_build(img.ctypes.data, w, h, C.byref(cfg), 1, C.byref(hnd))
        else:
            rc = self.lib.dor_build_scale_space(img.ctypes.data, w, h, C.byref(cfg), C.byref(hnd))
        if rc:
            raise OracleError(self.error())
        return self._wrap_ss(hnd.value, cfg.intervals)

    def _wrap_ss(self, hnd, s):
        n_oct, up = C.c_int32(), C.c_int32()
        dims = np.zeros(128, np.int32)
        self._f("ss_info")(C.c_void_p(hnd), C.byref(n_oct), C.byref(up), dims.ctypes.data)
        d = [(int(dims[2 * o]), int(dims[2 * o + 1])) for o in range(n_oct.value)]
        return ScaleSpace(self, hnd, n_oct.value, bool(up.value), d, s)

    def scale_space_from_levels(self, gauss, dog, s=3, sigma0=1.6, upsampled=False):
        """gauss[o][i], dog[o][i]: 2-D float32 arrays (handcrafted spaces, test_detect.cpp:14-30)."""
        n_oct = len(gauss)
        dims = np.array([v for o in range(n_oct) for v in (gauss[o][0].shape[1], gauss[o][0].shape[0])],
                        np.int32)
        g = [np.ascontiguousarray(a, np.float32) for o in range(n_oct) for a in gauss[o]]
        d = [np.ascontiguousarray(a, np.float32) for o in range(n_oct) for a in dog[o]]
        gp = (C.c_void_p * len(g))(*[a.ctypes.data for a in g])
        dp = (C.c_void_p * len(d))(*[a.ctypes.data for a in d])
        hnd = self._f("ss_from_levels")(n_oct, s, C.c_float(sigma0), int(upsampled), dims.ctypes.data, gp, dp)
        return self._wrap_ss(hnd, s)

    def find_extrema(self, ss: ScaleSpace, cfg=None) -> np.ndarray:
        cfg = cfg or make_config()
        args = [C.c_void_p(ss.handle), C.byref(cfg)] + ([1] if self.kind == "reference" else [])
        n = self._f("find_extrema")(*args, None, C.c_int64(0))
        out = np.zeros((max(n, 1), 5), np.int32)
        self._f("find_extrema")(*args, out.ctypes.data, C.c_int64(n))
        return out[:n]

    def refine(self, ss: ScaleSpace, e5, cfg=None):
        cfg = cfg or make_config()
        e = np.ascontiguousarray(e5, np.int32)
        kp = np.zeros(1, KEYPOINT_DTYPE)
        ok = self._f("refine")(C.c_void_p(ss.handle), e.ctypes.data, C.byref(cfg), kp.ctypes.data)
        return kp[0] if ok else None

    def detect(self, ss: ScaleSpace, cfg=None) -> np.ndarray:
        cfg = cfg or make_config()
        args = [C.c_void_p(ss.handle), C.byref(cfg)] + ([1] if self.kind == "reference" else [])
        n = self._f("detect")(*args, None, C.c_int64(0))
        out = np.zeros(max(n, 1), KEYPOINT_DTYPE)
        self._f("detect")(*args, out.ctypes.data, C.c_int64(n))
        return out[:n]

    def orientation_histogram(self, ss, kp, cfg=None) -> np.ndarray:
        cfg = cfg or make_config()
        k = np.array([kp], KEYPOINT_DTYPE)
        out = np.zeros(cfg.orientation_bins, np.float32)
        self._f("orientation_histogram")(C.c_void_p(ss.handle), k.ctypes.data, C.byref(cfg), out.ctypes.data)
        return out

    def assign_orientations(self, ss, kp, cfg=None) -> np.ndarray:
        cfg = cfg or make_config()
        k = np.array([kp], KEYPOINT_DTYPE)
        out = np.zeros(cfg.orientation_bins + 1, KEYPOINT_DTYPE)
        n = self._f("assign_orientations")(C.c_void_p(ss.handle), k.ctypes.data, C.byref(cfg), out.ctypes.data)
        return out[:n]

    def nearest_gauss_level(self, ss, sigma_rel) -> int:
        return self._f("nearest_gauss_level")(C.c_void_p(ss.handle), sigma_rel)

    def raw_descriptor(self, ss, kp, f, cfg=None) -> np.ndarray:
        cfg = cfg or make_config()
        k = np.array([kp], KEYPOINT_DTYPE)
        out = np.zeros(DESC_DIM, np.float32)
        rc = self._f("raw_descriptor")(C.c_void_p(ss.handle), k.ctypes.data, f, C.byref(cfg), out.ctypes.data)
        if rc:
            raise OracleError(self.error())
        return out

    def dsp_descriptor(self, ss, kp, cfg=None) -> np.ndarray:
        cfg = cfg or make_config()
        k = np.array([kp], KEYPOINT_DTYPE)
        out = np.zeros(DESC_DIM, np.float32)
        rc = self._f("dsp_descriptor")(C.c_void_p(ss.handle), k.ctypes.data, C.byref(cfg), out.ctypes.data)
        if rc:
            raise OracleError(self.error())
        return out

    def gaussian_kernel(self, sigma) -> np.ndarray:
        out = np.zeros(1024, np.float32)
        n = self._f("gaussian_kernel")(sigma, out.ctypes.data, 1024)
        if n < 0:
            raise OracleError(self.error())
        return out[:n]

    def tree_sum(self, v) -> np.float32:
        v = np.ascontiguousarray(v, np.float32)
        args = [v.ctypes.data, C.c_int64(len(v))] + ([1] if self.kind == "reference" else [])
        return np.float32(self._f("tree_sum")(*args))

    def tree_hist(self, bins, weights, bin_count) -> np.ndarray:
        b = np.ascontiguousarray(bins, np.int32)
        w = np.ascontiguousarray(weights, np.float32)
        out = np.zeros(bin_count, np.float32)
        args = [b.ctypes.data, w.ctypes.data, C.c_int64(len(b)), bin_count] + (
            [1] if self.kind == "reference" else [])
        rc = self._f("tree_hist")(*args, out.ctypes.data)
        if rc:
            raise OracleError(self.error())
        return out

    def config_validate(self, cfg) -> str | None:
        rc = self._f("config_validate")(C.byref(cfg))
        return self.error() if rc else None


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind])
