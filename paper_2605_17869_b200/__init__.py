"""paper_2605_17869_b200 — B200-native SIFT extraction behind the detsift API.

Python mirror of the reference's extraction surface (detsift::extract and the
stage functions its tests call: /root/reference/proj/include/detsift/*.hpp),
implemented over the C ABI in include/dsift.h (libdsift.so: hand-written
sm_100a CUDA kernels + C++ orchestration).  There is no CPU fallback: if the
library or a CUDA device is missing every entry point raises ``DsiftError``.

    from paper_2605_17869_b200 import SiftConfig, extract
    fs = extract(image_float32_hw, SiftConfig())      # FeatureSet
    fs.keypoints  # structured array (x, y, sigma, angle, response, octave, interval)
    fs.descriptors  # (n, 128) float32, canonical order (core.cpp:116-170)
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass, field

import numpy as np
from typing import NamedTuple

__all__ = [
    "SiftConfig", "FeatureSet", "KEYPOINT_DTYPE", "DsiftError", "Extractor", "extract",
    "library_path", "load_library",
]

HERE = os.path.dirname(os.path.abspath(__file__))
KEYPOINT_DTYPE = np.dtype(
    [("x", "<f4"), ("y", "<f4"), ("sigma", "<f4"), ("angle", "<f4"),
     ("response", "<f4"), ("octave", "<i4"), ("interval", "<i4")])
MATCH_DTYPE = np.dtype([("a", np.int32), ("b", np.int32), ("distance", np.float32)])   # detsift::Match
DESC_DIM = 128

(DSIFT_OK, DSIFT_EINVAL, DSIFT_ECAPACITY, DSIFT_ECUDA, DSIFT_ENOMEM, DSIFT_ESTATE, DSIFT_ERANGE, DSIFT_EIO,
 DSIFT_EGEOM) = range(9)
INPUT_HOST, INPUT_DEVICE = 0, 1


class DsiftError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class InvalidArgument(DsiftError, ValueError):
    """std::invalid_argument in the reference."""


class ImageIOError(DsiftError, RuntimeError):
    """std::runtime_error from load_image (io.cpp:49-81)."""


class GeometryError(DsiftError, RuntimeError):
    """std::runtime_error from the geometry code (geom.cpp: degenerate DLT,
    point mapped to infinity)."""


class OutOfRange(DsiftError, IndexError):
    """std::out_of_range in the reference (detsum.cpp:138-141)."""


class _Config(C.Structure):
    _fields_ = [
        ("sigma0", C.c_float), ("intervals", C.c_int32), ("assumed_blur", C.c_float),
        ("contrast_threshold", C.c_float), ("edge_ratio", C.c_float),
        ("max_refine_iters", C.c_int32), ("upsample_pixel_limit", C.c_int64),
        ("dsp_scales", C.POINTER(C.c_double)), ("n_dsp_scales", C.c_int32),
        ("descriptor_clip", C.c_float), ("orientation_bins", C.c_int32),
        ("orientation_peak_ratio", C.c_float), ("num_octaves", C.c_int32),
    ]


@dataclass
class SiftConfig:
    """detsift::SiftConfig (core.hpp:30-47), same defaults and field meaning."""
    sigma0: float = 1.6
    intervals_per_octave: int = 3
    assumed_input_blur: float = 0.5
    contrast_threshold: float = 0.04
    edge_ratio: float = 10.0
    max_refine_iters: int = 5
    upsample_pixel_limit: int = 4_000_000
    dsp_scales: tuple = (0.5, 1.0 / 1.4142135623730951, 1.0, 1.4142135623730951, 2.0)
    descriptor_clip: float = 0.2
    orientation_bins: int = 36
    orientation_peak_ratio: float = 0.8
    num_octaves: int = 0

    def to_c(self) -> _Config:
        arr = (C.c_double * max(1, len(self.dsp_scales)))(*self.dsp_scales)
        c = _Config(self.sigma0, self.intervals_per_octave, self.assumed_input_blur,
                    self.contrast_threshold, self.edge_ratio, self.max_refine_iters,
                    self.upsample_pixel_limit, C.cast(arr, C.POINTER(C.c_double)),
                    len(self.dsp_scales), self.descriptor_clip, self.orientation_bins,
                    self.orientation_peak_ratio, self.num_octaves)
        c._keep = arr
        return c

    def validate(self) -> None:
        """SiftConfig::validate (core.cpp:17-46); raises InvalidArgument."""
        lib = load_library()
        _check(lib, lib.dsift_config_validate(C.byref(self.to_c())))


@dataclass
class FeatureSet:
    """detsift::FeatureSet (core.hpp:66-78) + the uint8 export."""
    keypoints: np.ndarray = field(default_factory=lambda: np.zeros(0, KEYPOINT_DTYPE))
    descriptors: np.ndarray = field(default_factory=lambda: np.zeros((0, DESC_DIM), np.float32))
    descriptors_u8: np.ndarray | None = None
    dim: int = DESC_DIM

    def __len__(self) -> int:
        return len(self.keypoints)

    def size(self) -> int:
        return len(self.keypoints)

    def row(self, i: int) -> np.ndarray:
        return self.descriptors[i]


_LIB = None


def library_path() -> str:
    return os.path.join(HERE, "libdsift.so")


def load_library(path: str | None = None):
    """Loads the in-tree libdsift.so (fails loudly; no fallback).  `path` names
    another build of the same ABI explicitly (the test-only negative-control
    library); it must be given before the first load."""
    global _LIB
    if _LIB is not None:
        if path is not None and getattr(_LIB, "_path", None) != os.path.abspath(path):
            raise DsiftError(DSIFT_ESTATE, "load_library: a different library is already loaded")
        return _LIB
    path = os.path.abspath(path) if path is not None else library_path()
    if not os.path.exists(path):
        raise DsiftError(DSIFT_ECUDA, f"CUDA extension missing: {path} (run __graft_entry__.build())")
    lib = C.CDLL(path)
    vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int
    sig = {
        "dsift_abi_version": ([], C.c_int), "dsift_strerror": ([C.c_int], C.c_char_p),
        "dsift_last_error": ([], C.c_char_p), "dsift_config_default": ([vp], None),
        "dsift_config_validate": ([vp], C.c_int), "dsift_create": ([i32, vp, vp], C.c_int),
        "dsift_destroy": ([vp], None), "dsift_set_stream": ([vp, vp], C.c_int),
        "dsift_set_capacity": ([vp, i64], C.c_int),
        "dsift_extract_batch": ([vp, vp, i32, i32, i32, i32], C.c_int),
        "dsift_extract": ([vp, vp, i32, i32, i32], C.c_int),
        "dsift_extract_batch_u8": ([vp, vp, i32, i32, i32, i32, i32], C.c_int),
        "dsift_load_image": ([C.c_char_p, vp, vp, vp, vp, i64], C.c_int),
        "dsift_ratio_match": ([vp, vp, i64, vp, i64, i32, i32, C.c_float, i32, vp, i64, vp, vp, vp], C.c_int),
        "dsift_ingest_u8": ([vp, vp, i64, i32, i32, vp], C.c_int),
        "dsift_magsac_lite": ([vp, vp, i64, i32, C.c_double, C.c_uint64, vp, vp], C.c_int),
        "dsift_dlt_homography": ([vp, vp, i64, vp, vp], C.c_int),
        "dsift_corner_error": ([vp, vp, C.c_double, C.c_double, vp], C.c_int),
        "dsift_result_sync": ([vp, vp], C.c_int), "dsift_result_range": ([vp, i32, vp, vp], C.c_int),
        "dsift_result_copy": ([vp, vp, vp, vp, vp], C.c_int),
        "dsift_result_device": ([vp, vp, vp, vp, vp], C.c_int),
        "dsift_export_dlpack": ([vp, i32, vp], C.c_int),
        "dsift_result_sha256": ([vp, i32, C.c_char_p], C.c_int),
        "dsift_build_scale_space": ([vp, vp, i32, i32, i32], C.c_int),
        "dsift_load_scale_space": ([vp, i32, i32, vp, vp, vp], C.c_int),
        "dsift_scale_space_info": ([vp, vp, vp, vp], C.c_int),
        "dsift_scale_space_level": ([vp, i32, i32, i32, vp], C.c_int),
        "dsift_find_extrema": ([vp, vp, i64, vp], C.c_int),
        "dsift_detect": ([vp, vp, i64, vp], C.c_int),
        "dsift_orientation_histograms": ([vp, vp, i64, vp], C.c_int),
        "dsift_assign_orientations": ([vp, vp, i64, vp, i64, vp], C.c_int),
        "dsift_raw_descriptors": ([vp, vp, i64, C.c_double, vp], C.c_int),
        "dsift_dsp_descriptors": ([vp, vp, i64, vp, vp], C.c_int),
        "dsift_synth_value_noise": ([vp, vp, i32, i32, i32, C.c_uint64, i32, i32], C.c_int),
        "dsift_kernel_launches": ([vp], C.c_int64),
        "dsift_set_profiling": ([vp, i32], C.c_int), "dsift_stage_times": ([vp, vp], C.c_int),
        "dsift_set_option": ([vp, i32, i64], C.c_int), "dsift_stat": ([vp, i32], C.c_int64),
        "dsift_extract_images": ([vp, vp, i32, i32], C.c_int),
        "dsift_result_create": ([vp, vp], C.c_int), "dsift_result_destroy": ([vp], None),
        "dsift_result_select": ([vp, vp], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    lib._path = path
    _LIB = lib
    return lib


def _check(lib, rc: int) -> None:
    if rc != DSIFT_OK:
        msg = lib.dsift_last_error().decode()
        if rc == DSIFT_EINVAL:
            raise InvalidArgument(rc, msg)
        if rc == DSIFT_ERANGE:
            raise OutOfRange(rc, msg)
        if rc == DSIFT_EIO:
            raise ImageIOError(rc, msg)
        if rc == DSIFT_EGEOM:
            raise GeometryError(rc, msg)
        raise DsiftError(rc, f"{lib.dsift_strerror(rc).decode()}: {msg}")


def _f32(img) -> np.ndarray:
    a = np.ascontiguousarray(img, dtype=np.float32)
    if a.ndim != 2:
        raise InvalidArgument(DSIFT_EINVAL, "image must be a 2-D [h, w] float32 array")
    return a


class Extractor:
    """One dsift_ctx: a device, a stream, a config and the last result."""

    def __init__(self, cfg: SiftConfig | None = None, device: int = 0):
        self.lib = load_library()
        self.cfg = cfg or SiftConfig()
        self._ccfg = self.cfg.to_c()
        ctx = C.c_void_p()
        _check(self.lib, self.lib.dsift_create(device, C.byref(self._ccfg), C.byref(ctx)))
        self.ctx = ctx
        self.device = device
        self._batch = 0
        self._own_batch = 0
        self._selected = None
        self._stream = None

    @property
    def batch(self) -> int:
        return self._batch

    @batch.setter
    def batch(self, n: int) -> None:
        self._batch = n
        if getattr(self, "_selected", None) is not None:
            self._selected.batch = n
        else:
            self._own_batch = n

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.dsift_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- hot path ----------------------------------------------------------
    def set_stream(self, cuda_stream_handle: int | None) -> None:
        _check(self.lib, self.lib.dsift_set_stream(self.ctx, C.c_void_p(cuda_stream_handle or 0)))
        self._stream = cuda_stream_handle

    def set_capacity(self, per_image: int) -> None:
        _check(self.lib, self.lib.dsift_set_capacity(self.ctx, per_image))

    def submit(self, images, n: int | None = None, w: int | None = None, h: int | None = None,
               device_ptr: int | None = None) -> None:
        """Enqueue a batch: host array [n, h, w] / [h, w], or a device pointer."""
        if device_ptr is not None:
            _check(self.lib, self.lib.dsift_extract_batch(self.ctx, C.c_void_p(device_ptr), n, w, h,
                                                          INPUT_DEVICE))
            self.batch = n
            return
        a = np.ascontiguousarray(images, dtype=np.float32)
        if a.ndim == 2:
            a = a[None]
        if a.ndim != 3:
            raise InvalidArgument(DSIFT_EINVAL, "images must be [n, h, w] float32")
        self._pin = a
        _check(self.lib, self.lib.dsift_extract_batch(self.ctx, a.ctypes.data, a.shape[0], a.shape[2],
                                                      a.shape[1], INPUT_HOST))
        self.batch = a.shape[0]

    def submit_images(self, images, device: bool = False) -> None:
        """Enqueue a ragged batch (dsift_extract_images): a list of [h, w]
        float32 host arrays of any sizes, or (device_ptr, w, h) tuples."""
        n = len(images)
        arr = (_Image * max(1, n))()
        keep = []
        for i, im in enumerate(images):
            if device:
                ptr, w, h = im
                arr[i] = _Image(C.c_void_p(ptr), w, h)
            else:
                a = _f32(im)
                keep.append(a)
                arr[i] = _Image(C.c_void_p(a.ctypes.data), a.shape[1], a.shape[0])
        self._pin = (arr, keep)
        _check(self.lib, self.lib.dsift_extract_images(self.ctx, arr, n, INPUT_DEVICE if device else INPUT_HOST))
        self.batch = n

    def extract_images(self, images) -> list[FeatureSet]:
        """detsift::extract over images of any sizes in one call; results in batch order."""
        self.submit_images(images)
        return self.results()

    def new_result(self) -> "Result":
        """A result handle of this context (dsift_result_create)."""
        return Result(self)

    def select(self, result: "Result | None") -> None:
        """Route the following extract / result calls to `result` (None = the context's own)."""
        _check(self.lib, self.lib.dsift_result_select(self.ctx, result.handle if result else None))
        self._selected = result
        self._batch = result.batch if result else self._own_batch

    def sync(self) -> int:
        total = C.c_int64()
        _check(self.lib, self.lib.dsift_result_sync(self.ctx, C.byref(total)))
        return total.value

    def offsets(self) -> np.ndarray:
        """Per-image result offsets [batch + 1] of the last batch (host copy)."""
        self.sync()
        out = np.zeros(self.batch + 1, np.int64)
        for b in range(self.batch):
            beg, cnt = C.c_int64(), C.c_int64()
            _check(self.lib, self.lib.dsift_result_range(self.ctx, b, C.byref(beg), C.byref(cnt)))
            out[b], out[b + 1] = beg.value, beg.value + cnt.value
        return out

    def results(self, with_u8: bool = True) -> list[FeatureSet]:
        total = self.sync()
        kps = np.zeros(total, KEYPOINT_DTYPE)
        desc = np.zeros((total, DESC_DIM), np.float32)
        u8 = np.zeros((total, DESC_DIM), np.uint8) if with_u8 else None
        offs = np.zeros(self.batch + 1, np.int64)
        _check(self.lib, self.lib.dsift_result_copy(self.ctx, kps.ctypes.data, desc.ctypes.data,
                                                    u8.ctypes.data if with_u8 else None, offs.ctypes.data))
        out = []
        for b in range(self.batch):
            s, e = int(offs[b]), int(offs[b + 1])
            out.append(FeatureSet(kps[s:e], desc[s:e], u8[s:e] if with_u8 else None))
        return out

    def submit_u8(self, pixels) -> None:
        """Enqueue 8-bit images converted on the device exactly as load_image does
        (io.cpp:71-78): [h, w] or [n, h, w] gray (P5), [n, h, w, 3] RGB (P6)."""
        a = np.ascontiguousarray(pixels, dtype=np.uint8)
        if a.ndim == 2:
            a = a[None]
        if a.ndim == 3:
            ch = 1
        elif a.ndim == 4 and a.shape[-1] == 3:
            ch = 3
        else:
            raise InvalidArgument(DSIFT_EINVAL, "pixels must be [n, h, w] or [n, h, w, 3] uint8")
        self._pin = a
        _check(self.lib, self.lib.dsift_extract_batch_u8(self.ctx, a.ctypes.data, a.shape[0], a.shape[2],
                                                         a.shape[1], ch, INPUT_HOST))
        self.batch = a.shape[0]

    def extract_u8(self, pixels) -> list[FeatureSet]:
        """extract(load_image(...)) for a batch of 8-bit images."""
        self.submit_u8(pixels)
        return self.results()

    def ingest_u8(self, pixels) -> np.ndarray:
        """The float GrayImage load_image builds from these bytes, converted on the device."""
        import torch
        a = np.ascontiguousarray(pixels, dtype=np.uint8)
        ch = 3 if (a.ndim >= 3 and a.shape[-1] == 3) else 1
        n_px = a.size // ch
        out = torch.empty(n_px, dtype=torch.float32, device=f"cuda:{self.device}")
        _check(self.lib, self.lib.dsift_ingest_u8(self.ctx, a.ctypes.data, n_px, ch, INPUT_HOST,
                                                  C.c_void_p(out.data_ptr())))
        shape = a.shape[:-1] if ch == 3 else a.shape
        return out.cpu().numpy().reshape(shape)

    def ratio_match(self, desc_a, desc_b, ratio: float = 0.8):
        """detsift::ratio_match (match.cpp:77-119) on the device: returns
        (pairs structured [k] (a, b, distance), putative_a, putative_b).  Inputs are
        host arrays [n, 128] float32 or torch CUDA tensors (zero copy: contiguous
        float32 [n, 128] on this context's device; the call is ordered after the
        current torch stream)."""
        flags = INPUT_HOST
        stream = None
        if hasattr(desc_a, "data_ptr") and getattr(desc_a, "is_cuda", False):
            import torch
            for t in (desc_a, desc_b):
                if not (getattr(t, "is_cuda", False) and t.dtype == torch.float32 and t.is_contiguous()
                        and t.dim() == 2 and t.shape[1] == DESC_DIM and t.device.index == self.device):
                    raise InvalidArgument(DSIFT_EINVAL, "ratio_match: device descriptors must be contiguous "
                                          f"float32 [n, {DESC_DIM}] tensors on cuda:{self.device}")
            pa, na, da = desc_a.data_ptr(), desc_a.shape[0], desc_a.shape[1]
            pb, nb, db = desc_b.data_ptr(), desc_b.shape[0], desc_b.shape[1]
            flags = INPUT_DEVICE
            stream = torch.cuda.current_stream(self.device).cuda_stream
        else:
            a = np.ascontiguousarray(desc_a, np.float32)
            b = np.ascontiguousarray(desc_b, np.float32)
            self._pin_match = (a, b)
            pa, na, da = a.ctypes.data, a.shape[0], a.shape[1] if a.ndim == 2 else DESC_DIM
            pb, nb, db = b.ctypes.data, b.shape[0], b.shape[1] if b.ndim == 2 else DESC_DIM
        cap = max(1, min(na, nb))
        out = np.zeros(cap, MATCH_DTYPE)
        n, put_a, put_b = C.c_int64(), C.c_int64(), C.c_int64()
        if stream is not None:   # run on the producer's stream, then restore the context's own
            self.set_stream(stream)
        try:
            _check(self.lib, self.lib.dsift_ratio_match(self.ctx, C.c_void_p(pa), na, C.c_void_p(pb), nb, da, db,
                                                        C.c_float(ratio), flags, out.ctypes.data, cap, C.byref(n),
                                                        C.byref(put_a), C.byref(put_b)))
        finally:
            if stream is not None:
                self.set_stream(self._stream)
        return out[:n.value], put_a.value, put_b.value

    def magsac_lite(self, matches, iterations: int, tau: float, seed: int):
        """detsift::magsac_lite (geom.cpp:181-320) on the device.  matches: [n, 4]
        float64 (x1, y1, x2, y2) = detsift::Correspondence.  Returns a
        MagsacResult (success, h [3, 3], inlier_mask uint8 [n], score,
        best_iteration), bit-identical to the reference."""
        m = np.ascontiguousarray(matches, np.float64).reshape(-1, 4)
        res = _MagsacResult()
        mask = np.zeros(len(m), np.uint8)
        _check(self.lib, self.lib.dsift_magsac_lite(self.ctx, m.ctypes.data, len(m), int(iterations),
                                                    C.c_double(tau), C.c_uint64(seed), C.byref(res),
                                                    mask.ctypes.data))
        return MagsacResult(bool(res.success), np.array(res.h, np.float64).reshape(3, 3),
                            mask if res.success else np.zeros(0, np.uint8), float(res.score),
                            int(res.best_iteration))

    def dlt_homography(self, matches, weights=None) -> np.ndarray:
        """detsift::dlt_homography (geom.cpp:108-161) on the device: [3, 3]."""
        m = np.ascontiguousarray(matches, np.float64).reshape(-1, 4)
        w = None if weights is None else np.ascontiguousarray(weights, np.float64)
        if w is not None and len(w) != len(m):
            raise InvalidArgument(DSIFT_EINVAL, "dlt: weight count mismatch")
        out = np.zeros(9, np.float64)
        _check(self.lib, self.lib.dsift_dlt_homography(self.ctx, m.ctypes.data, len(m),
                                                       None if w is None else w.ctypes.data, out.ctypes.data))
        return out.reshape(3, 3)

    def extract(self, img) -> FeatureSet:
        """detsift::extract (io.cpp:111-142) for one image."""
        self.submit(_f32(img))
        return self.results()[0]

    def extract_batch(self, imgs) -> list[FeatureSet]:
        self.submit(imgs)
        return self.results()

    def sha256(self, image: int = 0) -> str:
        buf = C.create_string_buffer(65)
        _check(self.lib, self.lib.dsift_result_sha256(self.ctx, image, buf))
        return buf.value.decode()

    def set_profiling(self, on: bool = True) -> None:
        _check(self.lib, self.lib.dsift_set_profiling(self.ctx, int(on)))

    def stage_times(self) -> dict:
        ms = (C.c_float * 5)()
        _check(self.lib, self.lib.dsift_stage_times(self.ctx, ms))
        return dict(zip(("pyramid", "detect", "orient", "sort", "describe"), [float(v) for v in ms]))

    def set_force_exact(self, on: bool = True) -> None:
        """Route every descriptor through the exact scan-order kernel (test hook)."""
        _check(self.lib, self.lib.dsift_set_option(self.ctx, 1, int(on)))

    def set_capacity_scale(self, permille: int) -> None:
        """Scale of the automatic work-list capacities in 1/1000 (DSIFT_OPT_CAPACITY_SCALE)."""
        _check(self.lib, self.lib.dsift_set_option(self.ctx, 2, int(permille)))

    def set_texture_gathers(self, on: bool = True) -> None:
        """Descriptor bilinear footprints by texture gathers (default) or plain
        loads (DSIFT_OPT_TEXTURE_GATHERS); the results are identical."""
        _check(self.lib, self.lib.dsift_set_option(self.ctx, 3, int(on)))

    def replays(self) -> int:
        """Times the last result was replayed after an automatic capacity overflow."""
        return int(self.lib.dsift_stat(self.ctx, 2))

    def lattice_points(self) -> tuple[int, int]:
        """(all, in-range) descriptor lattice points of the last result, counted
        on the device (DSIFT_STAT_LATTICE_POINTS / _IN_RANGE)."""
        return int(self.lib.dsift_stat(self.ctx, 3)), int(self.lib.dsift_stat(self.ctx, 4))

    def exact_fallbacks(self) -> int:
        """Keypoints of the last result whose fast-path certificate failed."""
        return int(self.lib.dsift_stat(self.ctx, 1))

    def export_torch(self, which: int = 1):
        """Zero-copy DLPack export of the last result as a torch CUDA tensor
        (0 keypoints [n, 7] float32 view, 1 descriptors [n, 128] float32,
        2 descriptors [n, 128] uint8)."""
        import torch

        ptr = C.c_void_p()
        _check(self.lib, self.lib.dsift_export_dlpack(self.ctx, which, C.byref(ptr)))
        pyapi = C.pythonapi
        pyapi.PyCapsule_New.restype = C.py_object
        pyapi.PyCapsule_New.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]
        cap = pyapi.PyCapsule_New(ptr, b"dltensor", None)
        return torch.utils.dlpack.from_dlpack(cap)

    def kernel_launches(self) -> int:
        return int(self.lib.dsift_kernel_launches(self.ctx))

    def synth_value_noise(self, dev_ptr: int, n: int, w: int, h: int, seed0: int, octaves: int = 5,
                          cells: int = 8) -> None:
        _check(self.lib, self.lib.dsift_synth_value_noise(self.ctx, C.c_void_p(dev_ptr), n, w, h,
                                                          C.c_uint64(seed0), octaves, cells))

    # ---- stage level (scalespace.hpp / detect.hpp / orient.hpp / describe.hpp) ----
    def build_scale_space(self, img) -> dict:
        a = _f32(img)
        _check(self.lib, self.lib.dsift_build_scale_space(self.ctx, a.ctypes.data, a.shape[1], a.shape[0],
                                                          INPUT_HOST))
        return self.scale_space_info()

    def load_scale_space(self, gauss, dog, upsampled: bool = False) -> dict:
        n_oct = len(gauss)
        dims = np.array([v for o in range(n_oct) for v in (gauss[o][0].shape[1], gauss[o][0].shape[0])], np.int32)
        g = [np.ascontiguousarray(x, np.float32) for o in range(n_oct) for x in gauss[o]]
        d = [np.ascontiguousarray(x, np.float32) for o in range(n_oct) for x in dog[o]]
        gp = (C.c_void_p * len(g))(*[x.ctypes.data for x in g])
        dp = (C.c_void_p * len(d))(*[x.ctypes.data for x in d])
        _check(self.lib, self.lib.dsift_load_scale_space(self.ctx, n_oct, int(upsampled), dims.ctypes.data, gp, dp))
        return self.scale_space_info()

    def scale_space_info(self) -> dict:
        n, up = C.c_int32(), C.c_int32()
        dims = np.zeros(128, np.int32)
        _check(self.lib, self.lib.dsift_scale_space_info(self.ctx, C.byref(n), C.byref(up), dims.ctypes.data))
        return {"n_oct": n.value, "upsampled": bool(up.value),
                "dims": [(int(dims[2 * o]), int(dims[2 * o + 1])) for o in range(n.value)]}

    def level(self, octave: int, kind: str, level: int) -> np.ndarray:
        info = self.scale_space_info()
        w, h = info["dims"][octave]
        out = np.empty((h, w), np.float32)
        _check(self.lib, self.lib.dsift_scale_space_level(self.ctx, octave, 0 if kind == "gauss" else 1, level,
                                                          out.ctypes.data))
        return out

    def find_extrema(self) -> np.ndarray:
        n = C.c_int64()
        _check(self.lib, self.lib.dsift_find_extrema(self.ctx, None, 0, C.byref(n)))
        out = np.zeros((max(1, n.value), 5), np.int32)
        _check(self.lib, self.lib.dsift_find_extrema(self.ctx, out.ctypes.data, n.value, C.byref(n)))
        return out[:n.value]

    def detect(self) -> np.ndarray:
        n = C.c_int64()
        _check(self.lib, self.lib.dsift_detect(self.ctx, None, 0, C.byref(n)))
        out = np.zeros(max(1, n.value), KEYPOINT_DTYPE)
        _check(self.lib, self.lib.dsift_detect(self.ctx, out.ctypes.data, n.value, C.byref(n)))
        return out[:n.value]

    def orientation_histograms(self, kps) -> np.ndarray:
        k = np.ascontiguousarray(kps, KEYPOINT_DTYPE)
        out = np.zeros((len(k), self.cfg.orientation_bins), np.float32)
        _check(self.lib, self.lib.dsift_orientation_histograms(self.ctx, k.ctypes.data, len(k), out.ctypes.data))
        return out

    def assign_orientations(self, kps) -> np.ndarray:
        k = np.ascontiguousarray(kps, KEYPOINT_DTYPE)
        cap = max(1, len(k) * self.cfg.orientation_bins)
        out = np.zeros(cap, KEYPOINT_DTYPE)
        n = C.c_int64()
        _check(self.lib, self.lib.dsift_assign_orientations(self.ctx, k.ctypes.data, len(k), out.ctypes.data, cap,
                                                            C.byref(n)))
        return out[:n.value]

    def raw_descriptors(self, kps, scale_factor: float) -> np.ndarray:
        k = np.ascontiguousarray(kps, KEYPOINT_DTYPE)
        out = np.zeros((len(k), DESC_DIM), np.float32)
        _check(self.lib, self.lib.dsift_raw_descriptors(self.ctx, k.ctypes.data, len(k), scale_factor,
                                                        out.ctypes.data))
        return out

    def dsp_descriptors(self, kps, with_u8: bool = False):
        k = np.ascontiguousarray(kps, KEYPOINT_DTYPE)
        out = np.zeros((len(k), DESC_DIM), np.float32)
        u8 = np.zeros((len(k), DESC_DIM), np.uint8)
        _check(self.lib, self.lib.dsift_dsp_descriptors(self.ctx, k.ctypes.data, len(k), out.ctypes.data,
                                                        u8.ctypes.data))
        return (out, u8) if with_u8 else out


def load_image(path: str) -> np.ndarray:
    """The 8-bit payload of a binary PNM, parsed like detsift::load_image
    (io.cpp:49-81; same errors, raised as ImageIOError): [h, w] for P5,
    [h, w, 3] for P6.  Convert with Extractor.ingest_u8 / extract_u8."""
    lib = load_library()
    w, h, ch = C.c_int32(), C.c_int32(), C.c_int32()
    _check(lib, lib.dsift_load_image(os.fsencode(path), C.byref(w), C.byref(h), C.byref(ch), None, 0))
    out = np.empty((h.value, w.value, ch.value) if ch.value == 3 else (h.value, w.value), np.uint8)
    _check(lib, lib.dsift_load_image(os.fsencode(path), C.byref(w), C.byref(h), C.byref(ch),
                                     out.ctypes.data, out.size))
    return out


class _Image(C.Structure):
    _fields_ = [("data", C.c_void_p), ("width", C.c_int32), ("height", C.c_int32)]


class Result:
    """A dsift_result handle: one more batch in flight on the same context
    (select it, submit, select another, submit, select back, read)."""

    def __init__(self, ex: "Extractor"):
        self.ex = ex
        self.batch = 0
        h = C.c_void_p()
        _check(ex.lib, ex.lib.dsift_result_create(ex.ctx, C.byref(h)))
        self.handle = h

    def close(self) -> None:
        if self.handle:
            if self.ex._selected is self:
                self.ex.select(None)
            self.ex.lib.dsift_result_destroy(self.handle)
            self.handle = None


class _MagsacResult(C.Structure):
    _fields_ = [("success", C.c_int32), ("best_iteration", C.c_int32), ("score", C.c_double),
                ("h", C.c_double * 9)]


class MagsacResult(NamedTuple):
    """detsift::MagsacResult (geom.hpp:55-61)."""
    success: bool
    h: np.ndarray
    inlier_mask: np.ndarray
    score: float
    best_iteration: int


def corner_error(h_est, h_gt, width: float, height: float) -> float:
    """detsift::corner_error (geom.cpp:322-333): mean corner displacement."""
    lib = load_library()
    a = np.ascontiguousarray(h_est, np.float64).reshape(9)
    b = np.ascontiguousarray(h_gt, np.float64).reshape(9)
    out = C.c_double()
    _check(lib, lib.dsift_corner_error(a.ctypes.data, b.ctypes.data, float(width), float(height), C.byref(out)))
    return out.value


_TLS = threading.local()


def default_device() -> int:
    """The device the drop-in extract() runs on: $DSIFT_DEVICE, else 0."""
    return int(os.environ.get("DSIFT_DEVICE", "0"))


def extract(img, cfg: SiftConfig | None = None, workers: int = 1) -> FeatureSet:
    """FeatureSet detsift::extract(const GrayImage&, const SiftConfig&, int workers)
    (io.hpp:17-19) on a B200.  `workers` keeps the reference's meaning — host
    threads, 0 = all — and, as in the reference, never changes the output; the
    device parallelism is the GPU's.  The device is default_device().  Each
    host thread reuses one cached context per (device, config)."""
    cfg = cfg or SiftConfig()
    dev = default_device()
    key = (dev, repr(cfg))
    cached = getattr(_TLS, "ex", None)
    if cached is None or cached[0] != key:
        if cached is not None:
            cached[1].close()
        _TLS.ex = (key, Extractor(cfg, dev))
    return _TLS.ex[1].extract(img)


def quantize_u8(desc: np.ndarray) -> np.ndarray:
    """The uint8 export q(v) = min(255, lround(v * 255.0)) applied on the host."""
    v = np.asarray(desc, np.float64) * 255.0
    q = np.floor(np.abs(v) + 0.5) * np.sign(v)
    return np.clip(q, 0, 255).astype(np.uint8)
