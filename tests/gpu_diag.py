"""Stage-by-stage GPU-vs-oracle diagnostic (prints mismatch counts, never
fails).  Run on a GPU box:  python tests/gpu_diag.py [size ...]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_17869_b200 as ds  # noqa: E402
from oracle.oracle import Oracle, make_config  # noqa: E402


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def main():
    sizes = [(96, 64, 3, 6), (160, 120, 7, 8), (320, 240, 11, 16), (640, 480, 0x5EED0000, 32)]
    ref = Oracle("reference") if os.path.exists(os.path.join("oracle", "_ref", "libdetsift_ref.so")) else Oracle("port")
    port = Oracle("port")
    ex = ds.Extractor()
    for (w, h, seed, cells) in sizes:
        img = port.value_noise(w, h, seed, 5, cells)
        print(f"=== {w}x{h} cells={cells} ===", flush=True)
        # pyramid
        info = ex.build_scale_space(img)
        ss = port.scale_space(img)
        bad = 0
        tot = 0
        for o in range(ss.n_oct):
            for i in range(ss.s + 3):
                a, b = ex.level(o, "gauss", i), ss.level(o, "gauss", i)
                d = int((bits(a) != bits(b)).sum())
                bad += d
                tot += a.size
                if d and bad == d:
                    idx = np.argwhere(bits(a) != bits(b))[0]
                    print("  first gauss diff", o, i, idx, a[tuple(idx)], b[tuple(idx)])
            for i in range(ss.s + 2):
                a, b = ex.level(o, "dog", i), ss.level(o, "dog", i)
                bad += int((bits(a) != bits(b)).sum())
                tot += a.size
        print(f"  pyramid: octaves gpu={info['n_oct']} oracle={ss.n_oct} up={info['upsampled']} "
              f"mismatched px {bad}/{tot}", flush=True)
        # extrema
        eg = ex.find_extrema()
        eo = port.find_extrema(ss)
        print(f"  extrema: gpu={len(eg)} oracle={len(eo)} equal={np.array_equal(eg, eo)}", flush=True)
        kg = ex.detect()
        ko = port.detect(ss)
        same = len(kg) == len(ko) and kg.tobytes() == ko.tobytes()
        print(f"  detect: gpu={len(kg)} oracle={len(ko)} bitwise={same}", flush=True)
        if not same and len(kg) == len(ko):
            for f in ko.dtype.names:
                print("    field", f, int((kg[f] != ko[f]).sum()))
        if len(ko):
            hg = ex.orientation_histograms(ko)
            ho = np.stack([port.orientation_histogram(ss, k) for k in ko])
            print(f"  ori hist: mismatched bins {int((bits(hg) != bits(ho)).sum())}/{ho.size}", flush=True)
            og = ex.assign_orientations(ko)
            oo = np.concatenate([port.assign_orientations(ss, k) for k in ko])
            print(f"  assign: gpu={len(og)} oracle={len(oo)} bitwise={og.tobytes() == oo.tobytes()}", flush=True)
            sub = oo[: min(len(oo), 200)]
            for f in (1.0, 0.5, 2.0):
                rg = ex.raw_descriptors(sub, f)
                ro = np.stack([port.raw_descriptor(ss, k, f) for k in sub])
                print(f"  raw desc f={f}: mismatched {int((bits(rg) != bits(ro)).sum())}/{ro.size} "
                      f"maxabs {float(np.abs(rg - ro).max()):.3g}", flush=True)
            dg = ex.dsp_descriptors(sub)
            do = np.stack([port.dsp_descriptor(ss, k) for k in sub])
            print(f"  dsp desc: mismatched {int((bits(dg) != bits(do)).sum())}/{do.size}", flush=True)
        # full extract
        t0 = time.time()
        fs = ex.extract(img)
        t1 = time.time()
        kr, dr = ref.extract(img)
        t2 = time.time()
        print(f"  extract: gpu n={len(fs)} ({t1 - t0:.3f}s) {ref.kind} n={len(kr)} ({t2 - t1:.2f}s) "
              f"kps bitwise={fs.keypoints.tobytes() == kr.tobytes()} "
              f"desc bitwise={fs.descriptors.tobytes() == dr.tobytes()} "
              f"sha gpu={ex.sha256(0)[:16]} ref={ref.hash_features(kr, dr)[:16]}", flush=True)
        print(f"    exact fallbacks: {ex.exact_fallbacks()}", flush=True)
        ex.set_force_exact(True)
        fs2 = ex.extract(img)
        ex.set_force_exact(False)
        print(f"    forced-exact path identical: {fs2.descriptors.tobytes() == fs.descriptors.tobytes()} "
              f"(fallbacks {ex.exact_fallbacks()})", flush=True)
        if len(fs) == len(kr) and len(kr):
            q = ds.quantize_u8(dr)
            print(f"    u8 mismatch {int((fs.descriptors_u8 != q).sum())} desc float mism "
                  f"{int((bits(fs.descriptors) != bits(dr)).sum())}", flush=True)
    # batch + determinism
    imgs = np.stack([port.value_noise(320, 240, 100 + i, 5, 16) for i in range(4)])
    a = ex.extract_batch(imgs)
    h1 = [ex.sha256(i) for i in range(4)]
    b = ex.extract_batch(imgs)
    h2 = [ex.sha256(i) for i in range(4)]
    singles = []
    for i in range(4):
        ex.extract(imgs[i])
        singles.append(ex.sha256(0))
    print("batch run-to-run identical:", h1 == h2, " batch==single:", h1 == singles, [len(x) for x in a])


if __name__ == "__main__":
    main()
