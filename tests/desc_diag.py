"""Descriptor-kernel diagnostic (GPU box): fallback counts per kernel and, in
'trust' mode (certificate ignored), the raw fast-path sums vs the oracle.
python tests/desc_diag.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_17869_b200 as ds  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402


def main():
    port = Oracle("port")
    for (w, h, seed, cells) in [(160, 120, 7, 8), (640, 480, 0x5EED0000, 32)]:
        img = port.value_noise(w, h, seed, 5, cells)
        k_ref, d_ref = port.extract(img)
        with ds.Extractor() as ex:
            for kern in (1, 2):
                ex.set_desc_kernel(kern)
                fs = ex.extract(img)
                same = np.array_equal(fs.descriptors.view(np.uint32), d_ref.view(np.uint32))
                print(f"{w}x{h} kernel {kern}: n={len(fs)} fallbacks={ex.exact_fallbacks()} bitexact={same}",
                      flush=True)
            ex.set_desc_kernel(2)
            ex.lib.dsift_set_option(ex.ctx, 1, -1)     # trust mode
            fs = ex.extract(img)
            d = fs.descriptors
            diff = np.abs(d.astype(np.float64) - d_ref.astype(np.float64))
            nbad = int((d.view(np.uint32) != d_ref.view(np.uint32)).sum())
            print(f"   trust: mismatching floats {nbad}/{d.size}, max abs diff {diff.max():.3g}, "
                  f"nan {int(np.isnan(d).sum())}", flush=True)
            if nbad:
                i = int(np.argwhere((d.view(np.uint32) != d_ref.view(np.uint32)).any(1))[0][0])
                print("   first bad kp", i, fs.keypoints[i], "\n   gpu", d[i][:16], "\n   ref", d_ref[i][:16])
            ex.lib.dsift_set_option(ex.ctx, 1, 0)




def dump():
    port = Oracle("port")
    img = port.value_noise(160, 120, 7, 5, 8)
    np.set_printoptions(linewidth=200, precision=6)
    with ds.Extractor() as ex:
        ex.set_desc_kernel(2)
        ex.lib.dsift_set_option(ex.ctx, 1, -2)
        fs = ex.extract(img)
        d = fs.descriptors
        for fi in range(5):
            acc, lsb, kc, ok = d[fi * 4], d[fi * 4 + 1], d[fi * 4 + 2], d[fi * 4 + 3]
            bad = np.where(ok == 0)[0]
            print(f"scale {fi}: failing bins {len(bad)} kchain/npass {kc[0]}", flush=True)
            for b in bad[:6]:
                print("   bin", b, "acc", repr(float(acc[b])), "lsb", lsb[b])


if __name__ == "__main__":
    dump() if "dump" in sys.argv else main()
