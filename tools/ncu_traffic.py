"""Builds profiles/ncu_traffic.json (bench.py's roofline.traffic) from the ncu
per-launch CSV of one 32-image C3 extraction (profiles/capture_r02b.sh step 3):
DRAM bytes read + written by every K1 (blur), K2 (extrema) and K3 (refine)
launch, per image, beside SURVEY 8(d)'s algorithmic bytes.
usage: python tools/ncu_traffic.py profiles/r02/r02_k123_b32.csv [batch]"""
import csv
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    path = sys.argv[1]
    batch = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    lines = open(path).read().split("\n")
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    idc, kn, mn, mv = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    launches = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        if len(r) <= mv:
            continue
        launches[r[idc]][r[mn]] = float(r[mv].replace(",", ""))
        names[r[idc]] = r[kn].split("(")[0].split("<")[0].replace("void ", "").strip()
    # one extraction = the first launch of blur_level2 (or the first blur) up to the first refine
    ids = sorted(launches, key=int)
    first_refine = next(i for i in ids if names[i] == "refine_kernel")
    ids = [i for i in ids if int(i) <= int(first_refine)]
    per_kernel = collections.Counter()
    dfma = 0.0
    for i in ids:
        m = launches[i]
        per_kernel[names[i]] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        if "blur" in names[i]:
            dfma += m.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0.0)
    import bench
    total = sum(per_kernel.values())
    out = {
        "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over every K1 (blur), K2 "
                  f"(detect_count, detect_emit) and K3 (refine) launch of one {batch}-image C3 extraction "
                  f"({os.path.relpath(path)}, the benched batch); made by tools/ncu_traffic.py",
        "pyramid_detect_bytes_per_image": total / batch,
        "algorithmic_bytes_per_image": sum(bench.stage_bytes(1600, 1200)[:2]),
        "blur_dfma_per_image_executed": dfma / batch,
        "per_kernel_mb_per_image": {k: v / batch / 1e6 for k, v in sorted(per_kernel.items())},
        "note": "the level blurs write G and DoG (8 B/px) and read the previous level once; the first "
                "octave's bridge reads the input image; small octaves stay in the 126 MB L2 between launches",
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
