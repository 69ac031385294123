"""verify-determinism on the B200 path (reference: tools/detsift.cpp:170-200,
acceptance criterion 1, acceptance.cpp:72-101).

The reference extracts one image `runs` times for every worker count and exits
0 iff all DSF1 SHA-256 digests (detsum.cpp:129-132) are identical, 3 otherwise.
On the GPU the free variables are the run index and the batch composition: an
image is extracted alone, inside batches of several sizes (its neighbours
change the grid, the tile tickets and the compaction offsets).  Every digest
must be the same (tests/test_gpu_parity.py::test_verify_determinism also
checks it against the reference's own digest).

    python -m paper_2605_17869_b200.verify IMAGE.pgm [--runs 10] [--batches 1,2,4,8]
    python -m paper_2605_17869_b200.verify --synthetic 640x480 --seed 0x5EED0000
    python -m paper_2605_17869_b200.verify --sweep 10000    # C5: 10k mixed images, twice
    python -m paper_2605_17869_b200.verify --sweep 10000 --record c5.txt   # resumable record
    python -m paper_2605_17869_b200.verify --sweep 10000 --check c5.txt    # a later run against it

Prints one line per extraction (run, batch, digest) and a summary; exit code 0
(one digest) or 3 (several), like the reference.
"""
from __future__ import annotations

import argparse
import sys

import numpy as np

from . import Extractor, SiftConfig, load_image


def digests_for(img: np.ndarray, runs: int, batches: list[int], cfg: SiftConfig | None = None,
                device: int = 0, fillers: np.ndarray | None = None) -> dict[str, list[tuple[int, int]]]:
    """{digest: [(run, batch size), ...]} for `img` extracted `runs` times at
    every batch size (the image sits at a rotating position among fillers)."""
    out: dict[str, list[tuple[int, int]]] = {}
    with Extractor(cfg, device) as ex:
        for run in range(runs):
            for b in batches:
                if b == 1:
                    batch = img[None]
                    pos = 0
                else:
                    pos = run % b
                    fill = fillers if fillers is not None else np.stack([np.roll(img, k + 1, axis=1) for k in range(b)])
                    batch = np.array(fill[:b], np.float32, copy=True)
                    batch[pos] = img
                ex.submit(batch)
                ex.sync()
                d = ex.sha256(pos)
                out.setdefault(d, []).append((run, b))
    return out


C5_SIZES = [(640, 480), (800, 600), (1000, 750), (1024, 768), (1280, 720), (1600, 1200), (1920, 1080),
            (2048, 1536), (2560, 1440), (3840, 2160)]


def c5_sweep_sizes(n: int, seed: int = 0xC5) -> list[tuple[int, int]]:
    """resolutions of n images drawn by SplitMix64(seed) from
    the ten 480p-4K sizes."""
    s = seed & 0xFFFFFFFFFFFFFFFF
    out = []
    for _ in range(n):
        s = (s + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = ((s ^ (s >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        out.append(C5_SIZES[(z ^ (z >> 31)) % len(C5_SIZES)])
    return out


def sweep_digests(n: int, batch: int, device: int = 0, cfg: SiftConfig | None = None,
                  seed0: int = 0x5EED0000, skip: set | None = None, sink=None) -> list[str]:
    """DSF1 SHA-256 of each of the n C5 sweep images (image i: value noise of its
    drawn size, seed seed0 + i, generated on the device), extracted in same-size
    batches of up to `batch` images.  `skip`: indices already done (a resumed
    sweep; their entries stay ""); `sink(i, size, digest)` sees each result as
    soon as it exists."""
    import torch
    sizes = c5_sweep_sizes(n)
    out = [""] * n
    skip = skip or set()
    with Extractor(cfg, device) as ex:
        for size in sorted(set(sizes)):
            w, h = size
            idx = [i for i, s in enumerate(sizes) if s == size and i not in skip]
            for k in range(0, len(idx), batch):
                part = idx[k:k + batch]
                buf = torch.empty((len(part), h, w), dtype=torch.float32, device=f"cuda:{device}")
                for j, i in enumerate(part):   # per-image seeds, as the host generator
                    ex.synth_value_noise(buf[j].data_ptr(), 1, w, h, seed0 + i, 5, max(8, w // 20))
                torch.cuda.synchronize(device)
                ex.submit(None, n=len(part), w=w, h=h, device_ptr=buf.data_ptr())
                ex.sync()
                for j, i in enumerate(part):
                    out[i] = ex.sha256(j)
                    if sink:
                        sink(i, size, out[i])
    return out


def read_digests(path: str) -> dict[int, str]:
    """index -> digest from a sweep record ("index WxH sha256" per line)."""
    got = {}
    try:
        with open(path) as f:
            for line in f:
                parts = line.split()
                if len(parts) == 3:
                    got[int(parts[0])] = parts[2]
    except FileNotFoundError:
        pass
    return got


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("image", nargs="?", help="binary PNM (P5/P6)")
    ap.add_argument("--synthetic", help="WxH value-noise image instead of a file (synth.cpp:44-66)")
    ap.add_argument("--seed", type=lambda s: int(s, 0), default=0x5EED0000)
    ap.add_argument("--runs", type=int, default=10)
    ap.add_argument("--batches", default="1,2,4,8")
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--library", help="another build of libdsift (the test-only negative control)")
    ap.add_argument("--sweep", type=int, default=0,
                    help="C5: N mixed-resolution images, extracted twice (batches of 32, then 7); "
                         "every image's digest must repeat")
    ap.add_argument("--record", help="--sweep: append each image's digest to this file (resumes: images "
                                     "already recorded are skipped)")
    ap.add_argument("--check", help="--sweep: compare each image's digest with this record; exit 3 on a difference")
    args = ap.parse_args(argv)
    if args.sweep and (args.record or args.check):
        sizes = c5_sweep_sizes(args.sweep)
        if args.record:
            done = read_digests(args.record)
            with open(args.record, "a") as f:
                def sink(i, size, d):
                    f.write(f"{i} {size[0]}x{size[1]} {d}\n")
                    f.flush()
                sweep_digests(args.sweep, 32, args.device, skip=set(done), sink=sink)
            total = len(read_digests(args.record))
            print(f"recorded: {total} of {args.sweep} images in {args.record}")
            return 0
        ref = read_digests(args.check)
        bad = []

        def cmp(i, size, d):
            if ref.get(i) != d:
                bad.append(i)
        sweep_digests(args.sweep, 7, args.device, sink=cmp)
        print(f"sweep check: {args.sweep} images against {args.check}: {args.sweep - len(bad)} identical, "
              f"{len(bad)} differ")
        for i in bad[:10]:
            print(f"image {i} {sizes[i]}: recorded {ref.get(i)}")
        return 0 if not bad else 3
    if args.sweep:
        first = sweep_digests(args.sweep, 32, args.device)
        second = sweep_digests(args.sweep, 7, args.device)
        bad = [i for i in range(args.sweep) if first[i] != second[i]]
        sizes = c5_sweep_sizes(args.sweep)
        print(f"sweep: {args.sweep} images over {len(set(sizes))} sizes, 2 runs (batches 32 / 7): "
              f"{args.sweep - len(bad)} identical digests, {len(bad)} differ")
        for i in bad[:10]:
            print(f"image {i} {sizes[i]}: {first[i]} != {second[i]}")
        return 0 if not bad else 3
    if args.library:
        from . import load_library
        load_library(args.library)
    if args.synthetic:
        w, h = (int(v) for v in args.synthetic.lower().split("x"))
        import torch
        ex = Extractor(device=args.device)
        dev = torch.empty((1, h, w), dtype=torch.float32, device=f"cuda:{args.device}")
        ex.synth_value_noise(dev.data_ptr(), 1, w, h, args.seed, 5, max(8, w // 20))
        torch.cuda.synchronize()
        img = dev[0].cpu().numpy()
        ex.close()
    elif args.image:
        pix = load_image(args.image)
        with Extractor(device=args.device) as ex:
            img = ex.ingest_u8(pix)
    else:
        ap.error("an image path or --synthetic WxH is required")
    batches = [int(b) for b in args.batches.split(",") if b]
    table = digests_for(img, args.runs, batches, device=args.device)
    total = 0
    for d, occ in table.items():
        for run, b in occ:
            print(f"run={run} batch={b} sha256={d}")
            total += 1
    ok = len(table) == 1
    if len(table) == 1:
        print(f"1 unique digest over {total} runs")
    else:
        print(f"{len(table)} distinct digests over {total} runs")
    return 0 if ok else 3


if __name__ == "__main__":
    sys.exit(main())
