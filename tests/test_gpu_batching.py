"""GPU: the drop-in boundary beyond one same-size batch — ragged batches
(dsift_extract_images, the reference's any-size extract, io.cpp:111-142),
result handles (two batches in flight on one context), the automatic
capacity replay, and the drop-in extract(img, cfg, workers) with a cached
per-thread context (io.hpp:17-19; workers never changes the output,
parallel.hpp:12-16)."""
import os

import numpy as np
import pytest

import paper_2605_17869_b200 as ds

pytestmark = pytest.mark.gpu

C5_SIZES = [(640, 480), (800, 600), (1000, 750), (1024, 768), (1280, 720), (1600, 1200), (1920, 1080),
            (2048, 1536), (2560, 1440), (3840, 2160)]


def splitmix64(seed):
    s = [seed & 0xFFFFFFFFFFFFFFFF]

    def nxt():
        M = 0xFFFFFFFFFFFFFFFF
        s[0] = (s[0] + 0x9E3779B97F4A7C15) & M
        z = s[0]
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)
    return nxt


def c5_sizes(n):
    """C5 resolutions drawn by SplitMix64(0xC5); every size present."""
    rng = splitmix64(0xC5)
    sizes = [C5_SIZES[rng() % len(C5_SIZES)] for _ in range(n - len(C5_SIZES))]
    return sizes + C5_SIZES   # guarantee all ten


def test_c5_ragged_batch_matches_single_images_and_reference(port, ref):
    sizes = c5_sizes(64)
    imgs = [port.value_noise(w, h, 0x5EED0000 + i, 5, max(8, w // 20)) for i, (w, h) in enumerate(sizes)]
    with ds.Extractor() as ex:
        res = ex.extract_images(imgs)
        shas = [ex.sha256(i) for i in range(len(imgs))]
        assert len(res) == len(imgs)
        ex.extract_images(imgs)   # run to run
        assert [ex.sha256(i) for i in range(len(imgs))] == shas
        singles = []
        for im in imgs:
            ex.extract(im)
            singles.append(ex.sha256(0))
    assert shas == singles
    # the reference on a sample (small, mid, 4K)
    for i in (0, 5, len(imgs) - 1):
        k, d = ref.extract(imgs[i], None, os.cpu_count() or 1)
        assert shas[i] == ref.hash_features(k, d), sizes[i]
        assert res[i].keypoints.tobytes() == np.ascontiguousarray(k).tobytes()


def test_result_handles_two_batches_in_flight(port):
    a = np.stack([port.value_noise(320, 240, 0x5EED0100 + i, 5, 16) for i in range(3)])
    b = [port.value_noise(200, 150, 0x5EED0200, 5, 10), port.value_noise(321, 199, 0x5EED0201, 5, 16)]
    with ds.Extractor() as ex:
        want_a = [f.descriptors.tobytes() for f in ex.extract_batch(a)]
        want_b = [f.descriptors.tobytes() for f in ex.extract_images(b)]
        r1, r2 = ex.new_result(), ex.new_result()
        ex.select(r1)
        ex.submit(a)
        ex.select(r2)
        ex.submit_images(b)        # batch 2 enqueued while batch 1 is unread
        ex.select(r1)
        got_a = [f.descriptors.tobytes() for f in ex.results()]
        ex.select(r2)
        got_b = [f.descriptors.tobytes() for f in ex.results()]
        ex.select(None)
        r1.close()
        r2.close()
    assert got_a == want_a and got_b == want_b


def test_automatic_capacity_replays_instead_of_failing(port):
    # automatic capacities started at 1% of their size: the first pass
    # overflows, the batch is replayed with x4 lists until it fits, and the
    # caller still receives every keypoint (the reference has no such limit)
    img = port.value_noise(320, 240, 0x5EED0009, 5, 16)
    k, d = port.extract(img)
    with ds.Extractor() as ex:
        ex.set_capacity_scale(10)
        fs = ex.extract(img)
        assert ex.replays() >= 1
        assert fs.keypoints.tobytes() == k.tobytes()
        assert ex.sha256(0) == port.hash_features(k, d)
        ex.set_capacity(8)   # a fixed capacity still fails loudly
        with pytest.raises(ds.DsiftError) as e:
            ex.extract(img)
        assert e.value.code == ds.DSIFT_ECAPACITY


def test_drop_in_extract_workers_and_cached_context(port):
    img = port.value_noise(160, 120, 0x5EED0007, 5, 8)
    k, d = port.extract(img)
    want = port.hash_features(k, d)
    f1 = ds.extract(img, ds.SiftConfig(), 8)
    ctx1 = ds._TLS.ex[1].ctx.value
    f2 = ds.extract(img, ds.SiftConfig(), 0)
    assert ds._TLS.ex[1].ctx.value == ctx1   # reused, not re-created
    assert f1.keypoints.tobytes() == f2.keypoints.tobytes() == k.tobytes()
    assert f1.descriptors.tobytes() == d.tobytes()
    with ds.Extractor() as ex:
        ex.extract(img)
        assert ex.sha256(0) == want


def test_failed_submit_leaves_no_stale_result(port):
    img = port.value_noise(160, 120, 0x5EED0008, 5, 8)
    with ds.Extractor() as ex:
        ex.extract(img)
        with pytest.raises(ds.InvalidArgument):
            ex.submit(np.zeros((3, 3), np.float32))
        with pytest.raises(ds.DsiftError) as e:
            ex.sync()
        assert e.value.code == ds.DSIFT_ESTATE


def test_c5_sweep_twice_identical_and_reference_sample(ref):
    # C5's determinism check at sweep scale: 256 mixed-resolution images
    # (SplitMix64(0xC5) over the ten sizes, device-generated value noise) run
    # twice with different batch compositions give identical per-image digests;
    # a sample equals the reference's
    from paper_2605_17869_b200.verify import c5_sweep_sizes, sweep_digests
    n = 256
    a = sweep_digests(n, 32)
    b = sweep_digests(n, 7)
    assert a == b
    sizes = c5_sweep_sizes(n)
    assert len(set(sizes)) == 10
    for i in (0, 1, 2):
        w, h = sizes[i]
        img = ref.value_noise(w, h, 0x5EED0000 + i, 5, max(8, w // 20))
        k, d = ref.extract(img, None, os.cpu_count() or 1)
        assert a[i] == ref.hash_features(k, d), sizes[i]


def test_c5_sweep_record_resume_and_check(tmp_path):
    # the resumable sweep: a record interrupted after part of the images is
    # completed by a second --record run, and --check of a fresh run against it
    # passes (exit 0); a corrupted record entry makes --check exit 3
    from paper_2605_17869_b200 import verify
    rec = str(tmp_path / "c5.txt")
    n = 40
    part = verify.sweep_digests(n, 32, skip=set(range(20, n)))   # "interrupted": images 0..19 only
    sizes = verify.c5_sweep_sizes(n)
    with open(rec, "w") as f:
        for i in range(20):
            f.write(f"{i} {sizes[i][0]}x{sizes[i][1]} {part[i]}\n")
    assert verify.main(["--sweep", str(n), "--record", rec]) == 0
    assert len(verify.read_digests(rec)) == n
    assert verify.main(["--sweep", str(n), "--check", rec]) == 0
    lines = open(rec).read().splitlines()
    i0, size0, _ = lines[0].split()
    lines[0] = f"{i0} {size0} {'0' * 64}"
    open(rec, "w").write("\n".join(lines) + "\n")
    assert verify.main(["--sweep", str(n), "--check", rec]) == 3


def test_concurrent_drop_in_calls_from_host_threads(port):
    # calls on distinct images may run concurrently: 6 host threads
    # each call the drop-in extract (one cached context per thread, ctypes drops
    # the GIL) on their own images; every result equals the single-threaded one
    from concurrent.futures import ThreadPoolExecutor
    imgs = [port.value_noise(320, 240, 0x5EED0100 + i, 5, 16) for i in range(12)]
    want = []
    with ds.Extractor() as ex:
        for im in imgs:
            ex.extract(im)
            want.append(ex.sha256(0))

    def one(i):
        fs = ds.extract(imgs[i])
        k, d = fs.keypoints, fs.descriptors
        return port.hash_features(k, d)

    with ThreadPoolExecutor(max_workers=6) as pool:
        got = list(pool.map(one, range(len(imgs))))
    assert got == want


def test_c5_sweep_sample_matches_committed_record():
    # the committed 10,000-image C5 record of the final round-2 kernels
    # (profiles/r02/c5_record_final.txt.gz, verify --sweep 10000 --record): a
    # 64-image sample spread over all ten sizes, extracted now in batches of 5,
    # must reproduce its digests (a later kernel change that alters any output
    # bit at any C5 size fails here)
    import gzip
    from paper_2605_17869_b200 import verify
    rec = {}
    with gzip.open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r02",
                                "c5_record_final.txt.gz"), "rt") as f:
        for line in f:
            i, _, d = line.split()
            rec[int(i)] = d
    assert len(rec) == 10000
    sizes = verify.c5_sweep_sizes(10000)
    sample = set()
    for size in sorted(set(sizes)):   # the first 6-7 images of every size
        sample |= set([i for i, s in enumerate(sizes) if s == size][:7])
    sample = set(sorted(sample)[:64])
    got = verify.sweep_digests(10000, 5, skip=set(range(10000)) - sample)
    assert {i: got[i] for i in sample} == {i: rec[i] for i in sample}
