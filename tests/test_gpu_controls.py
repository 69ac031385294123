"""GPU: evidence that the determinism checks can fail and that the kernels are
race- and error-free.

* Negative control (reference acceptance criterion 2, acceptance.cpp:103-111,
  hook detsum.cpp:73-109): a test-only build of the same sources with
  DSIFT_NONDET_TEST_HOOK replaces the descriptor's fixed trees by float
  atomics in scheduling order when DSIFT_NONDET=1; verify-determinism must
  then exit 3, and exit 0 with the hook built in but not enabled.
* compute-sanitizer memcheck / racecheck / synccheck over a small batch that
  runs every extraction kernel (tests/native/sanitize_run.py)."""
import json
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NONDET = os.path.join(ROOT, "tests", "native", "libdsift_nondet.so")
BOUNDS = os.path.join(ROOT, "tests", "native", "libdsift_bounds.so")
PRODUCT = os.path.join(ROOT, "paper_2605_17869_b200", "libdsift.so")
SANITIZER = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"

pytestmark = pytest.mark.gpu


def _verify(env_extra, timeout=600):
    env = dict(os.environ)
    env.pop("DSIFT_NONDET", None)
    env.update(env_extra)
    cmd = [sys.executable, "-m", "paper_2605_17869_b200.verify", "--synthetic", "320x240", "--runs", "4",
           "--batches", "1,2,4,8", "--library", NONDET]
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


def test_negative_control_makes_verify_exit_3():
    if not os.path.exists(NONDET):
        pytest.fail("tests/native/libdsift_nondet.so missing (run __graft_entry__.build())")
    r = _verify({"DSIFT_NONDET": "1"})
    assert r.returncode == 3, (r.returncode, r.stdout[-2000:], r.stderr[-2000:])
    assert "distinct digests" in r.stdout


def test_hook_build_is_deterministic_when_disabled():
    r = _verify({})
    assert r.returncode == 0, (r.returncode, r.stdout[-2000:], r.stderr[-2000:])
    assert "1 unique digest" in r.stdout


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer_clean(tool):
    cmd = [SANITIZER, "--tool", tool, "--error-exitcode", "9", "--print-limit", "20"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    cmd += [sys.executable, os.path.join(ROOT, "tests", "native", "sanitize_run.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    if r.returncode != 0 and "closed on this pool" in out:
        # the GPU pool's wrapper refuses the tool (runs under it left GPUs needing a
        # reset); the clean runs of this same test are in
        # profiles/r02/pytest_gpu_final.log (earlier session, same test)
        pytest.skip("compute-sanitizer closed on this GPU pool: " + out.strip().splitlines()[0][:200])
    assert r.returncode == 0, out[-4000:]
    assert "sanitize workload ok" in out
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-2000:]


def test_gather_to_rank0_nccl_device_buffers():
    # shard.gather_to_rank0 on the exported device tensors through NCCL (one
    # rank on the one GPU: sizes all-gathered, rank-0 assembly on the device)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "native", "gather_nccl.py")], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    assert "nccl gather ok" in r.stdout


def _bounds_run(lib):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "native", "bounds_run.py"), lib], cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-4000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_bounds_build_clean():
    # the stand-in for compute-sanitizer memcheck (refused by this GPU pool): a
    # build of the same sources with device-side index checks (DSIFT_BOUND in
    # K1, K2, K4 and K5: ring / slot / table / staged-tile indices, the
    # unclamped interior sample footprints, full-tile stores) runs cases that
    # reach every indexed path; no condition may fail, and the digests must be
    # the product library's
    if not os.path.exists(BOUNDS):
        pytest.fail("tests/native/libdsift_bounds.so missing (run __graft_entry__.build())")
    chk = _bounds_run(BOUNDS)
    assert chk["selftest"] == [1, 999]   # a failing condition is counted (and then reset)
    assert set(chk["bounds"]) == {"pyramid", "detect", "orient", "describe"}, chk["bounds"]
    for unit, (count, site) in chk["bounds"].items():
        assert count == 0, f"{unit}: {count} failed index conditions, first at site {site}"
    prod = _bounds_run(PRODUCT)
    assert prod["bounds"] == {}
    assert chk["digests"] == prod["digests"]
