"""The intra-warp race detector (debug build, csrc/nrng_racecheck.cuh) over the hot kernels:
no unsynchronised cross-lane access to any shared window or scratch word -- and the detector's
negative control (one __syncwarp removed from B3's tail gather) is caught.

compute-sanitizer racecheck/synccheck is closed on this GPU pool; this is the substitute
(DESIGN.md §6).  The debug builds are compiled here (about a minute each)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(name, defines):
    from paper_1004_3105_b200 import build as B

    out = os.path.join(ROOT, "ab_libs", name)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    deps = B.DEPS + [os.path.join(ROOT, "paper_1004_3105_b200", "csrc", "nrng_racecheck.cuh")]
    if not (os.path.exists(out) and all(os.path.getmtime(out) >= os.path.getmtime(d) for d in deps)):
        B.build(force=True, out=out, defines=defines)
    return out


def _run(lib):
    env = dict(os.environ, NRNG_LIB_OVERRIDE=lib)
    return subprocess.run([sys.executable, os.path.join(ROOT, "tools", "racecheck_cases.py"), "--quick"],
                          capture_output=True, text=True, env=env, timeout=1200)


def test_no_intra_warp_races():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = _run(_build("rc.so", ["NRNG_RACECHECK=1"]))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "races 0" in r.stdout.splitlines()[-1]


def test_detector_catches_a_missing_syncwarp():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = _run(_build("rc_selftest.so", ["NRNG_RACECHECK=1", "NRNG_RACECHECK_SELFTEST=1"]))
    assert r.returncode == 1, r.stdout + r.stderr
    assert "RAW" in r.stdout
