"""The C ABI from a plain C program (examples/c_api_demo.c): B3 and Polar into host memory through
the library's own staging, per-stream partition invariance of two half calls bit for bit, sample
moments, and an argument error -- no Python or torch on the path."""
import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu

from test_abi import c_demo_cmd  # noqa: E402


def test_c_api_demo_runs(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    from paper_1004_3105_b200 import build

    lib = build.build()
    exe = str(tmp_path / "c_api_demo")
    res = subprocess.run(c_demo_cmd(exe, lib), capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    run = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert run.returncode == 0, run.stdout + run.stderr
    out = run.stdout
    assert "B3: n=16777216" in out and "P: n=16777216" in out
    assert out.count("partition-invariant=yes moments=ok") == 2
    assert "sigma<0 -> invalid argument" in out and out.strip().endswith("ok")
