"""The C-ABI library builds, loads and exports every symbol include/nrng.h declares (no GPU needed)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nrng.h")


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(nrng_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def libnrng():
    from paper_1004_3105_b200 import build

    path = build.build()
    return C.CDLL(path), path


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for f in ("nrng_create", "nrng_normal_boxmuller", "nrng_normal_polar", "nrng_destroy"):
        assert f in names


def test_every_declared_symbol_is_exported(libnrng):
    L, path = libnrng
    for name in declared_functions():
        assert hasattr(L, name), name
    nm = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (nrng_[a-z0-9_]+)", nm))
    assert set(declared_functions()) <= exported


def test_binding_mirrors_header():
    import paper_1004_3105_b200 as P

    assert set(P.SIGNATURES) == set(declared_functions())
    for name in declared_functions():
        assert callable(getattr(P, name)), name


def test_library_is_sm100a_only(libnrng):
    _, path = libnrng
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_error_paths_without_compute(libnrng):
    L, _ = libnrng
    L.nrng_error_string.restype = C.c_char_p
    assert L.nrng_error_string(-1) == b"invalid argument"
    L.nrng_create.restype = C.c_void_p
    L.nrng_create.argtypes = [C.c_uint64, C.c_uint32, C.c_int]
    # invalid arguments are rejected before any device work
    assert L.nrng_create(1, 0, 1) is None and L.nrng_last_error() == -1
    assert L.nrng_create(1, 16, 7) is None and L.nrng_last_error() == -1
    L.nrng_normal_polar.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_double, C.c_double]
    assert L.nrng_normal_polar(None, None, 10, 0.0, 1.0) == -1
    L.nrng_destroy.argtypes = [C.c_void_p]
    L.nrng_destroy(None)  # NULL-safe


def test_no_cpu_fallback_in_product_package():
    # the product package never imports the oracle
    pkg = os.path.join(ROOT, "paper_1004_3105_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "liboracle" not in src, f


def test_output_buffer_checks():
    # the binding refuses buffers the library would overrun: wrong dtype,
    # non-contiguous views, read-only arrays; it accepts float64 host arrays / CPU tensors
    import numpy as np
    import torch

    import paper_1004_3105_b200 as P

    a = np.empty(10)
    assert P.out_buffer(a) == (a.ctypes.data, 10)
    t = torch.empty(7, dtype=torch.float64)
    assert P.out_buffer(t) == (t.data_ptr(), 7)
    with pytest.raises(TypeError):
        P.out_buffer(np.empty(10, np.float32))
    with pytest.raises(TypeError):
        P.out_buffer(torch.empty(10, dtype=torch.float32))
    with pytest.raises(ValueError):
        P.out_buffer(np.empty(20)[::2])
    with pytest.raises(ValueError):
        P.out_buffer(torch.empty(20, dtype=torch.float64)[::2])
    ro = np.empty(4)
    ro.flags.writeable = False
    with pytest.raises(ValueError):
        P.out_buffer(ro)
    with pytest.raises(TypeError):
        P.out_buffer([0.0] * 4)


def c_demo_cmd(out_path, lib_path):
    lib_dir = os.path.dirname(lib_path)
    return ["gcc", "-std=c11", "-O2", "-Wall", "-Wextra", "-Werror", "-I" + os.path.join(ROOT, "include"),
            os.path.join(ROOT, "examples", "c_api_demo.c"), "-L" + lib_dir, "-lnrng", "-Wl,-rpath," + lib_dir,
            "-lm", "-o", out_path]


def test_c_example_builds_against_the_header(libnrng, tmp_path):
    # the header is plain C11 and the library links from a C program (no Python, no CUDA headers);
    # tests/test_gpu_c_api.py runs the program on a GPU
    import shutil

    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    _, path = libnrng
    exe = str(tmp_path / "c_api_demo")
    res = subprocess.run(c_demo_cmd(exe, path), capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    assert os.path.exists(exe)
