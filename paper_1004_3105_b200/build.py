"""Build libnrng.so in-tree with nvcc for sm_100a (the only target).

    python -m paper_1004_3105_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = os.path.join(PKG, "csrc", "nrng.cu")
DEPS = [SRC, os.path.join(PKG, "csrc", "nrng_kernels.cuh"), os.path.join(PKG, "csrc", "nrng_device.cuh"),
        os.path.join(PKG, "csrc", "nrng_coeffs.cuh"), os.path.join(PKG, "csrc", "nrng_racecheck.cuh"),
        os.path.join(ROOT, "include", "nrng.h")]
LIB = os.path.join(PKG, "libnrng.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false",          # no implicit contraction: every fma in the path is written out
    "-Xptxas", "-v",
    "-shared", "-Xcompiler", "-fPIC",
]


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    lib = out or LIB
    if not force and os.path.exists(lib) and all(os.path.getmtime(lib) >= os.path.getmtime(d) for d in DEPS):
        return lib
    tmp = lib + ".tmp%d" % os.getpid()
    cmd = [NVCC, *FLAGS, *["-D" + d for d in defines], "-o", tmp, SRC]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libnrng.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # python -m paper_1004_3105_b200.build [--force] [--out PATH] [-DNAME=VALUE ...]  (variants for A/B runs)
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else None
    defs = [a[2:] for a in args if a.startswith("-D")]
    print(build(force="--force" in args or out is not None, verbose=True, out=out, defines=defs))
