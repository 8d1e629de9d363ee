"""CPU oracle for the hot path of Brent (1993) -- ctypes shim over ``liboracle.so``.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_1004_3105_b200``) never imports it and
shares no code with it.  See ``oracle/nrng_oracle.c`` for what is computed and
the PAPER.md passages each function follows.

Parity status: every function here is pinned by ``-m "not gpu"``
tests in ``tests/test_oracle_*.py`` except the B1-vs-glibc ulp behaviour of
log/sin/cos, which is covered only by tolerance.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "nrng_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")
CFLAGS = ["-std=gnu11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC"]

R = 607  # long lag
N0 = 607 * 11  # absolute index of uniform #0 (10 warm-up rounds discarded)


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C11 + OpenMP)."""
    deps = [SRC, os.path.join(HERE, "oracle_coeffs.h")]
    if not force and os.path.exists(LIB) and all(os.path.getmtime(LIB) >= os.path.getmtime(d) for d in deps):
        return LIB
    tmp = LIB + ".tmp%d" % os.getpid()
    subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, SRC, "-lm"])
    os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        u64, u32, dbl, p = C.c_uint64, C.c_uint32, C.c_double, C.c_void_p
        sig = {
            "orc_sizeof_stream": ([], C.c_int),
            "orc_set_threads": ([C.c_int], None),
            "orc_max_threads": ([], C.c_int),
            "orc_splitmix64": ([u64, u64, u64, p], None),
            "orc_stream_init": ([p, u64, u64], None),
            "orc_streams_init": ([p, u64, u64, u32], None),
            "orc_word_to_uniform": ([u64], dbl),
            "orc_words": ([p, u32, p, u64], None),
            "orc_uniform": ([p, u32, p, u64], None),
            "orc_sincos16": ([dbl, p, p], None),
            "orc_eval_h": ([dbl], dbl),
            "orc_mobius": ([dbl], dbl),
            "orc_b1_pair": ([dbl, dbl, dbl, dbl, p], None),
            "orc_b2_pair": ([dbl, dbl, dbl, dbl, p], None),
            "orc_b3_pair": ([dbl, dbl, dbl, dbl, dbl, p], None),
            "orc_polar_pair": ([dbl, dbl, dbl, dbl, p, p], C.c_int),
            "orc_normal_boxmuller": ([p, u32, p, u64, dbl, dbl, C.c_int], C.c_int),
            "orc_normal_polar": ([p, u32, p, u64, dbl, dbl], C.c_int),
            "orc_normal_polar2": ([p, u32, p, u64, dbl, dbl], C.c_int),
            "orc_polar2_pair": ([dbl, dbl, dbl, dbl, p, p], C.c_int),
            "orc_polar_mask": ([p, u32, p, u64], None),
            "orc_ratio_candidate": ([dbl, dbl, p], C.c_int),
            "orc_normal_ratio": ([p, u32, p, u64, dbl, dbl, p], C.c_int),
            "orc_ratio1_pretest": ([dbl, dbl, p], C.c_int),
            "orc_normal_ratio1": ([p, u32, p, u64, dbl, dbl, p, p], C.c_int),
            "orc_transform_from_uniforms": ([p, u64, p, p, dbl, dbl, C.c_int], C.c_int),
            "orc_stats": ([p, u64, dbl, p, C.c_int, p, p], None),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


STREAM_DTYPE = np.dtype([("ring", np.uint64, (R,)), ("count", np.uint64)])


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def max_threads() -> int:
    return int(lib().orc_max_threads())


def splitmix64(seed: int, first: int, n: int) -> np.ndarray:
    out = np.empty(n, np.uint64)
    lib().orc_splitmix64(seed, first, n, _ptr(out))
    return out


def word_to_uniform(x: int) -> float:
    return lib().orc_word_to_uniform(int(x))


class Streams:
    """A set of S consecutive global LFG streams [first, first+S) (the oracle's generator)."""

    def __init__(self, seed: int, n_streams: int, first_stream: int = 0):
        assert lib().orc_sizeof_stream() == STREAM_DTYPE.itemsize
        self.seed, self.first, self.S = int(seed), int(first_stream), int(n_streams)
        self.st = np.zeros(self.S, STREAM_DTYPE)
        lib().orc_streams_init(_ptr(self.st), self.seed, self.first, self.S)

    # -- state access (for bit-exact state parity and checkpoint tests)
    @property
    def counts(self) -> np.ndarray:
        return self.st["count"].copy()

    @property
    def rings(self) -> np.ndarray:
        return self.st["ring"].copy()

    def words(self, n: int) -> np.ndarray:
        out = np.empty(n, np.uint64)
        lib().orc_words(_ptr(self.st), self.S, _ptr(out), n)
        return out

    def uniform(self, n: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        lib().orc_uniform(_ptr(self.st), self.S, _ptr(out), n)
        return out

    def normal_boxmuller(self, n: int, mu: float = 0.0, sigma: float = 1.0, variant: int = 1) -> np.ndarray:
        out = np.empty(n, np.float64)
        rc = lib().orc_normal_boxmuller(_ptr(self.st), self.S, _ptr(out), n, mu, sigma, variant)
        if rc != 0:
            raise ValueError("bad variant %r" % variant)
        return out

    def normal_polar(self, n: int, mu: float = 0.0, sigma: float = 1.0) -> np.ndarray:
        out = np.empty(n, np.float64)
        lib().orc_normal_polar(_ptr(self.st), self.S, _ptr(out), n, mu, sigma)
        return out

    def normal_polar2(self, n: int, mu: float = 0.0, sigma: float = 1.0) -> np.ndarray:
        out = np.empty(n, np.float64)
        lib().orc_normal_polar2(_ptr(self.st), self.S, _ptr(out), n, mu, sigma)
        return out

    def normal_ratio(self, n: int, mu: float = 0.0, sigma: float = 1.0) -> np.ndarray:
        """Algorithm R: n normals, one per accepted candidate, stream-major with
        exact stop; self.ratio_margin = min |a - b|/b over all candidates drawn (reading R27)."""
        out = np.empty(n, np.float64)
        mg = np.empty(1, np.float64)
        lib().orc_normal_ratio(_ptr(self.st), self.S, _ptr(out), n, mu, sigma, _ptr(mg))
        self.ratio_margin = float(mg[0])
        return out

    def normal_ratio1(self, n: int, mu: float = 0.0, sigma: float = 1.0) -> np.ndarray:
        """Algorithm R1 (R with step 2.5, reading R29): the same output as
        normal_ratio; self.ratio1_logs / self.ratio1_cands = logarithms evaluated / candidates."""
        out = np.empty(n, np.float64)
        nl, nc = np.zeros(1, np.uint64), np.zeros(1, np.uint64)
        lib().orc_normal_ratio1(_ptr(self.st), self.S, _ptr(out), n, mu, sigma, _ptr(nl), _ptr(nc))
        self.ratio1_logs, self.ratio1_cands = int(nl[0]), int(nc[0])
        return out

    def polar_mask(self, cand_per_stream: int) -> np.ndarray:
        m = np.empty(self.S * cand_per_stream, np.uint8)
        lib().orc_polar_mask(_ptr(self.st), self.S, _ptr(m), cand_per_stream)
        return m


def sincos16(v: float) -> tuple[float, float]:
    s, c = C.c_double(), C.c_double()
    lib().orc_sincos16(v, C.byref(s), C.byref(c))
    return s.value, c.value


def eval_h(v: float) -> float:
    return lib().orc_eval_h(v)


def mobius(u: float) -> float:
    return lib().orc_mobius(u)


def b1_pair(u, v, mu=0.0, sigma=1.0):
    xy = np.empty(2)
    lib().orc_b1_pair(u, v, mu, sigma, _ptr(xy))
    return float(xy[0]), float(xy[1])


def b2_pair(u, v, mu=0.0, sigma=1.0):
    xy = np.empty(2)
    lib().orc_b2_pair(u, v, mu, sigma, _ptr(xy))
    return float(xy[0]), float(xy[1])


def b3_pair(u1, u2, u3, mu=0.0, sigma=1.0):
    xy = np.empty(2)
    lib().orc_b3_pair(u1, u2, u3, mu, sigma, _ptr(xy))
    return float(xy[0]), float(xy[1])


def polar_pair(a, b, mu=0.0, sigma=1.0):
    """Returns (accepted, (x_out, y_out) or None, (x, y, s))."""
    xy, xys = np.empty(2), np.empty(3)
    acc = lib().orc_polar_pair(a, b, mu, sigma, _ptr(xy), _ptr(xys))
    return bool(acc), ((float(xy[0]), float(xy[1])) if acc else None), tuple(float(t) for t in xys)


def polar2_pair(a, b, mu=0.0, sigma=1.0):
    """Method P2 on one candidate: (accepted, (x_out, y_out) or None, (x, y, s))."""
    xy, xys = np.empty(2), np.empty(3)
    acc = lib().orc_polar2_pair(a, b, mu, sigma, _ptr(xy), _ptr(xys))
    return bool(acc), ((float(xy[0]), float(xy[1])) if acc else None), tuple(float(t) for t in xys)


def ratio_candidate(u, v):
    """Algorithm R steps 2-3 on one (u, v): (accepted, x, a = x^2, b = -4 ln(1-u)); reject iff a > b."""
    xab = np.empty(3)
    acc = lib().orc_ratio_candidate(u, v, _ptr(xab))
    return bool(acc), float(xab[0]), float(xab[1]), float(xab[2])


def ratio1_pretest(u, v):
    """Algorithm R1 step 2.5 on one (u, v): (class, x, a = x^2); class 1 = P1 (accept without
    a logarithm), 2 = P2 (reject), 0 = borderline (step 3 decides)."""
    xa = np.empty(2)
    cls = lib().orc_ratio1_pretest(u, v, _ptr(xa))
    return int(cls), float(xa[0]), float(xa[1])


def transform_from_uniforms(u: np.ndarray, method: int, mu=0.0, sigma=1.0):
    """method 1/2/3 = B1/B2/B3, 4 = Polar, 5 = P2, 6 = R (out[2j] = sigma x + mu or NaN,
    out[2j+1] = x), 7 = R1 (as 6; mask = accept | class << 1).  Returns (out[2*pairs], mask or None)."""
    u = np.ascontiguousarray(u, np.float64)
    per = 3 if method == 3 else 2
    npairs = u.size // per
    out = np.empty(2 * npairs)
    mask = np.empty(npairs, np.uint8) if method >= 4 else None
    rc = lib().orc_transform_from_uniforms(_ptr(u), npairs, _ptr(out), _ptr(mask) if mask is not None else None,
                                           mu, sigma, method)
    if rc != 0:
        raise ValueError("bad method")
    return out, mask


def stats(x: np.ndarray, center: float, edges: np.ndarray):
    """(sum d, sum d^2, sum d^3, sum d^4, min, max), histogram over `edges` (K-1 interior edges)."""
    x = np.ascontiguousarray(x, np.float64)
    edges = np.ascontiguousarray(edges, np.float64)
    K = edges.size + 1
    sums = np.empty(6)
    hist = np.empty(K, np.int64)
    lib().orc_stats(_ptr(x), x.size, center, _ptr(edges), K, _ptr(sums), _ptr(hist))
    return sums, hist
