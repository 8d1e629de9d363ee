"""Seeded synthetic workloads shared by tests and bench (no method arithmetic here).

This module holds only *inputs*: the BASELINE.json configurations (seed, number
of LFG streams, n, mu, sigma) and a seeded generator of explicit uniform arrays
for the ``transform_from_uniforms`` parity cases.  It computes nothing the paper
defines; both the CUDA path and the oracle receive what it produces.

Input recipe: the paper measures on no dataset ("a large number
of random numbers were generated, so that vector lengths were long"),
so every workload is synthetic by construction: uniforms are 53-bit dyadic
rationals in [0, 1), exactly the values the paper's generator can return
("may return exactly 0 but never exactly 1").
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    methods: tuple[str, ...]
    n: int  # normals per call (per GPU for the sharded config)
    streams: int  # LFG streams (per GPU for the sharded config)
    seed: int
    mu: float = 0.0
    sigma: float = 1.0
    note: str = ""


# BASELINE.json "configs", in order.
C1 = Config("C1", ("B1",), 1 << 20, 1 << 10, 1, note="configs[0]: B1, n=2^20, 1024 streams, seed 1")
C2 = Config("C2", ("P",), 1 << 24, 1 << 14, 7, note="configs[1]: Polar, n=2^24, 2^14 streams, seed 7")
C3 = Config("C3", ("B2", "B3"), 1 << 28, 1 << 16, 42, 2.5, 0.5,
            note="configs[2]: B2/B3, n=2^28, 2^16 streams, seed 42, mu=2.5, sigma=0.5")
C4_LENGTHS = (1 << 6, 1 << 10, 1 << 14, 1 << 18, 1 << 22, 1 << 26)
C4 = Config("C4", ("B1", "P"), 1 << 26, 1 << 16, 3, note="configs[3]: call-length sweep, 10^3 calls per length")
# configs[4]: 2^34 normals over 2^19 streams split into disjoint ranges at 1/2/4/8 GPUs,
# "2^31 per GPU" -> the per-GPU shard is 2^31 normals over 2^16 streams (weak scaling:
# N ranks own global streams [r*2^16, (r+1)*2^16) and each makes 2^31 normals).
C5_SHARD = Config("C5", ("B1", "B2", "B3", "P"), 1 << 31, 1 << 16, 11,
                  note="configs[4] per-GPU shard: 2^31 normals, 2^16 streams/GPU, seed 11")
C5_TOTAL_STREAMS = 1 << 19

ALL = (C1, C2, C3, C4, C5_SHARD)


def dyadic_uniforms(seed: int, n: int) -> np.ndarray:
    """n uniforms k * 2^-53, k uniform in [0, 2^53), from numpy's PCG64 (seeded)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    k = rng.integers(0, 1 << 53, size=n, dtype=np.uint64)
    return k.astype(np.float64) * 2.0 ** -53


def edge_uniforms() -> np.ndarray:
    """Boundary uniforms the methods treat specially (0, the largest value < 1, 1/2, tau=8/9 neighbours)."""
    e = 2.0 ** -53
    tau = 8.0 / 9.0
    vals = [0.0, e, 2 * e, 0.5 - e, 0.5, 0.5 + e, 0.25, 0.75, 1.0 - e, 1.0 - 2 * e,
            np.sqrt(tau), np.nextafter(np.sqrt(tau), 0), np.nextafter(np.sqrt(tau), 1),
            np.float64(int((1 - np.exp(-2.0)) * 2 ** 53)) * e, 11 / 16, 3 / 4, 31 / 32]
    return np.array(vals, np.float64)
