"""Small calls that reach every kernel nrng.cu launches: the ncu launch list of the dispatch
paths (tools/round_snapshot.sh; profiles/<tag>_dispatch_launches.txt).  (compute-sanitizer, which
it was first written for, is closed on this GPU pool: tools/racecheck_cases.py runs the same paths
on the library's own race-detector build.)

    python tools/dispatch_cases.py

Shapes (DESIGN.md §6 dispatch): >= 16 x 148 streams with > 128 pairs per stream: the
one-block-per-SM pw_kernel<M,16> / b3_kernel<16>; fewer streams: pw_kernel<M,4> / b3_kernel<4>
/ polar_kernel<4,2>; misaligned outputs: bm_kernel / polar_kernel (20-warp blocks at >= 20 x 148
streams); 12-128 pairs: mid_kernel; < 12: tiny_kernel; the sequential mode's epoch kernels;
the test hooks and the validation reductions.  Outputs are checked for finiteness only (the
parity tests check values).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1004_3105_b200 as P  # noqa: E402

METHODS = ("B1", "B2", "B3", "P", "P2", "R", "R1")


def run(g, m, n, misaligned=False):
    buf = torch.empty(n + 1, dtype=torch.float64, device="cuda")
    out = buf[1:] if misaligned else buf[:n]
    g.normal(m, out=out, mu=0.5, sigma=2.0)
    torch.cuda.synchronize()
    assert torch.isfinite(out).all(), (m, n, misaligned)


def main():
    wide = 2400 if len(sys.argv) < 2 else int(sys.argv[1])
    for m in METHODS:
        per = 1 if m in ("R", "R1") else 2
        g = P.Generator(7, wide)
        run(g, m, per * wide * 130 + 1)                 # 16-warp one-block-per-SM kernels
        g = P.Generator(7, 3000)
        run(g, m, per * 3000 * 140 + 3, misaligned=True)  # bm_kernel<V,20> / polar_kernel<20,M>
        g = P.Generator(8, 600)
        run(g, m, per * 600 * 140 + 1)                  # 4-warp-block kernels
        run(g, m, per * 600 * 140, misaligned=True)     # bm_kernel<V,4> / polar_kernel<4,M>
        g = P.Generator(9, 512)
        run(g, m, per * 512 * 40 + 1)                   # mid_kernel
        g = P.Generator(9, 64)
        run(g, m, per * 64 * 3 + 1)                     # tiny_kernel
    for m in ("B1", "B2", "B3", "P", "P2"):             # sequential mode, whole epochs (EP kernels)
        g = P.Generator(3, 3000)
        x = g.normal_seq(m, 3 * 2 * 3000 * 128 + 5)  # 3 whole epochs in one launch: the EP kernels
        torch.cuda.synchronize()
        assert torch.isfinite(x).all()
    g = P.Generator(4, 600)
    u = g.uniform(600 * 100 + 7)
    mask = g.polar_mask(100)
    h = np.empty(2 * 600 * 140 + 3)
    P.Generator(5, 600).normal("B1", out=h)             # host output through the staging buffers
    uu = torch.rand(3 * 4096, dtype=torch.float64, device="cuda")
    for method in range(1, 8):
        P.transform_from_uniforms(uu, method, 0.5, 2.0)
    x = torch.randn(1 << 20, dtype=torch.float64, device="cuda")
    P.stats(x, 0.0, [-1.0, 0.0, 1.0])
    P.gof_hist(x, 0.0, 1.0, 16)
    P.serial_corr(x, 0.0, 100)
    torch.cuda.synchronize()
    assert torch.isfinite(u).all() and mask.numel() == 60000 and np.isfinite(h).all()
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
