"""Run every dispatch path of nrng.cu on the race-detector debug build (NRNG_RACECHECK=1,
csrc/nrng_racecheck.cuh) and report, per case, the shared-memory accesses checked and the
intra-warp races found (unsynchronised cross-lane RAW / WAW / WAR on a window or scratch word).

    python -m paper_1004_3105_b200.build --out ab_libs/rc.so -DNRNG_RACECHECK=1
    NRNG_LIB_OVERRIDE=ab_libs/rc.so python tools/racecheck_cases.py

Exit status 1 if any race was found.  (compute-sanitizer --tool racecheck/synccheck is closed
on this GPU pool; this is the substitute.)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1004_3105_b200 as P  # noqa: E402

KIND = {1: "RAW", 2: "WAW", 3: "WAR"}
total_races, total_checks, rows = 0, 0, []


def report(name):
    global total_races, total_checks
    races, first, checks = P.nrng_racecheck_result()
    total_races += races
    total_checks += checks
    desc = ""
    if races:
        desc = " first: line %d %s thread %d vs thread %d" % (first >> 32, KIND.get((first >> 24) & 0xff, "?"),
                                                               (first >> 12) & 0xfff, first & 0xfff)
    rows.append("%-44s checks %12d  races %d%s" % (name, checks, races, desc))
    print(rows[-1], flush=True)


def run(g, m, n, misaligned=False):
    buf = torch.empty(n + 1, dtype=torch.float64, device="cuda")
    out = buf[1:] if misaligned else buf[:n]
    g.normal(m, out=out, mu=0.5, sigma=2.0)
    torch.cuda.synchronize()


def main():
    quick = "--quick" in sys.argv  # one shape per kernel family (the pytest leg)
    P.nrng_racecheck_result()  # clear (and fail early on a product build)
    if quick:
        for m in ("B1", "B3", "P", "P2", "R1"):
            per = 1 if m in ("R", "R1") else 2
            g = P.Generator(7, 2400)
            run(g, m, per * 2400 * 140 + 1)
            report("%s S=2400 x 140 (one block per SM kernels)" % m)
            g = P.Generator(8, 600)
            run(g, m, per * 600 * 140 + 1)
            run(g, m, per * 600 * 140, misaligned=True)
            report("%s S=600 x 140, aligned + misaligned" % m)
        print("TOTAL checks %d races %d" % (total_checks, total_races))
        return 1 if total_races else 0
    for m in ("B1", "B2", "B3", "P", "P2", "R", "R1"):
        per = 1 if m in ("R", "R1") else 2
        g = P.Generator(7, 2400)
        report("create (init_kernel) S=2400")
        run(g, m, per * 2400 * 300 + 1)
        report("%s S=2400 x 300 (one block per SM kernels)" % m)
        g = P.Generator(7, 3000)
        run(g, m, per * 3000 * 140 + 3, misaligned=True)
        report("%s S=3000 misaligned (bm/polar 20-warp)" % m)
        g = P.Generator(8, 600)
        run(g, m, per * 600 * 300 + 1)
        report("%s S=600 x 300 (4-warp blocks)" % m)
        run(g, m, per * 600 * 140, misaligned=True)
        report("%s S=600 misaligned (bm/polar 4-warp)" % m)
        g = P.Generator(9, 512)
        run(g, m, per * 512 * 40 + 1)
        report("%s S=512 x 40 (mid_kernel)" % m)
    for m in ("B1", "B2", "B3", "P", "P2"):
        g = P.Generator(3, 3000)
        g.normal_seq(m, 3 * 2 * 3000 * 128 + 5)
        torch.cuda.synchronize()
        report("%s sequential mode, 3 epochs (EP kernels)" % m)
    g = P.Generator(4, 600)
    g.uniform(600 * 1000 + 7)
    report("uniform (uniform_kernel)")
    g.polar_mask(700)
    report("polar_mask (polar_mask_kernel)")
    print("TOTAL checks %d races %d" % (total_checks, total_races))
    return 1 if total_races else 0


if __name__ == "__main__":
    sys.exit(main())
