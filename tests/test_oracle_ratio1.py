"""Pins for the oracle's Algorithm R1 (Algorithm R with step 2.5, the
pretests P1/P2 before the logarithm; reading R29).

What pins it, independently of its own code: the geometry the paper states (R1's accept
region lies inside the curve C, R2's reject region outside it, and the borderline region
R2 minus R1 is small: "R1 and R2 have almost the same area"), checked against the
plain step-3 test on brute-force grids and around the two tangency points of the bounds;
R1 returning exactly Algorithm R's output (step 2.5 only skips logarithms); and the
fraction of logarithms evaluated against the area of the borderline region, integrated
numerically from the closed-form boundaries.
"""
import math

import numpy as np
from scipy import integrate

import oracle as O

C8E = math.sqrt(8 / math.e)


def _region_classes(u, v):
    return np.array([O.ratio1_pretest(a, b)[0] for a, b in zip(u, v)])


def _step3_accepts(u, v):
    return np.array([O.ratio_candidate(a, b)[0] for a, b in zip(u, v)])


def test_pretests_never_contradict_step3_random():
    rng = np.random.default_rng(3)
    u = rng.integers(0, 2**53, 200000) * 2.0**-53
    v = rng.integers(0, 2**53, 200000) * 2.0**-53
    cls = _region_classes(u, v)
    acc = _step3_accepts(u, v)
    assert np.all(acc[cls == 1]) and not np.any(acc[cls == 2])
    # the three classes all occur, in the proportions of their areas (below)
    assert 0.60 < (cls == 1).mean() < 0.72 and 0.12 < (cls == 2).mean() < 0.22


def test_pretests_at_the_tangency_points():
    # P1's line touches -4 ln U at U = e^{-1/4} (a = 1), P2's curve at U = e^{-1.35}
    # (a = 5.4): on a fine v-grid through both boundaries the pretests stay on their side
    for U0 in (math.exp(-0.25), math.exp(-1.35)):
        u = 1.0 - U0
        xb = math.sqrt(-4 * math.log(U0))  # |x| on C at this U
        rels = np.concatenate([np.linspace(-1e-6, 1e-6, 401), [-3e-14, -1e-14, 0.0, 1e-14, 3e-14]])
        for rel in rels:
            x = xb * (1 + rel)
            v = 0.5 + x * U0 / C8E
            cls, xx, a = O.ratio1_pretest(u, v)
            acc = O.ratio_candidate(u, v)[0]
            assert (cls != 1 or acc) and (cls != 2 or not acc)
            assert (cls != 1 or rel < 0) and (cls != 2 or rel > 0)  # each pretest stays on its side of C
            if abs(rel) <= 3e-14:
                assert cls == 0  # inside the 2^-40 margin only step 3 decides
    # well inside / outside C near U = 1 and at the rectangle's corners
    assert O.ratio1_pretest(0.0, 0.5)[0] == 0  # U = 1: P1's line is negative there
    assert O.ratio1_pretest(0.5, 0.5)[0] == 1
    assert O.ratio1_pretest(0.999, 0.0)[0] == 2


def test_r1_output_equals_r_and_counts_logs():
    S, n = 64, 64 * 3000 + 17
    a = O.Streams(23, S)
    b = O.Streams(23, S)
    xa = a.normal_ratio(n, 0.5, 2.0)
    xb = b.normal_ratio1(n, 0.5, 2.0)
    assert np.array_equal(xa, xb)
    assert np.array_equal(a.counts, b.counts) and np.array_equal(a.rings, b.rings)
    cands = b.ratio1_cands
    assert cands == b.counts.sum() // 2
    # logarithms: only the borderline candidates (area of R2 \\ R1 over the rectangle)
    border = _borderline_area()
    frac = b.ratio1_logs / cands
    assert abs(frac - border) < 4 * math.sqrt(border * (1 - border) / cands)
    # per normal: 8/sqrt(pi e) / 2 = 1.37 candidates, ~0.23 logarithms with step 2.5
    assert abs(b.ratio1_logs / n - 1.3688 * border) < 0.01


def _borderline_area():
    # probability that a candidate is borderline; in (U, x') with x' = x U / C8E = v - 1/2 in [-1/2, 1/2): P1 holds for
    # x^2 <= 5 - 4 e^{1/4} U, P2 for x^2 >= 4 e^{-1.35}/U + 1.4 (margins 2^-40 negligible)
    def half_width(x2max, U):
        return min(0.5, math.sqrt(max(x2max, 0.0)) * U / C8E)

    def f(U):
        return 2 * (half_width(4 * math.exp(-1.35) / U + 1.4, U) - half_width(5 - 4 * math.exp(0.25) * U, U))

    val, _ = integrate.quad(f, 0.0, 1.0, limit=200, points=[math.exp(-0.25), math.exp(-1.35)])
    return val  # the unit (u, v) square has area 1: this is the probability of a borderline candidate


def test_borderline_area_is_small():
    # "R1 and R2 have almost the same area": the borderline band is ~17% of
    # the candidates, against 100% of them needing a logarithm in Algorithm R
    border = _borderline_area()
    assert 0.15 < border < 0.19
