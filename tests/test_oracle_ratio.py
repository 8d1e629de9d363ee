"""Pins for the oracle's Algorithm R, the ratio method (Algorithm R at
P:421-427): x = sqrt(8/e)(v - 1/2)/(1 - u), reject outside the curve C, return sigma x + mu,
one normal per accepted candidate, exact stop per stream (readings R24-R27).

What pins it, independently of its own code: the geometry of C (the region in which v/u is
normal: inside [0,1] x [-sqrt(2/e), +sqrt(2/e)]), the paper's consumption figures
(8/sqrt(pi e) ~ 2.74 uniforms and 1.37 logarithms per normal), and normality of
the output.  The printed step 3 ("-x^2 ln(1-u) > 4") is tested to be an erratum.
"""
import math

import mpmath as mp
import numpy as np
from scipy import stats as sps

import oracle as O


def test_constant_is_rn_sqrt_8_over_e():
    # u = 0, v = 3/4: x = RN(C8E / 4) = C8E / 4 exactly (a power-of-two scaling)
    with mp.workdps(40):
        c = float(mp.sqrt(8 / mp.e))
    acc, x, a, b = O.ratio_candidate(0.0, 0.5 + 0.25)
    assert x == c * 0.25  # v - 1/2 = 1/4 exactly, 1 - u = 1: a power-of-two scaling of RN(sqrt(8/e))


def test_curve_c_closed_form_boundary():
    # 1 - u = 1/e (u = 1 - 1/e): -4 ln(1-u) = 4, so C is |x| <= 2; x = sqrt(8/e) e (v - 1/2)
    u = 1.0 - math.exp(-1.0)
    scale = math.sqrt(8 / math.e) * math.e  # |x| = scale |v - 1/2|
    for xtarget, expect in [(0.0, True), (1.9, True), (1.999, True), (2.001, False), (2.5, False), (-1.9, True),
                            (-2.001, False)]:
        v = 0.5 + xtarget / scale
        acc, x, a, b = O.ratio_candidate(u, v)
        assert abs(x - xtarget) < 1e-12 and abs(b - 4.0) < 1e-14
        assert acc == expect, (xtarget, x, a, b)


def test_curve_c_bounds_the_rectangle():
    # C lies inside |x| (1-u) <= sqrt(2/e): x = sqrt(8/e)(v-1/2)/(1-u), |v-1/2| <= 1/2;
    # the widest point is x = +-sqrt2 at 1-u = e^{-1/2}: accepted; v at the rectangle edge
    w = math.exp(-0.5)
    for v, expect in [(0.0, True), (1 - 2**-53, True)]:
        acc, x, a, b = O.ratio_candidate(1 - w, v)
        assert abs(abs(x) - math.sqrt(2)) < 1e-12 and acc == expect
    # u = 0 (1 - u = 1): C is the single point x = 0
    assert O.ratio_candidate(0.0, 0.5)[0] and not O.ratio_candidate(0.0, 0.5 + 2**-20)[0]


def test_acceptance_and_consumption_match_paper():
    st = O.Streams(17, 64)
    n = 1 << 20
    x = st.normal_ratio(n)
    cand = st.counts.sum() / 2
    p = math.sqrt(math.pi * math.e) / 4  # area(C) / area(rectangle) = 0.7306
    se = math.sqrt(p * (1 - p) / cand)
    assert abs(n / cand - p) < 4 * se
    # 8/sqrt(pi e) ~ 2.74 uniforms and ~1.37 logarithms (= candidates) per normal
    assert abs(st.counts.sum() / n - 8 / math.sqrt(math.pi * math.e)) < 0.01
    assert abs(cand / n - 1.37) < 0.01
    assert np.isfinite(x).all()


def test_output_is_normal_and_moments():
    st = O.Streams(5, 32)
    n = 1 << 20
    x = st.normal_ratio(n, 2.5, 0.5)
    z = (x - 2.5) / 0.5
    assert sps.kstest(z, "norm").pvalue > 0.001
    assert abs(z.mean()) < 4 / math.sqrt(n) and abs(z.var() - 1) < 4 * math.sqrt(2 / n)
    assert abs(sps.skew(z)) < 4 * math.sqrt(6 / n) and abs(sps.kurtosis(z)) < 4 * math.sqrt(24 / n)


def test_printed_step3_is_an_erratum():
    # The test as printed, reject iff -x^2 ln(1-u) > 4, on the same uniforms: wrong acceptance
    # rate and a non-normal output -- so the oracle reads step 3 as x^2 > -4 ln(1-u) (R25).
    rng = np.random.default_rng(1)
    u = rng.integers(0, 2**53, 1 << 20) * 2.0**-53
    v = rng.integers(0, 2**53, 1 << 20) * 2.0**-53
    x = math.sqrt(8 / math.e) * (v - 0.5) / (1 - u)
    lg = -np.log1p(-u)
    printed = x * x * lg <= 4
    km = x * x <= 4 * lg
    p = math.sqrt(math.pi * math.e) / 4
    assert abs(km.mean() - p) < 0.003 and abs(printed.mean() - p) > 0.02
    assert sps.kstest(x[km], "norm").pvalue > 0.001 and sps.kstest(x[printed], "norm").pvalue < 1e-6


def test_stream_major_exact_stop_and_partition():
    # stream k's outputs are its accepted candidates in order, then it stops: the S-stream
    # call equals S one-stream calls on the same global streams, concatenated
    S, q = 8, 1000
    full = O.Streams(9, S).normal_ratio(S * q + 3)  # 3 remainder normals on streams 0..2
    parts = [O.Streams(9, 1, first_stream=k).normal_ratio(q + (1 if k < 3 else 0)) for k in range(S)]
    assert np.array_equal(full, np.concatenate(parts))
    # and the first normal of stream 0 is sigma x + mu of its first accepted (u, v) pair
    st = O.Streams(9, 1)
    w = st.uniform(40)
    for j in range(20):
        acc, x, a, b = O.ratio_candidate(w[2 * j], w[2 * j + 1])
        if acc:
            assert full[0] == x  # sigma = 1, mu = 0: fma(1, x, 0) = x
            break
