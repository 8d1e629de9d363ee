"""Pins for the oracle's B2/B3 machinery: the Chebyshev fitter, sincos16, h(v), Moebius map.

Paper: P:159-170 (B2), P:218-263 (B3: g, tau = 8/9, v = (6u-4)/(4-3u), deg-15 h with
"absolute error less than 2e-11", "about 30 terms" without the map, Chebyshev truncation).
"""
import json
import math
import os

import mpmath as mp
import numpy as np
import pytest

import oracle as O
from oracle import fit_coeffs as F

HERE = os.path.dirname(os.path.abspath(__file__))
COEFFS = json.load(open(os.path.join(os.path.dirname(HERE), "oracle", "oracle_coeffs.json")))
H = [float.fromhex(x) for x in COEFFS["h"]]
SIN = [float.fromhex(x) for x in COEFFS["sin"]]
COS = [float.fromhex(x) for x in COEFFS["cos"]]


@pytest.mark.parametrize("k", range(0, 9))
def test_chebyshev_coeff_matches_jacobi_anger(k):
    # Closed form: sin(a cos t) = 2 sum_{k odd} (-1)^((k-1)/2) J_k(a) cos(k t),
    #              cos(a cos t) = J_0(a) + 2 sum_{k even>0} (-1)^(k/2) J_k(a) cos(k t).
    with mp.workdps(50):
        a = mp.pi / 16
        cs = F.chebyshev_series_coeff(lambda x: mp.sin(a * x), k)
        cc = F.chebyshev_series_coeff(lambda x: mp.cos(a * x), k)
        jk = mp.besselj(k, a)
        if k % 2:
            es, ec = 2 * (-1) ** ((k - 1) // 2) * jk, 0
        else:
            es, ec = 0, 2 * (-1) ** (k // 2) * jk
        assert abs(cs - es) < mp.mpf(10) ** -40
        assert abs(cc - ec) < mp.mpf(10) ** -40


def test_chebyshev_T_coefficients():
    t = F.chebyshev_T_integer_coeffs(5)
    assert t[2] == [-1, 0, 2] and t[3] == [0, -3, 0, 4] and t[5] == [0, 5, 0, -20, 0, 16]
    # T_k(cos t) = cos(k t)
    for k in range(6):
        x = 0.3
        assert abs(sum(c * x**j for j, c in enumerate(t[k])) - math.cos(k * math.acos(x))) < 1e-13


def test_low_degree_series_is_exact_for_polynomials():
    # truncating the Chebyshev series of a degree-3 polynomial at degree 3 returns it exactly
    f = lambda x: 1 + 2 * x - 3 * x**2 + 0.5 * x**3
    b = F.truncated_series_monomials(f, 3)
    assert [float(v) for v in b] == pytest.approx([1, 2, -3, 0.5], abs=1e-30)


def test_h_certified_error_below_paper_bound():
    # deg-15 h on [-1,1] with absolute error < 2e-11
    assert COEFFS["h_cert_err"] < 2e-11
    # re-certify the committed doubles on an independent (odd-count, shifted) grid
    worst = 0.0
    with mp.workdps(30):
        for i in range(1001):
            v = mp.mpf(-1) + mp.mpf(2) * (i + 0.37) / 1001.37
            worst = max(worst, float(abs(F.horner_mp(H, v) - F.h_exact(v))))
    assert worst < 2e-11


def test_degree_three_h_fails_the_bound():
    # SPEC fit example: a degree-3 truncation is far above 2e-11
    b = [F.round_to_double(x) for x in F.truncated_series_monomials(F.h_exact, 3)]
    err = max(abs(float(F.horner_mp(b, v)) - float(F.h_exact(v))) for v in np.linspace(-1, 1, 101))
    assert err > 1e-5


@pytest.mark.slow
def test_about_30_terms_without_the_map():
    # "About 30 terms would be needed if we attempted to approximate g(u) to
    # the same accuracy by a polynomial on [0, tau]".  Unmapped g on [0, 8/9] via x in [-1,1].
    tau = mp.mpf(8) / 9
    g_on_x = lambda x: F.g_exact(tau * (x + 1) / 2)
    errs = {}
    for deg in (15, 29):
        b = F.truncated_series_monomials(g_on_x, deg)
        errs[deg] = max(abs(F.horner_mp(b, mp.mpf(x)) - g_on_x(mp.mpf(x))) for x in np.linspace(-1, 1, 301))
    assert errs[15] > 1e-8          # deg 15 is nowhere near 2e-11 without the map
    assert errs[29] < 4e-11         # ~30 terms reach the same order as the mapped deg 15


@pytest.mark.parametrize("v,expect", [(-1.0, 1.0), (-0.4, math.sqrt(2 * math.log(2))),
                                      (1.0, math.sqrt(9 / 8 * math.log(9)))])
def test_h_special_values(v, expect):
    # h(-1) = g(0) = 1; v = -0.4 <-> u = 1/2; v = 1 <-> u = tau = 8/9
    assert abs(O.eval_h(v) - expect) < 2e-11


def test_mobius_endpoints():
    # P:251 v = (6u-4)/(4-3u): u=0 -> -1, u=4/9 -> -1/2, u=8/9 -> 1
    assert O.mobius(0.0) == -1.0
    assert abs(O.mobius(4 / 9) + 0.5) < 1e-15
    assert abs(O.mobius(8 / 9) - 1.0) < 1e-15


def test_composite_sqrt_trick_bound():
    # S:175 / P:264-270: sqrt(u) h(v(u)) ~ f(u) = sqrt(-ln(1-u)) on [0, 8/9], well under 1e-10
    u = np.linspace(0, 8 / 9, 20001)
    worst = 0.0
    for x in u:
        approx = math.sqrt(x) * O.eval_h(O.mobius(x))
        exact = math.sqrt(-math.log1p(-x))
        worst = max(worst, abs(approx - exact))
    assert worst < 2e-11


@pytest.mark.parametrize("v,s,c", [(0.5, 0.0, 1.0), (0.75, 1.0, 0.0), (0.0, 0.0, -1.0), (0.25, -1.0, 0.0)])
def test_sincos16_special_angles(v, s, c):
    # y = (2 pi v - pi)/16; v = 1/2 -> angle 0, 3/4 -> pi/2, 0 -> -pi
    gs, gc = O.sincos16(v)
    assert abs(gs - s) < 1e-10 and abs(gc - c) < 1e-10


def test_sincos16_grid_error_and_pythagoras():
    # P:150-153 "absolute error considerably less than 1e-10" (reading R17)
    v = np.linspace(0, 1, 100001)[:-1]
    es = ec = ep = 0.0
    for x in v:
        s, c = O.sincos16(float(x))
        th = 2 * math.pi * x - math.pi
        es = max(es, abs(s - math.sin(th)))
        ec = max(ec, abs(c - math.cos(th)))
        ep = max(ep, abs(s * s + c * c - 1))
    assert es < 1e-11 and ec < 1e-11 and ep < 4e-12


def test_sincos_leading_coefficients():
    # s1 ~ 1, c0 ~ 1 within 1e-6; Taylor: s3 ~ -1/6, c2 ~ -1/2
    assert abs(SIN[0] - 1) < 1e-6 and abs(COS[0] - 1) < 1e-6
    assert abs(SIN[1] + 1 / 6) < 1e-6 and abs(COS[1] + 0.5) < 1e-6
    assert COEFFS["sin_base_err"] < 1e-13 and COEFFS["cos_base_err"] < 1e-12


def test_header_matches_json():
    hdr = open(os.path.join(os.path.dirname(HERE), "oracle", "oracle_coeffs.h")).read()
    for x in COEFFS["h"] + COEFFS["sin"] + COEFFS["cos"]:
        assert x in hdr


@pytest.mark.slow
def test_committed_coefficients_reproduce():
    s, c = F.fit_sincos()
    assert [x.hex() for x in s] == COEFFS["sin"] and [x.hex() for x in c] == COEFFS["cos"]
    assert [x.hex() for x in F.fit_h()] == COEFFS["h"]
