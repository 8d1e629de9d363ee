"""Pins for the oracle's method P2: Polar with step 4a (u = 1 - s) and
the B3 approximation h(v) of g(s) = sqrt(-ln(1-s)/s) on s <= 8/9, library ln/sqrt on s > 8/9."""
import math

import numpy as np
import pytest
from scipy import stats as sps

import oracle as O
from paper_1004_3105_b200.workloads import dyadic_uniforms


def _p2_exact(x, y, s, mu=0.0, sigma=1.0):
    # step 4a with u = 1 - s: r = sigma sqrt(-2 ln(1-s)/s), output r x + mu
    if s == 0:
        return mu, mu
    r = sigma * math.sqrt(-2 * math.log1p(-s) / s)
    return mu + r * x, mu + r * y


@pytest.mark.parametrize("a,b", [(11 / 16, 3 / 4), (0.9, 0.3), (0.1, 0.45), (0.99, 0.55), (0.5, 0.96875)])
def test_p2_closed_forms_within_paper_bound(a, b):
    acc, xy, (x, y, s) = O.polar2_pair(a, b, 0.5, 2.0)
    assert acc
    ex = _p2_exact(x, y, s, 0.5, 2.0)
    # |h - g| < 2e-11 scaled by sigma sqrt2 |x| <= 2 * 1.42
    assert abs(xy[0] - ex[0]) < 2e-11 * 2.0 * math.sqrt(2) + 1e-14
    assert abs(xy[1] - ex[1]) < 2e-11 * 2.0 * math.sqrt(2) + 1e-14


def test_p2_origin_and_rejections():
    # s = 0: v = -1, h(-1) ~ 1, x = y = 0 -> exactly (mu, mu) with no special case
    acc, xy, xys = O.polar2_pair(0.5, 0.5, 1.25, 3.0)
    assert acc and xys[2] == 0.0 and xy == (1.25, 1.25)
    for a, b in [(0.0, 0.0), (0.0, 0.5), (1 - 2**-53, 1 - 2**-53)]:
        assert not O.polar2_pair(a, b)[0]


def test_p2_tail_branch_is_library_exact():
    # s > 8/9 uses ln/sqrt directly: agrees with the definition to rounding
    u = dyadic_uniforms(40, 2 * 200000)
    out, mask = O.transform_from_uniforms(u, 5, 0.0, 1.0)
    a, b = u[0::2], u[1::2]
    x, y = 2 * a - 1, 2 * b - 1
    s = x * x + y * y
    tail = (s > 8 / 9) & (s < 1)
    r = np.sqrt(-2 * np.log1p(-s[tail]) / s[tail])
    assert np.allclose(out[0::2][tail], r * x[tail], rtol=0, atol=1e-13)


def test_p2_matches_exact_everywhere_within_bound_and_tau_continuity():
    u = dyadic_uniforms(41, 2 * 200000)
    out, mask = O.transform_from_uniforms(u, 5, 0.0, 1.0)
    a, b = u[0::2], u[1::2]
    x, y = 2 * a - 1, 2 * b - 1
    s = x * x + y * y
    acc = mask.astype(bool)
    assert np.array_equal(acc, s < 1)
    r = np.where(s[acc] > 0, np.sqrt(-2 * np.log1p(-s[acc]) / np.where(s[acc] > 0, s[acc], 1)), 0)
    assert np.max(np.abs(out[0::2][acc] - r * x[acc])) < 4e-11
    # fast/tail agreement across s = 8/9
    for sv in np.linspace(8 / 9 - 1e-6, 8 / 9 + 1e-6, 41):
        fast = math.sqrt(2) * O.eval_h(O.mobius(float(sv)))
        tail = math.sqrt(-2 * math.log1p(-sv) / sv)
        assert abs(fast - tail) < 1e-10


def test_p2_consumption_equals_polar_and_gates():
    # same candidate stream and acceptance as P: identical consumption, same output signs/angles
    n = 1 << 20
    a, b = O.Streams(77, 256), O.Streams(77, 256)
    p1 = a.normal_polar(n)
    p2 = b.normal_polar2(n)
    assert np.array_equal(a.counts, b.counts)
    assert np.array_equal(np.sign(p1), np.sign(p2))
    z = p2
    assert abs(z.mean()) < 4 / math.sqrt(n) and abs(z.var() - 1) < 4 * math.sqrt(2 / n)
    K = 64
    edges = sps.norm.ppf(np.arange(1, K) / K)
    _, hist = O.stats(z, 0.0, edges)
    chi2 = np.sum((hist - n / K) ** 2 / (n / K))
    assert chi2 < sps.chi2.ppf(0.99, K - 1)
