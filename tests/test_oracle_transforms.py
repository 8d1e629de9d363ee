"""Pins for the oracle's transforms B1, B2, B3, P and its stream-level driver.

Closed forms, invariants, special cases, the paper's error bounds and rates:
B1 P:67-86; B2 P:148-170; B3 P:226-295; P P:106-134.
"""
import math

import numpy as np
import pytest
from scipy import stats as sps

import oracle as O
from paper_1004_3105_b200.workloads import dyadic_uniforms

E = 2.0 ** -53


# ------------------------------------------------------------------ B1 --------

def test_b1_closed_form_radius_two():
    # u = 1 - e^-2 (to 53 bits) -> r = sqrt(-2 ln e^-2) = 2; v = 3/4 -> theta = pi/2
    u = math.floor((1 - math.exp(-2.0)) * 2**53) * E
    x, y = O.b1_pair(u, 0.75)
    r = math.sqrt(-2 * math.log1p(-u))
    assert abs(r - 2) < 1e-15
    assert abs(x - r) < 1e-15 and abs(y) < 1e-15


@pytest.mark.parametrize("u,v", [(0.25, 0.125), (0.5, 0.9375), (0.1, 0.3), (1 - E, 0.0)])
def test_b1_reduces_to_library(u, v):
    r = math.sqrt(-2 * math.log(1 - u))
    th = 2 * math.pi * v - math.pi
    x, y = O.b1_pair(u, v)
    assert abs(x - r * math.sin(th)) < 1e-14 and abs(y - r * math.cos(th)) < 1e-14


def test_b1_zero_radius_and_sigma_zero():
    assert O.b1_pair(0.0, 0.3, 1.5, 2.0) == (1.5, 1.5)
    for u, v in [(0.3, 0.1), (1 - E, 0.77)]:
        assert O.b1_pair(u, v, -3.25, 0.0) == (-3.25, -3.25)


def test_b1_radius_invariant():
    # (x-mu)^2 + (y-mu)^2 = -2 sigma^2 ln(1-u)
    u = dyadic_uniforms(1, 20000)
    mu, sigma = 2.5, 0.5
    out, _ = O.transform_from_uniforms(u, 1, mu, sigma)
    lhs = (out[0::2] - mu) ** 2 + (out[1::2] - mu) ** 2
    rhs = -2 * sigma**2 * np.log1p(-u[0::2])
    assert np.allclose(lhs, rhs, rtol=1e-13, atol=1e-15)


# ------------------------------------------------------------------ B2 --------

def test_b2_within_paper_bound_of_b1():
    # approximations with absolute error "considerably less than 1e-10" (R17)
    u = dyadic_uniforms(2, 200000)
    b1, _ = O.transform_from_uniforms(u, 1)
    b2, _ = O.transform_from_uniforms(u, 2)
    err = np.max(np.abs(b1 - b2))
    assert err < 1e-10
    assert err > 0  # it is an approximation


# ------------------------------------------------------------------ B3 --------

def _b3_exact(u1, u2, u3, mu=0.0, sigma=1.0):
    m = max(u1, u2)
    rad = sigma * math.sqrt(-2 * math.log1p(-m * m))
    th = 2 * math.pi * u3 - math.pi
    return mu + rad * math.cos(th), mu + rad * math.sin(th)


def test_b3_bulk_example_equals_b1_radius():
    # (0.5, 0.25, 0.75): u = 1/4 (bulk), radius sqrt(-2 ln 3/4) = B1's radius at u = 1/4
    x, y = O.b3_pair(0.5, 0.25, 0.75)
    assert abs(x) < 1e-10 and abs(y - math.sqrt(-2 * math.log(0.75))) < 1e-10


def test_b3_tail_example():
    # (31/32, 0.25, 0.75): u = 0.9384765625 > 8/9 -> library branch
    x, y = O.b3_pair(31 / 32, 0.25, 0.75)
    assert abs(x) < 1e-10
    assert abs(y - math.sqrt(-2 * math.log1p(-(31 / 32) ** 2))) < 1e-13


def test_b3_zero_radius():
    assert O.b3_pair(0.0, 0.0, 0.4, 7.0, 3.0) == (7.0, 7.0)


def test_b3_within_paper_bound_of_exact():
    u = dyadic_uniforms(3, 3 * 100000)
    out, _ = O.transform_from_uniforms(u, 3, 2.5, 0.5)
    worst = 0.0
    for j in range(0, 100000, 7):
        ex = _b3_exact(u[3 * j], u[3 * j + 1], u[3 * j + 2], 2.5, 0.5)
        worst = max(worst, abs(out[2 * j] - ex[0]), abs(out[2 * j + 1] - ex[1]))
    assert worst < 1e-10 * 0.5


def test_b3_max_squared_is_uniform():
    # u = max(u1,u2)^2 is uniform on [0,1); KS at alpha = 0.01
    u1, u2 = dyadic_uniforms(4, 10**6), dyadic_uniforms(5, 10**6)
    m2 = np.maximum(u1, u2) ** 2
    assert sps.kstest(m2, "uniform").pvalue > 0.01


def test_b3_tau_boundary_continuity():
    # fast/tail agreement across u = 8/9 (S:318 analogue for B3)
    m0 = math.sqrt(8 / 9)
    for m in [np.nextafter(m0, 0) - k * E for k in range(3)] + [np.nextafter(m0, 1) + k * E for k in range(3)]:
        x, y = O.b3_pair(float(m), 0.0, 0.75)
        assert abs(y - math.sqrt(-2 * math.log1p(-m * m))) < 1e-10


# ------------------------------------------------------------------ P ---------

def test_polar_closed_form():
    # (a,b) = (11/16, 3/4) -> x = 3/8, y = 1/2, s = 25/64 exactly
    acc, xy, xys = O.polar_pair(11 / 16, 3 / 4)
    assert acc and xys == (0.375, 0.5, 25 / 64)
    r = math.sqrt(-2 * math.log(25 / 64) / (25 / 64))
    assert abs(xy[0] - 0.375 * r) < 1e-15 and abs(xy[1] - 0.5 * r) < 1e-15
    acc, xy, _ = O.polar_pair(11 / 16, 3 / 4, 2.5, 0.5)
    assert abs(xy[0] - (2.5 + 0.5 * 0.375 * r)) < 1e-15


@pytest.mark.parametrize("a,b,acc", [(0.0, 0.0, False), (0.0, 0.5, False), (0.5, 0.0, False),
                                     (0.5, 0.5, True), (1 - E, 1 - E, False), (0.5 + E, 1 - E, True)])
def test_polar_accept_boundaries(a, b, acc):
    # s >= 1 rejects: x=-1,y=0 gives s = 1 exactly -> reject; s = 0 accepted -> (mu, mu)
    got, xy, xys = O.polar_pair(a, b, 1.25, 3.0)
    assert got == acc
    if got and xys[2] == 0.0:
        assert xy == (1.25, 1.25)


def test_polar_invariants():
    u = dyadic_uniforms(6, 2 * 100000)
    mu, sigma = -1.0, 2.0
    out, mask = O.transform_from_uniforms(u, 4, mu, sigma)
    a, b = u[0::2], u[1::2]
    x, y = 2 * a - 1, 2 * b - 1
    s = x * x + y * y
    assert np.array_equal(mask.astype(bool), s < 1)
    sel = mask.astype(bool) & (s > 0)
    xo, yo = out[0::2][sel] - mu, out[1::2][sel] - mu
    # (xo^2 + yo^2) = -2 sigma^2 ln s ; xo/yo = x/y
    assert np.allclose(xo**2 + yo**2, -2 * sigma**2 * np.log(s[sel]), rtol=1e-13)
    assert np.allclose(xo * y[sel], yo * x[sel], rtol=1e-12, atol=1e-14)


def test_polar_acceptance_rate_and_s_uniform():
    # accepted s uniform on [0,1); acceptance pi/4
    m = 10**6
    msk = O.Streams(7, 8).polar_mask(m // 8)
    p = msk.mean()
    assert abs(p - math.pi / 4) < 4 * math.sqrt(math.pi / 4 * (1 - math.pi / 4) / m)
    u = dyadic_uniforms(8, 2 * 200000)
    x, y = 2 * u[0::2] - 1, 2 * u[1::2] - 1
    s = x * x + y * y
    assert sps.kstest(s[s < 1], "uniform").pvalue > 0.01


# ------------------------------------------------------ stream-level driver ----

@pytest.mark.parametrize("variant,per_pair", [(1, 2), (2, 2), (3, 3)])
def test_boxmuller_consumption_and_layout(variant, per_pair):
    S, n = 6, 2 * 6 * 5 + 2 * 4 + 1  # P = 39 pairs: q = 6, rem = 3; odd n drops the last deviate
    st = O.Streams(13, S)
    out = st.normal_boxmuller(n, 0.5, 2.0, variant)
    P = (n + 1) // 2
    q, rem = divmod(P, S)
    assert list(st.counts) == [per_pair * (q + (k < rem)) for k in range(S)]
    for k in range(S):
        one = O.Streams(13, 1, first_stream=k)
        cnt = q + (k < rem)
        off = 2 * (k * q + min(k, rem))
        ref = one.normal_boxmuller(2 * cnt, 0.5, 2.0, variant)
        m = min(2 * cnt, n - off)
        assert np.array_equal(out[off:off + m], ref[:m])


def test_boxmuller_uses_stream_uniforms_in_order():
    st = O.Streams(21, 3)
    u = O.Streams(21, 3).uniform(3 * 2 * 4)  # 4 pairs per stream
    out = st.normal_boxmuller(3 * 2 * 4)
    ref, _ = O.transform_from_uniforms(u, 1)
    assert np.array_equal(out, ref)


def test_polar_exact_stop_and_order():
    S, n = 4, 2 * 4 * 9
    st = O.Streams(7, S)
    out = st.normal_polar(n, 1.0, 0.5)
    for k in range(S):
        # replay stream k's uniforms through the pairwise definition, stop at the 9th accept
        ref_st = O.Streams(7, 1, first_stream=k)
        used = int(st.counts[k])
        u = ref_st.uniform(used)
        tr, mask = O.transform_from_uniforms(u, 4, 1.0, 0.5)
        acc = np.flatnonzero(mask)
        assert acc.size == 9 and acc[-1] == used // 2 - 1  # last candidate consumed was accepted
        exp = tr.reshape(-1, 2)[acc].ravel()
        assert np.array_equal(out[18 * k:18 * (k + 1)], exp)


def test_polar_uniforms_per_normal():
    # 4/pi ~ 1.27 uniforms per normal on average
    st = O.Streams(99, 64)
    n = 64 * 2 * 4000
    st.normal_polar(n)
    rate = st.counts.sum() / n
    # 2 uniforms per candidate, candidates geometric with p = pi/4; 4 SE
    se = 2 * math.sqrt((1 - math.pi / 4) / (math.pi / 4) ** 2 / (n / 2)) / 2
    assert abs(rate - 4 / math.pi) < 4 * se


def test_n_smaller_than_two_streams_and_zero():
    st = O.Streams(3, 64)
    out = st.normal_boxmuller(64)  # 32 pairs -> only streams 0..31 advance
    assert list(st.counts) == [2] * 32 + [0] * 32
    assert st.normal_polar(0).size == 0 and st.normal_boxmuller(0).size == 0


def test_partition_invariance_per_stream():
    # one call of n vs k calls of n/k (each call gives every stream the same quota)
    S = 8
    for fn in ("normal_polar", "normal_boxmuller"):
        a, b = O.Streams(5, S), O.Streams(5, S)
        one = getattr(a, fn)(2 * S * 12).reshape(S, 24)
        parts = [getattr(b, fn)(2 * S * 4).reshape(S, 8) for _ in range(3)]
        assert np.array_equal(one, np.concatenate(parts, axis=1))
        assert np.array_equal(a.counts, b.counts)


# ------------------------------------------------------ statistical gates ------

@pytest.mark.parametrize("method", ["B1", "B2", "B3", "P"])
def test_moment_and_chi_square_gates(method):
    n, mu, sigma = 1 << 20, 2.5, 0.5
    st = O.Streams(1234, 1024)
    if method == "P":
        x = st.normal_polar(n, mu, sigma)
    else:
        x = st.normal_boxmuller(n, mu, sigma, int(method[1]))
    z = (x - mu) / sigma
    m1, m2 = z.mean(), z.var()
    sk = np.mean((z - m1) ** 3) / m2**1.5
    ku = np.mean((z - m1) ** 4) / m2**2 - 3
    assert abs(m1) < 4 / math.sqrt(n)
    assert abs(m2 - 1) < 4 * math.sqrt(2 / n)
    assert abs(sk) < 4 * math.sqrt(6 / n)
    assert abs(ku) < 4 * math.sqrt(24 / n)
    K = 64
    edges = mu + sigma * sps.norm.ppf(np.arange(1, K) / K)
    sums, hist = O.stats(x, mu, edges)
    assert hist.sum() == n
    chi2 = np.sum((hist - n / K) ** 2 / (n / K))
    assert chi2 < sps.chi2.ppf(0.99, K - 1)
    assert abs(sums[0] / n / sigma - m1) < 1e-12


def test_stats_against_numpy():
    x = dyadic_uniforms(10, 5000) * 6 - 3
    edges = np.array([-1.0, 0.0, 0.5, 2.0])
    sums, hist = O.stats(x, 0.25, edges)
    d = x - 0.25
    assert np.allclose(sums[:4], [d.sum(), (d**2).sum(), (d**3).sum(), (d**4).sum()], rtol=1e-12)
    assert sums[4] == x.min() and sums[5] == x.max()
    assert list(hist) == list(np.histogram(x, bins=np.concatenate([[-np.inf], edges, [np.inf]]))[0])
