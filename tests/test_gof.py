"""The histogram-based KS / Anderson-Darling gates (paper_1004_3105_b200/gof.py) against the
exact order-statistic formulas, and their power."""
import math

import numpy as np
import pytest
from scipy import stats as sps

import oracle as O
from paper_1004_3105_b200 import gof


def _hist(x, K):
    p = sps.norm.cdf(x)
    return np.bincount(np.minimum((p * K).astype(np.int64), K - 1), minlength=K)


def _exact(x):
    p = np.sort(sps.norm.cdf(x))
    n = p.size
    i = np.arange(1, n + 1)
    d = max(np.max(i / n - p), np.max(p - (i - 1) / n))
    a2 = -n - np.mean((2 * i - 1) * (np.log(p) + np.log1p(-p[::-1])))
    return d, a2


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_histogram_statistics_match_exact(seed):
    x = np.random.default_rng(seed).standard_normal(400000)
    r = gof.ks_ad(_hist(x, 1 << 18))
    d, a2 = _exact(x)
    assert r["ks_d"] <= d + 1e-12 <= r["ks_d_max"] + 1e-12
    assert abs(r["ad_a2"] - a2) < 0.01 * max(1.0, a2)


def test_gates_pass_on_oracle_output_and_fail_on_wrong_laws():
    n = 1 << 20
    for m in (1, 3):
        x = O.Streams(5, 256).normal_boxmuller(n, 0.0, 1.0, m)
        r = gof.ks_ad(_hist(x, 1 << 18))
        assert r["ks_pass"] and r["ad_pass"], r
    x = O.Streams(5, 256).normal_polar(n)
    r = gof.ks_ad(_hist(x, 1 << 18))
    assert r["ks_pass"] and r["ad_pass"]
    # uniforms labelled normal and a slightly heavy tail both fail
    rng = np.random.default_rng(9)
    assert not gof.ks_ad(_hist(rng.uniform(-2, 2, n), 1 << 18))["ad_pass"]
    t = gof.ks_ad(_hist(rng.standard_t(25, n), 1 << 18))
    assert not t["ad_pass"]


def test_kolmogorov_sf():
    assert abs(gof.kolmogorov_sf(gof.KS_CRIT_001) - 0.01) < 2e-4
    assert gof.kolmogorov_sf(0.1) == 1.0


# ---------------------------------------------------------------- serial correlation

def _lag_sums(x, c, K):
    d = x - c
    return np.array([np.dot(d[: d.size - k], d[k:]) for k in range(K + 1)])


def test_serial_gate_passes_iid_and_catches_ma1():
    rng = np.random.default_rng(7)
    z = rng.standard_normal(1_000_001)
    n = 1_000_000
    assert gof.serial_corr_gate(_lag_sums(z[1:], 0.0, 100), n)["serial_pass"]
    # MA(1): x_i = z_i + 0.05 z_{i-1} has r_1 = 0.05 / 1.0025 ~ 0.0499 >> 4/sqrt(n) = 0.004
    x = z[1:] + 0.05 * z[:-1]
    g = gof.serial_corr_gate(_lag_sums(x, 0.0, 100), n)
    assert not g["serial_pass"] and g["serial_lag_max"] == 1 and abs(g["serial_r_max"] - 0.05 / 1.0025) < 0.005


def test_serial_gate_on_oracle_uniform_stream():
    # serial correlation at lags 1..100 of 10^6 draws of one stream within 4/sqrt(10^6)
    st = O.Streams(2024, 1)
    u = st.uniform(1_000_000)
    g = gof.serial_corr_gate(_lag_sums(u, 0.5, 100), u.size)
    assert g["serial_pass"], g
