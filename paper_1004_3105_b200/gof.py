"""Kolmogorov-Smirnov and Anderson-Darling gates from a fine probability-space histogram.

The device (nrng_gof_hist) bins p = Phi((x - mu)/sigma) into K = 2^log2K equal-probability
bins; with counts c_j and cumulative C_j = sum_{i<j} c_i:
  KS: D_edges = max_j |C_j / n - j / K| (the exact statistic D satisfies
      D_edges <= D <= D_edges + max_j c_j / n, reported as `ks_d_max`);
  AD: A^2 = n int_0^1 (F_n(p) - p)^2 / (p (1-p)) dp with F_n linear inside each bin
      (samples spread uniformly in a bin), integrated exactly per bin.
Gates at alpha = 0.01 with fully specified parameters: KS critical 1.6276 / sqrt(n)
(asymptotic Kolmogorov), AD critical 3.857 (asymptotic, Stephens).  No method arithmetic.
"""
from __future__ import annotations

import math

import numpy as np

KS_CRIT_001 = 1.6276
AD_CRIT_001 = 3.857


def kolmogorov_sf(lam: float) -> float:
    """P(sqrt(n) D > lam) for the limiting Kolmogorov distribution."""
    if lam < 0.2:
        return 1.0
    k = np.arange(1, 101)
    return float(min(1.0, max(0.0, 2 * np.sum((-1.0) ** (k - 1) * np.exp(-2 * k * k * lam * lam)))))


def ks_ad(hist) -> dict:
    c = np.asarray(hist, dtype=np.float64)
    n = c.sum()
    K = c.size
    C = np.concatenate([[0.0], np.cumsum(c)])  # C[j] = count below edge j/K
    edges = np.arange(K + 1) / K
    Fe = C / n
    d_edges = float(np.max(np.abs(Fe - edges)))
    d_max = d_edges + float(c.max() / n)
    # A^2: per bin, G(p) = F_n(p) - p is linear: G(a) = Fe[j]-a, G(b) = Fe[j+1]-b.
    # int_a^b G^2/(p(1-p)) dp with G = alpha + beta p: expand G^2/(p(1-p)) via partial fractions.
    a, b = edges[:-1], edges[1:]
    ga, gb = Fe[:-1] - a, Fe[1:] - b
    beta = (gb - ga) * K
    alpha = ga - beta * a
    # (alpha + beta p)^2 / (p (1 - p)) = alpha^2 / p + (alpha + beta)^2 / (1 - p) - beta^2
    with np.errstate(divide="ignore", invalid="ignore"):
        lnb_a = np.where(a > 0, np.log(b / np.where(a > 0, a, 1)), 0.0)
        ln1 = np.log((1 - a) / np.where(b < 1, 1 - b, 1))
    integ = np.zeros(K)
    mid = (a > 0) & (b < 1)
    integ[mid] = alpha[mid] ** 2 * lnb_a[mid] + (alpha[mid] + beta[mid]) ** 2 * ln1[mid] - beta[mid] ** 2 / K
    # end bins: F_n is a step near p = 0 and p = 1; the integrand is finite only if
    # alpha = 0 at p=0 (resp. alpha + beta = 0 at p=1) -- use the midpoint rule instead
    for j in (0, K - 1):
        pm = (a[j] + b[j]) / 2
        g = alpha[j] + beta[j] * pm
        integ[j] = g * g / (pm * (1 - pm)) / K
    A2 = float(n * np.sum(integ))
    lam = d_edges * math.sqrt(n)
    return {"n": int(n), "bins": K, "ks_d": d_edges, "ks_d_max": d_max, "ks_p": kolmogorov_sf(lam),
            "ks_pass": bool(d_max < KS_CRIT_001 / math.sqrt(n)), "ad_a2": A2, "ad_pass": bool(A2 < AD_CRIT_001)}


def serial_corr_gate(sums, n: int, z: float = 4.0) -> dict:
    """Serial-correlation gate: from S_k = sum_i d_i d_{i+k} (k = 0..K, d = x - c),
    r_k = (S_k / (n - k)) / (S_0 / n); each |r_k| of independent draws is ~N(0, 1/n), gate
    |r_k| <= z / sqrt(n) for every lag k = 1..K (z = 4 as the SPEC)."""
    s = np.asarray(sums, dtype=np.float64)
    K = s.size - 1
    k = np.arange(1, K + 1)
    r = (s[1:] / (n - k)) / (s[0] / n)
    bound = z / math.sqrt(n)
    worst = int(np.argmax(np.abs(r))) + 1
    return {"serial_r_max": float(np.max(np.abs(r))), "serial_lag_max": worst, "serial_bound": bound,
            "serial_pass": bool(np.all(np.abs(r) <= bound))}
