"""Multi-GPU plumbing: stream sharding and the validation all-reduce.

Generation needs no communication: rank r of W owns the contiguous global stream range
[r * S_r, (r+1) * S_r) and generates its own outputs.  The only exchange is the
validation reduction -- per-rank sums of (x - mu)^k (k = 1..4), min, max and a K-bin
histogram -- all-reduced with torch.distributed (NCCL on GPUs; gloo in the CPU tests).
"""
from __future__ import annotations

import math


def shard_streams(rank: int, streams_per_rank: int) -> tuple[int, int]:
    """(first global stream id, stream count) owned by `rank` (weak scaling)."""
    return rank * streams_per_rank, streams_per_rank


def allreduce_stats(sums, hist, group=None):
    """In-place all-reduce of one rank's (sums[6], hist[K]) torch tensors: SUM over the four
    power sums and the histogram, MIN of sums[4], MAX of sums[5].  Returns (sums, hist)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return sums, hist
    packed = torch.cat([sums[:4], hist.to(sums.dtype)])
    dist.all_reduce(packed, group=group)
    mn, mx = sums[4:5].clone(), sums[5:6].clone()
    dist.all_reduce(mn, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    out = torch.cat([packed[:4], mn, mx])
    return out, packed[4:].round().to(hist.dtype)


def moments(sums, n: int, sigma: float = 1.0) -> dict:
    """Mean, variance, skewness and excess kurtosis (in units of sigma) from the power sums
    about mu, with the 4-standard-error gates (mean 4/sqrt(n), var 4 sqrt(2/n), skew
    4 sqrt(6/n), kurt 4 sqrt(24/n))."""
    s1, s2, s3, s4 = (float(sums[i]) for i in range(4))
    m1 = s1 / n
    var = s2 / n - m1 * m1
    mu3 = s3 / n - 3 * m1 * s2 / n + 2 * m1 ** 3
    mu4 = s4 / n - 4 * m1 * s3 / n + 6 * m1 * m1 * s2 / n - 3 * m1 ** 4
    skew = mu3 / var ** 1.5
    kurt = mu4 / var ** 2 - 3
    mean_s, var_s = m1 / sigma, var / sigma ** 2
    ok = (abs(mean_s) < 4 / math.sqrt(n) and abs(var_s - 1) < 4 * math.sqrt(2 / n)
          and abs(skew) < 4 * math.sqrt(6 / n) and abs(kurt) < 4 * math.sqrt(24 / n))
    return {"mean": mean_s, "var": var_s, "skew": skew, "exkurt": kurt, "moments_4se_pass": bool(ok)}


def chi_square(hist, n: int) -> float:
    """Pearson statistic of an equiprobable-bin histogram."""
    K = len(hist)
    e = n / K
    return float(sum((float(h) - e) ** 2 / e for h in hist))


def cross_rank_lag_sums(tail, head_next, lags: int):
    """Lagged products sum_i d_i d_{i+k}, k = 0..lags, over the pairs (i, i+k) that straddle
    a rank boundary: i among the last `lags` deviates of rank r (`tail`, centred), i+k among
    the first `lags` of rank r+1 (`head_next`, centred).  k = 0 has none."""
    import numpy as np

    t = np.asarray(tail, np.float64)
    h = np.asarray(head_next, np.float64)
    out = np.zeros(lags + 1)
    L = t.size
    for k in range(1, lags + 1):
        # i = L - a (a = 1..min(k, L)) pairs with head index k - a
        a = np.arange(1, min(k, L) + 1)
        a = a[k - a < h.size]
        out[k] = float(np.dot(t[L - a], h[k - a]))
    return out


def validate(x, n_local: int, mu: float, sigma: float, *, stats, gof_hist, serial, world: int = 1,
             rank: int = 0, K: int = 256, log2K: int = 20, lags: int = 100, group=None) -> dict:
    """The bench's validation of one method's output, identical on every rank count: each
    rank's deviates `x` are the contiguous slice [rank n_local, (rank+1) n_local) of the
    global stream-major output (Q6), so the gates see the whole 2^34-deviate sequence.
      * moments + K-bin chi-square: per-rank power sums / histogram (`stats`), all-reduced;
      * KS / Anderson-Darling: per-rank 2^log2K-bin probability histogram (`gof_hist`), summed;
      * serial correlation, lags 1..`lags`: per-rank lagged sums (`serial`) plus the products
        that straddle each rank boundary (first `lags` deviates all-gathered), summed.
    `stats(x, center, edges) -> (sums[6], hist[K])` tensors, `gof_hist(x, mu, sigma, log2K)`
    -> int tensor, `serial(x, center, lags)` -> numpy (lags + 1) -- the device kernels in
    bench.py, CPU stand-ins in the gloo test.  The only exchanges are these reductions."""
    from statistics import NormalDist

    import numpy as np
    import torch
    import torch.distributed as dist

    from . import gof as G

    multi = world > 1 and dist.is_available() and dist.is_initialized()
    edges = [mu + sigma * NormalDist().inv_cdf(i / K) for i in range(1, K)]
    sums, hist = stats(x, mu, edges)
    sums, hist = allreduce_stats(sums, hist, group=group)
    fine = gof_hist(x, mu, sigma, log2K).to(torch.int64)
    if multi:
        dist.all_reduce(fine, group=group)
    gofr = G.ks_ad(fine.cpu().numpy())
    lag = np.asarray(serial(x, mu, lags), np.float64)
    if multi:
        m = min(lags, n_local)
        head = (x[:m].to(torch.float64) - mu).contiguous()
        heads = [torch.empty_like(head) for _ in range(world)]
        dist.all_gather(heads, head, group=group)
        if rank + 1 < world:
            tail = (x[n_local - m:].to(torch.float64) - mu).cpu().numpy()
            lag = lag + cross_rank_lag_sums(tail, heads[rank + 1].cpu().numpy(), lags)
        lt = torch.from_numpy(lag).to(x.device)
        dist.all_reduce(lt, group=group)
        lag = lt.cpu().numpy()
    n = world * n_local
    serial_r = G.serial_corr_gate(lag, n)
    sums, hist = sums.cpu().numpy(), hist.cpu().numpy()
    v = moments(sums, n, sigma)
    v.update({"chi2": chi_square(hist, n), "dof": K - 1, "min": float(sums[4]), "max": float(sums[5]),
              "ks_d": gofr["ks_d"], "ks_pass": gofr["ks_pass"], "ad_a2": gofr["ad_a2"], "ad_pass": gofr["ad_pass"],
              "serial_r_max": serial_r["serial_r_max"], "serial_lag_max": serial_r["serial_lag_max"],
              "serial_pass": serial_r["serial_pass"]})
    return v
