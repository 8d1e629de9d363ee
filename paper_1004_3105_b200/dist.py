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
