"""Validation of the whole BASELINE configs[4] sequence on ONE GPU: 2^34 fp64 normals over 2^19
streams, generated as the 8 rank shards of `bench.py --gpus 8` (rank r: global streams
[r 2^16, (r+1) 2^16), 2^31 normals), one after another, with the gate sums combined exactly as
`dist.validate`'s all-reduce combines them (SUM of power sums and histograms, MIN / MAX, the lag
products that straddle each shard boundary).  No collective and no second GPU: the same
reduction, evaluated in one process.  Per method: moments, 256-bin chi-square, KS and
Anderson-Darling on the 2^20-bin probability histogram, serial correlation lags 1..100 -- all
over the full 2^34-deviate sequence.

    python tools/validate_c5_full.py [--methods B1,B2,B3,P,P2] [--out FILE]
"""
import argparse
import json
import os
import sys
import time
from statistics import NormalDist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1004_3105_b200 as P  # noqa: E402
from paper_1004_3105_b200 import dist as D  # noqa: E402
from paper_1004_3105_b200 import gof as G  # noqa: E402
from paper_1004_3105_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--methods", default="B1,B2,B3,P,P2")
ap.add_argument("--out", default=None)
args = ap.parse_args()

c = W.C5_SHARD
RANKS, LAGS, K, LOG2K = 8, 100, 256, 20
n_total = RANKS * c.n
edges = [c.mu + c.sigma * NormalDist().inv_cdf(i / K) for i in range(1, K)]
out = torch.empty(c.n, dtype=torch.float64, device="cuda")
res = {"config": "BASELINE configs[4]: %d normals over %d streams (8 shards of %d streams), seed %d, mu %g, sigma %g"
                 % (n_total, RANKS * c.streams, c.streams, c.seed, c.mu, c.sigma),
       "note": "one GPU, shards generated in sequence; gate sums combined as dist.validate's all-reduce"}
for m in args.methods.split(","):
    t0 = time.time()
    sums = np.zeros(6)
    sums[4], sums[5] = np.inf, -np.inf
    hist = np.zeros(K, np.int64)
    fine = None
    lag = np.zeros(LAGS + 1)
    prev_tail = None
    for r in range(RANKS):
        g = P.Generator(c.seed, c.streams, first_stream=r * c.streams)
        g.normal(m, out=out, mu=c.mu, sigma=c.sigma)
        s, h = P.stats(out, c.mu, edges)
        s = s.cpu().numpy()
        sums[:4] += s[:4]
        sums[4], sums[5] = min(sums[4], s[4]), max(sums[5], s[5])
        hist += h.cpu().numpy().astype(np.int64)
        f = P.gof_hist(out, c.mu, c.sigma, LOG2K).to(torch.int64).cpu().numpy()
        fine = f if fine is None else fine + f
        lag += np.asarray(P.serial_corr(out, c.mu, LAGS), np.float64)
        head = (out[:LAGS] - c.mu).cpu().numpy()
        if prev_tail is not None:
            lag += D.cross_rank_lag_sums(prev_tail, head, LAGS)
        prev_tail = (out[c.n - LAGS:] - c.mu).cpu().numpy()
        g.close()
    torch.cuda.synchronize()
    v = D.moments(sums, n_total, c.sigma)
    gofr = G.ks_ad(fine)
    ser = G.serial_corr_gate(lag, n_total)
    v.update({"chi2": D.chi_square(hist, n_total), "dof": K - 1, "min": float(sums[4]), "max": float(sums[5]),
              "ks_d": gofr["ks_d"], "ks_p": gofr["ks_p"], "ks_pass": gofr["ks_pass"], "ad_a2": gofr["ad_a2"], "ad_pass": gofr["ad_pass"],
              "serial_r_max": ser["serial_r_max"], "serial_lag_max": ser["serial_lag_max"], "serial_bound": ser["serial_bound"],
              "serial_pass": ser["serial_pass"], "n": n_total, "seconds": round(time.time() - t0, 1)})
    res[m] = v
    print(m, json.dumps(v), flush=True)
del out
if args.out:
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)
