"""Per-config throughput on one GPU for every BASELINE.json config (C1-C5), incl. the C4 sweep.

Not the driver's bench line (that is bench.py, the C5 shard step); this reports each config's
own shape: normals/s per method, us per call, and fraction of the roofline floor.

    python tools/bench_configs.py [--calls N] > profiles/<tag>_configs.json
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1004_3105_b200 as P  # noqa: E402
from paper_1004_3105_b200 import workloads as W  # noqa: E402

HBM = 6554.6e9  # MEASURED_PEAKS.json hbm_gbs (copy)


def time_calls(g, method, n, mu, sigma, out, calls, warm=3, graph=False):
    stream = torch.cuda.current_stream()
    for _ in range(warm):
        g.normal(method, out=out[:n], mu=mu, sigma=sigma)
    if graph:
        gr = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(stream)
        with torch.cuda.stream(s):
            with torch.cuda.graph(gr, stream=s):
                for _ in range(calls):
                    g.normal(method, out=out[:n], mu=mu, sigma=sigma)
        stream.wait_stream(s)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        gr.replay()
        b.record(stream)
    else:
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(calls):
            g.normal(method, out=out[:n], mu=mu, sigma=sigma)
        b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / calls
    return {"n": n, "us_per_call": ms * 1e3, "normals_per_s": n / (ms / 1e3),
            "hbm_floor_frac": (8 * n / HBM) / (ms / 1e3)}


def time_seq(g, method, n, out, calls):
    stream = torch.cuda.current_stream()
    g.normal_seq(method, out=out[:n])
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(calls):
        g.normal_seq(method, out=out[:n])
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / calls
    return {"n": n, "us_per_call": ms * 1e3, "normals_per_s": n / (ms / 1e3),
            "hbm_floor_frac": (8 * n / HBM) / (ms / 1e3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=20)
    ap.add_argument("--sweep-calls", type=int, default=1000)
    args = ap.parse_args()
    res = {}
    big = torch.empty(1 << 31, dtype=torch.float64, device="cuda")
    for c in (W.C1, W.C2, W.C3):
        g = P.Generator(c.seed, c.streams)
        for m in c.methods + (("P2", "R", "R1") if c.name == "C2" else ()):
            res["%s_%s" % (c.name, m)] = time_calls(g, m, c.n, c.mu, c.sigma, big, args.calls)
        g.close()
    c = W.C4
    g = P.Generator(c.seed, c.streams)
    for m in c.methods:
        for L in W.C4_LENGTHS:
            calls = args.sweep_calls if L <= (1 << 22) else 50
            r = time_calls(g, m, L, c.mu, c.sigma, big, calls)
            r["calls"] = calls
            res["C4_%s_n%d" % (m, L)] = r
            rg = time_calls(g, m, L, c.mu, c.sigma, big, calls, graph=True)
            res["C4_%s_n%d_graph" % (m, L)] = dict(rg, calls=calls, note="CUDA graph of the calls")
    g.close()
    c = W.C5_SHARD
    g = P.Generator(c.seed, c.streams)
    for m in c.methods + ("P2", "R", "R1"):
        res["C5shard_%s" % m] = time_calls(g, m, c.n, c.mu, c.sigma, big, 5)
    # the sequential (RANN3-style, partition-invariant) mode at the shard
    # shape: one whole-epoch call of 2^31 deviates, and 10^3 short calls of 10^4 deviates
    for m in ("B1", "P"):
        P.nrng_seq_reset(g.h)
        res["seq_%s_bulk" % m] = time_seq(g, m, c.n, big, 3)
        res["seq_%s_n10000" % m] = dict(time_seq(g, m, 10000, big, args.sweep_calls), calls=args.sweep_calls)
    g.close()
    # the validation reductions on 2^31 deviates (untimed in bench.py; HBM
    # read-bound in principle: 16 GiB at the copy bandwidth is the floor)
    import statistics
    edges = [statistics.NormalDist().inv_cdf(i / 256) for i in range(1, 256)]
    for name, fn in (("stats_256bins", lambda: P.stats(big, 0.0, edges)),
                     ("gof_hist_2^20bins", lambda: P.gof_hist(big, 0.0, 1.0, 20)),
                     ("serial_corr_lags100", lambda: P.serial_corr(big, 0.0, 100))):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        res["validate_%s" % name] = {"n": big.numel(), "ms_per_call": ms,
                                      "read_gbs": 8 * big.numel() / (ms / 1e3) / 1e9,
                                      "hbm_floor_frac": (8 * big.numel() / HBM) / (ms / 1e3)}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
