"""Multi-process (world size 2, gloo, CPU) checks of the sharding and validation plumbing
that bench.py runs over NCCL."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1004_3105_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


EDGES = np.array([-1.5, -0.5, 0.0, 0.5, 1.5])


def _local_stats(x, center):
    sums, hist = O.stats(x, center, EDGES)
    return torch.tensor(sums, dtype=torch.float64), torch.tensor(hist, dtype=torch.int64)


def _worker(rank, world, port, streams_per_rank, per_stream, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, count = D.shard_streams(rank, streams_per_rank)
    st = O.Streams(5, count, first_stream=first)
    x = st.normal_polar(count * per_stream, 0.25, 2.0)
    sums, hist = _local_stats(x, 0.25)
    sums, hist = D.allreduce_stats(sums, hist)
    if rank == 0:
        q.put((sums.numpy(), hist.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_reduction_equals_single_process():
    world, spr, per = 2, 8, 2 * 50
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, spr, per, q)) for r in range(world)]
    for p in procs:
        p.start()
    sums, hist = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # single process over the union of the shards: the same global streams [0, 16)
    full = O.Streams(5, world * spr).normal_polar(world * spr * per, 0.25, 2.0)
    ref_sums, ref_hist = O.stats(full, 0.25, EDGES)
    assert np.allclose(sums[:4], ref_sums[:4], rtol=1e-12)
    assert sums[4] == ref_sums[4] and sums[5] == ref_sums[5]
    assert np.array_equal(hist, ref_hist)


def test_shard_ranges_are_disjoint_and_cover():
    ranges = [D.shard_streams(r, 1 << 16) for r in range(8)]
    assert ranges[0] == (0, 1 << 16)
    assert all(ranges[i][0] + ranges[i][1] == ranges[i + 1][0] for i in range(7))
    assert ranges[-1][0] + ranges[-1][1] == 1 << 19  # BASELINE configs[4]: 2^19 streams at 8 GPUs


def test_moments_and_gates():
    x = O.Streams(1, 64).normal_boxmuller(1 << 18, 0.0, 1.0, 1)
    sums, hist = O.stats(x, 0.0, EDGES)
    m = D.moments(sums, x.size)
    assert abs(m["mean"] - x.mean()) < 1e-12 and abs(m["var"] - x.var()) < 1e-12
    z = (x - x.mean()) / x.std()
    assert abs(m["skew"] - np.mean(z**3)) < 1e-9 and abs(m["exkurt"] - (np.mean(z**4) - 3)) < 1e-9
    assert m["moments_4se_pass"]
    bad = D.moments(sums * np.array([1, 1.1, 1, 1, 1, 1]), x.size)  # variance off by 10%
    assert not bad["moments_4se_pass"]
    flat = D.chi_square([100] * 6, 600)
    assert flat == 0.0 and D.chi_square([200, 0, 100, 100, 100, 100], 600) > 100


# ---------------------------------------------------------------- bench.py's validation leg
# dist.validate is what bench.py runs after its timed region (over NCCL); here the same code
# runs over gloo with CPU stand-ins for the three device reductions, and world size 2 must
# give the single-process result on the concatenated output (including the lagged products
# that straddle the rank boundary).

def _cpu_stats(x, center, edges):
    sums, hist = O.stats(x.numpy(), center, np.asarray(edges))
    return torch.tensor(sums, dtype=torch.float64), torch.tensor(hist, dtype=torch.int64)


def _cpu_gof_hist(x, mu, sigma, log2K):
    from scipy.stats import norm

    K = 1 << log2K
    b = np.minimum((norm.cdf((x.numpy() - mu) / sigma) * K).astype(np.int64), K - 1)
    return torch.from_numpy(np.bincount(b, minlength=K))


def _cpu_serial(x, center, lags):
    d = x.numpy() - center
    return np.array([np.dot(d[: d.size - k], d[k:]) for k in range(lags + 1)])


def _validate_worker(rank, world, port, per_rank, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    st = O.Streams(11, 64, first_stream=64 * rank)
    x = torch.from_numpy(st.normal_polar(per_rank, 0.0, 1.0))
    v = D.validate(x, per_rank, 0.0, 1.0, stats=_cpu_stats, gof_hist=_cpu_gof_hist, serial=_cpu_serial,
                   world=world, rank=rank, log2K=12, lags=100)
    if rank == 0:
        q.put(v)
    dist.barrier()
    dist.destroy_process_group()


def test_validate_world2_equals_single_process():
    world, per_rank = 2, 64 * 2 * 1000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_validate_worker, args=(r, world, port, per_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    v2 = q.get(timeout=180)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    full = torch.from_numpy(O.Streams(11, 128).normal_polar(world * per_rank, 0.0, 1.0))
    v1 = D.validate(full, world * per_rank, 0.0, 1.0, stats=_cpu_stats, gof_hist=_cpu_gof_hist,
                    serial=_cpu_serial, log2K=12, lags=100)
    for key in ("mean", "var", "skew", "exkurt", "chi2", "ks_d", "ad_a2", "serial_r_max"):
        assert math.isclose(v1[key], v2[key], rel_tol=1e-9, abs_tol=1e-15), key
    for key in ("min", "max", "serial_lag_max", "ks_pass", "ad_pass", "serial_pass", "moments_4se_pass"):
        assert v1[key] == v2[key], key


def test_cross_rank_lag_sums_brute_force():
    rng = np.random.default_rng(1)
    a, b = rng.standard_normal(37), rng.standard_normal(50)

    def lagsum(v, k):
        return float(np.dot(v[: v.size - k], v[k:])) if k < v.size else 0.0

    for lags in (1, 5, 36, 40):
        ab = np.concatenate([a, b])
        full = np.array([lagsum(ab, k) for k in range(lags + 1)])
        sep = np.array([lagsum(a, k) + lagsum(b, k) for k in range(lags + 1)])
        m = min(lags, 37)
        cross = D.cross_rank_lag_sums(a[a.size - m:], b[:lags], lags)
        assert np.allclose(sep + cross, full, rtol=1e-13, atol=1e-12)


def test_bench_relaunches_itself_under_torchrun(monkeypatch):
    # `python bench.py --gpus N` without a launcher re-executes under torch.distributed.run with
    # N ranks on 127.0.0.1 (the flag used to be ignored outside torchrun)
    import subprocess
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    seen = {}

    def fake_call(cmd):
        seen["cmd"] = cmd
        return 0

    monkeypatch.setattr(subprocess, "call", fake_call)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])
    assert bench.relaunch(4) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert cmd[cmd.index("--nproc-per-node") + 1] == "4" and cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"] and cmd[-5].endswith("bench.py")
