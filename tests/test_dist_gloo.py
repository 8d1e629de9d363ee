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
