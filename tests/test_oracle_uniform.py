"""Pins for the oracle's uniform source (splitmix64 seeding + additive LFG(607,273)).

The paper uses RANU4, a "generalised Fibonacci random number generator"
whose lags it does not state; reading R1 takes the SPEC's additive
x_n = x_{n-607} + x_{n-273} mod 2^64 and splitmix64 seeding (BASELINE.json).
"""
import math

import numpy as np
import pytest

import oracle as O

MASK = (1 << 64) - 1


def test_splitmix64_published_vector():
    # First three outputs of splitmix64 seeded with 0, as published with the reference
    # implementation (Vigna, splitmix64.c); an external pin for the seeding mixer.
    got = [int(x) for x in O.splitmix64(0, 0, 3)]
    assert got == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_splitmix64_offsets_are_one_sequence():
    a = O.splitmix64(12345, 0, 20)
    b = np.concatenate([O.splitmix64(12345, 0, 7), O.splitmix64(12345, 7, 13)])
    assert np.array_equal(a, b)


def _literal_lfg_words(seed, stream_id, count):
    """Brute force: the whole sequence x_0, x_1, ... as a Python list (no ring)."""
    x = [int(w) for w in O.splitmix64(seed, 607 * stream_id, 607)]
    if not any(w & 1 for w in x):
        x[0] |= 1
    n_total = 607 * 11 + count
    while len(x) < n_total:
        n = len(x)
        x.append((x[n - 607] + x[n - 273]) & MASK)
    return x[607 * 11:]


def _round_lfg_words(seed, stream_id, count):
    """Round-based update (three dependency phases 273/273/61) on whole 607-word tables."""
    old = O.splitmix64(seed, 607 * stream_id, 607).astype(np.uint64)
    if not (old & np.uint64(1)).any():
        old[0] |= np.uint64(1)
    out = []
    with np.errstate(over="ignore"):
        for _ in range(11 + (count + 606) // 607):
            new = np.empty_like(old)
            new[0:273] = old[0:273] + old[334:607]
            new[273:546] = old[273:546] + new[0:273]
            new[546:607] = old[546:607] + new[273:334]
            old = new
            out.append(new)
    seq = np.concatenate(out)
    # the first 10 rounds are the warm-up
    return [int(w) for w in seq[607 * 10: 607 * 10 + count]]


@pytest.mark.parametrize("seed,stream", [(1, 0), (1, 1), (7, 12345), (0, 0), (2**64 - 1, 3)])
def test_lfg_matches_literal_recurrence_and_round_update(seed, stream):
    count = 3 * 607 + 11
    st = O.Streams(seed, 1, first_stream=stream)
    got = [int(w) for w in st.words(count)]
    assert got == _literal_lfg_words(seed, stream, count)
    assert got == _round_lfg_words(seed, stream, count)
    assert int(st.counts[0]) == count


def test_ring_holds_last_607_words():
    st = O.Streams(5, 1)
    w = st.words(1000)
    ring = st.rings[0]
    lit = _literal_lfg_words(5, 0, 1000)
    # x_n sits at ring[n mod 607]; uniform #i is x_{6677+i} and 6677 = 11 * 607
    for i in range(1000 - 607, 1000):
        assert int(ring[i % 607]) == lit[i] == int(w[i])


@pytest.mark.parametrize("word,expect", [(0, 0.0), (0x7FF, 0.0), (0x800, 2.0**-53), (1 << 63, 0.5),
                                         (MASK, 1.0 - 2.0**-53), ((1 << 64) - 2048, 1.0 - 2.0**-53)])
def test_word_to_uniform_edges(word, expect):
    # u = (x >> 11) 2^-53: 0 possible, 1 impossible
    assert O.word_to_uniform(word) == expect


def test_fill_partition_invariance():
    # S:56 / S:69: fill(3) then fill(5) == fill(8) from the same state
    a = O.Streams(9, 1)
    b = O.Streams(9, 1)
    x = np.concatenate([a.uniform(3), a.uniform(5)])
    y = b.uniform(8)
    assert np.array_equal(x, y)
    assert np.array_equal(a.rings, b.rings) and np.array_equal(a.counts, b.counts)


def test_stream_major_quota_layout():
    S, n = 5, 23  # q = 4, rem = 3 -> streams 0..2 get 5 uniforms, 3..4 get 4
    st = O.Streams(3, S)
    u = st.uniform(n)
    assert list(st.counts) == [5, 5, 5, 4, 4]
    for k in range(S):
        one = O.Streams(3, 1, first_stream=k)
        cnt = 5 if k < 3 else 4
        off = k * 4 + min(k, 3)
        assert np.array_equal(u[off:off + cnt], one.uniform(cnt))


def test_zero_fill_is_noop():
    st = O.Streams(3, 4)
    r0 = st.rings
    assert st.uniform(0).size == 0
    assert np.array_equal(st.rings, r0) and not st.counts.any()


def test_streams_differ_and_seeds_differ():
    a = O.Streams(1, 2).uniform(2000)
    b = O.Streams(2, 2).uniform(2000)
    assert np.mean(a != b) > 0.99
    s0, s1 = a[:1000], a[1000:]
    assert np.mean(s0 != s1) > 0.99


def test_uniform_statistics_1e6():
    n = 10**6
    u = O.Streams(2024, 16).uniform(n)
    assert u.min() >= 0.0 and u.max() < 1.0
    # mean 0.5 +- 4 sqrt(1/12/n)
    assert abs(u.mean() - 0.5) < 4 * math.sqrt(1 / 12 / n)
    # KS against U[0,1) at alpha = 0.01: D_crit ~ 1.628/sqrt(n)
    us = np.sort(u)
    i = np.arange(1, n + 1)
    d = max(np.max(i / n - us), np.max(us - (i - 1) / n))
    assert d < 1.628 / math.sqrt(n)


def test_serial_correlation_single_stream():
    # lag-1..100 serial correlation of 10^6 draws bounded by 4/sqrt(10^6)
    n = 10**6
    u = O.Streams(77, 1).uniform(n) - 0.5
    var = np.dot(u, u) / n
    worst = max(abs(np.dot(u[:-L], u[L:]) / (n - L) / var) for L in range(1, 101))
    # 100 lags at 4 SE: family-wise false-alarm ~100 * 6e-5
    assert worst < 4 / math.sqrt(n)


def test_shard_ranges_concatenate():
    # reading R5/R6 (Q6): streams [0, 8) == [0, 4) ++ [4, 8) when the per-stream quota is equal
    full = O.Streams(11, 8).normal_boxmuller(8 * 6)
    lo = O.Streams(11, 4, first_stream=0).normal_boxmuller(4 * 6)
    hi = O.Streams(11, 4, first_stream=4).normal_boxmuller(4 * 6)
    assert np.array_equal(full, np.concatenate([lo, hi]))
