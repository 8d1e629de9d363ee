"""GPU parity for every dispatch path of nrng.cu, against the CPU oracle.

Each case names the kernel instantiation the dispatcher picks for its shape (DESIGN.md §6:
one-block-per-SM kernels at >= 16 x 148 streams, 4-warp blocks below; misaligned outputs on
bm_kernel / polar_kernel; the sequential mode's epoch layout; host outputs through the
staging buffers, in per-stream pieces when a stream's slots exceed a staging buffer), so
that no shipped kernel goes untested.  Bars as in test_gpu_parity.py: outputs element by
element within 1e-13 (B2's sincos16 and B3's bulk branch are bit-exact given identical
coefficients), per-stream consumption and the written-back generator state bit-exact.

The edge-word cases craft the generator state (nrng_set_state, and the same state in the
oracle) so that the next 273 words of every stream are chosen boundary uniforms: the bulk
kernels' U = 4 compacted transforms (b3_pairs_compact, p2_transform_compact, the Polar
ranking) then see u = 0, 1 - 2^-53, sqrt(8/9) neighbours, s = 0, s = 1, s near 8/9 ...
(P:78-81 exact 0; P:114 s >= 1 reject; P:282-285 B3's tau; P:375-378 P2's tau).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
import paper_1004_3105_b200 as P  # noqa: E402
from paper_1004_3105_b200 import workloads as W  # noqa: E402

TOL = 1e-13
SMS = 148


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1004_3105_b200 import build as B

    B.build()
    yield
    torch.cuda.synchronize()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def ora(st, method, n, mu, sigma):
    if method == "U":
        return st.uniform(n)
    if method == "P":
        return st.normal_polar(n, mu, sigma)
    if method == "P2":
        return st.normal_polar2(n, mu, sigma)
    if method in ("R", "R1"):
        return st.normal_ratio(n, mu, sigma)  # R1 returns R's output (reading R29)
    return st.normal_boxmuller(n, mu, sigma, P.METHODS[method])


def gen(g, method, n, mu, sigma, out=None):
    if method == "U":
        return g.uniform(n, out=out)
    return g.normal(method, n, mu, sigma, out=out)


def assert_state_equal(g, st):
    ring, cnt = g.get_state()
    assert np.array_equal(cnt, st.counts)
    assert np.array_equal(ring, st.rings)


def check(d, o, method, what=""):
    assert d.shape == o.shape, what
    if method in ("U", "R", "R1"):
        assert np.array_equal(d, o), what  # uniforms bit-exact; R's IEEE x bit-exact (R27 margin checked)
    else:
        err = float(np.max(np.abs(d - o))) if d.size else 0.0
        assert err <= TOL, (what, err)


# ---------------------------------------------------------------- few-stream host outputs
# slots per stream > 2^24 (one staging buffer): one stream per chunk, in pieces (ADVICE r1:
# the clamp to one stream per chunk used to overrun the staging buffer here)

@pytest.mark.parametrize("S", [1, 3, 8])
@pytest.mark.parametrize("method", ["U", "B1", "B2", "B3", "P", "P2", "R", "R1"])
def test_host_output_few_streams(S, method):
    n = (1 << 25) + 3
    if method in ("R", "R1") and S == 8:
        n = (1 << 27) + 5  # one normal per unit: 2^24 slots per stream need a longer call
    g, st = P.Generator(5, S, first_stream=9), O.Streams(5, S, first_stream=9)
    h = np.full(n, np.nan)
    gen(g, method, n, 0.5, 2.0, out=h)
    o = ora(st, method, n, 0.5, 2.0)
    if method in ("R", "R1"):
        assert st.ratio_margin > 1e-12
    check(h, o, method, (S, method))
    assert_state_equal(g, st)
    # and a pinned host buffer, continuing the same streams
    pin = torch.empty(n, dtype=torch.float64).pin_memory()
    gen(g, method, n, 0.5, 2.0, out=pin)
    check(pin.numpy(), ora(st, method, n, 0.5, 2.0), method, (S, method, "pinned"))
    assert_state_equal(g, st)


@pytest.mark.parametrize("method", ["R", "B1", "P"])
def test_device_output_long_quota_pieces(method):
    # a per-stream quota above 2^28 units runs as consecutive pieces (32-bit per-launch
    # counters in every kernel; ADVICE r1 for R/R1): equal to a sequence of shorter calls
    # (per-stream partition invariance), which the oracle-checked paths produce
    per = 1 if method == "R" else 2
    n = per * ((1 << 28) + 777) + 1
    free = torch.cuda.mem_get_info()[0]
    if free < 2 * n * 8 + (4 << 30):
        pytest.skip("not enough device memory")
    a, b = P.Generator(3, 1), P.Generator(3, 1)
    x = a.normal(method, n)
    parts, left = [], n
    while left > 0:
        m = min(left, per * (1 << 27))
        parts.append(b.normal(method, m))
        left -= m
    y = torch.cat(parts)
    torch.cuda.synchronize()
    assert torch.equal(x, y)
    assert np.array_equal(a.stream_counts(), b.stream_counts())
    del x, y, parts


def test_sequential_mode_long_run_pieces():
    # a device-output sequential call over few streams and many epochs: 3 x 2^30 + 768
    # deviates from one stream are 1.5 x 2^30 + 384 B3 pairs, 4.8e9 words -- past the kernels'
    # 32-bit per-launch word counts (round 2 found the sequential mode bypassing the pieces
    # of run_bulk: this call failed) -- so it runs as launches of at most 2^28 pairs per
    # stream; equal to a sequence of shorter calls (the canonical sequence is partition
    # invariant), which the oracle-checked sequential tests pin.  One stream = one warp: ~40 s
    method = "B3"
    n = 3 * (1 << 30) + 768
    free = torch.cuda.mem_get_info()[0]
    if free < 2 * n * 8 + (4 << 30):
        pytest.skip("not enough device memory")
    a, b = P.Generator(5, 1), P.Generator(5, 1)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    a.normal_seq(method, out=x)
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    step = 1 << 30
    for s in range(0, n, step):
        b.normal_seq(method, out=y[s:min(n, s + step)])
    torch.cuda.synchronize()
    assert torch.equal(x, y)
    assert np.array_equal(a.stream_counts(), b.stream_counts())
    del x, y


# ---------------------------------------------------------------- 4-warp-block bulk kernels
# fewer streams than 16 x 148 one-block-per-SM slots, > 128 units per stream (above mid_kernel)

@pytest.mark.parametrize("method,S,pairs", [
    ("B1", 1024, 300),   # pw_kernel<1,4>
    ("B2", 1024, 300),   # pw_kernel<2,4>
    ("B3", 1024, 300),   # b3_kernel<4>
    ("P", 2048, 4096),   # pw_kernel<4,4>
    ("P", 37, 1000),     # pw_kernel<4,4>, a partial block
    ("P2", 1024, 300),   # polar_kernel<4,2>
])
def test_few_stream_bulk_kernels(method, S, pairs):
    g, st = P.Generator(13, S, first_stream=100), O.Streams(13, S, first_stream=100)
    for n in (2 * S * pairs + 2 * (S // 3) + 1, 2 * S * 200 + 2 * 5, 2 * S * pairs):
        d = host(g.normal(method, n, -1.25, 0.75))
        o = ora(st, method, n, -1.25, 0.75)
        check(d, o, method, (method, S, n))
        assert_state_equal(g, st)


# ---------------------------------------------------------------- misaligned device outputs
# 8-byte aligned only: bm_kernel<V,20> / polar_kernel<20,M> at >= 20 x 148 streams,
# bm_kernel<V,4> / polar_kernel<4,M> below

@pytest.mark.parametrize("S", [4160, 1024])
@pytest.mark.parametrize("method", ["B1", "B2", "B3", "P", "P2"])
def test_misaligned_wide(S, method):
    g, st = P.Generator(19, S, first_stream=3), O.Streams(19, S, first_stream=3)
    for pairs, extra in ((150, 2 * 99 + 1), (260, 0)):
        n = 2 * S * pairs + extra
        buf = torch.empty(n + 1, dtype=torch.float64, device="cuda")
        view = buf[1:]
        g.normal(method, out=view, mu=0.25, sigma=1.5)
        check(host(view), ora(st, method, n, 0.25, 1.5), method, (S, method, n))
    assert_state_equal(g, st)


# ---------------------------------------------------------------- sequential mode, P2 wide
def test_sequential_p2_wide_epoch_kernel():
    # >= 16 x 148 streams: whole P2 epochs on the pair-window kernel pw_kernel<5,16,true>
    # (polar_kernel<20,2,true> only in a -DNRNG_P2_PW=0 build)
    S, E = 3000, 128
    ep = 2 * S * E
    total = 2 * ep + 999
    a = P.Generator(31, S)
    one = host(a.normal_seq("P2", total, -0.5, 1.5))
    st = O.Streams(31, S)
    o = np.concatenate([st.normal_polar2(ep, -0.5, 1.5) for _ in range(3)])[:total]
    check(one, o, "P2")


# ---------------------------------------------------------------- edge words through the bulk kernels
def _edge_values(method):
    e = list(W.edge_uniforms())
    if method in ("P", "P2", "R", "R1"):
        r = np.sqrt(8.0 / 9.0)
        k = np.floor((1.0 + r) / 2.0 * 2.0 ** 53)  # x = 2a - 1 ~ sqrt(8/9), y = 0: s ~ 8/9 (P2's tau)
        e += [(k + d) * 2.0 ** -53 for d in (-2, -1, 0, 1, 2)]
        e += [0.5 + 2.0 ** -53 * d for d in (-3, 3)]
    return np.array(e)


def _crafted(seed, S, first, method):
    """Generator + oracle with the same state, crafted so that the next 273 words of every
    stream are boundary uniforms (combinations of the edge list, shifted per stream)."""
    g, st = P.Generator(seed, S, first_stream=first), O.Streams(seed, S, first_stream=first)
    ring, cnt = g.get_state()
    vals = _edge_values(method)
    per = 3 if method == "B3" else 2
    if per == 2:
        combos = np.array([[a, b] for a in vals for b in vals])
    else:
        combos = np.array([[a, b, c] for a in vals for b in vals for c in vals[:6]])
    rng = np.random.default_rng(seed)
    flat = combos.ravel()
    nper = 273 // per * per
    for k in range(S):
        start = (k * nper) % flat.size
        u = np.resize(np.roll(flat, -start), 273)
        u[nper:] = rng.integers(0, 1 << 53, 273 - nper) * 2.0 ** -53
        words = (np.round(u * 2.0 ** 53).astype(np.uint64) << np.uint64(11)) | \
            rng.integers(0, 1 << 11, 273).astype(np.uint64)  # low 11 bits must not matter
        base = int(cnt[k]) % 607
        j = np.arange(273)
        ring[k, (base + j) % 607] = words - ring[k, (base + j + 334) % 607]  # x_{C+j} = words[j]
    g.set_state(ring, cnt)
    s = st.st
    s["ring"] = ring
    s["count"] = cnt
    assert_state_equal(g, st)
    return g, st


@pytest.mark.parametrize("method", ["U", "B1", "B2", "B3", "P", "P2", "R", "R1"])
def test_edge_words_through_bulk_kernels(method):
    # S = 2400 >= 16 x 148: pw_kernel<M,16> / b3_kernel<16> (U = 4 compacted transforms)
    S = 2400
    g, st = _crafted(41, S, 7, method)
    per = 1 if method in ("U", "R", "R1") else 2
    n = per * S * 300 + 1
    d = host(gen(g, method, n, 2.5, 0.5))
    o = ora(st, method, n, 2.5, 0.5)
    if method in ("R", "R1"):
        assert st.ratio_margin > 1e-12
    check(d, o, method, method)
    assert_state_equal(g, st)
    if method in ("B1", "B2", "B3", "P", "P2"):
        # the crafted specials really reached the outputs: s = 0 (P/P2) and u = 0 (B1/B2) give (mu, mu)
        if method != "B3":
            e = d[:-1]
            assert np.any((e[0::2] == 2.5) & (e[1::2] == 2.5))


@pytest.mark.parametrize("aligned", [True, False])
def test_edge_words_few_stream_kernels(aligned):
    # the same through the 4-warp-block kernels (S < 2368: pw_kernel<M,4>, b3_kernel<4>,
    # polar_kernel<4,2>) and the misaligned paths (bm_kernel<V,4>, polar_kernel<4,M>)
    S = 600
    for method in ("B1", "B2", "B3", "P", "P2"):
        g, st = _crafted(43, S, 0, method)
        n = 2 * S * 300
        buf = torch.empty(n + 1, dtype=torch.float64, device="cuda")
        view = buf[:n] if aligned else buf[1:]
        g.normal(method, out=view, mu=-1.0, sigma=3.0)
        check(host(view), ora(st, method, n, -1.0, 3.0), method, (method, aligned))
        assert_state_equal(g, st)


# ---------------------------------------------------------------- independent handles
def test_two_handles_on_two_streams_concurrently():
    # distinct handles share no state (include/nrng.h "Concurrency"): two generators enqueued
    # alternately on two CUDA streams, their kernels free to overlap, give exactly what each
    # gives alone; consecutive calls and a Polar call included
    S, n = 4096, 2 * 4096 * 300
    ref = {}
    for seed in (3, 4):
        g = P.Generator(seed, S)
        ref[seed] = [host(g.normal(m, n)) for m in ("B1", "P", "B3")]
        g.close()
    ga, gb = P.Generator(3, S), P.Generator(4, S)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    outs = {3: [], 4: []}
    for m in ("B1", "P", "B3"):
        with torch.cuda.stream(sa):
            outs[3].append(ga.normal(m, n))
        with torch.cuda.stream(sb):
            outs[4].append(gb.normal(m, n))
    torch.cuda.synchronize()
    for seed in (3, 4):
        for got, want in zip(outs[seed], ref[seed]):
            assert np.array_equal(got.cpu().numpy(), want)
