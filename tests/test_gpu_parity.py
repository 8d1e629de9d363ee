"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bars (BASELINE.json north_star): uniforms, Polar accept masks, output order, per-stream
consumption counters and the generator state bit-exact; B1/P normals within 1e-13
absolute.  North star allows B2/B3 1e-13 + the paper's 1e-10 bound (reading
R17), but both sides evaluate the same approximations with identical coefficients and
operation order (B2's sincos16 and B3's bulk branch are bit-exact; only ln in B2's radius
and B3's tail differs by ulps), so B2/B3/P2 are held to the same 1e-13: a regression in
the coefficients or the doubling at the 1e-11 level fails.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
import paper_1004_3105_b200 as P  # noqa: E402
from paper_1004_3105_b200 import workloads as W  # noqa: E402

TOL = 1e-13
TOL_APPROX = 1e-13  # B2/B3/P2: same bar as B1/P (see the module docstring)


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


def gen_normals(g, method, n, mu, sigma):
    return host(g.normal(method, n, mu, sigma))


def ora_normals(st, method, n, mu, sigma):
    if method == "R":
        return st.normal_ratio(n, mu, sigma)
    if method == "P":
        return st.normal_polar(n, mu, sigma)
    if method == "P2":
        return st.normal_polar2(n, mu, sigma)
    return st.normal_boxmuller(n, mu, sigma, P.METHODS[method])


def tol_for(method):
    return TOL if method in ("B1", "P") else TOL_APPROX


def test_c2_polar2_full():
    # method P2 on config 2's shape: same candidates as P
    c = W.C2
    g, st = P.Generator(c.seed, c.streams), O.Streams(c.seed, c.streams)
    d = gen_normals(g, "P2", c.n, 2.5, 0.5)
    o = ora_normals(st, "P2", c.n, 2.5, 0.5)
    assert np.max(np.abs(d - o)) <= TOL_APPROX
    assert_state_equal(g, st)


def test_p2_shard_all_streams():
    # method P2 at the bench shape (2^31 normals over 2^16 streams): every output and counter
    c = W.C5_SHARD
    g = P.Generator(c.seed, c.streams)
    out = torch.empty(c.n, dtype=torch.float64, device="cuda")
    g.normal("P2", out=out)
    per_stream = c.n // c.streams
    check_stream_blocks(out, c.seed, 0, per_stream, "P2", 0.0, 1.0, g.stream_counts(),
                        [(k, 8192) for k in range(0, c.streams, 8192)])
    del out


def assert_state_equal(g, st):
    ring, cnt = g.get_state()
    assert np.array_equal(cnt, st.counts)
    assert np.array_equal(ring, st.rings)


# ---------------------------------------------------------------- uniforms / state

@pytest.mark.parametrize("cfg", W.ALL, ids=lambda c: c.name)
def test_seeded_state_bit_exact(cfg):
    g = P.Generator(cfg.seed, cfg.streams)
    st = O.Streams(cfg.seed, cfg.streams)
    assert_state_equal(g, st)


@pytest.mark.parametrize("seed,S,n", [(1, 1024, 1024 * 1500 + 77), (7, 1 << 14, (1 << 14) * 70 + 5),
                                      (42, 1 << 16, (1 << 16) * 3 + 1), (3, 37, 37 * 2000 + 36)])
def test_uniforms_bit_exact(seed, S, n):
    g = P.Generator(seed, S)
    st = O.Streams(seed, S)
    for m in (n, 3, n // 3):  # several calls: ragged tails, < S, and window reuse
        assert np.array_equal(host(g.uniform(m)), st.uniform(m))
    assert_state_equal(g, st)


def test_polar_mask_bit_exact():
    S = 1 << 14
    g = P.Generator(7, S)
    st = O.Streams(7, S)
    for cand in (651, 1, 333):
        assert np.array_equal(host(g.polar_mask(cand)), st.polar_mask(cand))
    assert_state_equal(g, st)


# ---------------------------------------------------------------- configs, full size

def test_c1_b1_full():
    c = W.C1
    g, st = P.Generator(c.seed, c.streams), O.Streams(c.seed, c.streams)
    for _ in range(2):
        d = gen_normals(g, "B1", c.n, c.mu, c.sigma)
        o = ora_normals(st, "B1", c.n, c.mu, c.sigma)
        assert np.max(np.abs(d - o)) <= TOL
    assert_state_equal(g, st)


def test_c2_polar_full():
    c = W.C2
    g, st = P.Generator(c.seed, c.streams), O.Streams(c.seed, c.streams)
    d = gen_normals(g, "P", c.n, c.mu, c.sigma)
    o = ora_normals(st, "P", c.n, c.mu, c.sigma)
    assert np.max(np.abs(d - o)) <= TOL  # element-wise => stream-major, accepted-pair order exact
    assert_state_equal(g, st)  # exact stop: consumed uniforms per stream bit-exact


def check_stream_blocks(d, seed, first, per_stream, method, mu, sigma, counts, blocks):
    """Streams [k, k + B) of a full-size call against the oracle run on exactly those streams
    (the oracle's stream ids are global: first + k), element by element, with their counters."""
    for k, B in blocks:
        st = O.Streams(seed, B, first_stream=first + k)
        o = ora_normals(st, method, B * per_stream, mu, sigma)
        dk = host(d[k * per_stream:(k + B) * per_stream])
        assert np.max(np.abs(dk - o)) <= tol_for(method), (method, k, B)
        assert np.array_equal(counts[k:k + B], st.counts), (method, k, B)


def sample_blocks(S, B, n_random, seed):
    # the first and last B streams, B around the middle, and n_random single streams
    rng = np.random.default_rng(seed)
    ks = sorted(set(int(k) for k in rng.integers(B, S - 2 * B, n_random)))
    return [(0, B), (S // 2 - B // 2, B), (S - B, B)] + [(k, 1) for k in ks]


@pytest.mark.parametrize("method", ["B2", "B3"])
def test_c3_full_size_all_streams(method):
    # 2^28 normals over 2^16 streams: all of them, every element and counter (2 GB per side)
    c = W.C3
    g = P.Generator(c.seed, c.streams)
    d = g.normal(method, c.n, c.mu, c.sigma)
    per_stream = c.n // c.streams
    check_stream_blocks(d, c.seed, 0, per_stream, method, c.mu, c.sigma, g.stream_counts(),
                        [(0, c.streams)])


@pytest.mark.parametrize("method", ["B1", "B2", "B3", "P"])
def test_c5_shard_bench_launch_all_streams(method):
    # the exact launch bench.py times: 2^31 normals over 2^16 streams (global ids of rank 1);
    # all of them, every element and counter, in blocks of 8192 streams (2 GB of host memory
    # per side at a time)
    c = W.C5_SHARD
    first = c.streams  # rank 1 of the sharded run
    g = P.Generator(c.seed, c.streams, first_stream=first)
    out = torch.empty(c.n, dtype=torch.float64, device="cuda")
    g.normal(method, out=out)
    per_stream = c.n // c.streams
    check_stream_blocks(out, c.seed, first, per_stream, method, c.mu, c.sigma, g.stream_counts(),
                        [(k, 8192) for k in range(0, c.streams, 8192)])
    del out


def test_short_calls_partial_state_load():
    # per-stream quotas of 5..100 pairs: warp kernel reading only the state words it needs
    S = 512
    for m in ("B1", "B2", "B3"):
        g, st = P.Generator(31, S), O.Streams(31, S)
        for pairs in (5, 17, 100, 3, 140):
            d = gen_normals(g, m, 2 * S * pairs, 0.0, 1.0)
            o = ora_normals(st, m, 2 * S * pairs, 0.0, 1.0)
            assert np.max(np.abs(d - o)) <= tol_for(m)
        assert_state_equal(g, st)


def test_c4_sweep_sequence():
    c = W.C4
    g, st = P.Generator(c.seed, c.streams), O.Streams(c.seed, c.streams)
    for L in W.C4_LENGTHS:
        for method in ("B1", "P", "B1"):
            d = gen_normals(g, method, L, c.mu, c.sigma)
            o = ora_normals(st, method, L, c.mu, c.sigma)
            assert np.max(np.abs(d - o)) <= TOL, (L, method)
    assert_state_equal(g, st)


# ---------------------------------------------------------------- transforms on given uniforms

@pytest.mark.parametrize("method", [1, 2, 3, 4, 5])
def test_transform_from_uniforms(method):
    per = 3 if method == 3 else 2
    u = W.dyadic_uniforms(100 + method, per * 300001)
    e = W.edge_uniforms()
    grid = np.array([[a, b] for a in e for b in e]).ravel() if per == 2 else \
        np.array([[a, b, c] for a in e for b in e for c in e[:5]]).ravel()
    u = np.concatenate([grid, u])
    mu, sigma = 2.5, 0.5
    d_out, d_mask = P.transform_from_uniforms(torch.from_numpy(u).cuda(), method, mu, sigma)
    o_out, o_mask = O.transform_from_uniforms(u, method, mu, sigma)
    d_out = host(d_out)
    if method >= 4:
        assert np.array_equal(host(d_mask), o_mask)
        acc = np.repeat(o_mask.astype(bool), 2)
        assert np.all(np.isnan(d_out[~acc]))
        d_out, o_out = d_out[acc], o_out[acc]
    assert np.max(np.abs(d_out - o_out)) <= (TOL if method in (1, 4) else TOL_APPROX)
    if method == 3:
        # the bulk branch (u <= 8/9) has no library call: bit-exact
        m = np.maximum(u[0::3], u[1::3])
        bulk = np.repeat(m * m <= 8 / 9, 2)
        assert np.array_equal(d_out[bulk], o_out[bulk])
    if method == 5:
        # P2's bulk branch (s <= 8/9): bit-exact
        x, y = 2 * u[0::2] - 1, 2 * u[1::2] - 1
        s = x * x + y * y
        acc = s < 1
        bulk = np.repeat(s[acc] <= 8 / 9, 2)
        assert np.array_equal(d_out[bulk], o_out[bulk])


# ---------------------------------------------------------------- Algorithm R (the ratio method)

def _ratio_margin(u, v):
    # |a - b| / b of reading R27, recomputed from the definition (b = 0 at u = 0 is exact)
    x = (float.fromhex("0x1.b72cd3f331398p+0") * (v - 0.5)) / (1.0 - u)
    b = -4.0 * np.log(1.0 - u)
    with np.errstate(divide="ignore", invalid="ignore"):
        return np.where(b > 0, np.abs(x * x - b) / np.where(b > 0, b, 1.0), np.inf)


def test_ratio_transform_from_uniforms():
    u = W.dyadic_uniforms(106, 2 * 400001)
    e = W.edge_uniforms()
    u = np.concatenate([np.array([[a, b] for a in e for b in e]).ravel(), u])
    mu, sigma = -0.75, 1.5
    d_out, d_mask = P.transform_from_uniforms(torch.from_numpy(u).cuda(), 6, mu, sigma)
    o_out, o_mask = O.transform_from_uniforms(u, 6, mu, sigma)
    d_out, d_mask = host(d_out), host(d_mask)
    # x = RN(RN(C (v - 1/2)) / (1 - u)) uses IEEE operations only: bit-exact everywhere
    assert np.array_equal(d_out[1::2], o_out[1::2])
    # the accept decision depends on ln (free to 1 ulp, R27): equal wherever it cannot flip
    safe = _ratio_margin(u[0::2], u[1::2]) > 1e-12
    assert safe.mean() > 0.99999
    assert np.array_equal(d_mask[safe], o_mask[safe])
    acc = o_mask.astype(bool) & safe
    assert np.array_equal(d_out[0::2][acc], o_out[0::2][acc])
    assert np.all(np.isnan(d_out[0::2][~d_mask.astype(bool)]))


@pytest.mark.parametrize("S,ns", [(64, [1, 3, 2 * 64 + 1, 64 * 33 + 5, 64 * 700 + 17]),
                                  (1000, [1000 * 130 + 999, 7]),
                                  (4160, [4160 * 40 + 2345, 4160 * 3 + 7, 4160 * 129])])
def test_ratio_bulk_parity(S, ns):
    # tiny quotas (thread per stream), 4-warp and one-block-per-SM pair-window kernels, with
    # remainders and consecutive calls; every stream against the oracle, state bit-exact
    g, st = P.Generator(21, S, first_stream=5), O.Streams(21, S, first_stream=5)
    for n in ns:
        d = gen_normals(g, "R", n, -1.0, 2.0)
        o = ora_normals(st, "R", n, -1.0, 2.0)
        assert st.ratio_margin > 1e-12  # no decision of this run could depend on ln's last bits
        assert d.size == n and np.array_equal(d, o), (S, n)
    assert_state_equal(g, st)


def check_ratio_blocks(out, seed, per, counts, blocks):
    # R / R1 outputs of blocks of streams, bit for bit against the oracle's Algorithm R; the
    # oracle's smallest decision margin over the block must exceed 1e-12 (reading R27)
    for k, B in blocks:
        st = O.Streams(seed, B, first_stream=k)
        o = st.normal_ratio(B * per)
        assert st.ratio_margin > 1e-12, (k, B, st.ratio_margin)
        assert np.array_equal(host(out[k * per:(k + B) * per]), o), (k, B)
        assert np.array_equal(counts[k:k + B], st.counts), (k, B)


def test_ratio_bench_shape_all_streams_and_host_output():
    # bench shape (2^31 normals over 2^16 streams): every output and counter, in blocks of 8192 streams
    c = W.C5_SHARD
    g = P.Generator(c.seed, c.streams)
    out = torch.empty(c.n, dtype=torch.float64, device="cuda")
    g.normal("R", out=out)
    check_ratio_blocks(out, c.seed, c.n // c.streams, g.stream_counts(), [(k, 8192) for k in range(0, c.streams, 8192)])
    del out
    # host output (chunked staging, one normal per unit)
    g1, g2 = P.Generator(3, 2048), P.Generator(3, 2048)
    h = np.empty((1 << 22) + 5)
    g1.normal("R", out=h, mu=0.5, sigma=3.0)
    assert np.array_equal(h, gen_normals(g2, "R", h.size, 0.5, 3.0))


# ---------------------------------------------------------------- Algorithm R1 (R + step 2.5)

def test_ratio1_transform_from_uniforms():
    u = W.dyadic_uniforms(107, 2 * 400001)
    e = W.edge_uniforms()
    u = np.concatenate([np.array([[a, b] for a in e for b in e]).ravel(), u])
    mu, sigma = 0.25, 2.0
    d_out, d_mask = P.transform_from_uniforms(torch.from_numpy(u).cuda(), 7, mu, sigma)
    o_out, o_mask = O.transform_from_uniforms(u, 7, mu, sigma)
    r_out, r_mask = O.transform_from_uniforms(u, 6, mu, sigma)
    d_out, d_mask = host(d_out), host(d_mask)
    # step 2.5 classes: P1 / P2 / borderline, as the oracle classifies them; each pretest
    # agrees with step 3 (R's oracle decision), and all three classes occur
    assert np.array_equal(d_mask >> 1, o_mask >> 1)
    cls, acc_r = d_mask >> 1, r_mask.astype(bool)
    assert np.all(acc_r[cls == 1]) and not np.any(acc_r[cls == 2])
    assert 0.12 < (cls == 0).mean() < 0.22 and (cls == 1).mean() > 0.6
    # x bit-exact; decisions and outputs equal R's wherever ln's last bits cannot matter (R27)
    assert np.array_equal(d_out[1::2], r_out[1::2])
    safe = _ratio_margin(u[0::2], u[1::2]) > 1e-12
    assert np.array_equal((d_mask & 1)[safe], r_mask[safe])
    acc = acc_r & safe
    assert np.array_equal(d_out[0::2][acc], r_out[0::2][acc])
    assert np.all(np.isnan(d_out[0::2][~(d_mask & 1).astype(bool)]))


@pytest.mark.parametrize("S,ns", [(64, [1, 3, 2 * 64 + 1, 64 * 33 + 5, 64 * 700 + 17]),
                                  (1000, [1000 * 130 + 999, 7]),
                                  (4160, [4160 * 40 + 2345, 4160 * 3 + 7, 4160 * 129])])
def test_ratio1_bulk_parity(S, ns):
    # R1 returns exactly Algorithm R's output (reading R29): against the oracle's R and R1,
    # tiny, 4-warp and one-block-per-SM kernels, consecutive calls, state bit-exact
    g, st, st1 = P.Generator(21, S, first_stream=5), O.Streams(21, S, first_stream=5), O.Streams(21, S, first_stream=5)
    for n in ns:
        d = gen_normals(g, "R1", n, -1.0, 2.0)
        o = ora_normals(st, "R", n, -1.0, 2.0)
        assert st.ratio_margin > 1e-12
        assert d.size == n and np.array_equal(d, o), (S, n)
        assert np.array_equal(st1.normal_ratio1(n, -1.0, 2.0), o)
    assert_state_equal(g, st)


def test_ratio1_bench_shape_all_streams():
    c = W.C5_SHARD
    g = P.Generator(c.seed, c.streams)
    out = torch.empty(c.n, dtype=torch.float64, device="cuda")
    g.normal("R1", out=out)
    check_ratio_blocks(out, c.seed, c.n // c.streams, g.stream_counts(), [(k, 8192) for k in range(0, c.streams, 8192)])
    del out


# ---------------------------------------------------------------- serial correlation gate

def test_serial_corr_kernel_matches_numpy():
    from paper_1004_3105_b200 import gof as G

    rng = np.random.default_rng(3)
    for n, K in [(1_000_003, 100), (4096 * 3 + 17, 127), (50, 100), (1, 5)]:
        x = rng.standard_normal(n) * 2 + 1
        d = P.serial_corr(torch.from_numpy(x).cuda(), 1.0, K)
        dx = x - 1.0
        ref = np.array([np.dot(dx[: max(0, n - k)], dx[k:]) if k < n else 0.0 for k in range(K + 1)])
        assert np.allclose(d, ref, rtol=1e-12, atol=1e-9 * max(1.0, abs(ref[0])))


@pytest.mark.parametrize("what", ["uniform", "B1", "B3", "P", "R"])
def test_serial_corr_gate_on_generated_streams(what):
    from paper_1004_3105_b200 import gof as G

    g = P.Generator(77, 1 << 14)
    n = 1 << 26
    x = g.uniform(n) if what == "uniform" else g.normal(what, n)
    r = G.serial_corr_gate(P.serial_corr(x, 0.5 if what == "uniform" else 0.0, 100), n)
    assert r["serial_pass"], r


# ---------------------------------------------------------------- edge cases of the API

def test_zero_n_is_noop_and_sigma_zero():
    g = P.Generator(9, 64)
    r0, c0 = g.get_state()
    for m in ("B1", "B2", "B3", "P"):
        assert g.normal(m, 0).numel() == 0
    r1, c1 = g.get_state()
    assert np.array_equal(r0, r1) and np.array_equal(c0, c1)
    for m in ("B1", "B2", "B3", "P"):
        x = host(g.normal(m, 1001, -4.5, 0.0))
        assert np.all(x == -4.5)


@pytest.mark.parametrize("n", [1, 2, 3, 63, 64, 65, 127, 129, 2 * 64 * 4 + 1, 2 * 64 * 5 - 1, 2 * 64 * 33 + 1])
@pytest.mark.parametrize("method", ["B1", "B2", "B3", "P", "P2"])
def test_small_and_odd_n(n, method):
    # n <= 2 * 64 * 4: one thread per stream (tiny quotas); larger: warp per stream
    S = 64
    g, st = P.Generator(4, S), O.Streams(4, S)
    for _ in range(2):
        d = gen_normals(g, method, n, 1.0, 2.0)
        o = ora_normals(st, method, n, 1.0, 2.0)
        assert d.size == n and np.max(np.abs(d - o)) <= tol_for(method)
    assert_state_equal(g, st)


@pytest.mark.parametrize("method", ["B1", "B2", "B3", "P", "P2"])
def test_wide_ragged_calls(method):
    # >= 28 x 148 streams: the one-block-per-SM kernels (B3's triple-row kernel included)
    # with ragged per-stream quotas (remainder streams, a partial last row, a dropped odd
    # deviate) over consecutive calls, every stream against the oracle, state bit-exact.
    S = 4160
    g, st = P.Generator(12, S, first_stream=77), O.Streams(12, S, first_stream=77)
    for n in (2 * S * 70 + 2 * 1234 + 1, 2 * S * 37 + 2 * 4000, 2 * S * 64 + 2 * 17 + 1):
        d = gen_normals(g, method, n, -0.25, 1.5)
        o = ora_normals(st, method, n, -0.25, 1.5)
        assert d.size == n and np.max(np.abs(d - o)) <= tol_for(method), (method, n)
    assert_state_equal(g, st)


@pytest.mark.parametrize("method", ["B1", "B2", "B3", "P"])
def test_wide_multi_block_calls_state_continuity(method):
    # The one-block-per-SM kernels with several steady blocks per stream, ending in every
    # window phase (B3: 128-pair iterations, 3 phases of its 12-row window; pw kernels:
    # 128-pair blocks, 4 phases), then a partial row, over consecutive calls: outputs
    # against the oracle and the written-back state bit-exact after every call.
    S = 2400
    g, st = P.Generator(21, S, first_stream=5), O.Streams(21, S, first_stream=5)
    for pairs in (128 * 4 + 17, 128 * 2 + 5, 128 * 3 + 100, 128 * 5 + 31, 128):
        n = 2 * S * pairs + 2 * 7
        d = gen_normals(g, method, n, 0.5, 2.0)
        o = ora_normals(st, method, n, 0.5, 2.0)
        assert d.size == n and np.max(np.abs(d - o)) <= tol_for(method), (method, pairs)
        assert_state_equal(g, st)


@pytest.mark.parametrize("method", ["B1", "B2", "B3", "P", "P2", "R", "R1"])
def test_mid_quota_calls(method):
    # per-stream quotas of 12..128 pairs run one warp per stream straight through the HBM ring
    # (mid_kernel): ragged quotas, odd n, partial last steps, consecutive calls, state bit-exact
    S = 512
    g, st = P.Generator(17, S, first_stream=3), O.Streams(17, S, first_stream=3)
    per = 1 if method in ("R", "R1") else 2  # R's unit is a normal
    for pairs, extra in ((12, 0), (31, 2 * 100 + 1), (33, 2 * 511), (64, 7), (100, 2 * 5), (128, 0), (45, 1)):
        n = per * S * pairs + extra
        d = gen_normals(g, method, n, 0.5, 2.0)
        o = ora_normals(st, "R" if method == "R1" else method, n, 0.5, 2.0)
        assert d.size == n and np.max(np.abs(d - o)) <= tol_for(method), (method, pairs, extra)
    assert_state_equal(g, st)


def test_invalid_arguments():
    g = P.Generator(1, 8)
    out = torch.empty(16, dtype=torch.float64, device="cuda")
    bad = [dict(mu=0.0, sigma=-1.0), dict(mu=float("nan"), sigma=1.0), dict(mu=0.0, sigma=float("inf"))]
    r0, c0 = g.get_state()
    for kw in bad:
        with pytest.raises(P.NrngError) as e:
            P.nrng_normal_boxmuller(g.h, out.data_ptr(), 16, kw["mu"], kw["sigma"], 1)
        assert e.value.code == P.NRNG_EINVAL
        with pytest.raises(P.NrngError):
            P.nrng_normal_polar(g.h, out.data_ptr(), 16, kw["mu"], kw["sigma"])
    with pytest.raises(P.NrngError):
        P.nrng_normal_boxmuller(g.h, out.data_ptr(), 16, 0.0, 1.0, 5)
    with pytest.raises(P.NrngError):
        P.nrng_normal_boxmuller(g.h, None, 16, 0.0, 1.0, 1)
    r1, c1 = g.get_state()
    assert np.array_equal(r0, r1) and np.array_equal(c0, c1)


def test_misaligned_device_output():
    S, n = 32, 2 * 32 * 40
    g, st = P.Generator(8, S), O.Streams(8, S)
    buf = torch.empty(n + 1, dtype=torch.float64, device="cuda")
    view = buf[1:]  # 8-byte aligned only
    for m in ("B1", "P"):
        g.normal(m, out=view)
        o = ora_normals(st, m, n, 0.0, 1.0)
        assert np.max(np.abs(host(view) - o)) <= TOL


@pytest.mark.parametrize("method", ["B1", "B3", "P"])
def test_host_output_path(method):
    # out is host memory: chunked generation into staging buffers + overlapped D2H copies
    c = W.C3
    S, n = c.streams, (1 << 25) + 3
    g, g2 = P.Generator(c.seed, S), P.Generator(c.seed, S)
    h = np.empty(n)
    g.normal(method, out=h, mu=c.mu, sigma=c.sigma)
    pinned = torch.empty(n, dtype=torch.float64).pin_memory()
    d = gen_normals(g2, method, n, c.mu, c.sigma)
    assert np.array_equal(h, d)
    g.normal(method, out=pinned, mu=c.mu, sigma=c.sigma)
    d = gen_normals(g2, method, n, c.mu, c.sigma)
    assert np.array_equal(pinned.numpy(), d)
    assert np.array_equal(g.stream_counts(), g2.stream_counts())


def test_partition_invariance_per_stream():
    S = 256
    for m in ("B1", "B2", "B3", "P"):
        a, b = P.Generator(17, S), P.Generator(17, S)
        one = gen_normals(a, m, 2 * S * 96, 0.0, 1.0).reshape(S, 192)
        parts = [gen_normals(b, m, 2 * S * 32, 0.0, 1.0).reshape(S, 64) for _ in range(3)]
        assert np.array_equal(one, np.concatenate(parts, axis=1))
        assert np.array_equal(a.stream_counts(), b.stream_counts())


def test_fake_shards_concatenate():
    # multi-GPU partition emulated on one GPU: G handles over disjoint ranges
    S, G, per = 1 << 12, 4, 2 * 40
    full = gen_normals(P.Generator(11, S), "P", S * per, 0.0, 1.0)
    parts = [gen_normals(P.Generator(11, S // G, first_stream=r * S // G), "P", S // G * per, 0.0, 1.0)
             for r in range(G)]
    assert np.array_equal(full, np.concatenate(parts))


def test_checkpoint_resume():
    S = 512
    a = P.Generator(23, S)
    a.normal("B1", 2 * S * 50)
    ring, cnt = a.get_state()
    x1 = gen_normals(a, "P", 2 * S * 70, 0.0, 1.0)
    b = P.Generator(99, S)  # other seed, then restored
    b.set_state(ring, cnt)
    x2 = gen_normals(b, "P", 2 * S * 70, 0.0, 1.0)
    assert np.array_equal(x1, x2)


def test_above_2_32_outputs():
    # 64-bit indexing: n = 2^32 + 6 over 2^16 streams; sample the first and last streams
    S, n = 1 << 16, (1 << 32) + 6
    free = torch.cuda.mem_get_info()[0]
    if free < n * 8 + (2 << 30):
        pytest.skip("not enough device memory")
    g = P.Generator(5, S)
    out = g.normal("B1", n)
    pairs = (n + 1) // 2
    q, rem = divmod(pairs, S)
    for k in (0, rem - 1, rem, S - 1):
        cnt = q + (k < rem)
        off = 2 * (k * q + min(k, rem))
        st = O.Streams(5, 1, first_stream=k)
        o = st.normal_boxmuller(2 * cnt)
        m = min(2 * cnt, n - off)
        assert np.max(np.abs(host(out[off:off + m]) - o[:m])) <= TOL
    del out


# ---------------------------------------------------------------- validation reduction

@pytest.mark.parametrize("K", [2, 3, 64, 256, 1024])
def test_stats_histogram_bins_exact(K):
    # bin(v) = #edges <= v, exactly (numpy searchsorted side='right'), for uneven edges, values
    # equal to edges and their neighbours, and values outside the edge range
    rng = np.random.default_rng(K)
    edges = np.sort(np.concatenate([rng.standard_normal(K - 1 - (K - 1) // 3) * 2.0,
                                    np.linspace(-0.5, 0.5, (K - 1) // 3)]))
    x = np.concatenate([rng.standard_normal(300001) * 3.0, edges, np.nextafter(edges, -np.inf),
                        np.nextafter(edges, np.inf), [-1e300, 1e300, edges[0] - 1e-3, edges[-1] + 1e-3]])
    sums, hist = P.stats(torch.from_numpy(x).cuda(), 0.25, edges)
    ref = np.bincount(np.searchsorted(edges, x, side="right"), minlength=K)
    assert np.array_equal(host(hist), ref)
    assert host(sums)[4] == x.min() and host(sums)[5] == x.max()
    xm = x[:300001]  # moments without the +-1e300 extremes
    sums, _ = P.stats(torch.from_numpy(xm).cuda(), 0.25, edges)
    d, s = xm - 0.25, host(sums)
    assert np.allclose(s[:4], [d.sum(), (d ** 2).sum(), (d ** 3).sum(), (d ** 4).sum()], rtol=1e-9, atol=1e-6)


def test_stats_sums_are_compensated():
    # (1e16, 1, -1e16) repeated: every 1 is lost to rounding in a plain fp64 running sum, while
    # the compensated sums (Neumaier) recover sum d = number of ones
    x = np.tile([1e16, 1.0, -1e16], 100003)
    sums, _ = P.stats(torch.from_numpy(x).cuda(), 0.0, [-1.0, 0.0, 1.0])
    assert abs(host(sums)[0] - 100003) < 1e-3


def test_stats_kernel_matches_oracle_stats():
    c = W.C1
    from scipy import stats as sps

    K = 64
    edges = c.mu + c.sigma * sps.norm.ppf(np.arange(1, K) / K)
    g, st = P.Generator(c.seed, c.streams), O.Streams(c.seed, c.streams)
    d = g.normal("B1", c.n, c.mu, c.sigma)
    o = st.normal_boxmuller(c.n, c.mu, c.sigma, 1)
    sums, hist = P.stats(d, c.mu, edges)
    osums, ohist = O.stats(o, c.mu, edges)
    sums, hist = host(sums), host(hist)
    assert np.allclose(sums[:4], osums[:4], rtol=1e-9, atol=1e-9)
    assert abs(sums[4] - osums[4]) <= TOL and abs(sums[5] - osums[5]) <= TOL
    assert np.sum(np.abs(hist - ohist)) <= 2 and hist.sum() == c.n


@pytest.mark.parametrize("method", ["B1", "B2", "B3", "P"])
def test_statistical_gates_at_c3_size(method):
    from scipy import stats as sps

    c = W.C3
    g = P.Generator(c.seed + 1, c.streams)
    x = g.normal(method, c.n, c.mu, c.sigma)
    K = 256
    edges = c.mu + c.sigma * sps.norm.ppf(np.arange(1, K) / K)
    sums, hist = P.stats(x, c.mu, edges)
    sums, hist = host(sums), host(hist)
    n = c.n
    m1 = sums[0] / n / c.sigma
    m2 = sums[1] / n / c.sigma**2
    assert abs(m1) < 4 / math.sqrt(n)
    assert abs(m2 - 1) < 4 * math.sqrt(2 / n)
    chi2 = np.sum((hist - n / K) ** 2 / (n / K))
    assert chi2 < sps.chi2.ppf(0.999, K - 1)


# ---------------------------------------------------------------- sequential (RANN3-style) mode

def _oracle_seq(seed, S, E, method, total, mu, sigma):
    st = O.Streams(seed, S)
    parts, got = [], 0
    while got < total:
        parts.append(ora_normals(st, method, 2 * S * E, mu, sigma))
        got += 2 * S * E
    return np.concatenate(parts)[:total]


@pytest.mark.parametrize("method", ["B1", "B3", "P", "P2"])
def test_sequential_mode_partition_invariant(method):
    S, E = 256, 128
    ep = 2 * S * E
    total = 2 * ep + 12345
    splits = [1, 6, ep - 3, ep + 1000, 0]
    splits[-1] = total - sum(splits)
    a, b = P.Generator(29, S), P.Generator(29, S)
    one = host(a.normal_seq(method, total, 0.5, 2.0))
    parts = [host(b.normal_seq(method, m, 0.5, 2.0)) for m in splits]
    assert np.array_equal(one, np.concatenate(parts))  # any call partition: same sequence
    o = _oracle_seq(29, S, E, method, total, 0.5, 2.0)
    assert np.max(np.abs(one - o)) <= tol_for(method)
    assert P.nrng_seq_buffered(a.h) == 3 * ep - total


@pytest.mark.parametrize("method,E", [("B1", 128), ("B2", 256), ("B3", 128), ("P", 128), ("P", 512), ("P2", 128)])
def test_sequential_mode_wide_epoch_kernels(method, E):
    # >= 16 x 148 streams: whole epochs go through the one-block-per-SM kernels with the
    # epoch-layout store (EP); against the oracle's epoch sequence, and partition-invariant
    S = 2400
    ep = 2 * S * E
    total = 3 * ep + 4321
    a, b = P.Generator(31, S), P.Generator(31, S)
    P.nrng_seq_configure(a.h, E)
    P.nrng_seq_configure(b.h, E)
    one = host(a.normal_seq(method, total, -0.5, 1.5))
    parts = [host(b.normal_seq(method, m, -0.5, 1.5)) for m in (ep + 7, 2 * ep - 7, total - 3 * ep)]
    assert np.array_equal(one, np.concatenate(parts))
    o = _oracle_seq(31, S, E, method, total, -0.5, 1.5)
    assert np.max(np.abs(one - o)) <= tol_for(method)


@pytest.mark.parametrize("method", ["B1", "B2", "B3", "P", "P2"])
def test_sequential_mode_bench_shape_sampled(method):
    # the sequential mode at the bench shape: 2^31 deviates over 2^16 streams in one call, E = 128
    # (128 whole epochs, the EP kernels); the output is epoch-major, so viewed as
    # [epoch][stream][2E] and transposed it is every stream's own sequence, which the oracle
    # gives stream by stream: 3 blocks of 1024 streams and 16 single ones (all 2^16 streams pass
    # too, ~20 s per method: run r2zz2), every element
    c = W.C5_SHARD
    E = 128
    g = P.Generator(c.seed, c.streams)
    out = g.normal_seq(method, c.n)
    per = c.n // c.streams
    by_stream = out.view(per // (2 * E), c.streams, 2 * E).transpose(0, 1)  # [stream][epoch][2E]
    counts = g.stream_counts()
    for k, B in sample_blocks(c.streams, 1024, 16, 13):
        st = O.Streams(c.seed, B, first_stream=k)
        o = ora_normals(st, method, B * per, 0.0, 1.0)
        d = host(by_stream[k:k + B].reshape(-1))
        assert np.max(np.abs(d - o)) <= tol_for(method), (method, k, B)
        assert np.array_equal(counts[k:k + B], st.counts), (method, k, B)
    del out, by_stream


def test_sequential_mode_params_and_host_output():
    S = 128
    g = P.Generator(3, S)
    g.normal_seq("B1", 1001)
    with pytest.raises(P.NrngError):  # other method while B1 deviates are buffered
        g.normal_seq("P", 10)
    P.nrng_seq_reset(g.h)
    g.normal_seq("P", 10)
    a, b = P.Generator(4, S), P.Generator(4, S)
    h = np.empty(3 * 2 * S * 128 + 77)
    a.normal_seq("B2", out=h)
    d = host(b.normal_seq("B2", h.size))
    assert np.array_equal(h, d)


# ---------------------------------------------------------------- goodness-of-fit histogram

def test_gof_hist_matches_numpy():
    from scipy import stats as sps

    x = torch.from_numpy(W.dyadic_uniforms(90, 1 << 20) * 8 - 4).cuda()
    for mu, sigma in ((0.0, 1.0), (0.3, 1.7)):
        h = host(P.gof_hist(x, mu, sigma, 16)).astype(np.int64)
        p = sps.norm.cdf((host(x) - mu) / sigma)
        ref = np.bincount(np.minimum((p * (1 << 16)).astype(np.int64), (1 << 16) - 1), minlength=1 << 16)
        assert h.sum() == x.numel()
        assert np.sum(np.abs(h - ref)) <= 4  # Phi differs by ulps only at bin edges


@pytest.mark.parametrize("method", ["B1", "B2", "B3", "P", "P2"])
def test_ks_ad_gates_at_c3_size(method):
    from paper_1004_3105_b200 import gof

    c = W.C3
    g = P.Generator(c.seed + 7, c.streams)
    x = g.normal(method, c.n, c.mu, c.sigma)
    r = gof.ks_ad(host(P.gof_hist(x, c.mu, c.sigma, 20)))
    assert r["n"] == c.n and r["ks_pass"] and r["ad_pass"], r
