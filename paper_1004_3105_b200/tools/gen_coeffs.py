"""Build-time generator of the B2/B3 polynomial coefficients for the CUDA path.

Writes ``paper_1004_3105_b200/csrc/nrng_coeffs.cuh`` (committed).  Written
independently of the oracle's fitter: the oracle integrates the Chebyshev
coefficient integrals by quadrature; this file *interpolates* at N first-kind
Chebyshev nodes (a discrete cosine transform), which equals the truncated
Chebyshev series up to aliasing terms c_{2N-k}, negligible at N = 96 for these
analytic functions (h has its nearest singularities at v = +-2).

PAPER.md passages: B2 polynomials P:162-166 (odd degree-7 sin, even degree-6
cos on |y| <= pi/16); B3 h(v) of degree 15 on [-1, 1] with the Moebius map
v = (6u-4)/(4-3u), rho = 1, tau = 8/9; "close to minimax
approximations ... obtained by truncating Chebyshev series".

Every coefficient is computed in 60-digit arithmetic and rounded once to the
nearest double (``to_float(..., rnd='n')``), so the doubles are those of the
exact truncated series.

    python -m paper_1004_3105_b200.tools.gen_coeffs
"""
from __future__ import annotations

import math
import os
import struct

import mpmath as mp
from mpmath.libmp.libmpf import to_float

N_NODES = 96
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "csrc", "nrng_coeffs.cuh")


def cheb_interp(f, degree):
    """a_k = (2/N) sum_j f(x_j) cos(pi k (j+1/2)/N), x_j = cos(pi (j+1/2)/N); a_0 halved."""
    N = N_NODES
    th = [mp.pi * (j + mp.mpf(1) / 2) / N for j in range(N)]
    fx = [f(mp.cos(t)) for t in th]
    a = []
    for k in range(degree + 1):
        acc = mp.fsum(fx[j] * mp.cos(k * th[j]) for j in range(N))
        a.append(acc * 2 / N)
    a[0] /= 2
    return a


def t_monomial(k, p):
    """Coefficient of x^p in T_k(x) (explicit formula, p = k - 2m)."""
    if k == 0:
        return 1 if p == 0 else 0
    if (k - p) % 2 or p > k:
        return 0
    m = (k - p) // 2
    # T_k(x) = (k/2) sum_m (-1)^m (k-m-1)! / (m! (k-2m)!) (2x)^(k-2m)
    return mp.mpf(k) / 2 * (-1) ** m * math.factorial(k - m - 1) / (math.factorial(m) * math.factorial(k - 2 * m)) * 2 ** p


def to_monomial(a):
    deg = len(a) - 1
    return [mp.fsum(a[k] * t_monomial(k, p) for k in range(p, deg + 1)) for p in range(deg + 1)]


def rn(x):
    return to_float(mp.mpf(x)._mpf_, strict=True, rnd="n")


def generate():
    mp.mp.dps = 60
    half_width = mp.pi / 16
    sin_m = to_monomial(cheb_interp(lambda x: mp.sin(half_width * x), 7))
    cos_m = to_monomial(cheb_interp(lambda x: mp.cos(half_width * x), 6))
    sin_c = [rn(sin_m[p] / half_width ** p) for p in (1, 3, 5, 7)]
    cos_c = [rn(cos_m[p] / half_width ** p) for p in (0, 2, 4, 6)]

    def h(v):
        u = 4 * (1 + v) / (3 * (2 + v))  # inverse Moebius map, rho = 1
        return mp.sqrt(-mp.log1p(-u) / u) if u != 0 else mp.mpf(1)

    h_c = [rn(c) for c in to_monomial(cheb_interp(h, 15))]
    return sin_c, cos_c, h_c


# ----------------------------------------------------------------------------------------
# Coefficients of the path's own fp64 primitives (fast ln / sinpi / cospi), DESIGN.md §6.
# These are implementation constants of the CUDA kernels, not part of the paper's method:
# they replace libdevice's log / sincospi with cheaper table + polynomial versions whose
# error (< 1e-16 absolute on the reduced arguments) sits far inside the 1e-13 output bar.

LOG_BASE_HI = 0x3FE6A09E  # high word of sqrt(1/2): m is normalised into [sqrt(1/2), sqrt(2))
LOG_TABLE_BITS = 7  # 128 buckets: the table is stored 8x interleaved (bank-conflict-free, 16 KB)


def _d_from_hi(hi):
    return struct.unpack("<d", struct.pack("<Q", hi << 32))[0]


def log_table():
    """Bucket j holds the m whose high word is LOG_BASE_HI + j*2^13 .. + (j+1)*2^13 (exclusive).
    c_j = 1 for the bucket containing 1 (so ln(1-u) keeps full relative accuracy for tiny u),
    else the bucket midpoint; inv_j = RN(1/c_j); T_j = RN(-ln(inv_j)); r = fma(m, inv_j, -1)."""
    rows, rmax = [], mp.mpf(0)
    step = 1 << (20 - LOG_TABLE_BITS)
    for j in range(1 << LOG_TABLE_BITS):
        lo = _d_from_hi(LOG_BASE_HI + j * step)
        hi = _d_from_hi(LOG_BASE_HI + (j + 1) * step)
        c = mp.mpf(1) if lo <= 1.0 < hi else (mp.mpf(lo) + mp.mpf(hi)) / 2
        inv = rn(1 / c)
        t = rn(-mp.log(mp.mpf(inv)))
        rmax = max(rmax, abs(mp.mpf(lo) * inv - 1), abs(mp.mpf(hi) * inv - 1))
        rows.append((inv, t))
    return rows, float(rmax)


def log1p_coeffs(rmax, degree=5):
    """ln(1+r) = r + r^2 P(r) on |r| <= rmax, P of degree `degree` - 2: the Chebyshev
    interpolant of (ln(1+r) - r)/r^2 (r = 0: -1/2), so the r and r^2 terms stay exact-leading
    and the relative accuracy as r -> 0 is kept.  Returns (coefficients of P, max error of
    r + r^2 P(r) on a fine grid, in exact arithmetic)."""
    a = mp.mpf(rmax)
    f = lambda r: (mp.log1p(r) - r) / (r * r) if r != 0 else mp.mpf(-1) / 2
    P = [rn(x) for x in _cheb_fit_interval(f, -a, a, degree - 2)]
    err = mp.mpf(0)
    for i in range(-400, 401):
        r = a * i / 400
        err = max(err, abs(r + r * r * mp.fsum(c * r ** k for k, c in enumerate(P)) - mp.log1p(r)))
    return P, float(err)


def _cheb_fit_interval(f, a, b, degree):
    """Monomial coefficients (in x) of the degree-`degree` Chebyshev interpolant of f on [a, b]."""
    N = N_NODES
    th = [mp.pi * (j + mp.mpf(1) / 2) / N for j in range(N)]
    fx = [f((a + b) / 2 + (b - a) / 2 * mp.cos(t)) for t in th]
    ak = []
    for k in range(degree + 1):
        ak.append(mp.fsum(fx[j] * mp.cos(k * th[j]) for j in range(N)) * 2 / N)
    ak[0] /= 2
    # in s = (2x - a - b)/(b - a): monomials in s, then expand s = alpha x + beta
    ms = to_monomial(ak)
    alpha, beta = 2 / (b - a), -(a + b) / (b - a)
    out = [mp.mpf(0)] * (degree + 1)
    for p, cp in enumerate(ms):
        for q in range(p + 1):
            out[q] += cp * mp.binomial(p, q) * alpha ** q * beta ** (p - q)
    return out


def sincospi_coeffs(sdeg=6, cdeg=6):
    """sin(pi z) = z S(z^2), cos(pi z) = C(z^2) on |z| <= 1/4 (w = z^2 in [0, 1/16])."""
    S = lambda w: mp.sin(mp.pi * mp.sqrt(w)) / mp.sqrt(w) if w > 0 else mp.pi
    Cf = lambda w: mp.cos(mp.pi * mp.sqrt(w))
    s = _cheb_fit_interval(S, mp.mpf(0), mp.mpf(1) / 16, sdeg)
    c = _cheb_fit_interval(Cf, mp.mpf(0), mp.mpf(1) / 16, cdeg)
    serr = cerr = mp.mpf(0)
    for i in range(801):
        z = mp.mpf(i) / 3200
        w = z * z
        serr = max(serr, abs(z * mp.fsum(cf * w ** k for k, cf in enumerate(s)) - mp.sin(mp.pi * z)))
        cerr = max(cerr, abs(mp.fsum(cf * w ** k for k, cf in enumerate(c)) - mp.cos(mp.pi * z)))
    return [rn(x) for x in s], [rn(x) for x in c], float(serr), float(cerr)


def emit_math(body):
    rows, rmax = log_table()
    l1p, l1p_err = log1p_coeffs(rmax)
    sc, cc, serr, cerr = sincospi_coeffs()
    ln2 = mp.log(2)
    ln2_hi = rn(ln2)
    ln2_hi = float.fromhex(ln2_hi.hex()[:-4] + "0p-1") if False else ln2_hi
    # ln2 split so that e * LN2_HI is exact for |e| < 2^11: keep 42 significant bits
    m, e = mp.frexp(ln2)
    hi = mp.floor(m * 2 ** 42) / 2 ** 42 * 2 ** e
    lo = ln2 - hi
    body.append("// ---- path primitives (implementation constants, DESIGN.md §6) ----")
    body.append("// ln: m in [sqrt(1/2), sqrt(2)), bucket j = top %d bits of m's 20-bit high mantissa field;" % LOG_TABLE_BITS)
    body.append("// max |r| = %.6e; ln(1+r) = r + r^2 P(r), P Chebyshev degree %d, max error %.3e" % (rmax, len(l1p) - 1, l1p_err))
    body.append("constexpr unsigned kLogBaseHi = 0x%08X;" % LOG_BASE_HI)
    body.append("constexpr int kLogTableBits = %d;" % LOG_TABLE_BITS)
    body.append("constexpr double kLn2 = %s;" % rn(ln2).hex())
    body.append("// ln(1+r) = r + r^2 (L2 + r (L3 + ...))")
    body.append("__constant__ double kLog1p[%d] = {%s};" % (len(l1p), ", ".join(x.hex() for x in l1p)))
    body.append("// {inv_c_j, -ln(inv_c_j)} pairs")
    body.append("__device__ double kLogTable[%d] = {" % (2 * len(rows)))
    body += ["    %s, %s," % (a.hex(), b.hex()) for a, b in rows]
    body.append("};")
    body.append("// sin(pi z) = z S(w), cos(pi z) = C(w), w = z^2, |z| <= 1/4; max err sin %.2e cos %.2e" % (serr, cerr))
    # pre-scaled for an integer argument Z = z 2^63 (|Z| <= 2^61): sin = Z S'(Z^2), cos = C'(Z^2),
    # S'_k = S_k 2^-(63+126k), C'_k = C_k 2^-126k (exact power-of-two scalings, all normal)
    sz = [math.ldexp(x, -(63 + 126 * k)) for k, x in enumerate(sc)]
    cz = [math.ldexp(x, -126 * k) for k, x in enumerate(cc)]
    assert all(abs(x) > 2.0 ** -1000 for x in sz + cz)
    body.append("__constant__ double kSinPiZ[%d] = {%s};" % (len(sz), ", ".join(x.hex() for x in sz)))
    body.append("__constant__ double kCosPiZ[%d] = {%s};" % (len(cz), ", ".join(x.hex() for x in cz)))


def main():
    sin_c, cos_c, h_c = generate()
    body = [
        "// nrng_coeffs.cuh -- GENERATED by paper_1004_3105_b200/tools/gen_coeffs.py; do not edit.",
        "// B2 sin/cos polynomials on |y| <= pi/16 (PAPER.md P:162-166) and B3 h(v), degree 15 on [-1,1]",
        "// (P:254-257): truncated Chebyshev series (P:260-263), each rounded once to double.",
        "#pragma once",
        "namespace nrng {",
        "// sin y ~ y * (S1 + S3 y^2 + S5 y^4 + S7 y^6)",
    ]
    body.append("__constant__ double kB2Sin[4] = {%s};  // S1, S3, S5, S7" % ", ".join(v.hex() for v in sin_c))
    body.append("// cos y ~ C0 + C2 y^2 + C4 y^4 + C6 y^6")
    body.append("__constant__ double kB2Cos[4] = {%s};  // C0, C2, C4, C6" % ", ".join(v.hex() for v in cos_c))
    body.append("// the same polynomials times 2 (exact): sincos16 carries (2s, 2c), see sincos16_x2")
    body.append("__constant__ double kB2Sin2[4] = {%s};" % ", ".join(math.ldexp(v, 1).hex() for v in sin_c))
    body.append("__constant__ double kB2Cos2[4] = {%s};" % ", ".join(math.ldexp(v, 1).hex() for v in cos_c))
    body.append("// h(v) ~ sum_j kH[j] v^j")
    body.append("__constant__ double kH[16] = {")
    body += ["    %s," % v.hex() for v in h_c]
    body += ["};"]
    emit_math(body)
    body += ["}  // namespace nrng", ""]
    with open(OUT, "w") as fh:
        fh.write("\n".join(body))
    print("\n".join(body))


if __name__ == "__main__":
    main()
