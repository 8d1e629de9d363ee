"""Oracle-side coefficient fitter for methods B2 and B3.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / reference leg may import anything under
``oracle/``.  The CUDA product path has its own, independently written
generator (``paper_1004_3105_b200/tools/gen_coeffs.py``) and shares no code
with this file.

What it computes (§3):

* B2, P:162-166 -- "approximate sin y by a polynomial of the form
  s1 y + s3 y^3 + s5 y^5 + s7 y^7, and cos y by ... c0 + c2 y^2 + c4 y^4 +
  c6 y^6" on |y| <= pi/16 (the P:166 "c^4y^4" is read as c4 y^4, DESIGN.md
  reading R8).
* B3, P:226-259 -- h(v) = g(u), g(u) = sqrt(-ln(1-u)/u), with the Moebius
  change of variable v = (6u-4)/(4-3u) (rho = 1, tau = 8/9), so
  u(v) = 4(1+v) / (3(2+v)); "a polynomial of the form h0 + h1 v + ... +
  h15 v^15 ... with absolute error less than 2e-11 on [-1, 1]".
* How: "close to minimax approximations. These may easily be obtained by
  truncating Chebyshev series".  The Chebyshev series of f on
  [-1, 1] is f(x) = sum' c_k T_k(x) with the defining integral
  c_k = (2/pi) * int_0^pi f(cos t) cos(k t) dt (sum' halves c_0).  This
  file evaluates that integral by quadrature in 50-digit arithmetic,
  truncates at the stated degree, rewrites sum' c_k T_k in the monomial
  basis (exact integer T_k coefficients), and rounds each monomial
  coefficient once to the nearest double.  Nothing here is blocked, fused
  or reordered.

The result is a well-defined set of doubles (the exact truncated series,
correctly rounded), so any independent correct computation reproduces it
bit for bit.  Run ``python -m oracle.fit_coeffs`` to regenerate
``oracle/oracle_coeffs.h`` and ``oracle/oracle_coeffs.json``.
"""
from __future__ import annotations

import json
import os
from fractions import Fraction

import mpmath as mp

DPS = 50
HERE = os.path.dirname(os.path.abspath(__file__))


def chebyshev_T_integer_coeffs(kmax: int) -> list[list[int]]:
    """T_k(x) = sum_j t[k][j] x^j, from T_0=1, T_1=x, T_{k+1} = 2x T_k - T_{k-1}."""
    t = [[1], [0, 1]]
    for k in range(1, kmax):
        nxt = [0] * (k + 2)
        for j, a in enumerate(t[k]):
            nxt[j + 1] += 2 * a
        for j, a in enumerate(t[k - 1]):
            nxt[j] -= a
        t.append(nxt)
    return t[: kmax + 1]


def chebyshev_series_coeff(f, k: int):
    """c_k = (2/pi) int_0^pi f(cos t) cos(k t) dt  (the definition; P:260-263 / [Cle61])."""
    with mp.workdps(DPS):
        integrand = lambda t: f(mp.cos(t)) * mp.cos(k * t)
        # split at multiples of pi/(2k+2) so each piece holds < 1 oscillation
        pieces = 2 * k + 2
        pts = [mp.pi * i / pieces for i in range(pieces + 1)]
        return 2 / mp.pi * mp.quad(integrand, pts)


def truncated_series_monomials(f, degree: int, parity: str | None = None):
    """Monomial coefficients (mpf) of sum'_{k<=degree} c_k T_k(x)."""
    t = chebyshev_T_integer_coeffs(degree)
    ks = range(degree + 1)
    if parity == "odd":
        ks = [k for k in ks if k % 2 == 1]
    elif parity == "even":
        ks = [k for k in ks if k % 2 == 0]
    with mp.workdps(DPS):
        b = [mp.mpf(0)] * (degree + 1)
        for k in ks:
            ck = chebyshev_series_coeff(f, k)
            if k == 0:
                ck = ck / 2
            for j, a in enumerate(t[k]):
                if a:
                    b[j] += ck * a
        return b


def round_to_double(x) -> float:
    """Round an mpf to the nearest double exactly once (via an exact rational)."""
    sign, man, exp, _ = mp.mpf(x)._mpf_
    q = Fraction(man) * (Fraction(2) ** exp)
    return float(-q if sign else q)


# ---- B3: g(u), u(v), h(v) -------------------------------------

def g_exact(u):
    """g(u) = sqrt(-ln(1-u)/u), g(0) = 1."""
    with mp.workdps(DPS):
        u = mp.mpf(u)
        if u == 0:
            return mp.mpf(1)
        return mp.sqrt(-mp.log1p(-u) / u)


def u_of_v(v):
    """Inverse of v = (6u-4)/(4-3u): u = 4(1+v)/(3(2+v))."""
    with mp.workdps(DPS):
        v = mp.mpf(v)
        return 4 * (1 + v) / (3 * (2 + v))


def h_exact(v):
    return g_exact(u_of_v(v))


# ---- B2: sin / cos on |y| <= pi/16 ------------------------------

def fit_sincos():
    with mp.workdps(DPS):
        a = mp.pi / 16
        bs = truncated_series_monomials(lambda x: mp.sin(a * x), 7, "odd")
        bc = truncated_series_monomials(lambda x: mp.cos(a * x), 6, "even")
        s = [bs[j] / a ** j for j in (1, 3, 5, 7)]
        c = [bc[j] / a ** j for j in (0, 2, 4, 6)]
    return [round_to_double(x) for x in s], [round_to_double(x) for x in c]


def fit_h():
    b = truncated_series_monomials(h_exact, 15)
    return [round_to_double(x) for x in b]


def horner_mp(coeffs, x):
    with mp.workdps(DPS):
        acc = mp.mpf(0)
        for cf in reversed(coeffs):
            acc = acc * x + mp.mpf(cf)
        return acc


def certify_h(h, npts=4001):
    """max |sum h_j v^j - h(v)| on an equispaced grid of [-1, 1] (exact arithmetic on the doubles)."""
    worst = mp.mpf(0)
    with mp.workdps(30):
        for i in range(npts):
            v = mp.mpf(-1) + mp.mpf(2) * i / (npts - 1)
            worst = max(worst, abs(horner_mp(h, v) - h_exact(v)))
    return float(worst)


def certify_sincos(s, c, npts=2001):
    """max base error of the two polynomials on |y| <= pi/16 (before doubling)."""
    ws = wc = mp.mpf(0)
    with mp.workdps(30):
        a = mp.pi / 16
        for i in range(npts):
            y = -a + 2 * a * i / (npts - 1)
            y2 = y * y
            ps = y * horner_mp(s, y2)
            pc = horner_mp(c, y2)
            ws = max(ws, abs(ps - mp.sin(y)))
            wc = max(wc, abs(pc - mp.cos(y)))
    return float(ws), float(wc)


def main():
    s, c = fit_sincos()
    h = fit_h()
    herr = certify_h(h)
    serr, cerr = certify_sincos(s, c)
    data = {
        "source": "oracle/fit_coeffs.py: truncated Chebyshev series by quadrature (P:260-263)",
        "sin": [x.hex() for x in s],
        "cos": [x.hex() for x in c],
        "h": [x.hex() for x in h],
        "h_cert_err": herr,
        "sin_base_err": serr,
        "cos_base_err": cerr,
    }
    with open(os.path.join(HERE, "oracle_coeffs.json"), "w") as fh:
        json.dump(data, fh, indent=1)
        fh.write("\n")
    lines = [
        "/* oracle_coeffs.h -- GENERATED by oracle/fit_coeffs.py; do not edit.",
        " * TEST INFRASTRUCTURE: the CPU oracle's own B2/B3 coefficients (PAPER.md P:162-166,",
        " * P:254-263), truncated Chebyshev series rounded once to double. */",
        "#ifndef ORACLE_COEFFS_H",
        "#define ORACLE_COEFFS_H",
        "/* sin y ~ s1 y + s3 y^3 + s5 y^5 + s7 y^7 on |y| <= pi/16 */",
        "static const double ORC_SIN[4] = {" + ", ".join(x.hex() for x in s) + "};",
        "/* cos y ~ c0 + c2 y^2 + c4 y^4 + c6 y^6 */",
        "static const double ORC_COS[4] = {" + ", ".join(x.hex() for x in c) + "};",
        "/* h(v) ~ h0 + h1 v + ... + h15 v^15 on [-1, 1]; certified max error %.3e */" % herr,
        "static const double ORC_H[16] = {",
    ]
    lines += ["    " + x.hex() + "," for x in h]
    lines += ["};", "#endif", ""]
    with open(os.path.join(HERE, "oracle_coeffs.h"), "w") as fh:
        fh.write("\n".join(lines))
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
