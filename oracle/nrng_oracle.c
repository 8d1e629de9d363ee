/*
 * nrng_oracle.c -- plain, slow, obviously-correct CPU oracle for the hot path of
 * R. P. Brent, "Fast Normal Random Number Generators for Vector Processors"
 * (ANU TR-CS-93-04, 1993) = /root/reference/PAPER.md ("P:n" = line n).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_1004_3105_b200/);
 * its B2/B3 coefficients come from its own fitter (oracle/fit_coeffs.py).
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 * (-ffp-contract=off: no multiply-add is fused unless written as fma() below).
 * Parallelism: OpenMP over streams only; every stream is plain sequential code.
 *
 * What it computes (readings R1..R20 are listed in DESIGN.md §3):
 *   uniform source  additive lagged Fibonacci x_n = x_{n-607} + x_{n-273} mod 2^64
 *                   (the paper's RANU4 "generalised Fibonacci" generator, P:176-181,
 *                   lags unstated -> SPEC S:74 lags), table seeded by splitmix64,
 *                   10*607 warm-up outputs discarded, u = (x >> 11) * 2^-53 in [0,1)
 *                   ("may return exactly 0 but never exactly 1").
 *   B1  P:67-74   r = sigma sqrt(-2 ln(1-u)), x = r sin(theta)+mu, y = r cos(theta)+mu,
 *                 theta = 2 pi v - pi in [-pi, pi) (reading R6).
 *   B2  P:159-170 as B1 with sin/cos from the two polynomials + 4 angle doublings.
 *   B3  P:280-295 m = max(u1,u2), u = m^2, tail u > 8/9 -> library ln/sqrt,
 *                 else v = (6u-4)/(4-3u), r = sigma m h(v); return mu + c r sqrt2,
 *                 mu + s r sqrt2.
 *   P   P:108-119 x,y in [-1,1), s = x^2+y^2, reject s >= 1,
 *                 r = sigma sqrt(-2 ln(s)/s), return r x + mu, r y + mu.
 *   P2  P:367-385 as P, but s > 8/9 -> r = sigma sqrt(-ln(1-s)/s), else r = sigma h(v(s));
 *                 return x r sqrt2 + mu, y r sqrt2 + mu.
 *   R   P:421-427 (the ratio method, Algorithm R): x = sqrt(8/e)(v - 1/2)/(1 - u), reject
 *                 if x^2 > -4 ln(1-u) (the printed "-x^2 ln(1-u) > 4" is an erratum,
 *                 reading R25), return sigma x + mu -- ONE normal per accepted candidate.
 *   R1  P:452-468 R with step 2.5 (pretests P1/P2 before the logarithm, reading R29).
 * Work partition (stream-major, exact-stop; R5/R18): P = ceil(n/2) pairs,
 * stream k yields p_k = q + [k < rem] pairs at out[off_k + 2j], off_k = 2(kq+min(k,rem)).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "oracle_coeffs.h"

#define ORC_R 607 /* long lag */
#define ORC_S 273 /* short lag */
#define ORC_WARM_ROUNDS 10 /* discard 10*607 outputs (reading R3) */

/* Per-stream state: x_n is held at ring[n mod 607] for the 607 most recent n.
 * count = uniforms already delivered; the next uniform is x_{N0 + count} where
 * N0 = 607 + 10*607 = 6677 (first output after the warm-up). */
typedef struct {
    uint64_t ring[ORC_R];
    uint64_t count;
} orc_stream;

#define ORC_N0 ((uint64_t)ORC_R * (1 + ORC_WARM_ROUNDS))

int orc_sizeof_stream(void) { return (int)sizeof(orc_stream); }

void orc_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---------------------------------------------------------------- splitmix64 ---
 * Reading R2: the Weyl state advances by gamma = 0x9E3779B97F4A7C15; output #i
 * (0-based) of the sequence seeded with `seed` is mix(seed + (i+1)*gamma). */
static uint64_t splitmix64_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

void orc_splitmix64(uint64_t seed, uint64_t first, uint64_t n, uint64_t* out) {
    for (uint64_t i = 0; i < n; ++i)
        out[i] = splitmix64_mix(seed + (first + i + 1) * 0x9E3779B97F4A7C15ULL);
}

/* ------------------------------------------------------------- LFG stream ----- */

/* x_n = x_{n-607} + x_{n-273} (mod 2^64).  `n` is the absolute index. */
static uint64_t lfg_next_word(orc_stream* st, uint64_t n) {
    uint64_t x = st->ring[n % ORC_R] + st->ring[(n - ORC_S) % ORC_R];
    st->ring[n % ORC_R] = x;
    return x;
}

/* Table of global stream k: x_j = splitmix64 output #(607k + j), j = 0..606 (R2);
 * if every word is even, set bit 0 of x_0 (R4); then discard 10*607 outputs (R3). */
void orc_stream_init(orc_stream* st, uint64_t seed, uint64_t stream_id) {
    orc_splitmix64(seed, (uint64_t)ORC_R * stream_id, ORC_R, st->ring);
    uint64_t any_odd = 0;
    for (int j = 0; j < ORC_R; ++j) any_odd |= st->ring[j] & 1u;
    if (!any_odd) st->ring[0] |= 1u;
    for (uint64_t n = ORC_R; n < ORC_N0; ++n) lfg_next_word(st, n);
    st->count = 0;
}

void orc_streams_init(orc_stream* st, uint64_t seed, uint64_t first_stream, uint32_t S) {
#pragma omp parallel for schedule(static)
    for (long k = 0; k < (long)S; ++k) orc_stream_init(&st[k], seed, first_stream + (uint64_t)k);
}

/* u = (x >> 11) * 2^-53: exact, in [0, 1), 0 possible, 1 impossible. */
double orc_word_to_uniform(uint64_t x) { return (double)(x >> 11) * 0x1p-53; }

static uint64_t next_word(orc_stream* st) {
    uint64_t x = lfg_next_word(st, ORC_N0 + st->count);
    st->count += 1;
    return x;
}

static double next_uniform(orc_stream* st) { return orc_word_to_uniform(next_word(st)); }

/* ------------------------------------------------------ work partition (R5) --- */
static void quota(uint64_t units, uint32_t S, uint32_t k, uint64_t* cnt, uint64_t* off) {
    uint64_t q = units / S, rem = units % S;
    *cnt = q + (k < rem ? 1 : 0);
    *off = (uint64_t)k * q + (k < rem ? k : rem);
}

/* Raw 64-bit words, 1 per slot, stream-major (test hook for the LFG itself). */
void orc_words(orc_stream* st, uint32_t S, uint64_t* out, uint64_t n) {
#pragma omp parallel for schedule(static)
    for (long k = 0; k < (long)S; ++k) {
        uint64_t cnt, off;
        quota(n, S, (uint32_t)k, &cnt, &off);
        for (uint64_t j = 0; j < cnt; ++j) out[off + j] = next_word(&st[k]);
    }
}

/* Uniforms, 1 per slot, stream-major. */
void orc_uniform(orc_stream* st, uint32_t S, double* out, uint64_t n) {
#pragma omp parallel for schedule(static)
    for (long k = 0; k < (long)S; ++k) {
        uint64_t cnt, off;
        quota(n, S, (uint32_t)k, &cnt, &off);
        for (uint64_t j = 0; j < cnt; ++j) out[off + j] = next_uniform(&st[k]);
    }
}

/* --------------------------------------------------- fast functions (B2/B3) --- */

/* sincos16: y = (2 pi v - pi)/16, |y| <= pi/16; s = s1 y + s3 y^3 + s5 y^5 +
 * s7 y^7, c = c0 + c2 y^2 + c4 y^4 + c6 y^6; then four times sin2y = 2 sin y cos y,
 * cos2y = 1 - 2 sin^2 y.  Rounding (readings R7, R9): t = 2v-1 (exact),
 * y = RN(t * RN(pi)/16), y2 = RN(y*y), s = RN(y * Horner_fma(y2)), c = Horner_fma(y2),
 * doubling: s' = RN((s+s)*c), c' = fma(-(s+s), s, 1). */
void orc_sincos16(double v, double* sout, double* cout) {
    const double pi16 = M_PI / 16.0; /* RN(pi)/16, exact scaling */
    double t = 2.0 * v - 1.0;
    double y = t * pi16;
    double y2 = y * y;
    double ps = fma(fma(fma(ORC_SIN[3], y2, ORC_SIN[2]), y2, ORC_SIN[1]), y2, ORC_SIN[0]);
    double s = y * ps;
    double c = fma(fma(fma(ORC_COS[3], y2, ORC_COS[2]), y2, ORC_COS[1]), y2, ORC_COS[0]);
    for (int i = 0; i < 4; ++i) {
        double s2 = s + s;
        double sn = s2 * c;
        double cn = fma(-s2, s, 1.0);
        s = sn;
        c = cn;
    }
    *sout = s;
    *cout = c;
}

/* h(v) = h0 + h1 v + ... + h15 v^15, Horner with fma. */
double orc_eval_h(double v) {
    double acc = ORC_H[15];
    for (int j = 14; j >= 0; --j) acc = fma(acc, v, ORC_H[j]);
    return acc;
}

/* Moebius map with rho = 1: v = (6u-4)/(4-3u), reading R15:
 * v = RN(fma(6,u,-4) / fma(-3,u,4)). */
double orc_mobius(double u) { return fma(6.0, u, -4.0) / fma(-3.0, u, 4.0); }

/* ------------------------------------------------------ pair transforms ------- */

/* B1, P:67-74 on one (u, v): exact arithmetic except log/sqrt/sin/cos. */
static void b1_pair(double u, double v, double mu, double sigma, double* x, double* y) {
    double L = log(1.0 - u);              /* 1-u is exact for u a multiple of 2^-53 */
    double r = sigma * sqrt(-2.0 * L);
    double t = 2.0 * v - 1.0;             /* theta = pi t = 2 pi v - pi (R6) */
    double th = M_PI * t;
    *x = fma(r, sin(th), mu);
    *y = fma(r, cos(th), mu);
}

/* B2: B1 with sin/cos replaced by sincos16. */
static void b2_pair(double u, double v, double mu, double sigma, double* x, double* y) {
    double L = log(1.0 - u);
    double r = sigma * sqrt(-2.0 * L);
    double s, c;
    orc_sincos16(v, &s, &c);
    *x = fma(r, s, mu);
    *y = fma(r, c, mu);
}

/* B3, steps 1-5 in order. */
static const double ORC_TAU = 8.0 / 9.0;                   /* RN(8/9) */
static const double ORC_SQRT2 = 0x1.6a09e667f3bcdp+0;      /* RN(sqrt 2) */
static void b3_pair(double u1, double u2, double u3, double mu, double sigma, double* x, double* y) {
    double m = u1 > u2 ? u1 : u2;                          /* step 2 */
    double u = m * m;
    double r;
    if (u > ORC_TAU) {                                     /* step 3.1, reading R14 */
        double w = fma(-m, m, 1.0);
        r = sigma * sqrt(-log(w));
    } else {                                               /* step 3.2 */
        double v = orc_mobius(u);
        double hv = orc_eval_h(v);
        r = sigma * (m * hv);
    }
    double s, c;
    orc_sincos16(u3, &s, &c);                              /* step 4 */
    double A = r * ORC_SQRT2;                              /* step 5, reading R11 */
    *x = fma(c, A, mu);
    *y = fma(s, A, mu);
}

/* Polar acceptance test: s = RN(RN(x*x) + RN(y*y)), accept iff s < 1. */
static int polar_candidate(double a, double b, double* x, double* y, double* s) {
    *x = 2.0 * a - 1.0;
    *y = 2.0 * b - 1.0;
    double xx = *x * *x, yy = *y * *y;
    *s = xx + yy;
    return *s < 1.0;
}

/* Polar step 4; s == 0 -> (mu, mu) (reading R12). */
static void polar_transform(double x, double y, double s, double mu, double sigma, double* ox, double* oy) {
    if (s == 0.0) {
        *ox = mu;
        *oy = mu;
        return;
    }
    double q = (-2.0 * log(s)) / s;
    double r = sigma * sqrt(q);
    *ox = fma(r, x, mu);
    *oy = fma(r, y, mu);
}

/* Method P2, P:367-385 (step 4a: r = sigma sqrt(-2 ln(u)/s) with u = 1 - s):
 * 4.1 s > 8/9: r = sigma sqrt(-ln(1-s)/s) (library ln/sqrt; 1-s exact by Sterbenz);
 * 4.2 else: v = (6s-4)/(4-3s) (reading R15's rounding), r = sigma h(v);
 * 5.  return x r sqrt2 + mu, y r sqrt2 + mu, A = RN(r sqrt2) (reading R22).
 * s == 0 needs no special case: v = -1, h(-1) ~ 1 and x = y = 0 give (mu, mu). */
static void p2_transform(double x, double y, double s, double mu, double sigma, double* ox, double* oy) {
    double r;
    if (s > ORC_TAU) {
        double w = 1.0 - s;
        double q = -log(w) / s;
        r = sigma * sqrt(q);
    } else {
        double v = orc_mobius(s);
        r = sigma * orc_eval_h(v);
    }
    double A = r * ORC_SQRT2;
    *ox = fma(x, A, mu);
    *oy = fma(y, A, mu);
}

/* Exported single-pair transforms for closed-form pins (no stream involved). */
void orc_b1_pair(double u, double v, double mu, double sigma, double* xy) { b1_pair(u, v, mu, sigma, &xy[0], &xy[1]); }
void orc_b2_pair(double u, double v, double mu, double sigma, double* xy) { b2_pair(u, v, mu, sigma, &xy[0], &xy[1]); }
void orc_b3_pair(double u1, double u2, double u3, double mu, double sigma, double* xy) {
    b3_pair(u1, u2, u3, mu, sigma, &xy[0], &xy[1]);
}
int orc_polar2_pair(double a, double b, double mu, double sigma, double* xy, double* xys) {
    int acc = polar_candidate(a, b, &xys[0], &xys[1], &xys[2]);
    if (acc) p2_transform(xys[0], xys[1], xys[2], mu, sigma, &xy[0], &xy[1]);
    return acc;
}
/* returns accept; xy = outputs when accepted; xys = (x, y, s) */
int orc_polar_pair(double a, double b, double mu, double sigma, double* xy, double* xys) {
    int acc = polar_candidate(a, b, &xys[0], &xys[1], &xys[2]);
    if (acc) polar_transform(xys[0], xys[1], xys[2], mu, sigma, &xy[0], &xy[1]);
    return acc;
}

/* ------------------------------------------------- bulk, stream-major --------- */
enum { ORC_B1 = 1, ORC_B2 = 2, ORC_B3 = 3 };

static void put_pair(double* out, uint64_t n, uint64_t idx, double x, double y) {
    if (idx < n) out[idx] = x;
    if (idx + 1 < n) out[idx + 1] = y; /* odd n: the very last deviate is dropped (R18) */
}

int orc_normal_boxmuller(orc_stream* st, uint32_t S, double* out, uint64_t n, double mu, double sigma,
                         int variant) {
    if (variant < 1 || variant > 3) return -1;
    uint64_t P = (n + 1) / 2;
#pragma omp parallel for schedule(static)
    for (long k = 0; k < (long)S; ++k) {
        uint64_t cnt, off;
        quota(P, S, (uint32_t)k, &cnt, &off);
        for (uint64_t j = 0; j < cnt; ++j) {
            double x, y;
            if (variant == ORC_B3) {
                double u1 = next_uniform(&st[k]);
                double u2 = next_uniform(&st[k]);
                double u3 = next_uniform(&st[k]);
                b3_pair(u1, u2, u3, mu, sigma, &x, &y);
            } else {
                double u = next_uniform(&st[k]);
                double v = next_uniform(&st[k]);
                if (variant == ORC_B1)
                    b1_pair(u, v, mu, sigma, &x, &y);
                else
                    b2_pair(u, v, mu, sigma, &x, &y);
            }
            put_pair(out, n, 2 * (off + j), x, y);
        }
    }
    return 0;
}

/* Algorithm P with exact stop (reading R5): stream k draws candidates until p_k are
 * accepted; rejected candidates are consumed, nothing after the last accepted one. */
int orc_normal_polar(orc_stream* st, uint32_t S, double* out, uint64_t n, double mu, double sigma) {
    uint64_t P = (n + 1) / 2;
#pragma omp parallel for schedule(static)
    for (long k = 0; k < (long)S; ++k) {
        uint64_t cnt, off;
        quota(P, S, (uint32_t)k, &cnt, &off);
        uint64_t j = 0;
        while (j < cnt) {
            double a = next_uniform(&st[k]);
            double b = next_uniform(&st[k]);
            double x, y, s;
            if (!polar_candidate(a, b, &x, &y, &s)) continue; /* step 3: reject */
            double ox, oy;
            polar_transform(x, y, s, mu, sigma, &ox, &oy);
            put_pair(out, n, 2 * (off + j), ox, oy);
            ++j;
        }
    }
    return 0;
}

/* Method P2 with the same candidate stream, acceptance and exact stop as Algorithm P. */
int orc_normal_polar2(orc_stream* st, uint32_t S, double* out, uint64_t n, double mu, double sigma) {
    uint64_t P = (n + 1) / 2;
#pragma omp parallel for schedule(static)
    for (long k = 0; k < (long)S; ++k) {
        uint64_t cnt, off;
        quota(P, S, (uint32_t)k, &cnt, &off);
        uint64_t j = 0;
        while (j < cnt) {
            double a = next_uniform(&st[k]);
            double b = next_uniform(&st[k]);
            double x, y, s;
            if (!polar_candidate(a, b, &x, &y, &s)) continue;
            double ox, oy;
            p2_transform(x, y, s, mu, sigma, &ox, &oy);
            put_pair(out, n, 2 * (off + j), ox, oy);
            ++j;
        }
    }
    return 0;
}

/* Algorithm R, readings R24-R27: C8E = RN(sqrt(8/e));
 * x = RN(RN(C8E (v - 1/2)) / (1 - u)) (v - 1/2 and 1 - u exact, left to right as written);
 * step 3 with the erratum read as the Kinderman-Monahan test (R25): with a = RN(x x) and
 * b = -4 log(1 - u) (the factor 4 is exact), reject iff a > b; output fma(sigma, x, mu).
 * As printed, "-x^2 ln(1-u) > 4", the test accepts 76% of the candidates instead of the
 * sqrt(pi e)/4 = 73.1% that the paper's own 8/sqrt(pi e) = 2.74 uniforms per normal
 * implies, and its output is not normal (tests/test_oracle_ratio.py).  `ab` receives (a, b). */
static const double ORC_C8E = 0x1.b72cd3f331398p+0; /* RN(sqrt(8/e)) = 1.7155277699214136 */
static int ratio_candidate(double u, double v, double* x, double* ab) {
    *x = (ORC_C8E * (v - 0.5)) / (1.0 - u);
    ab[0] = *x * *x;
    ab[1] = -4.0 * log(1.0 - u);
    return !(ab[0] > ab[1]);
}
/* xab = (x, a, b) */
int orc_ratio_candidate(double u, double v, double* xab) { return ratio_candidate(u, v, &xab[0], &xab[1]); }

/* Algorithm R with exact stop (reading R5 with normals as the unit, R26): stream k draws
 * candidates until its quota of n/S (+1 for k < n mod S) normals is accepted, one normal
 * per accepted candidate at out[off_k + j].  *margin (if given) receives the smallest
 * |a - b| / b over every candidate drawn with b > 0 (b = 0 means u = 0, where ln is
 * exactly 0 everywhere): how close the closest accept decision came to depending on the
 * last bits of the logarithm, which the GPU parity tests check (reading R27). */
int orc_normal_ratio(orc_stream* st, uint32_t S, double* out, uint64_t n, double mu, double sigma, double* margin) {
    double mg = INFINITY;
#pragma omp parallel for schedule(static) reduction(min : mg)
    for (long k = 0; k < (long)S; ++k) {
        uint64_t cnt, off;
        quota(n, S, (uint32_t)k, &cnt, &off);
        uint64_t j = 0;
        while (j < cnt) {
            double u = next_uniform(&st[k]);
            double v = next_uniform(&st[k]);
            double x, ab[2];
            int acc = ratio_candidate(u, v, &x, ab);
            if (ab[1] > 0.0) {
                double d = fabs(ab[0] - ab[1]) / ab[1];
                if (d < mg) mg = d;
            }
            if (!acc) continue; /* step 3: reject */
            out[off + j] = fma(sigma, x, mu);
            ++j;
        }
    }
    if (margin) *margin = mg;
    return 0;
}

/* Algorithm R1 = Algorithm R with step 2.5: if P1(u, v), go to step 4 (accept
 * without a logarithm); else if P2(u, v), reject; else step 3.  The paper only says P1 and
 * P2 are "easily-computed conditions" whose regions R1 (inside C) and R2 (enclosing C) have
 * almost the same area, citing Kinderman-Monahan and Leva.  Reading R29: the two
 * tangent-line bounds of the logarithm, with U = 1 - u and a = x^2 as in step 3:
 *   ln is concave, so ln U <= ln c + (U - c)/c; at c = e^{-1/4}:  -4 ln U >= 5 - 4 e^{1/4} U;
 *   ln y <= y - 1 at y = c'/U gives -ln U <= c'/U - 1 - ln c'; at c' = e^{-1.35}:
 *                                                                -4 ln U <= 4 e^{-1.35}/U + 1.4.
 * P1: a <= 5 - 4 e^{1/4} U - d;  P2: a >= (4 e^{-1.35} / U)(1 + d) + 1.4 + d,  d = 2^-40.
 * The margin d (absolute, and relative on the 1/U term) exceeds every rounding error in
 * these expressions and in step 3's a and b = -4 log U (|b| <= 4 ln 2^53 < 148) by orders
 * of magnitude, so step 2.5 never decides differently from step 3: R1 returns exactly R's
 * output, and only the number of logarithms changes.
 * Returns 1 (P1: accept), 2 (P2: reject) or 0 (borderline: step 3 decides); x and a as in R. */
static const double ORC_R1_D = 0x1p-40;
static int ratio1_pretest(double u, double v, double* x, double* a) {
    *x = (ORC_C8E * (v - 0.5)) / (1.0 - u);
    *a = *x * *x;
    const double U = 1.0 - u;
    if (*a <= 5.0 - 4.0 * exp(0.25) * U - ORC_R1_D) return 1;
    if (*a >= (4.0 * exp(-1.35) / U) * (1.0 + ORC_R1_D) + 1.4 + ORC_R1_D) return 2;
    return 0;
}
/* xa = (x, a) */
int orc_ratio1_pretest(double u, double v, double* xa) { return ratio1_pretest(u, v, &xa[0], &xa[1]); }

/* Algorithm R1 with exact stop, the same partition as orc_normal_ratio; *logs (if given)
 * receives the number of logarithms evaluated (step 3 runs only for borderline candidates),
 * *cands the number of candidates drawn. */
int orc_normal_ratio1(orc_stream* st, uint32_t S, double* out, uint64_t n, double mu, double sigma, uint64_t* logs,
                      uint64_t* cands) {
    uint64_t nl = 0, nc = 0;
#pragma omp parallel for schedule(static) reduction(+ : nl, nc)
    for (long k = 0; k < (long)S; ++k) {
        uint64_t cnt, off;
        quota(n, S, (uint32_t)k, &cnt, &off);
        uint64_t j = 0;
        while (j < cnt) {
            double u = next_uniform(&st[k]);
            double v = next_uniform(&st[k]);
            double x, a;
            ++nc;
            int cls = ratio1_pretest(u, v, &x, &a); /* step 2.5 */
            if (cls == 2) continue;                  /* P2: reject */
            if (cls == 0) {                          /* step 3 */
                ++nl;
                if (a > -4.0 * log(1.0 - u)) continue;
            }
            out[off + j] = fma(sigma, x, mu); /* step 4 */
            ++j;
        }
    }
    if (logs) *logs = nl;
    if (cands) *cands = nc;
    return 0;
}

/* Accept mask of exactly `cand` candidates per stream (2 uniforms each), stream-major. */
void orc_polar_mask(orc_stream* st, uint32_t S, uint8_t* mask, uint64_t cand) {
#pragma omp parallel for schedule(static)
    for (long k = 0; k < (long)S; ++k) {
        for (uint64_t j = 0; j < cand; ++j) {
            double a = next_uniform(&st[k]);
            double b = next_uniform(&st[k]);
            double x, y, s;
            mask[(uint64_t)k * cand + j] = (uint8_t)polar_candidate(a, b, &x, &y, &s);
        }
    }
}

/* Transforms on caller-given uniforms: B1/B2/P/P2/R/R1 use 2 per pair, B3 3 per pair.
 * method: 1,2,3 = B1,B2,B3; 4 = P, 5 = P2 (rejected candidates give NaN, NaN and mask 0);
 * 6 = R: out[2j] = sigma x + mu (NaN if rejected), out[2j+1] = x (always);
 * 7 = R1: as 6, and mask = accept | (step-2.5 class << 1). */
int orc_transform_from_uniforms(const double* u, uint64_t n_pairs, double* out, uint8_t* mask, double mu,
                                double sigma, int method) {
    if (method < 1 || method > 7) return -1;
#pragma omp parallel for schedule(static)
    for (long j = 0; j < (long)n_pairs; ++j) {
        double x = NAN, y = NAN;
        if (method == 1) b1_pair(u[2 * j], u[2 * j + 1], mu, sigma, &x, &y);
        else if (method == 2) b2_pair(u[2 * j], u[2 * j + 1], mu, sigma, &x, &y);
        else if (method == 3) b3_pair(u[3 * j], u[3 * j + 1], u[3 * j + 2], mu, sigma, &x, &y);
        else if (method == 6) {
            double ab[2];
            int acc = ratio_candidate(u[2 * j], u[2 * j + 1], &y, ab);
            if (mask) mask[j] = (uint8_t)acc;
            if (acc) x = fma(sigma, y, mu);
        }
        else if (method == 7) {
            double a;
            int cls = ratio1_pretest(u[2 * j], u[2 * j + 1], &y, &a);
            int acc = cls == 1 || (cls == 0 && !(a > -4.0 * log(1.0 - u[2 * j])));
            if (mask) mask[j] = (uint8_t)(acc | (cls << 1));
            if (acc) x = fma(sigma, y, mu);
        } else {
            double cx, cy, s;
            int acc = polar_candidate(u[2 * j], u[2 * j + 1], &cx, &cy, &s);
            if (mask) mask[j] = (uint8_t)acc;
            if (acc) {
                if (method == 4) polar_transform(cx, cy, s, mu, sigma, &x, &y);
                else p2_transform(cx, cy, s, mu, sigma, &x, &y);
            }
        }
        out[2 * j] = x;
        out[2 * j + 1] = y;
    }
    return 0;
}

/* --------------------------------------------------- validation statistics ---- */
/* Sums of x^k (k=1..4) about `center`, min, max and a histogram over caller-given
 * ascending edges (K-1 interior edges -> K bins), in long double.  Used to pin the
 * GPU stats reduction. */
void orc_stats(const double* x, uint64_t n, double center, const double* edges, int K, double* sums /*6*/,
               int64_t* hist /*K*/) {
    long double s1 = 0, s2 = 0, s3 = 0, s4 = 0;
    double mn = INFINITY, mx = -INFINITY;
    for (int b = 0; b < K; ++b) hist[b] = 0;
    for (uint64_t i = 0; i < n; ++i) {
        long double d = (long double)x[i] - center;
        s1 += d;
        s2 += d * d;
        s3 += d * d * d;
        s4 += d * d * d * d;
        if (x[i] < mn) mn = x[i];
        if (x[i] > mx) mx = x[i];
        int b = 0; /* bin b holds edges[b-1] <= x < edges[b] */
        while (b < K - 1 && x[i] >= edges[b]) ++b;
        hist[b] += 1;
    }
    sums[0] = (double)s1;
    sums[1] = (double)s2;
    sums[2] = (double)s3;
    sums[3] = (double)s4;
    sums[4] = mn;
    sums[5] = mx;
}
