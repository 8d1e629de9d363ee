/*
 * nrng.h -- C ABI of libnrng.so: bulk fp64 normal random numbers on B200 (sm_100a)
 * by the vectorised generators of R. P. Brent, "Fast Normal Random Number
 * Generators for Vector Processors", ANU TR-CS-93-04 (1993).
 * "P:n" = line n of that paper's text; "Rk" = reading k
 * in DESIGN.md §3 (where the paper is silent or ambiguous).
 *
 * Methods
 *   B1  Box-Muller: r = sigma sqrt(-2 ln(1-u)), x = r sin(theta) + mu,
 *       y = r cos(theta) + mu, theta = 2 pi v - pi (R6).
 *   B2  B1 with sin/cos from the odd/even polynomials on |y| <= pi/16 and four
 *       angle doublings.
 *   B3  P:280-295: m = max(u1,u2), u = m^2; u > 8/9 -> r = sigma sqrt(-ln(1-u)),
 *       else r = sigma m h((6u-4)/(4-3u)); returns mu + c r sqrt2, mu + s r sqrt2.
 *   P   Polar (Box-Muller-Marsaglia, Knuth's Algorithm P): x, y uniform in
 *       [-1,1), s = x^2 + y^2, reject s >= 1, r = sigma sqrt(-2 ln(s)/s), returns
 *       r x + mu, r y + mu; rejected candidates are compacted out.
 * Uniform source (the paper's RANU4 "generalised Fibonacci" generator, P:176-181;
 * lags unstated -> R1): per stream x_n = x_{n-607} + x_{n-273} mod 2^64, the 607-word
 * table of global stream k = splitmix64 outputs #607k..#607k+606 of `seed` (R2),
 * 10*607 warm-up outputs discarded (R3), u = (x >> 11) 2^-53 in [0,1).
 *
 * Work partition (R5, R18) -- identical for every call below that fills `n` slots:
 *   units U (pairs for the normal calls, P = ceil(n/2); uniforms for nrng_uniform);
 *   q = U / S, rem = U % S; stream k yields q + [k < rem] units, written at unit offset
 *   k*q + min(k, rem) ("stream-major, then accepted-pair index").  Pair j of stream k
 *   goes to out[2(off_k + j)] (first deviate) and out[2(off_k + j) + 1].  If n is odd
 *   the very last deviate is not written (its uniforms are still consumed).  Polar
 *   stops each stream exactly after its p_k-th accepted candidate.
 *   The result is a pure function of (seed, global stream ids, per-stream cumulative
 *   consumption, method, mu, sigma): independent of grid shape, GPU count or of how
 *   the caller splits calls, per stream.
 *
 * Memory and ownership
 *   A handle owns its device state (S x 608 u64 ring + S u64 counters) on the device
 *   current at create time.  `out` for the normal/uniform calls may be a DEVICE pointer
 *   (the fast path: asynchronous on the handle's stream; one kernel launch, or one per
 *   2^28 units of a stream's quota when a stream's quota is longer) or a HOST pointer
 *   (pinned or pageable: generated into two handle-owned 128 MiB device staging buffers
 *   -- ranges of whole streams, or pieces of one stream when its output exceeds a staging
 *   buffer -- and copied back overlapped with the next piece; the call returns after the
 *   host data is complete).  Device outputs should be 16-byte aligned (8-byte aligned
 *   is accepted on a slower store path).  `out` must hold n doubles; the library cannot
 *   check it (the Python binding checks dtype, contiguity and device).  No call
 *   allocates host memory for outputs.
 *
 * Errors: functions return NRNG_OK (0) or a negative code; the same code is kept as a
 * thread-local "last error" (nrng_last_error).  Argument errors are detected before
 * anything is launched and leave the state unchanged.  Device faults surface at the
 * next synchronising call as NRNG_ECUDA.
 *
 * Concurrency: one handle = one owner; do not use a handle from two host threads or
 * two CUDA streams at once.  Distinct handles are independent.
 */
#ifndef NRNG_H
#define NRNG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nrng_gen* nrng_handle;

enum { NRNG_DEFAULT = 0, NRNG_B1 = 1, NRNG_B2 = 2, NRNG_B3 = 3, NRNG_POLAR = 4, NRNG_POLAR2 = 5 };
enum { NRNG_OK = 0, NRNG_EINVAL = -1, NRNG_ENOMEM = -2, NRNG_ECUDA = -3, NRNG_ENODEV = -4 };

#define NRNG_LAG_R 607        /* long lag: words of state per stream */
#define NRNG_RING_PITCH 608   /* u64 words per stream in the state layout (padded) */

/* Create S = n_streams streams (global ids 0..S-1) seeded from `seed`, run the
 * splitmix64 fill and the 10-round warm-up on the current device (one kernel).
 * variant in {0,1,2,3}: the Box-Muller variant used when a call passes 0 (0 -> B1).
 * Returns NULL on error (see nrng_last_error()). */
nrng_handle nrng_create(uint64_t seed, uint32_t n_streams, int variant);

/* As nrng_create for the global stream range [first_stream, first_stream+n_streams):
 * the shard a rank owns.  The streams are bit-identical to the same
 * ids of a single larger handle. */
nrng_handle nrng_create_range(uint64_t seed, uint64_t first_stream, uint32_t n_streams, int variant);

/* Synchronise the handle's stream, free its device memory.  NULL-safe. */
void nrng_destroy(nrng_handle h);

/* Enqueue subsequent work on `cuda_stream` (a cudaStream_t, e.g. torch's
 * current_stream().cuda_stream; NULL = legacy default stream). */
int nrng_set_stream(nrng_handle h, void* cuda_stream);

/* n N(mu, sigma^2) deviates by Box-Muller variant 1/2/3 (0 = handle default) into out.
 * EINVAL: h NULL, out NULL with n>0, sigma<0, non-finite mu/sigma, bad variant,
 * wrong device.  n == 0: no-op.  sigma == 0: all outputs == mu. */
int nrng_normal_boxmuller(nrng_handle h, double* out, size_t n, double mu, double sigma, int variant);

/* n deviates by the Polar method P with rejection compaction and exact stop. */
int nrng_normal_polar(nrng_handle h, double* out, size_t n, double mu, double sigma);

/* n deviates by method P2: the same candidates, acceptance
 * and exact stop as nrng_normal_polar (identical uniform consumption), with step 4a
 * (u = 1 - s): s <= 8/9 -> r = sigma h((6s-4)/(4-3s)) (B3's polynomial, bit-exact
 * with the definition), s > 8/9 -> r = sigma sqrt(-ln(1-s)/s); returns x r sqrt2 + mu,
 * y r sqrt2 + mu.  Errors as nrng_normal_polar. */
int nrng_normal_polar2(nrng_handle h, double* out, size_t n, double mu, double sigma);

/* Algorithm R, the ratio method of Kinderman and Monahan:
 * for consecutive uniforms (u, v) of a stream, x = RN(RN(sqrt(8/e) (v - 1/2)) / (1 - u));
 * reject iff RN(x x) > -4 ln(1 - u) (the printed step 3 is an erratum, R25);
 * accepted candidates give ONE normal each, fma(sigma, x, mu).  Unlike the pair methods the
 * unit is a normal: stream k yields n/S (+1 for k < n mod S) normals at out[off_k + j],
 * exact stop (R26), no dropped deviate for odd n.  The step-2.5 pretests are not used (they
 * change no output, R28).  Uses 8/sqrt(pi e) = 2.74 uniforms per normal on average.
 * Errors as nrng_normal_polar.  Not available in the sequential mode. */
int nrng_normal_ratio(nrng_handle h, double* out, size_t n, double mu, double sigma);

/* Algorithm R1: Algorithm R with step 2.5, the pretests P1
 * (accept without a logarithm) and P2 (reject) before step 3 -- reading R29: the tangent-line
 * bounds of ln with a 2^-40 safety margin, so they never decide differently from step 3.
 * Same arguments, layout, exact stop, output and uniform consumption as nrng_normal_ratio
 * (identical results); only ~17% of the candidates (the borderline region) evaluate the
 * logarithm, gathered into one pass per warp step.  Errors as nrng_normal_polar. */
int nrng_normal_ratio1(nrng_handle h, double* out, size_t n, double mu, double sigma);

/* ---- sequential mode: RANN3-style buffering ----
 * One canonical, partition-invariant sequence per handle and method: epoch e is the output
 * of every stream making E more pairs, stream-major (2 S E deviates; E = epoch_pairs, a
 * power of two in [128, 2^20], default 128).  nrng_normal_seq(h, out, n, ...) returns the
 * next n deviates of that sequence: it first drains the deviates left over from the last
 * partially used epoch (kept in a handle-owned device buffer of 2 S E doubles), then writes
 * whole epochs straight into `out` (one launch per at most 2^28 pairs per stream), then
 * generates one more epoch into the buffer for the remainder.  Any split of a total into calls gives the same concatenated
 * output; odd counts and Polar's exact-count requirement need no dropped deviates.
 * EINVAL if deviates of another (method, mu, sigma) are still buffered (nrng_seq_reset
 * discards them; their uniforms stay consumed).  method: 1/2/3 = B1/B2/B3, 4 = P, 5 = P2.
 * out: device or host pointer, as for the bulk calls.  The state checkpoint
 * (nrng_get_state) does not include the buffer: reset or drain before checkpointing. */
int nrng_seq_configure(nrng_handle h, uint32_t epoch_pairs);
int nrng_normal_seq(nrng_handle h, double* out, size_t n, double mu, double sigma, int method);
size_t nrng_seq_buffered(nrng_handle h);
int nrng_seq_reset(nrng_handle h);

/* Thread-local status of the last nrng_* call on this thread, and its text. */
int nrng_last_error(void);
const char* nrng_error_string(int code);

/* ---- accessors / checkpoint (state = ring + per-stream consumed-uniform counter) ---- */
uint32_t nrng_num_streams(nrng_handle h);
uint64_t nrng_first_stream(nrng_handle h);
/* Copy per-stream consumed-uniform counters (S u64) to host memory; synchronises. */
int nrng_stream_counts(nrng_handle h, uint64_t* host_counts);
/* Copy the full state to host: ring S x 607 u64 (x_n at [k][n mod 607]) and counters.
 * Either pointer may be NULL.  Synchronises. */
int nrng_get_state(nrng_handle h, uint64_t* host_ring, uint64_t* host_counts);
/* Restore a state produced by nrng_get_state (same S); either pointer may be NULL.  Any
 * deviates the sequential mode still buffers are discarded (they came from the old state).
 * Synchronises. */
int nrng_set_state(nrng_handle h, const uint64_t* host_ring, const uint64_t* host_counts);
/* Block until all work enqueued by the handle has completed. */
int nrng_synchronize(nrng_handle h);
/* Number of kernels this handle has launched since creation (instrumentation). */
uint64_t nrng_kernel_launches(nrng_handle h);
/* Race-detector result of a DEBUG build (-DNRNG_RACECHECK=1, csrc/nrng_racecheck.cuh: every
 * shared-memory window / scratch access of the warp-per-stream kernels is checked against the
 * __syncwarp() epochs of the other lanes): host_out3[0] = races seen since the last call,
 * [1] = the first one (source line << 32 | kind << 16 | lane << 8 | other lane; kind 1 RAW,
 * 2 WAW, 3 WAR), [2] = accesses checked; the counters are then cleared.  Synchronises the
 * device.  The product build has no detector: zeros and NRNG_EINVAL. */
int nrng_racecheck_result(uint64_t* host_out3);

/* ---- test hooks (same partition rule; used by the parity tests) ---- */
/* n uniforms in [0,1), one per slot, stream-major (bit-exact with the oracle). */
int nrng_uniform(nrng_handle h, double* out, size_t n);
/* Advance EVERY stream by exactly cand_per_stream Polar candidates (2 uniforms each);
 * dev_mask[k*cand_per_stream + j] = 1 iff candidate j of stream k is accepted (s < 1). */
int nrng_polar_mask(nrng_handle h, uint8_t* dev_mask, size_t cand_per_stream);
/* Transforms on caller-given device uniforms (no generator state involved):
 * method 1/2/3 = B1/B2/B3 (2/2/3 uniforms per pair), 4 = Polar candidate, 5 = P2 candidate
 * (2 uniforms; rejected -> NaN outputs and dev_mask 0; dev_mask may be NULL), 6 = R
 * candidate (2 uniforms: out[2j] = sigma x + mu, NaN if rejected; out[2j+1] = x), 7 = R1
 * candidate (as 6; dev_mask = accepted | step-2.5 class << 1, class 1 = P1, 2 = P2,
 * 0 = borderline).
 * out: 2*n_pairs.
 * Enqueued on cuda_stream. */
int nrng_transform_from_uniforms(const double* dev_u, size_t n_pairs, double* dev_out, uint8_t* dev_mask,
                                 double mu, double sigma, int method, void* cuda_stream);

/* ---- validation reduction (the only data a multi-GPU run exchanges) ----
 * Over dev_x[0..n): dev_sums[0..3] = sum (x-center)^k, k=1..4; dev_sums[4] = min,
 * dev_sums[5] = max; dev_hist[b] (K bins, int64) counts x with edges[b-1] <= x < edges[b]
 * for the K-1 ascending device edges (bin 0 below edges[0], bin K-1 at/above edges[K-2]).
 * 2 <= K <= 1024.  Results are written (not accumulated).  Enqueued on cuda_stream. */
int nrng_stats(const double* dev_x, size_t n, double center, const double* dev_edges, int K, double* dev_sums,
               int64_t* dev_hist, void* cuda_stream);

/* Goodness-of-fit histogram (gates as SPEC S:409-426): dev_hist[b]
 * (2^log2K u32 counters, 4 <= log2K <= 24) counts x with Phi((x - mu)/sigma) in
 * [b/K, (b+1)/K), K = 2^log2K.  The host computes the Kolmogorov-Smirnov and
 * Anderson-Darling statistics from it (paper_1004_3105_b200/gof.py), after summing the
 * histograms of all ranks.  Results are written, not accumulated.  sigma > 0. */
int nrng_gof_hist(const double* dev_x, size_t n, double mu, double sigma, int log2K, uint32_t* dev_hist,
                  void* cuda_stream);

/* Serial-correlation gate ("serial correlation at lags 1..100
 * bounded by 4/sqrt(n)"): for d_i = dev_x[i] - center, dev_partial[b*(K+1) + k] =
 * sum over the i of the 4096-element tiles block b visits (tile b, b + blocks, ...; i + k < n) of d_i d_{i+k}, k = 0..K,
 * 1 <= K <= 127; nrng_serial_corr_blocks(n) blocks.  The host sums the blocks in order
 * (deterministic) and forms r_k = S_k / S_0 (paper_1004_3105_b200/gof.py).  Written, not
 * accumulated; enqueued on cuda_stream.  Validation only. */
int nrng_serial_corr(const double* dev_x, size_t n, double center, int K, double* dev_partial, void* cuda_stream);
size_t nrng_serial_corr_blocks(size_t n);

#ifdef __cplusplus
}
#endif
#endif /* NRNG_H */
