// nrng_kernels.cuh -- the sm_100a kernels of the hot path.
//
// One warp owns one LFG stream at a time (607 x u64 of state is too large for a
// thread; the lag structure gives 256 independent words per refill).  Warps stride
// over streams, persistent grid sized to the SM count x resident blocks.
#pragma once
#include <utility>

#include "nrng_device.cuh"

namespace nrng {

// Parameters shared by the bulk kernels.  Streams [s_begin, s_end) of the handle are
// processed; `units` = pairs (normal kernels) or uniforms (uniform kernel) over ALL S
// streams of the handle (so off_k is global), out + (g - shift) is where global deviate
// index g goes, n = number of valid output slots.
struct BulkParams {
    uint64_t* ring;     // S x kPitch
    uint64_t* count;    // S
    double* out;
    uint64_t units, q, rem, shift, n;
    // a piece of every stream's quota (host-side splitting of very long per-stream quotas):
    // units [jb, jb + jcap) of stream k's quota, at their own output slots; jcap = 0: whole quota
    uint64_t jb, jcap;
    uint32_t s_begin, s_end;
    TParams tp;
    int aligned;
    // epoch layout (sequential mode, nrng_normal_seq): 0 = plain stream-major.  Otherwise
    // every stream makes q = (#epochs) E pairs, E = 2^log2E, and pair j of stream k goes to
    // pair slot (j / E) S E + k E + j mod E: the output is epoch-major, stream-major within
    // an epoch, so consecutive calls continue one canonical sequence.
    uint32_t log2E, S;
};

__device__ __forceinline__ Quota quota(const BulkParams& p, uint64_t k) {
    Quota r = quota(p.q, p.rem, k);
    if (p.jcap) {
        const uint64_t left = r.cnt > p.jb ? r.cnt - p.jb : 0;
        r.cnt = left < p.jcap ? left : p.jcap;
        r.off += p.jb;
    }
    return r;
}

__device__ __forceinline__ uint64_t pair_slot(const BulkParams& p, uint64_t off, uint32_t k, uint64_t j) {
    if (p.log2E == 0) return off + j;
    const uint64_t E = 1ull << p.log2E;
    return (j >> p.log2E) * ((uint64_t)p.S << p.log2E) + (uint64_t)k * E + (j & (E - 1));
}

// Per-block shared memory: [NW x kWinAlloc u64 windows][tables][per-kernel extras].
// The bulk kernels come in two block shapes: NW = 4 warps (small stream counts: spread
// over all SMs) and NW = kBigBlock warps, one block per SM (the tables are stored once per
// SM instead of once per 4 warps, which is what lets 20 windows fit in 227 KB).
constexpr size_t win_bytes(int nw) { return (size_t)nw * kWinAlloc * sizeof(uint64_t); }
// The rejection methods' pair-window kernels (P, P2, R, R1) stage the warp's NEXT stream -- its
// ring row and counter -- in shared memory with cp.async while the current one computes:
// kStageWords after the 1024-word window, in place of the mirror they do not use.  Measured
// (interleaved, r2y/r2z/r2zp/r2zs): C2 (2^14 streams) P 64.3 -> 60.0 us, P2 79.6 -> 74.5 us,
// R 100.9 -> 96.8, R1 113.3 -> 108.8, the bench shape within noise; for B2 it cost 1-2% at the
// bench shape and in C3, so it keeps the L2 prefetch (B1 and B3 use their mirrors).
#ifndef NRNG_STAGE_NEXT
#define NRNG_STAGE_NEXT 1
#endif
constexpr int kStageWords = kPitch + 2;  // ring row (608) + counter + pad (16-byte multiple)
__host__ __device__ constexpr bool pw_staged(int M, bool EP) { return NRNG_STAGE_NEXT && M >= 4 && !EP; }
__host__ __device__ constexpr int pw_stride(int M, bool EP) { return pw_staged(M, EP) ? kWin + kStageWords : kWinAlloc; }
constexpr size_t pw_smem(int M, bool EP, int nw) {
    return (size_t)nw * pw_stride(M, EP) * sizeof(uint64_t) + kTabBytes +
           ((M == 5 || M == 7) ? (size_t)nw * 32 * sizeof(double) : 0);
}
// Issue the cp.async copies of stream kn's ring row and counter into stg (one commit group).
__device__ __forceinline__ void stage_state(uint64_t* stg, const BulkParams& p, uint32_t kn, int lane) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(stg);
    const uint64_t* row = p.ring + (uint64_t)kn * kPitch;
    for (int c = lane; c < kPitch / 2; c += 32)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s + 16 * c), "l"(row + 2 * c) : "memory");
    if (lane == 0)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s + 8 * kPitch), "l"(p.count + kn) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void stage_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// The pair window's XOR swizzle (see pw_kernel): logical word p at physical word swz(p).
__device__ __forceinline__ uint32_t swz(uint32_t p) { return p ^ ((p >> 4) & 1u); }

#ifndef NRNG_STAGE_RUNS
#define NRNG_STAGE_RUNS 1
#endif
// A stream's state into its window: src = the ring row in ring order (global memory, or the
// staging copy), cnt = its counter C; ring slot q holds word j = (q - C) mod 607 of the state,
// which goes to buf + phys(W - 607 + j), phys = the pair window's swizzle (kSwz) or the identity.
// A lane's slots q = lane + 32 t lie on two runs (q < C mod 607 and q >= it) whose window
// positions advance by 32 words per t, and swz(p + 32 t) = swz(p) + 32 t (the swizzle flips bit 0
// as a function of bit 4 only), so every store is one of two per-lane pointers plus an immediate.
template <bool kSwz, int W>
__device__ __forceinline__ uint64_t load_state_runs(const uint64_t* __restrict__ src, const uint64_t* cnt,
                                                    uint64_t* buf, int lane) {
    constexpr int T = (kLagR + 31) / 32;
    uint64_t v[T];
    const uint64_t C = *cnt;
#pragma unroll
    for (int t = 0; t < T; ++t)
        if (lane + 32 * t < kLagR) v[t] = src[lane + 32 * t];
    const int base = (int)(C % kLagR);
    auto phys = [](int p) { return kSwz ? (int)swz((uint32_t)p) : p; };
    uint64_t* const pa = buf + phys(W - base + lane);          // q < base: j = q + 607 - base
    uint64_t* const pb = buf + phys(W - kLagR + lane - base);  // q >= base: j = q - base
#pragma unroll
    for (int t = 0; t < T; ++t)
        if (lane + 32 * t < kLagR) NRNG_ST((lane + 32 * t >= base ? pb : pa) + 32 * t, v[t]);
    return C;
}
__device__ __forceinline__ uint64_t load_staged_state(const uint64_t* stg, uint64_t* buf, int lane) {
    return load_state_runs<true, kWin>(stg, stg + kPitch, buf, lane);
}

#ifndef NRNG_BIGBLOCK
#define NRNG_BIGBLOCK 20
#endif
constexpr int kBigBlock = NRNG_BIGBLOCK;
constexpr int kBigBlockPolar = 20;

// ------------------------------------------------------------------ seeding + warm-up
// Word j of global stream g = splitmix64 output #(607 g + j) of seed (R2); all-even fix
// (R4); 10 rounds of the round update (3 dependency phases 273/273/61) discarded (R3).
// L2 prefetch of the state of stream kn (its 4864-byte ring row = 38 lines, and its counter),
// issued when a warp starts a stream, for the stream it will take next: that stream's state
// load then hits L2 instead of paying an HBM round trip at the head of its serial chain (the
// mid-size configs run only a few blocks per stream, so that latency is not hidden).
#ifndef NRNG_PREFETCH_STATE  // 0: off, 1: when the warp starts a stream, 2: after its state load
#define NRNG_PREFETCH_STATE 2  // measured (us per call, off -> 2): C3 B2 603 -> 536, B3 806 -> 723, C4 B1 n=2^26
#endif                         // 278 -> 214, C1 11.3 -> 11.3, C2 P 70.5 -> 72.2; bench shape within +-2%
#ifndef NRNG_PREFETCH_B1
#define NRNG_PREFETCH_B1 1
#endif
template <int MODE>
__device__ __forceinline__ void prefetch_state(const BulkParams& p, uint32_t kn, int lane) {
    if (NRNG_PREFETCH_STATE != MODE || kn >= p.s_end) return;
    static_assert(kPitch * 8 == 38 * 128, "ring row = 38 lines");
    const char* row = reinterpret_cast<const char*>(p.ring + (uint64_t)kn * kPitch);
    for (int l = lane; l < 38; l += 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(row + 128 * l));
    if (lane == 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.count + kn));
}

// The first stream of each warp: its state prefetch is issued before the block loads its ln table,
// so the two global latencies overlap (calls with few streams per warp are latency-bound).
__device__ __forceinline__ void prefetch_first_state(const BulkParams& p, uint32_t k, int lane) {
    if (k >= p.s_end) return;
    const char* row = reinterpret_cast<const char*>(p.ring + (uint64_t)k * kPitch);
    for (int l = lane; l < 38; l += 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(row + 128 * l));
    if (lane == 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.count + k));
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32) init_kernel(uint64_t* __restrict__ ring,
                                                                   uint64_t* __restrict__ count, uint64_t seed,
                                                                   uint64_t first_stream, uint32_t S) {
    extern __shared__ __align__(16) uint64_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* buf = smem + warp * kPitch;
    for (uint32_t k = blockIdx.x * kWarpsPerBlock + warp; k < S; k += gridDim.x * kWarpsPerBlock) {
        const uint64_t g = first_stream + k;
        uint64_t odd = 0;
        for (int j = lane; j < kLagR; j += 32) {
            uint64_t x = splitmix64_mix(seed + ((uint64_t)kLagR * g + j + 1) * kGamma);
            NRNG_ST(&buf[j], x);
            odd |= x & 1;
        }
        const bool any_odd = __any_sync(kFull, odd != 0);
        NRNG_SYNCWARP();
        if (!any_odd && lane == 0) NRNG_ST(&buf[0], NRNG_LD(&buf[0]) | 1);
        NRNG_SYNCWARP();
        for (int r = 0; r < 10; ++r) {
            for (int i = lane; i < kLagS; i += 32) NRNG_ST(&buf[i], NRNG_LD(&buf[i]) + NRNG_LD(&buf[i + (kLagR - kLagS)]));
            NRNG_SYNCWARP();
            for (int i = kLagS + lane; i < 2 * kLagS; i += 32) NRNG_ST(&buf[i], NRNG_LD(&buf[i]) + NRNG_LD(&buf[i - kLagS]));
            NRNG_SYNCWARP();
            for (int i = 2 * kLagS + lane; i < kLagR; i += 32) NRNG_ST(&buf[i], NRNG_LD(&buf[i]) + NRNG_LD(&buf[i - kLagS]));
            NRNG_SYNCWARP();
        }
        uint64_t* rk = ring + (uint64_t)k * kPitch;
        for (int j = lane; j < kPitch; j += 32) rk[j] = j < kLagR ? NRNG_LD(&buf[j]) : 0;
        if (lane == 0) count[k] = 0;
        NRNG_SYNCWARP();
    }
}

// ------------------------------------------------------------------ Box-Muller B1/B2/B3
// Main loop: 64 pairs of stream k per warp iteration, two per lane (pairs j0+l and
// j0+32+l: independent dependency chains for latency hiding, and every constant-bank
// load and loop step amortised over two pairs); each store instruction writes 512
// contiguous bytes with a 16-byte streaming store.  Streams whose outputs are all in
// range and 16-byte aligned take this path; the tail (< 64 pairs), misaligned outputs
// and the stream holding the dropped last deviate of an odd n take the 32-pair path.
// U pairs per lane: pair u reads its words at src + u * 32 * per (lane-interleaved).
template <int V, int U>
__device__ __forceinline__ void bm_pairs(const uint64_t* src, const TParams& tp, const Tables& tab, double (&x)[U],
                                         double (&y)[U]) {
    constexpr int per = (V == 3) ? 3 : 2;
    if (V == 3) {
        uint64_t w1[U], w2[U], w3[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            w1[u] = NRNG_LD(&src[32 * per * u]);
            w2[u] = NRNG_LD(&src[32 * per * u + 1]);
            w3[u] = NRNG_LD(&src[32 * per * u + 2]);
        }
        b3_pairs<U>(w1, w2, w3, tp, tab, x, y);
    } else {
        uint64_t wu[U], wv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const ulonglong2 xw = NRNG_LD(reinterpret_cast<const ulonglong2*>(src + 32 * per * u));
            wu[u] = xw.x;
            wv[u] = xw.y;
        }
        if (V == 1)
            b1_pairs<U>(wu, wv, tp, tab, x, y);
        else
            b2_pairs<U>(wu, wv, tp, tab, x, y);
    }
}

template <int V, int NW>
__global__ void __launch_bounds__(NW * 32, NW == kBigBlock ? 1 : 5) bm_kernel(BulkParams p) {
    extern __shared__ __align__(16) uint64_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr uint32_t per = (V == 3) ? 3 : 2;
#ifndef NRNG_B3_U
#define NRNG_B3_U 2
#endif
    constexpr int kU = (V == 3) ? NRNG_B3_U : 4;       // pairs per lane per main-loop iteration
    constexpr int kB = 128;                            // refill batch
    constexpr uint32_t kNeedU = 32 * kU * per;         // words per main-loop iteration
    static_assert(kNeedU - 1 + kB <= kWin - kLagR, "lookahead would clobber the write-back words");
    static_assert(kNeedU <= kMirror, "unmasked reads must stay inside the mirror");
    prefetch_first_state(p, p.s_begin + blockIdx.x * NW + (threadIdx.x >> 5), threadIdx.x & 31);
    const Tables tab = load_tables<NW * 32>(reinterpret_cast<double2*>(smem + NW * kWinAlloc));
    __syncthreads();
    WarpLFG L;
    L.buf = smem + warp * kWinAlloc;
    for (uint32_t k = p.s_begin + blockIdx.x * NW + warp; k < p.s_end; k += gridDim.x * NW) {
        const Quota qk = quota(p, k);
        if (qk.cnt == 0) continue;
        prefetch_state<1>(p, k + gridDim.x * NW, lane);
        const uint64_t C = p.count[k];
        uint64_t* rk = p.ring + (uint64_t)k * kPitch;
        lfg_load(L, rk, C, lane, qk.cnt * per < (uint64_t)kLagR ? (uint32_t)(qk.cnt * per) : (uint32_t)kLagR);
        prefetch_state<2>(p, k + gridDim.x * NW, lane);
        uint64_t j0 = 0;
        if (p.aligned && 2 * (qk.off + qk.cnt) <= p.n) {
            double2* o = reinterpret_cast<double2*>(p.out + (2 * qk.off - p.shift)) + lane;
            const uint64_t full = qk.cnt - qk.cnt % (32 * kU);
            // B1: pair rows; B2: word-wise (measured faster for B2, whose sincos16 has no
            // integer work to hide the generator's latencies behind)
            constexpr bool kPairRows = V == 1;
            if constexpr (V == 2 && !kPairRows) if (full > 0) {
                // B2 phased steady state: iteration b transforms block b from the window and
                // generates block b + 1 word-wise (measured faster than pair rows for B2).
                lfg_generate<kBlk>(L, lane);  // block 0
                uint64_t* bl = L.buf + lane;
                uint32_t ph = 0;
                for (; j0 < full; j0 += 32 * kU, o += 32 * kU) {
                    if (p.log2E)
                        o = reinterpret_cast<double2*>(p.out + (2 * pair_slot(p, qk.off, k, j0) - p.shift)) + lane;
                    const uint32_t nb = (ph + 1) & 3;
                    uint64_t g[kBlkW];
                    phase_gen_load(bl, nb, g);
                    double x[kU], y[kU];
                    bm_pairs<V, kU>(L.buf + kBlk * ph + per * lane, p.tp, tab, x, y);
                    phase_gen_store(bl, nb, g);
#pragma unroll
                    for (int u = 0; u < kU; ++u) __stcs(o + 32 * u, make_double2(x[u], y[u]));
                    NRNG_SYNCWARP();
                    ph = nb;
                }
                L.wc = kW0 + (uint32_t)(per * full);
                L.wg = L.wc + kBlk;
            }
            if constexpr (kPairRows) if (full > 0) {
                // B1 phased steady state: iteration b generates block b (positions 256 (b
                // mod 4) ..) as four pair rows and transforms it from registers.
                static_assert(kU == 4 && kNeedU == kBlk, "one pair row per transform slot");
                uint64_t carry = block_first_word(L.buf, 0);
                uint32_t ph = 0;
                for (; j0 < full; j0 += 32 * kU, o += 32 * kU) {
                    if (p.log2E)
                        o = reinterpret_cast<double2*>(p.out + (2 * pair_slot(p, qk.off, k, j0) - p.shift)) + lane;
                    uint64_t wu[kU], wv[kU];
#ifndef NRNG_EXP_NOLFG
                    const PairRowPtrs r = pair_row_ptrs(L.buf, ph, lane);
                    gen_pair_rows<kU>(r.sa, r.sb, r.d, ph == 0, lane, carry, wu, wv);
#else  // experiment: transform cost alone (words from a counter, no window traffic)
#pragma unroll
                    for (int t = 0; t < kU; ++t) { wu[t] = (j0 + t) * 0x9E3779B97F4A7C15ull + lane; wv[t] = wu[t] * 0xBF58476D1CE4E5B9ull; }
#endif
                    double x[kU], y[kU];
#ifndef NRNG_EXP_NOTRANSFORM
                    if (V == 1)
                        b1_pairs<kU>(wu, wv, p.tp, tab, x, y);
                    else
                        b2_pairs<kU>(wu, wv, p.tp, tab, x, y);
#else  // experiment: generator + stores alone
#pragma unroll
                    for (int t = 0; t < kU; ++t) { x[t] = __longlong_as_double(wu[t] >> 2); y[t] = __longlong_as_double(wv[t] >> 2); }
#endif
#if defined(NRNG_EXP_PLAINSTORE)
#pragma unroll
                    for (int u = 0; u < kU; ++u) o[32 * u] = make_double2(x[u], y[u]);
#elif !defined(NRNG_EXP_NOSTORE)
#pragma unroll
                    for (int u = 0; u < kU; ++u) __stcs(o + 32 * u, make_double2(x[u], y[u]));
#else  // experiment: no output traffic (a never-taken store keeps the transform alive)
#pragma unroll
                    for (int u = 0; u < kU; ++u)
                        if (x[u] == 1234.5 && y[u] == 1234.5) __stcs(o + 32 * u, make_double2(x[u], y[u]));
#endif
                    NRNG_SYNCWARP();
                    ph = (ph + 1) & 3;
                }
                L.wc = L.wg = kW0 + (uint32_t)(per * full);
            }
            for (; j0 < full; j0 += 32 * kU, o += 32 * kU) {
                if (p.log2E)  // epochs are multiples of 32 kU pairs: one slot computation per step
                    o = reinterpret_cast<double2*>(p.out + (2 * pair_slot(p, qk.off, k, j0) - p.shift)) + lane;
                lfg_ensure<kB>(L, lane, kNeedU);
                double x[kU], y[kU];
                bm_pairs<V, kU>(L.at(per * lane), p.tp, tab, x, y);
#pragma unroll
                for (int u = 0; u < kU; ++u) __stcs(o + 32 * u, make_double2(x[u], y[u]));
                L.wc += kNeedU;
                NRNG_SYNCWARP();
            }
        }
        for (; j0 < qk.cnt; j0 += 32) {
            lfg_ensure<kB>(L, lane, 32 * per);
            const uint64_t left = qk.cnt - j0;
            const uint32_t active = left < 32 ? (uint32_t)left : 32u;
            if ((uint32_t)lane < active) {
                double x[1], y[1];
                bm_pairs<V, 1>(L.at(per * lane), p.tp, tab, x, y);
                store_pair(p.out, 2 * pair_slot(p, qk.off, k, j0 + lane), p.shift, p.n, x[0], y[0], p.aligned);
            }
            L.wc += per * active;
            NRNG_SYNCWARP();
        }
        lfg_store(L, rk, C, lane);
        if (lane == 0) p.count[k] = C + (L.wc - kW0);
        NRNG_SYNCWARP();
    }
}

// ------------------------------------------------------------------ B3, triple rows
// B3 consumes the stream in word triples (u1, u2, u3).  Here each lane
// GENERATES the three consecutive words it consumes: lane l makes x_{R+3l+i}, i < 3, of
// the 96-word row starting at R from x_{R+3l+i-607} and x_{R+3l+i-273} (rows are shorter
// than the 273 lag, so every source is older than the row), stores them and transforms
// them from registers.  A 64-bit access at a 3-word lane stride is bank-conflict-free (the
// 16 lanes of a half-warp hit bank pairs 6l mod 32, all distinct), so a row costs 6 loads
// and 3 stores of 256 B each: 24 B of shared traffic per word, against 34 B for a
// word-wise refill plus the consumer's re-read.  An iteration makes 4 rows (128 pairs) in
// two halves of 2 rows (rows 2-3 read rows 0-1 at lag 273, so a __syncwarp separates the
// halves).  The window is 12 rows (1152 words >= 607 + the 4 rows of an iteration) plus a
// 2-row mirror of rows 0-1 for the sources that run past its end (10.5 KB per warp).  12
// rows are 3 iterations, so the steady loop is unrolled over the 3 iteration phases: every
// load and store address is the lane's base pointer plus an immediate, and the mirror
// stores appear in phase 0 only (measured against an 11-row window with runtime positions:
// the wrap arithmetic and predicated mirror stores were ~5% of the issue slots).
// Word i of the call (i < 0: the loaded state) sits at window position i mod 1152.
constexpr int kTriRow = 96;
constexpr int kTriWin = 12 * kTriRow;
constexpr int kTriMirror = 2 * kTriRow;
constexpr int kTriAlloc = kTriWin + kTriMirror;
constexpr int kTriScratch = 32;  // per-warp tail-compaction slots (doubles)
#ifndef NRNG_TRI_WARPS
#define NRNG_TRI_WARPS 16  // measured (11-row window): 16 warps 5.79 ms, 20 warps 5.94, 12 warps 5.82; 12-row window:
                           // 12 warps 5.89-5.96 vs 16 warps 5.80-5.84 (sustained); 20 warps no longer fit in 227 KB
#endif
constexpr int kTriWarps = NRNG_TRI_WARPS;
static_assert(kTriWin >= kLagR + 4 * kTriRow && 2 * kTriRow < kLagS && kTriWin % (4 * kTriRow) == 0,
              "triple-row window");
constexpr size_t tri_smem(int nw) {
    return (size_t)nw * (kTriAlloc + kTriScratch) * sizeof(uint64_t) + kTabBytes;
}

__device__ __forceinline__ uint32_t tri_wrap(uint32_t x) { return x >= (uint32_t)kTriWin ? x - kTriWin : x; }

// Window positions of a row and of its two source runs (the partial last rows of a call).
struct TriPos {
    uint32_t d, a, b;  // row at d; sources x_{w-607} at a, x_{w-273} at b (row t at +96 t, via the mirror)
    __device__ __forceinline__ void advance(uint32_t rows) {
        d = tri_wrap(d + kTriRow * rows);
        a = tri_wrap(a + kTriRow * rows);
        b = tri_wrap(b + kTriRow * rows);
    }
};

// Generate R (<= 2) consecutive rows at `ps`.  All loads are issued before any store (the
// rows' sources are all older than the rows).
template <int R>
__device__ __forceinline__ void gen_tri_rows(uint64_t* buf, const TriPos& ps, int lane, uint64_t (&w1)[R],
                                             uint64_t (&w2)[R], uint64_t (&w3)[R]) {
    static_assert(R <= 2, "mirror covers two rows of source overrun");
    uint64_t a[R][3], b[R][3];
    const uint64_t* sa = buf + ps.a + 3 * lane;
    const uint64_t* sb = buf + ps.b + 3 * lane;
#pragma unroll
    for (int t = 0; t < R; ++t) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            a[t][i] = NRNG_LD(&sa[kTriRow * t + i]);
            b[t][i] = NRNG_LD(&sb[kTriRow * t + i]);
        }
    }
#pragma unroll
    for (int t = 0; t < R; ++t) {
        w1[t] = a[t][0] + b[t][0];
        w2[t] = a[t][1] + b[t][1];
        w3[t] = a[t][2] + b[t][2];
        const uint32_t pd = t == 0 ? ps.d : tri_wrap(ps.d + kTriRow * t);
        uint64_t* d = buf + pd + 3 * lane;
        NRNG_ST(&d[0], w1[t]);
        NRNG_ST(&d[1], w2[t]);
        NRNG_ST(&d[2], w3[t]);
        if (pd < (uint32_t)kTriMirror) {  // rows 0-1 are mirrored past the end
            NRNG_ST(&d[kTriWin], w1[t]);
            NRNG_ST(&d[kTriWin + 1], w2[t]);
            NRNG_ST(&d[kTriWin + 2], w3[t]);
        }
    }
}

// The two rows 2H, 2H+1 of a steady iteration in phase PH (row 0 at window position
// 384 PH), at compile-time offsets from the lane's base pointer lb = buf + 3 lane.
template <int PH, int H>
__device__ __forceinline__ void gen_tri_half(uint64_t* lb, uint64_t (&w1)[4], uint64_t (&w2)[4], uint64_t (&w3)[4]) {
    constexpr int d = 4 * kTriRow * PH + 2 * kTriRow * H;
    constexpr int a = (d + kTriWin - kLagR) % kTriWin, b = (d + kTriWin - kLagS) % kTriWin;
    static_assert(a + 2 * kTriRow <= kTriAlloc && b + 2 * kTriRow <= kTriAlloc, "source runs inside the mirror");
    uint64_t sa[2][3], sb[2][3];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            sa[t][i] = NRNG_LD(&lb[a + kTriRow * t + i]);
            sb[t][i] = NRNG_LD(&lb[b + kTriRow * t + i]);
        }
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int r = 2 * H + t;
        w1[r] = sa[t][0] + sb[t][0];
        w2[r] = sa[t][1] + sb[t][1];
        w3[r] = sa[t][2] + sb[t][2];
        NRNG_ST(&lb[d + kTriRow * t], w1[r]);
        NRNG_ST(&lb[d + kTriRow * t + 1], w2[r]);
        NRNG_ST(&lb[d + kTriRow * t + 2], w3[r]);
        if constexpr (d < kTriMirror) {
            NRNG_ST(&lb[d + kTriWin + kTriRow * t], w1[r]);
            NRNG_ST(&lb[d + kTriWin + kTriRow * t + 1], w2[r]);
            NRNG_ST(&lb[d + kTriWin + kTriRow * t + 2], w3[r]);
        }
    }
}

// One steady iteration (4 rows, 128 pairs) in phase PH.
template <int PH>
__device__ __forceinline__ void b3_iter(uint64_t* lb, const TParams& tp, const Tables& tab, double* scr, int lane,
                                        unsigned lt, double2* o) {
    uint64_t w1[4], w2[4], w3[4];
    gen_tri_half<PH, 0>(lb, w1, w2, w3);
    NRNG_SYNCWARP();  // rows 2-3 read rows 0-1 (lag 273)
    gen_tri_half<PH, 1>(lb, w1, w2, w3);
    double x[4], y[4];
    b3_pairs_compact<4>(w1, w2, w3, tp, tab, scr, lane, lt, x, y);
#pragma unroll
    for (int u = 0; u < 4; ++u) __stcs(o + 32 * u, make_double2(x[u], y[u]));
#if !NRNG_SCR_SYNC_MIN
    NRNG_SYNCWARP();  // (with NRNG_SCR_SYNC_MIN the gather's __syncwarp, after every window access of
#endif             // this iteration, orders them before the next iteration's window writes)
}

// Aligned, plain-layout B3 calls (the dispatcher sends the rest to bm_kernel<3>).
template <int NW, bool EP = false>  // EP: the sequential mode's epoch layout (see pw_kernel)
__global__ void __launch_bounds__(NW * 32, 1) b3_kernel(BulkParams p) {
    extern __shared__ __align__(16) uint64_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* const buf = smem + warp * (kTriAlloc + kTriScratch);
    prefetch_first_state(p, p.s_begin + blockIdx.x * NW + warp, lane);
    const Tables tab = load_tables<NW * 32>(reinterpret_cast<double2*>(smem + NW * (kTriAlloc + kTriScratch)));
    __syncthreads();
    double* const scr = reinterpret_cast<double*>(buf + kTriAlloc);
    const unsigned lt = lanemask_lt(lane);
    for (uint32_t k = p.s_begin + blockIdx.x * NW + warp; k < p.s_end; k += gridDim.x * NW) {
        const Quota qk = quota(p, k);
        if (qk.cnt == 0) continue;
        prefetch_state<1>(p, k + gridDim.x * NW, lane);
        uint64_t* rk = p.ring + (uint64_t)k * kPitch;
        // x_{C-607+j} -> position 1152 - 607 + j
        const uint64_t C = load_state_rot(rk, p.count + k, lane, [&](uint32_t j) { return buf + (kTriWin - kLagR) + j; });
        NRNG_SYNCWARP();
        prefetch_state<2>(p, k + gridDim.x * NW, lane);
        // pairs whose 16-byte outputs are all in range (odd n: the very last pair is not)
        const uint64_t safe_cnt = 2 * (qk.off + qk.cnt) <= p.n ? qk.cnt : qk.cnt - 1;
        const uint32_t nit = (uint32_t)(safe_cnt / 128);  // full 4-row iterations (a 32-bit count: no
        double2* o = EP ? reinterpret_cast<double2*>(p.out) + pair_slot(p, qk.off, k, 0) + lane
                        : reinterpret_cast<double2*>(p.out + (2 * qk.off - p.shift)) + lane;  // per-iteration
        auto adv = [&](uint32_t itn) {  // o -> the first pair of iteration itn (+ lane)
            if constexpr (EP)  // +128 pairs inside an epoch chunk (E >= 128, 128 | E), else to the next epoch's
                o += ((128u * itn) & ((1u << p.log2E) - 1)) ? 128 : ((uint64_t)p.S << p.log2E) - (1u << p.log2E) + 128;
            else
                o += 128;
        };
        uint64_t* const lb = buf + 3 * lane;
        for (uint32_t it = 0;;) {  // unrolled over the 3 phases of the 12-row window
            if (it == nit) break;
            b3_iter<0>(lb, p.tp, tab, scr, lane, lt, o);
            adv(it + 1);
            if (++it == nit) break;
            b3_iter<1>(lb, p.tp, tab, scr, lane, lt, o);
            adv(it + 1);
            if (++it == nit) break;
            b3_iter<2>(lb, p.tp, tab, scr, lane, lt, o);
            adv(it + 1);
            ++it;
        }
        const uint32_t d0 = 4 * kTriRow * (nit % 3);
        TriPos ps{d0, tri_wrap(d0 + kTriWin - kLagR), tri_wrap(d0 + kTriWin - kLagS)};
        // Re-derive the per-stream values from k (kernel parameters live in the constant
        // bank): nothing but k and `nit` has to stay live across the loop, which kept
        // the compiler from rematerialising the quota inside every iteration.
        const Quota qk2 = quota(p, k);
        for (uint64_t j0 = 128ull * nit; j0 < qk2.cnt; j0 += 32) {  // last rows, partial, unsafe pair
            uint64_t w1[1], w2[1], w3[1];
            gen_tri_rows<1>(buf, ps, lane, w1, w2, w3);
            double x[1], y[1];
            b3_pairs<1>(w1, w2, w3, p.tp, tab, x, y);
            if ((uint64_t)lane < qk2.cnt - j0)
                store_pair(p.out, 2 * (EP ? pair_slot(p, qk2.off, k, j0 + lane) : qk2.off + j0 + lane), p.shift, p.n,
                           x[0], y[0], true);
            NRNG_SYNCWARP();
            ps.advance(1);
        }
        // write back the last min(3 cnt, 607) consumed words (relative index i at i mod 1152)
        const uint64_t C2 = p.count[k];
        uint64_t* rk2 = p.ring + (uint64_t)k * kPitch;
        const uint64_t used = 3 * qk2.cnt;
        const uint32_t nw = used < (uint64_t)kLagR ? (uint32_t)used : (uint32_t)kLagR;
        const uint32_t pos0 = (uint32_t)((used - nw) % kTriWin);  // used - nw >= 0
        const uint32_t slot0 = (uint32_t)((C2 + used - nw) % kLagR);
        store_state(rk2, slot0, nw, lane, [&](uint32_t j) {
            uint32_t pp = pos0 + j;
            return &buf[pp >= (uint32_t)kTriWin ? pp - kTriWin : pp];
        });
        NRNG_SYNCWARP();  // every lane has read count[k] before lane 0 updates it
        if (lane == 0) p.count[k] = C2 + used;
        NRNG_SYNCWARP();
    }
}

// ------------------------------------------------------------------ Polar P
// 64 candidates (128 uniforms) per warp step, two per lane: candidate i of the step is
// lane i%32's (i < 32: words wc + 2i, i >= 32: wc + 64 + 2(i-32)).  Accepts are ranked
// with __ballot_sync/__popc in candidate order and trimmed at the stream's remaining quota
// (exact stop, R5: the last step consumes candidates only up to the p_k-th accept); each
// survivor's rank is its pair index, so the output is stream-major then accepted-pair
// order with no gaps.
// The survivors are compacted in the OUTPUT only: the warp transforms all 64 candidates
// of a step and rejected lanes are predicated off at the store.  On the VP2200 the
// compress made vector lengths full; on a GPU the 21.5% of lanes doing wasted
// work cost less than a survivor queue's per-candidate bookkeeping (measured: a shared-
// memory queue with dense 64-wide transforms ran 6.4 ms vs 5.7 ms per 2^31 normals; on the
// pair-window kernel, a 256-entry ring with dense 128-wide batches 4.75 vs 4.36 ms).
// M = 1: Algorithm P (= the paper's P1); M = 2: method P2, same candidates.
#ifndef NRNG_POLAR_U
#define NRNG_POLAR_U 4
#endif
constexpr int kPU = NRNG_POLAR_U;  // candidates per lane per step (32 kPU per warp)
#ifndef NRNG_POLAR_DIRECT_SPLIT
#define NRNG_POLAR_DIRECT_SPLIT 1  // pw_kernel: a Polar step loop specialised for in-range outputs
#endif
#ifndef NRNG_POLAR_SPLIT_STOP
#define NRNG_POLAR_SPLIT_STOP 1  // pw_polar_block: the exact-stop trim only in the stream's last step
#endif
constexpr int kPB = 128; // refill batch: lookahead 64 kPU - 1 + kPB <= 417
static_assert(64 * kPU - 1 + kPB <= kWin - kLagR && 64 * kPU <= kMirror, "polar window bounds");

// Rank the accepts of one step (candidate i = 32 u + lane) and, if the step reaches the
// remaining quota `need`, keep only the first `need` of them (exact stop, R5).  m[u] =
// kept accept masks; returns the candidates consumed (32 kPU unless the step stops).
__device__ __forceinline__ uint32_t polar_rank(const bool (&ok)[kPU], unsigned (&m)[kPU], uint32_t need, unsigned lt,
                                               bool& stop) {
    uint32_t tot = 0;
#pragma unroll
    for (int u = 0; u < kPU; ++u) {
        m[u] = __ballot_sync(kFull, ok[u]);
        tot += __popc(m[u]);
    }
    uint32_t used = 32 * kPU;
    stop = tot >= need;
    if (stop) {
        uint32_t rem = need;
#pragma unroll
        for (int u = 0; u < kPU; ++u) {
            const uint32_t nu = __popc(m[u]);
            if (rem == 0) {
                m[u] = 0;
            } else if (nu >= rem) {
                const unsigned last = __ballot_sync(kFull, ok[u] && (uint32_t)__popc(m[u] & lt) == rem - 1);
                const int l = __ffs(last) - 1;
                m[u] &= (l == 31) ? kFull : ((2u << l) - 1u);
                used = 32 * u + l + 1;
                rem = 0;
            } else {
                rem -= nu;
            }
        }
    }
    return used;
}

template <int NW, int M, bool EP = false>  // EP: the sequential mode's whole-epoch layout (see pw_kernel)
__global__ void __launch_bounds__(NW * 32, NW == kBigBlockPolar ? 1 : 4) polar_kernel(BulkParams p) {
    extern __shared__ __align__(16) uint64_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    prefetch_first_state(p, p.s_begin + blockIdx.x * NW + (threadIdx.x >> 5), threadIdx.x & 31);
    const Tables tab = load_tables<NW * 32>(reinterpret_cast<double2*>(smem + NW * kWinAlloc));
    __syncthreads();
    WarpLFG L;
    L.buf = smem + warp * kWinAlloc;
    const unsigned lt = lanemask_lt(lane);
    double* const scr = reinterpret_cast<double*>(smem + NW * kWinAlloc + kTabBytes / 8) + 32 * warp;  // P2 tails
    for (uint32_t k = p.s_begin + blockIdx.x * NW + warp; k < p.s_end; k += gridDim.x * NW) {
        const Quota qk = quota(p, k);
        if (qk.cnt == 0) continue;
        prefetch_state<1>(p, k + gridDim.x * NW, lane);
        const uint64_t C = p.count[k];
        uint64_t* rk = p.ring + (uint64_t)k * kPitch;
        lfg_load(L, rk, C, lane);
        prefetch_state<2>(p, k + gridDim.x * NW, lane);
        const bool fast = p.aligned && 2 * (qk.off + qk.cnt) <= p.n;
        const bool direct = fast && (EP || p.log2E == 0);
        const bool phased = direct && qk.cnt < (1ull << 31);
        if (phased) {
            // Phased steady state: every step but the stream's last consumes exactly one
            // 256-word block (128 candidates) and generates the next; the last step (exact
            // stop) generates nothing, so the lookahead stays <= 256 for the write-back.
            static_assert(64 * kPU == kBlk, "one block per polar step");
            double2* o = reinterpret_cast<double2*>(p.out + (2 * qk.off - p.shift));
            const uint32_t cnt = (uint32_t)qk.cnt;
            uint32_t ph = 0, acc = 0, it = 0;
            lfg_generate<kBlk>(L, lane);  // block 0
            uint64_t* bl = L.buf + lane;
            for (;;) {
                PolarCand c[kPU];
                bool ok[kPU];
                unsigned m[kPU];
                const uint32_t nb = (ph + 1) & 3;
                uint64_t g[kBlkW];
                phase_gen_load(bl, nb, g);
#ifndef NRNG_EXP_P_NOCONSUME
#pragma unroll
                for (int u = 0; u < kPU; ++u) {
                    const ulonglong2 w = NRNG_LD(reinterpret_cast<const ulonglong2*>(L.buf + kBlk * ph + 64 * u + 2 * lane));
                    ok[u] = polar_candidate(w.x, w.y, c[u]);
                }
#else  // experiment: candidates from the freshly generated words (no window re-read; wrong stream order)
#pragma unroll
                for (int u = 0; u < kPU; ++u) ok[u] = polar_candidate(g[2 * u], g[2 * u + 1], c[u]);
#endif
                bool stop;
                const uint32_t used = polar_rank(ok, m, cnt - acc, lt, stop);
                if (!stop) phase_gen_store(bl, nb, g);
                double ox[kPU], oy[kPU];
                if (M == 2)
                    p2_transform_compact<kPU>(c, ok, p.tp, tab, scr, lane, lt, ox, oy);
                else
                    polar_transform<kPU>(c, p.tp, tab, ox, oy);
                if constexpr (EP) {  // at most two epoch chunks per step (as pw_polar_block)
                    const uint32_t e0 = acc >> p.log2E, jb = e0 << p.log2E, E = 1u << p.log2E;
                    double2* const ob = reinterpret_cast<double2*>(p.out) + pair_slot(p, qk.off, k, jb);
                    const uint64_t jump = ((uint64_t)p.S << p.log2E) - E;
#pragma unroll
                    for (int u = 0; u < kPU; ++u) {
                        const uint32_t jj = acc + __popc(m[u] & lt) - jb;
                        if ((m[u] >> lane) & 1u) __stcs(ob + jj + (jj >= E ? jump : 0), make_double2(ox[u], oy[u]));
                        acc += __popc(m[u]);
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < kPU; ++u) {
                        if ((m[u] >> lane) & 1u) __stcs(o + (acc + __popc(m[u] & lt)), make_double2(ox[u], oy[u]));
                        acc += __popc(m[u]);
                    }
                }
                NRNG_SYNCWARP();
                if (stop) {
                    L.wc = kW0 + kBlk * it + 2 * used;
                    L.wg = kW0 + kBlk * (it + 1);
                    break;
                }
                ++it;
                ph = (ph + 1) & 3;
            }
        }
        for (uint64_t base = 0; !phased && base < qk.cnt;) {  // general path
            const uint32_t cnt = (uint32_t)(qk.cnt - base < (1ull << 31) ? qk.cnt - base : (1ull << 31));
            double2* o = reinterpret_cast<double2*>(p.out + (2 * (qk.off + base) - p.shift));
            uint32_t acc = 0;  // accepted pairs of this chunk
            while (acc < cnt) {
                lfg_ensure<kPB>(L, lane, 64 * kPU);
                PolarCand c[kPU];
                bool ok[kPU];
                unsigned m[kPU];
#pragma unroll
                for (int u = 0; u < kPU; ++u) {
                    const ulonglong2 w = NRNG_LD(reinterpret_cast<const ulonglong2*>(L.at(64 * u + 2 * lane)));
                    ok[u] = polar_candidate(w.x, w.y, c[u]);
                }
                bool stop;
                const uint32_t used = polar_rank(ok, m, cnt - acc, lt, stop);
                double ox[kPU], oy[kPU];
                if (M == 2)
                    p2_transform_compact<kPU>(c, ok, p.tp, tab, scr, lane, lt, ox, oy);
                else
                    polar_transform<kPU>(c, p.tp, tab, ox, oy);
                uint32_t j = acc;
                if (direct) {  // common case: one predicated 16-byte store per kept lane
#pragma unroll
                    for (int u = 0; u < kPU; ++u) {
                        if ((m[u] >> lane) & 1u) __stcs(o + j + __popc(m[u] & lt), make_double2(ox[u], oy[u]));
                        j += __popc(m[u]);
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < kPU; ++u) {
                        const uint32_t ju = j + __popc(m[u] & lt);
                        if ((m[u] >> lane) & 1u) {
                            if (p.log2E)
                                __stcs(reinterpret_cast<double2*>(p.out +
                                                                  (2 * pair_slot(p, qk.off, k, base + ju) - p.shift)),
                                       make_double2(ox[u], oy[u]));
                            else
                                store_pair(p.out, 2 * (qk.off + base + ju), p.shift, p.n, ox[u], oy[u], p.aligned);
                        }
                        j += __popc(m[u]);
                    }
                }
                acc = j;
                L.wc += 2 * used;
                NRNG_SYNCWARP();
            }
            base += cnt;
        }
        lfg_store(L, rk, C, lane);
        if (lane == 0) p.count[k] = C + (L.wc - kW0);
        NRNG_SYNCWARP();
    }
}

// ------------------------------------------------------------------ swizzled pair window
// B1, B2, P and P2 consume the stream in word pairs (x_{2i}, x_{2i+1}).  Here each lane
// GENERATES the pair it consumes, from four 64-bit loads (the sources x_{w-607}, x_{w-606},
// x_{w-273}, x_{w-272} of an even w start at odd positions, so they are two unaligned
// pairs), stores it with two 64-bit stores and transforms it from registers: no consumer
// re-read, no shuffle.  A lane stride of 2 words would put lanes l and l+8 of a half-warp
// on the same bank pair; the window is therefore XOR-swizzled, logical position p held at
// physical word swz(p) = p ^ ((p >> 4) & 1) (bit 0 flipped in every other 16-word row),
// which makes every stride-2 half-warp access hit 16 distinct bank pairs, keeps each
// aligned pair inside its 16-byte slot and keeps contiguous 32-word accesses a
// permutation of their row.  Because the per-lane part of every address (2l + a constant
// whose low 6 bits are fixed) is the same in every row, the swizzle is six per-lane
// offsets computed once; rows only add a uniform multiple of 64.  Window: 1024 words +
// the 256-word mirror of positions [0, 256) (sources of a row run up to 63 words past
// the end).  Word i of the call (i < 0: the loaded state) is at logical position i mod 1024.
// Used for aligned, plain-layout calls filling the GPU; the rest go to bm_kernel /
// polar_kernel.  M: 1 = B1, 2 = B2, 4 = P (P2 keeps polar_kernel: here it spilled), 6 = R
// (Algorithm R, the only path for it besides the tiny-quota kernel), 7 = R1 (R with the
// step-2.5 pretests; needs 32 more doubles of shared scratch per warp, pw_smem).
#ifndef NRNG_PW_WARPS
#define NRNG_PW_WARPS 16  // measured (ms per 2^31, B1/B2/P): 16 warps 3.68/3.88/4.52, 12: 4.09/3.83/4.54, 14: 4.28/4.21/4.72, 18: 4.06/4.44/4.73, 20 (another box): 3.79/4.19/4.30
#endif
constexpr int kPwWarps = NRNG_PW_WARPS;
#ifndef NRNG_B1_UNROLL
#define NRNG_B1_UNROLL 0
#endif
#ifndef NRNG_B1_MIRROR_BRANCH
#define NRNG_B1_MIRROR_BRANCH 1
#endif

#ifndef NRNG_PW_NOMIRROR
#define NRNG_PW_NOMIRROR 1  // compile-time generator: no mirror; straddling runs read through lane-wrapped pointers
#endif
struct PwLane {  // physical offsets of this lane's words in a row whose base is 0
    uint32_t a0, a1, b0, b1, d0, d1;
};
__device__ __forceinline__ PwLane pw_lane(int lane) {
    const uint32_t l2 = 2 * lane;
    return PwLane{swz(kWin - kLagR + l2), swz(kWin - kLagR + 1 + l2), swz(kWin - kLagS + l2),
                  swz(kWin - kLagS + 1 + l2), swz(l2), swz(l2 + 1)};
}

// Generate R consecutive pair rows starting at logical row base K (a multiple of 64 below
// 1024; rows at K + 64 t must not cross 1024): lane l makes (x_{K+64t+2l}, x_{K+64t+2l+1}).
// The source runs are masked once per call (a run of R rows may extend up to 255 words past
// 1023, into the mirror), so every row is the same four per-lane pointers plus an immediate.
// All loads are issued before any store (all sources are older than the rows: 64 R <= 273).
template <int R, bool kNoMirror = NRNG_PW_NOMIRROR>
__device__ __forceinline__ void pw_gen(uint64_t* buf, uint32_t K, const PwLane& o, uint64_t (&w0)[R],
                                       uint64_t (&w1)[R], int lane) {
    static_assert(64 * R <= kLagS && 64 * R <= kMirror, "rows of one call must be independent");
    uint64_t a0[R], a1[R], b0[R], b1[R];
    if constexpr (kNoMirror) {
        // every source position wrapped per lane (the short-call tail path: no mirror reads)
        const uint32_t l2 = 2 * lane;
#pragma unroll
        for (int t = 0; t < R; ++t) {
            const uint32_t pa = K + 64 * t + (kWin - kLagR) + l2, pb = K + 64 * t + (kWin - kLagS) + l2;
            a0[t] = NRNG_LD(&buf[swz(pa & kWinMask)]);
            a1[t] = NRNG_LD(&buf[swz((pa + 1) & kWinMask)]);
            b0[t] = NRNG_LD(&buf[swz(pb & kWinMask)]);
            b1[t] = NRNG_LD(&buf[swz((pb + 1) & kWinMask)]);
        }
    } else {
        const int ka = (int)((K + (kWin - kLagR)) & kWinMask) - (kWin - kLagR);  // multiple of 64
        const int kb = (int)((K + (kWin - kLagS)) & kWinMask) - (kWin - kLagS);
        const uint64_t* pa0 = buf + (ka + (int)o.a0);
        const uint64_t* pa1 = buf + (ka + (int)o.a1);
        const uint64_t* pb0 = buf + (kb + (int)o.b0);
        const uint64_t* pb1 = buf + (kb + (int)o.b1);
#pragma unroll
        for (int t = 0; t < R; ++t) {
            a0[t] = NRNG_LD(&pa0[64 * t]);
            a1[t] = NRNG_LD(&pa1[64 * t]);
            b0[t] = NRNG_LD(&pb0[64 * t]);
            b1[t] = NRNG_LD(&pb1[64 * t]);
        }
    }
    uint64_t* pd0 = buf + (K + o.d0);
    uint64_t* pd1 = buf + (K + o.d1);
#pragma unroll
    for (int t = 0; t < R; ++t) {
        w0[t] = a0[t] + b0[t];
        w1[t] = a1[t] + b1[t];
        NRNG_ST(&pd0[64 * t], w0[t]);
        NRNG_ST(&pd1[64 * t], w1[t]);
    }
    if (!kNoMirror && K < (uint32_t)kMirror) {  // rows in [0, 256): mirrored at +1024
#pragma unroll
        for (int t = 0; t < R; ++t) {
            NRNG_ST(&pd0[kWin + 64 * t], w0[t]);
            NRNG_ST(&pd1[kWin + 64 * t], w1[t]);
        }
    }
}

// The same for a block at a compile-time base K (the steady loops are unrolled over the 4
// block positions): every address is a per-lane pointer plus an immediate.
struct PwPtrs {
    const uint64_t *a0, *a1, *b0, *b1;
    uint64_t *d0, *d1;
    // the same source pointers minus one window (1024 words) on the lanes whose word of the one
    // row per lag that straddles the window's end lies past it (NRNG_PW_NOMIRROR): lag-607 run
    // at position 993 (+2l, +1: lanes >= 16 / >= 15), lag-273 run at 1007 (lanes >= 9 / >= 8)
    const uint64_t *a0x, *a1x, *b0x, *b1x;
};
__device__ __forceinline__ PwPtrs pw_ptrs(uint64_t* buf, const PwLane& o, int lane = 0) {
    return PwPtrs{buf + o.a0, buf + o.a1, buf + o.b0, buf + o.b1, buf + o.d0, buf + o.d1,
                  buf + o.a0 - (lane >= 16 ? kWin : 0), buf + o.a1 - (lane >= 15 ? kWin : 0),
                  buf + o.b0 - (lane >= 9 ? kWin : 0), buf + o.b1 - (lane >= 8 ? kWin : 0)};
}
// Row T of a compile-time block at K without the mirror: run starts (logical window positions of
// lane 0's words) past the end are read one window lower; the one straddling run per lag goes
// through the lane-wrapped pointers.
template <int K, int T>
__device__ __forceinline__ void pw_load_row(const PwPtrs& pp, uint64_t& a0, uint64_t& a1, uint64_t& b0, uint64_t& b1) {
    constexpr int ka = ((K + (kWin - kLagR)) & kWinMask) - (kWin - kLagR);
    constexpr int kb = ((K + (kWin - kLagS)) & kWinMask) - (kWin - kLagS);
    constexpr int sa = ((K + (kWin - kLagR)) & kWinMask) + 64 * T;
    constexpr int sb = ((K + (kWin - kLagS)) & kWinMask) + 64 * T;
    static_assert((sa >= kWin || sa + 64 <= kWin || sa == kWin - 31) &&
                      (sb >= kWin || sb + 64 <= kWin || sb == kWin - 17),
                  "the lane-wrapped pointers cover exactly these straddling runs");
    constexpr int oa = ka + 64 * T - (sa >= kWin ? kWin : 0);
    constexpr int ob = kb + 64 * T - (sb >= kWin ? kWin : 0);
    constexpr bool xa = sa < kWin && sa + 64 > kWin, xb = sb < kWin && sb + 64 > kWin;
    a0 = NRNG_LD(&(xa ? pp.a0x : pp.a0)[oa]);
    a1 = NRNG_LD(&(xa ? pp.a1x : pp.a1)[oa]);
    b0 = NRNG_LD(&(xb ? pp.b0x : pp.b0)[ob]);
    b1 = NRNG_LD(&(xb ? pp.b1x : pp.b1)[ob]);
}
template <int K, int R, int... T>
__device__ __forceinline__ void pw_load_rows(const PwPtrs& pp, uint64_t (&a0)[R], uint64_t (&a1)[R], uint64_t (&b0)[R],
                                             uint64_t (&b1)[R], std::integer_sequence<int, T...>) {
    (pw_load_row<K, T>(pp, a0[T], a1[T], b0[T], b1[T]), ...);
}

template <int R, int K>
__device__ __forceinline__ void pw_gen_c(const PwPtrs& pp, uint64_t (&w0)[R], uint64_t (&w1)[R]) {
    static_assert(64 * R <= kLagS && 64 * R <= kMirror && K % 64 == 0 && K + 64 * R <= kWin, "row geometry");
    constexpr int ka = ((K + (kWin - kLagR)) & kWinMask) - (kWin - kLagR);
    constexpr int kb = ((K + (kWin - kLagS)) & kWinMask) - (kWin - kLagS);
    uint64_t a0[R], a1[R], b0[R], b1[R];
    if constexpr (NRNG_PW_NOMIRROR) {
        pw_load_rows<K>(pp, a0, a1, b0, b1, std::make_integer_sequence<int, R>{});
    } else {
#pragma unroll
        for (int t = 0; t < R; ++t) {
            a0[t] = NRNG_LD(&pp.a0[ka + 64 * t]);
            a1[t] = NRNG_LD(&pp.a1[ka + 64 * t]);
            b0[t] = NRNG_LD(&pp.b0[kb + 64 * t]);
            b1[t] = NRNG_LD(&pp.b1[kb + 64 * t]);
        }
    }
#pragma unroll
    for (int t = 0; t < R; ++t) {
        w0[t] = a0[t] + b0[t];
        w1[t] = a1[t] + b1[t];
        NRNG_ST(&pp.d0[K + 64 * t], w0[t]);
        NRNG_ST(&pp.d1[K + 64 * t], w1[t]);
        if (!NRNG_PW_NOMIRROR && K < kMirror) {
            NRNG_ST(&pp.d0[K + kWin + 64 * t], w0[t]);
            NRNG_ST(&pp.d1[K + kWin + 64 * t], w1[t]);
        }
    }
}

// Source-run offsets (words, relative to the per-lane pointers) of the block at position
// 256 ph: a warp-uniform constant-bank load per block instead of per-block mask arithmetic.
__constant__ int2 kPwPhaseOff[4] = {
    {((0 + (kWin - kLagR)) & kWinMask) - (kWin - kLagR), ((0 + (kWin - kLagS)) & kWinMask) - (kWin - kLagS)},
    {((256 + (kWin - kLagR)) & kWinMask) - (kWin - kLagR), ((256 + (kWin - kLagS)) & kWinMask) - (kWin - kLagS)},
    {((512 + (kWin - kLagR)) & kWinMask) - (kWin - kLagR), ((512 + (kWin - kLagS)) & kWinMask) - (kWin - kLagS)},
    {((768 + (kWin - kLagR)) & kWinMask) - (kWin - kLagR), ((768 + (kWin - kLagS)) & kWinMask) - (kWin - kLagS)}};
template <int R>
__device__ __forceinline__ void pw_gen_r(const PwPtrs& pp, uint32_t ph, uint64_t (&w0)[R], uint64_t (&w1)[R]) {
    static_assert(64 * R <= kLagS && 64 * R <= kMirror, "row geometry");
    const int2 kk = kPwPhaseOff[ph];
    const int K = (int)(kBlk * ph);
    uint64_t a0[R], a1[R], b0[R], b1[R];
#pragma unroll
    for (int t = 0; t < R; ++t) {
        a0[t] = NRNG_LD(&pp.a0[kk.x + 64 * t]);
        a1[t] = NRNG_LD(&pp.a1[kk.x + 64 * t]);
        b0[t] = NRNG_LD(&pp.b0[kk.y + 64 * t]);
        b1[t] = NRNG_LD(&pp.b1[kk.y + 64 * t]);
    }
#pragma unroll
    for (int t = 0; t < R; ++t) {
        w0[t] = a0[t] + b0[t];
        w1[t] = a1[t] + b1[t];
        NRNG_ST(&pp.d0[K + 64 * t], w0[t]);
        NRNG_ST(&pp.d1[K + 64 * t], w1[t]);
    }
#if NRNG_B1_MIRROR_BRANCH  // a real branch: the mirror stores are skipped in 3 blocks of 4
    if (__builtin_expect(ph == 0, 0)) {
        asm volatile("" ::: "memory");
#pragma unroll
        for (int t = 0; t < R; ++t) {
            NRNG_ST(&pp.d0[kWin + 64 * t], w0[t]);
            NRNG_ST(&pp.d1[kWin + 64 * t], w1[t]);
        }
        NRNG_SYNCWARP();
    }
#else
    if (ph == 0) {
#pragma unroll
        for (int t = 0; t < R; ++t) {
            NRNG_ST(&pp.d0[kWin + 64 * t], w0[t]);
            NRNG_ST(&pp.d1[kWin + 64 * t], w1[t]);
        }
    }
#endif
}

// One steady-state B1/B2 block (128 pairs) at compile-time window base K.
template <int M, int K>
__device__ __forceinline__ void pw_bm_block(const PwPtrs& pp, const TParams& tp, const Tables& tab, double2* o) {
    uint64_t wu[4], wv[4];
    pw_gen_c<4, K>(pp, wu, wv);
    double x[4], y[4];
    if (M == 1)
        b1_pairs<4>(wu, wv, tp, tab, x, y);
    else
        b2_pairs<4>(wu, wv, tp, tab, x, y);
#pragma unroll
    for (int u = 0; u < 4; ++u) __stcs(o + 32 * u, make_double2(x[u], y[u]));
    NRNG_SYNCWARP();
}

// The accepts of one step trimmed to the remaining quota `need` (exact stop, R5): m[u] keeps
// only the first `need` accepts in candidate order; returns the candidates consumed.  Called
// only for the step that reaches the quota (tot >= need).
__device__ __forceinline__ uint32_t polar_trim(const bool (&ok)[kPU], unsigned (&m)[kPU], uint32_t need,
                                               unsigned lt) {
    uint32_t used = 32 * kPU, rem = need;
#pragma unroll
    for (int u = 0; u < kPU; ++u) {
        const uint32_t nu = __popc(m[u]);
        if (rem == 0) {
            m[u] = 0;
        } else if (nu >= rem) {
            const unsigned last = __ballot_sync(kFull, ok[u] && (uint32_t)__popc(m[u] & lt) == rem - 1);
            const int l = __ffs(last) - 1;
            m[u] &= (l == 31) ? kFull : ((2u << l) - 1u);
            used = 32 * u + l + 1;
            rem = 0;
        } else {
            rem -= nu;
        }
    }
    return used;
}

// Stores of one Polar step: accepted candidate i (mask bit) -> output pair acc + its rank.
template <bool EP>
__device__ __forceinline__ void pw_polar_stores(const unsigned (&m)[kPU], const double (&ox)[kPU],
                                                const double (&oy)[kPU], const BulkParams& p, const Quota& qk,
                                                double2*& o, bool direct, uint32_t& acc, int lane, unsigned lt,
                                                uint32_t& jb) {
    if (EP) {  // the sequential mode's epoch layout (whole epochs: every pair is in range)
        // o = the slot of pair jb, the first of the epoch chunk (E >= 128 pairs) holding pair
        // acc; a step's <= 128 pairs span at most two chunks: pair j goes to o + (j - jb), plus
        // the jump to the next chunk once j - jb >= E
        const uint32_t E = 1u << p.log2E;
        const uint64_t jump = ((uint64_t)p.S << p.log2E) - E;
#pragma unroll
        for (int u = 0; u < kPU; ++u) {
            const uint32_t jj = acc + __popc(m[u] & lt) - jb;
            if ((m[u] >> lane) & 1u) __stcs(o + jj + (jj >= E ? jump : 0), make_double2(ox[u], oy[u]));
            acc += __popc(m[u]);
        }
        if (acc - jb >= E) {
            jb += E;
            o += jump + E;
        }
    } else if (direct) {
#pragma unroll
        for (int u = 0; u < kPU; ++u) {
            if ((m[u] >> lane) & 1u) __stcs(o + (acc + __popc(m[u] & lt)), make_double2(ox[u], oy[u]));
            acc += __popc(m[u]);
        }
    } else {
#pragma unroll
        for (int u = 0; u < kPU; ++u) {
            if ((m[u] >> lane) & 1u)
                store_pair(p.out, 2 * (qk.off + acc + __popc(m[u] & lt)), p.shift, p.n, ox[u], oy[u], true);
            acc += __popc(m[u]);
        }
    }
}

// One Polar step (128 candidates, one block) at compile-time base K; returns whether the
// quota was reached (exact stop: `used` = candidates consumed of this block).  The steady
// path (the step does not reach the quota: every step of a stream but its last) touches no
// mask after the ballots; the trim runs only in the last step.
template <int M, int K, bool EP = false, bool kDirect = false>  // kDirect: `direct` known true
__device__ __forceinline__ bool pw_polar_block(const PwPtrs& pp, const TParams& tp, const Tables& tab,
                                               const BulkParams& p, const Quota& qk, double2*& o, bool direct,
                                               uint32_t cnt, uint32_t& acc, uint32_t& used, int lane, unsigned lt,
                                               double* scr, uint32_t& jb) {
    if (kDirect) direct = true;
    uint64_t wa[kPU], wb[kPU];
    pw_gen_c<kPU, K>(pp, wa, wb);
    PolarCand c[kPU];
    bool ok[kPU];
    unsigned m[kPU];
#pragma unroll
    for (int u = 0; u < kPU; ++u) ok[u] = polar_candidate(wa[u], wb[u], c[u]);
#if NRNG_POLAR_SPLIT_STOP
    uint32_t tot = 0;
#pragma unroll
    for (int u = 0; u < kPU; ++u) {
        m[u] = __ballot_sync(kFull, ok[u]);
        tot += __popc(m[u]);
    }
    const bool stop = tot >= cnt - acc;
#else
    bool stop;
    used = polar_rank(ok, m, cnt - acc, lt, stop);
#endif
    double ox[kPU], oy[kPU];
    if constexpr (M == 5)
        p2_transform_compact<kPU>(c, ok, tp, tab, scr, lane, lt, ox, oy);
    else
        polar_transform<kPU>(c, tp, tab, ox, oy);
#if NRNG_POLAR_SPLIT_STOP
    if (__builtin_expect(!stop, 1)) {
        pw_polar_stores<EP>(m, ox, oy, p, qk, o, direct, acc, lane, lt, jb);
        used = 32 * kPU;
    } else {
        used = polar_trim(ok, m, cnt - acc, lt);
        pw_polar_stores<EP>(m, ox, oy, p, qk, o, direct, acc, lane, lt, jb);
    }
#else
    pw_polar_stores<EP>(m, ox, oy, p, qk, o, direct, acc, lane, lt, jb);
#endif
    NRNG_SYNCWARP();
    return stop;
}

// One Algorithm R step (128 candidates, one block) at compile-time base K: one normal per
// accepted candidate, ranked by ballot in candidate order, exact stop (R26).  `o` points at
// this stream's first output slot.
template <int K>
__device__ __forceinline__ bool pw_ratio_block(const PwPtrs& pp, const TParams& tp, const Tables& tab, double* o,
                                               uint32_t cnt, uint32_t& acc, uint32_t& used, int lane, unsigned lt) {
    uint64_t wa[kPU], wb[kPU];
    pw_gen_c<kPU, K>(pp, wa, wb);
    double x[kPU];
    bool ok[kPU];
    unsigned m[kPU];
    ratio_candidates<kPU>(wa, wb, tab, x, ok);
    bool stop;
    used = polar_rank(ok, m, cnt - acc, lt, stop);
#pragma unroll
    for (int u = 0; u < kPU; ++u) {
        if ((m[u] >> lane) & 1u) __stcs(o + (acc + __popc(m[u] & lt)), __fma_rn(tp.sigma, x[u], tp.mu));
        acc += __popc(m[u]);
    }
    NRNG_SYNCWARP();
    return stop;
}

// One Algorithm R1 step (128 candidates) at compile-time base K: R's step with the step-2.5
// pretests and the borderline logarithms gathered (ratio1_decide); the same output.
template <int K>
__device__ __forceinline__ bool pw_ratio1_block(const PwPtrs& pp, const TParams& tp, const Tables& tab, double* o,
                                                double* scr, uint32_t cnt, uint32_t& acc, uint32_t& used, int lane,
                                                unsigned lt) {
    uint64_t wa[kPU], wb[kPU];
    pw_gen_c<kPU, K>(pp, wa, wb);
    double Nu[kPU], x[kPU], a[kPU];
    int cls[kPU];
    ratio1_pretest<kPU>(wa, wb, Nu, x, a, cls);
    bool ok[kPU];
    ratio1_decide<kPU>(Nu, a, cls, tab, scr, lane, lt, ok);
    unsigned m[kPU];
    bool stop;
    used = polar_rank(ok, m, cnt - acc, lt, stop);
#pragma unroll
    for (int u = 0; u < kPU; ++u) {
        if ((m[u] >> lane) & 1u) __stcs(o + (acc + __popc(m[u] & lt)), __fma_rn(tp.sigma, x[u], tp.mu));
        acc += __popc(m[u]);
    }
    NRNG_SYNCWARP();
    return stop;
}

// EP: the sequential mode's epoch layout (pair j of stream k at slot (j >> log2E) S E + k E +
// (j & (E-1)), E >= 128 a power of two, equal quotas, whole 128-pair blocks): each block's 128
// pairs are still contiguous, only the block pointer (and Polar's per-pair slot) changes.
template <int M, int NW, bool EP = false>
__global__ void __launch_bounds__(NW * 32, 1) pw_kernel(BulkParams p) {
    extern __shared__ __align__(16) uint64_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr bool kStaged = pw_staged(M, EP);
    constexpr int kStride = pw_stride(M, EP);
    uint64_t* const buf = smem + warp * kStride;
    uint64_t* const stg = buf + kWin;  // kStaged: the next stream's ring row and counter
    if constexpr (kStaged) {
        if (p.s_begin + blockIdx.x * NW + warp < p.s_end) stage_state(stg, p, p.s_begin + blockIdx.x * NW + warp, lane);
    } else {
        prefetch_first_state(p, p.s_begin + blockIdx.x * NW + warp, lane);
    }
    const Tables tab = load_tables<NW * 32>(reinterpret_cast<double2*>(smem + NW * kStride));
    __syncthreads();
    const PwLane ol = pw_lane(lane);
    const PwPtrs pp = pw_ptrs(buf, ol, lane);
    const unsigned lt = lanemask_lt(lane);
    double* const scr = reinterpret_cast<double*>(smem + NW * kStride + kTabBytes / 8) + 32 * warp;  // M = 5, 7
    for (uint32_t k = p.s_begin + blockIdx.x * NW + warp; k < p.s_end; k += gridDim.x * NW) {
        const Quota qk = quota(p, k);
        if constexpr (kStaged) {
            stage_wait();
            NRNG_SYNCWARP();  // every lane's copies of stream k are visible to the warp
            if (qk.cnt == 0) {
                if (k + gridDim.x * NW < p.s_end) stage_state(stg, p, k + gridDim.x * NW, lane);
                continue;
            }
        } else {
            if (qk.cnt == 0) continue;
        }
        if constexpr (!kStaged && (M != 1 || NRNG_PREFETCH_B1)) prefetch_state<1>(p, k + gridDim.x * NW, lane);
        uint64_t* rk = p.ring + (uint64_t)k * kPitch;
        // x_{C-607+j} -> logical position 417 + j.  (Ring and counter loaded together; except in
        // B1's one-block-per-SM kernel, whose schedule came out 4% slower with it: measured.)
        auto win = [&](uint32_t j) { return buf + swz((kWin - kLagR) + j); };
        uint64_t C;
        if constexpr (kStaged) {
            if constexpr (NRNG_STAGE_RUNS && M >= 6)  // R, R1 (measured: R -3 to -4%; P, P2 within noise)
                C = load_staged_state(stg, buf, lane);
            else
                C = load_state_rot(stg, stg + kPitch, lane, win);
        } else if constexpr (M == 1 && NW == kPwWarps) {
            C = p.count[k];
            load_state(rk, C, lane, win, all_state_words);
        } else {
            C = load_state_rot(rk, p.count + k, lane, win);
        }
        NRNG_SYNCWARP();
        if constexpr (kStaged) {  // every lane has read the staging area: refill it with the next stream
            if (k + gridDim.x * NW < p.s_end) stage_state(stg, p, k + gridDim.x * NW, lane);
        } else if constexpr (M != 1 || NRNG_PREFETCH_B1) {
            prefetch_state<2>(p, k + gridDim.x * NW, lane);
        }
        uint64_t used;  // words consumed by this call
        if constexpr (M <= 2) {
            // pairs whose 16-byte outputs are all in range (odd n: the very last pair is not)
            const uint64_t safe_cnt = 2 * (qk.off + qk.cnt) <= p.n ? qk.cnt : qk.cnt - 1;
            const uint32_t nblk = (uint32_t)(safe_cnt / 128);
            double2* o = EP ? reinterpret_cast<double2*>(p.out) + pair_slot(p, qk.off, k, 0) + lane
                            : reinterpret_cast<double2*>(p.out + (2 * qk.off - p.shift)) + lane;
            uint32_t b = 0;
            auto adv = [&](uint32_t bn) {  // o -> the first pair of block bn (+ lane)
                if constexpr (EP)  // +128 pairs inside an epoch chunk (E >= 128, 128 | E), else to the next epoch's
                    o += ((128u * bn) & ((1u << p.log2E) - 1)) ? 128 : ((uint64_t)p.S << p.log2E) - (1u << p.log2E) + 128;
                else
                    o += 128;
            };
            // B2: unrolled over the 4 block positions (compile-time window offsets); B1: one
            // block body with the offsets from the constant bank (measured faster for B1: the
            // unrolled body issued 16% fewer instructions but scheduled worse, 79% vs 92% of
            // the issue bound)
            if constexpr (M == 2 || (M == 1 && NRNG_B1_UNROLL)) while (b < nblk) {  // 4 block positions per pass, compile-time window offsets
                pw_bm_block<M, 0>(pp, p.tp, tab, o);
                adv(b + 1);
                if (++b == nblk) break;
                pw_bm_block<M, 256>(pp, p.tp, tab, o);
                adv(b + 1);
                if (++b == nblk) break;
                pw_bm_block<M, 512>(pp, p.tp, tab, o);
                adv(b + 1);
                if (++b == nblk) break;
                pw_bm_block<M, 768>(pp, p.tp, tab, o);
                adv(b + 1);
                ++b;
            }
            else for (; b < nblk; ++b, adv(b)) {
                uint64_t wu[4], wv[4];
                pw_gen_r<4>(pp, b & 3, wu, wv);
                double x[4], y[4];
                if (M == 1)
                    b1_pairs<4>(wu, wv, p.tp, tab, x, y);
                else
                    b2_pairs<4>(wu, wv, p.tp, tab, x, y);
#pragma unroll
                for (int u = 0; u < 4; ++u) __stcs(o + 32 * u, make_double2(x[u], y[u]));
                NRNG_SYNCWARP();
            }
            uint32_t K = (256 * b) & kWinMask;
            for (uint64_t j0 = 128ull * b; j0 < qk.cnt; j0 += 32) {  // last rows, partial, unsafe pair
                uint64_t wu[1], wv[1];
                pw_gen<1, (M != 1 || NRNG_B1_UNROLL) && NRNG_PW_NOMIRROR>(buf, K, ol, wu, wv, lane);  // B1's runtime body keeps its mirror
                double x[1], y[1];
                if (M == 1)
                    b1_pairs<1>(wu, wv, p.tp, tab, x, y);
                else
                    b2_pairs<1>(wu, wv, p.tp, tab, x, y);
                if ((uint64_t)lane < qk.cnt - j0)
                    store_pair(p.out, 2 * (EP ? pair_slot(p, qk.off, k, j0 + lane) : qk.off + j0 + lane), p.shift, p.n,
                               x[0], y[0], true);
                NRNG_SYNCWARP();
                K = (K + 64) & kWinMask;
            }
            used = 2 * qk.cnt;
        } else if constexpr (M == 7) {
            // Algorithm R1: R with the step-2.5 pretests (reading R29); the same output.
            double* const o = p.out + (qk.off - p.shift);
            const uint32_t cnt = (uint32_t)qk.cnt;
            uint32_t acc = 0, blocks = 0, usedc = 0;
            for (;;) {
                if (pw_ratio1_block<0>(pp, p.tp, tab, o, scr, cnt, acc, usedc, lane, lt)) break;
                ++blocks;
                if (pw_ratio1_block<256>(pp, p.tp, tab, o, scr, cnt, acc, usedc, lane, lt)) break;
                ++blocks;
                if (pw_ratio1_block<512>(pp, p.tp, tab, o, scr, cnt, acc, usedc, lane, lt)) break;
                ++blocks;
                if (pw_ratio1_block<768>(pp, p.tp, tab, o, scr, cnt, acc, usedc, lane, lt)) break;
                ++blocks;
            }
            used = (uint64_t)kBlk * blocks + 2 * usedc;
        } else if constexpr (M == 6) {
            // Algorithm R: 128 candidates per step, one normal per accepted candidate (R26).
            double* const o = p.out + (qk.off - p.shift);
            const uint32_t cnt = (uint32_t)qk.cnt;
            uint32_t acc = 0, blocks = 0, usedc = 0;
            for (;;) {
                if (pw_ratio_block<0>(pp, p.tp, tab, o, cnt, acc, usedc, lane, lt)) break;
                ++blocks;
                if (pw_ratio_block<256>(pp, p.tp, tab, o, cnt, acc, usedc, lane, lt)) break;
                ++blocks;
                if (pw_ratio_block<512>(pp, p.tp, tab, o, cnt, acc, usedc, lane, lt)) break;
                ++blocks;
                if (pw_ratio_block<768>(pp, p.tp, tab, o, cnt, acc, usedc, lane, lt)) break;
                ++blocks;
            }
            used = (uint64_t)kBlk * blocks + 2 * usedc;
        } else {
            // Polar: 128 candidates (one 4-row block) per step, ranked by ballot, exact stop (R5).
            const bool direct = 2 * (qk.off + qk.cnt) <= p.n;
            double2* o = EP ? reinterpret_cast<double2*>(p.out) + pair_slot(p, qk.off, k, 0)
                            : reinterpret_cast<double2*>(p.out + (2 * qk.off - p.shift));
            const uint32_t cnt = (uint32_t)qk.cnt;
            uint32_t acc = 0, blocks = 0, usedc = 0, jb = 0;  // jb: EP's current epoch chunk
            // the steps of a stream whose outputs are all in range (every stream but perhaps a
            // call's last) run without the per-step range test
            auto steps = [&](auto kd) {
                constexpr bool KD = decltype(kd)::value;
                for (;;) {
                    if (pw_polar_block<M, 0, EP, KD>(pp, p.tp, tab, p, qk, o, direct, cnt, acc, usedc, lane, lt, scr, jb)) break;
                    ++blocks;
                    if (pw_polar_block<M, 256, EP, KD>(pp, p.tp, tab, p, qk, o, direct, cnt, acc, usedc, lane, lt, scr, jb)) break;
                    ++blocks;
                    if (pw_polar_block<M, 512, EP, KD>(pp, p.tp, tab, p, qk, o, direct, cnt, acc, usedc, lane, lt, scr, jb)) break;
                    ++blocks;
                    if (pw_polar_block<M, 768, EP, KD>(pp, p.tp, tab, p, qk, o, direct, cnt, acc, usedc, lane, lt, scr, jb)) break;
                    ++blocks;
                }
            };
            if (!EP && NRNG_POLAR_DIRECT_SPLIT && direct)
                steps(std::integral_constant<bool, true>{});
            else
                steps(std::integral_constant<bool, false>{});
            used = (uint64_t)kBlk * blocks + 2 * usedc;
        }
        // write back the last min(used, 607) consumed words (word i at logical i mod 1024)
        const uint32_t nw = used < (uint64_t)kLagR ? (uint32_t)used : (uint32_t)kLagR;
        const uint32_t pos0 = (uint32_t)((used - nw) & kWinMask);
        const uint32_t slot0 = (uint32_t)((C + used - nw) % kLagR);
        store_state(rk, slot0, nw, lane, [&](uint32_t j) { return &buf[swz((pos0 + j) & kWinMask)]; });
        if (lane == 0) p.count[k] = C + used;
        NRNG_SYNCWARP();
    }
}

// ------------------------------------------------------------------ tiny quotas
// Calls that give every stream only a few pairs (the C4 sweep: n <= 2^22 over 2^16 streams
// gives 1-32 pairs per stream) are bound by per-stream latency and state traffic, not
// arithmetic, and a warp would spend most of its time on one stream's state round trip.
// Here one THREAD owns a stream and generates its words straight through the HBM ring in
// the canonical layout: x_{C+i} = ring[(C+i) mod 607] + ring[(C+i+334) mod 607], written
// back in place (exactly the recurrence), in chunks of 4 pairs whose 2 x 4 per source
// words are loaded together (ILP) and transformed as one 4-wide batch.  Only the words
// actually used are touched; unconsumed words of a Polar chunk are not written back.
constexpr int kTinyThreads = 128;
#ifndef NRNG_TINY_MAX
#define NRNG_TINY_MAX 32
#endif
constexpr uint64_t kTinyMaxPairs = NRNG_TINY_MAX;  // per-stream quota routed here

// x_{n+t}, t < CW, where ring position a holds x_{n-607} (valid for CW <= 273).
template <int CW>
__device__ __forceinline__ void ring_peek(const uint64_t* __restrict__ r, uint32_t a, uint64_t (&w)[CW]) {
    uint32_t b = a + (kLagR - kLagS);
    b = b >= (uint32_t)kLagR ? b - kLagR : b;
    uint64_t xa[CW], xb[CW];
#pragma unroll
    for (int t = 0; t < CW; ++t) {
        uint32_t pa = a + t, pb = b + t;
        pa = pa >= (uint32_t)kLagR ? pa - kLagR : pa;
        pb = pb >= (uint32_t)kLagR ? pb - kLagR : pb;
        xa[t] = r[pa];
        xb[t] = r[pb];
    }
#pragma unroll
    for (int t = 0; t < CW; ++t) w[t] = xa[t] + xb[t];
}
// Write back the first `used` words (x_n at its own slot) and advance the cursor.
template <int CW>
__device__ __forceinline__ void ring_commit(uint64_t* __restrict__ r, uint32_t& a, const uint64_t (&w)[CW],
                                            uint32_t used) {
#pragma unroll
    for (int t = 0; t < CW; ++t) {
        uint32_t pa = a + t;
        pa = pa >= (uint32_t)kLagR ? pa - kLagR : pa;
        if ((uint32_t)t < used) r[pa] = w[t];
    }
    a += used;
    a = a >= (uint32_t)kLagR ? a - kLagR : a;
}

template <int V>  // 1, 2, 3 = B1, B2, B3; 4 = Polar; 5 = P2; 6 = R (units: normals, one per accept)
__global__ void __launch_bounds__(kTinyThreads) tiny_kernel(BulkParams p) {
    __shared__ double2 tabs[kTabBytes / 16];
    const Tables tab = load_tables<kTinyThreads>(tabs);
    __syncthreads();
    const uint32_t k = p.s_begin + blockIdx.x * kTinyThreads + threadIdx.x;
    if (k >= p.s_end) return;
    const Quota qk = quota(p, k);
    if (qk.cnt == 0) return;
    const uint64_t C = p.count[k];
    uint64_t* r = p.ring + (uint64_t)k * kPitch;
    uint32_t a = (uint32_t)(C % kLagR);
    uint64_t used = 0;
    constexpr int per = (V == 3) ? 3 : 2;
    constexpr int CW = 4 * per;
    uint32_t j = 0;  // pairs done
    while (j < qk.cnt) {
        uint64_t w[CW];
        ring_peek<CW>(r, a, w);
        double x[4], y[4];
        uint32_t take, words;
        if (V == 6) {
            uint64_t wu[4], wv[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                wu[t] = w[2 * t];
                wv[t] = w[2 * t + 1];
            }
            double xr[4];
            bool ok[4];
            ratio_candidates<4>(wu, wv, tab, xr, ok);
            uint32_t got = 0, cand = 4;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                if (ok[t] && j + got < qk.cnt) {
                    const uint64_t g = qk.off + j + got;
                    if (g < p.n) p.out[g - p.shift] = __fma_rn(p.tp.sigma, xr[t], p.tp.mu);
                    if (j + ++got == qk.cnt) cand = t + 1;  // exact stop
                }
            }
            take = got;
            words = 2 * cand;
        } else if (V >= 4) {
            PolarCand c[4];
            bool ok[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) ok[t] = polar_candidate(w[2 * t], w[2 * t + 1], c[t]);
            if (V == 5)
                p2_transform<4>(c, p.tp, tab, x, y);
            else
                polar_transform<4>(c, p.tp, tab, x, y);
            uint32_t got = 0, cand = 4;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                if (ok[t] && j + got < qk.cnt) {
                    store_pair(p.out, 2 * pair_slot(p, qk.off, k, j + got), p.shift, p.n, x[t], y[t], p.aligned);
                    if (j + ++got == qk.cnt) cand = t + 1;  // exact stop: nothing after the last accept
                }
            }
            take = got;
            words = 2 * cand;
        } else {
            if (V == 3) {
                uint64_t w1[4], w2[4], w3[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    w1[t] = w[3 * t];
                    w2[t] = w[3 * t + 1];
                    w3[t] = w[3 * t + 2];
                }
                b3_pairs<4>(w1, w2, w3, p.tp, tab, x, y);
            } else {
                uint64_t wu[4], wv[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    wu[t] = w[2 * t];
                    wv[t] = w[2 * t + 1];
                }
                if (V == 1)
                    b1_pairs<4>(wu, wv, p.tp, tab, x, y);
                else
                    b2_pairs<4>(wu, wv, p.tp, tab, x, y);
            }
            take = qk.cnt - j < 4 ? (uint32_t)(qk.cnt - j) : 4u;
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if ((uint32_t)t < take)
                    store_pair(p.out, 2 * pair_slot(p, qk.off, k, j + t), p.shift, p.n, x[t], y[t], p.aligned);
            words = per * take;
        }
        ring_commit<CW>(r, a, w, words);
        used += words;
        j += take;
    }
    p.count[k] = C + used;
}

// ------------------------------------------------------------------ mid-size quotas
// Per-stream quotas of a few dozen pairs (the C4 sweep at n = 2^21..2^23 over 2^16 streams):
// too short for the shared-memory window (the full 4.8 KB state load would dominate) and too
// long for one thread per stream (whose 8-byte ring accesses are uncoalesced).  One WARP owns a
// stream and steps through the HBM ring in the canonical layout, 32 units per step (a pair for
// B1/B2, a candidate for Polar; lane l takes the step's words 2l, 2l+1): x_{C+i} =
// ring[(C+i) mod 607] + ring[(C+i+334) mod 607], written back in place.  Within a step the
// lanes' words are 64 apart at most (< 273), so every source is older than the step: loads
// first, then the new words, then a __syncwarp before the next step reads them.  Only the words
// a call consumes are read or written (Polar's exact stop leaves later candidates untouched).
constexpr int kMidWarps = 4;
#ifndef NRNG_MID_MIN
#define NRNG_MID_MIN 12
#endif
#ifndef NRNG_MID_MAX
#define NRNG_MID_MAX 128
#endif
constexpr uint64_t kMidMinPairs = NRNG_MID_MIN, kMidMaxPairs = NRNG_MID_MAX;  // per-stream quota routed here

template <int V>  // 1, 2, 3 = B1, B2, B3; 4 = Polar; 5 = P2; 6 = R (units: normals, one per accept)
__global__ void __launch_bounds__(kMidWarps * 32) mid_kernel(BulkParams p) {
    __shared__ double2 tabs[kTabBytes / 16];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t k0 = p.s_begin + blockIdx.x * kMidWarps + warp, stride = gridDim.x * kMidWarps;
    // the counters of the warp's next 32 streams, one per lane (a stream's ring reads need its
    // counter: loading them a batch ahead leaves one memory latency per stream, not two); the
    // first batch is in flight while the block loads its ln table
    auto counters = [&](uint32_t kb) {
        const uint64_t kk = kb + (uint64_t)lane * stride;
        return kk < p.s_end ? p.count[kk] : 0ull;
    };
    uint64_t cbatch = counters(k0);
    const Tables tab = load_tables<kMidWarps * 32>(tabs);
    __syncthreads();
    const unsigned lt = lanemask_lt(lane);
    uint32_t i = 0;
    for (uint32_t k = k0; k < p.s_end; k += stride, ++i) {
        if (i == 32) {
            cbatch = counters(k);
            i = 0;
        }
        const Quota qk = quota(p, k);
        if (qk.cnt == 0) continue;
        const uint64_t C = __shfl_sync(kFull, cbatch, i);
        uint64_t* r = p.ring + (uint64_t)k * kPitch;
        const uint32_t c0 = (uint32_t)(C % kLagR);
        uint32_t i0 = 0;  // words of the call consumed before this step
        if constexpr (V <= 3) {
        uint32_t j = 0;   // pairs delivered
        while (j < qk.cnt) {
            // this lane's words: call-relative i0 + per l + t (per = 3 for B3, else 2)
            constexpr int per = V == 3 ? 3 : 2;
            uint32_t pa[per], pb[per];
            uint64_t w[per];
            {
                uint32_t a = (c0 + i0 + per * lane) % kLagR;
                uint32_t b = a + (kLagR - kLagS);
                b = b >= (uint32_t)kLagR ? b - kLagR : b;
#pragma unroll
                for (int t = 0; t < per; ++t) {
                    pa[t] = a;
                    pb[t] = b;
                    a = a + 1 == (uint32_t)kLagR ? 0 : a + 1;
                    b = b + 1 == (uint32_t)kLagR ? 0 : b + 1;
                }
                uint64_t xa[per], xb[per];
#pragma unroll
                for (int t = 0; t < per; ++t) xa[t] = r[pa[t]], xb[t] = r[pb[t]];
#pragma unroll
                for (int t = 0; t < per; ++t) w[t] = xa[t] + xb[t];
            }
            uint32_t words;  // words this step consumes (stores only those)
            if constexpr (V <= 3) {
                double x[1], y[1];
                if constexpr (V == 3) {
                    const uint64_t w1[1] = {w[0]}, w2[1] = {w[1]}, w3[1] = {w[per - 1]};
                    b3_pairs<1>(w1, w2, w3, p.tp, tab, x, y);
                } else {
                    const uint64_t wu[1] = {w[0]}, wv[1] = {w[1]};
                    if (V == 1)
                        b1_pairs<1>(wu, wv, p.tp, tab, x, y);
                    else
                        b2_pairs<1>(wu, wv, p.tp, tab, x, y);
                }
                const uint32_t take = qk.cnt - j < 32 ? (uint32_t)(qk.cnt - j) : 32u;
                if ((uint32_t)lane < take)
                    store_pair(p.out, 2 * pair_slot(p, qk.off, k, j + lane), p.shift, p.n, x[0], y[0], p.aligned);
                words = per * take;
                j += take;
            }
            if ((uint32_t)(per * lane) < words) {  // write back the consumed words in place
#pragma unroll
                for (int t = 0; t < per; ++t) r[pa[t]] = w[t];
            }
            i0 += words;
            NRNG_SYNCWARP();
        }
        } else {
        uint32_t j = 0;   // accepted units delivered
        // Polar/P2/R: a lane's words of the step starting at call word s are s + 2l, s + 2l + 1;
        // the next step's sources are loaded while this step transforms, once its ballot shows
        // another step is needed: they are never words of this step (those are < 64 words
        // behind; the lags are 273 and 607), so one memory latency per stream, not per step.
        auto sources = [&](uint32_t s, uint32_t (&pa)[2], uint64_t (&xa)[2], uint64_t (&xb)[2]) {
            uint32_t a = (c0 + s + 2 * lane) % kLagR;
            uint32_t b = a + (kLagR - kLagS);
            b = b >= (uint32_t)kLagR ? b - kLagR : b;
            uint32_t pb[2];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                pa[t] = a;
                pb[t] = b;
                a = a + 1 == (uint32_t)kLagR ? 0 : a + 1;
                b = b + 1 == (uint32_t)kLagR ? 0 : b + 1;
            }
#pragma unroll
            for (int t = 0; t < 2; ++t) xa[t] = r[pa[t]], xb[t] = r[pb[t]];
        };
        uint32_t pa[2];
        uint64_t xa[2], xb[2];
        sources(0, pa, xa, xb);
        for (;;) {
            const uint64_t w[2] = {xa[0] + xb[0], xa[1] + xb[1]};
            bool ok;
            double x[1], y[1];
            PolarCand c[1];
            if constexpr (V == 6) {
                const uint64_t wu[1] = {w[0]}, wv[1] = {w[1]};
                bool okr[1];
                ratio_candidates<1>(wu, wv, tab, x, okr);
                ok = okr[0];
            } else {
                ok = polar_candidate(w[0], w[1], c[0]);
            }
            const unsigned m = __ballot_sync(kFull, ok);
            const uint32_t need = (uint32_t)(qk.cnt - j), rank = __popc(m & lt), got = __popc(m);
            const bool more = got < need;
            uint32_t npa[2];
            uint64_t nxa[2], nxb[2];
            if (more) sources(i0 + 64, npa, nxa, nxb);
            if constexpr (V == 5)
                p2_transform<1>(c, p.tp, tab, x, y);
            else if constexpr (V == 4)
                polar_transform<1>(c, p.tp, tab, x, y);
            if (ok && rank < need) {
                if constexpr (V == 6) {
                    const uint64_t g = qk.off + j + rank;  // one normal per accepted candidate
                    if (g < p.n) p.out[g - p.shift] = __fma_rn(p.tp.sigma, x[0], p.tp.mu);
                } else {
                    store_pair(p.out, 2 * pair_slot(p, qk.off, k, j + rank), p.shift, p.n, x[0], y[0], p.aligned);
                }
            }
            uint32_t words;  // words this step consumes (stores only those)
            if (!more) {  // exact stop: nothing after the need-th accept is consumed
                const unsigned last = __ballot_sync(kFull, ok && rank == need - 1);
                words = 2 * (uint32_t)__ffs(last);
                j += need;
            } else {
                words = 64;
                j += got;
            }
            if ((uint32_t)(2 * lane) < words) r[pa[0]] = w[0], r[pa[1]] = w[1];  // write back in place
            i0 += words;
            NRNG_SYNCWARP();
            if (!more) break;
#pragma unroll
            for (int t = 0; t < 2; ++t) pa[t] = npa[t], xa[t] = nxa[t], xb[t] = nxb[t];
        }
        }
        if (lane == 0) p.count[k] = C + i0;
        NRNG_SYNCWARP();
    }
}

// ------------------------------------------------------------------ test hooks
// nrng_uniform: one uniform per slot, stream-major (units = uniforms).
__global__ void __launch_bounds__(kWarpsPerBlock * 32) uniform_kernel(BulkParams p) {
    extern __shared__ __align__(16) uint64_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpLFG L;
    L.buf = smem + warp * kWinAlloc;
    for (uint32_t k = p.s_begin + blockIdx.x * kWarpsPerBlock + warp; k < p.s_end;
         k += gridDim.x * kWarpsPerBlock) {
        const Quota qk = quota(p, k);
        if (qk.cnt == 0) continue;
        const uint64_t C = p.count[k];
        uint64_t* rk = p.ring + (uint64_t)k * kPitch;
        lfg_load(L, rk, C, lane);
        for (uint64_t j0 = 0; j0 < qk.cnt; j0 += 32) {
            lfg_ensure(L, lane, 32);
            const uint64_t left = qk.cnt - j0;
            const uint32_t active = left < 32 ? (uint32_t)left : 32u;
            if ((uint32_t)lane < active) {
                const uint64_t g = qk.off + j0 + lane;
                p.out[g - p.shift] = (double)ukey(NRNG_LD(&L.buf[(L.wc + lane) & kWinMask])) * 0x1p-53;  // exact
            }
            L.wc += active;
            NRNG_SYNCWARP();
        }
        lfg_store(L, rk, C, lane);
        if (lane == 0) p.count[k] = C + (L.wc - kW0);
        NRNG_SYNCWARP();
    }
}

// nrng_polar_mask: every stream advances exactly `cand` candidates.
__global__ void __launch_bounds__(kWarpsPerBlock * 32) polar_mask_kernel(BulkParams p, uint8_t* __restrict__ mask,
                                                                         uint64_t cand) {
    extern __shared__ __align__(16) uint64_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpLFG L;
    L.buf = smem + warp * kWinAlloc;
    for (uint32_t k = p.s_begin + blockIdx.x * kWarpsPerBlock + warp; k < p.s_end;
         k += gridDim.x * kWarpsPerBlock) {
        const uint64_t C = p.count[k];
        uint64_t* rk = p.ring + (uint64_t)k * kPitch;
        lfg_load(L, rk, C, lane);
        for (uint64_t j0 = 0; j0 < cand; j0 += 32) {
            lfg_ensure(L, lane, 64);
            const uint64_t left = cand - j0;
            const uint32_t active = left < 32 ? (uint32_t)left : 32u;
            if ((uint32_t)lane < active) {
                const ulonglong2 xw = NRNG_LD(reinterpret_cast<const ulonglong2*>(&L.buf[(L.wc + 2 * lane) & kWinMask]));
                PolarCand pc;
                mask[(uint64_t)k * cand + j0 + lane] = polar_candidate(xw.x, xw.y, pc) ? 1 : 0;
            }
            L.wc += 2 * active;
            NRNG_SYNCWARP();
        }
        lfg_store(L, rk, C, lane);
        if (lane == 0) p.count[k] = C + (L.wc - kW0);
        NRNG_SYNCWARP();
    }
}

// nrng_transform_from_uniforms: one thread per pair; the given uniforms (multiples of
// 2^-53 in [0,1)) are turned back into the words the stream would hold, so this runs
// exactly the device code of the bulk kernels.
constexpr int kTransformThreads = 256;
__device__ __forceinline__ uint64_t word_of(double u) { return __double2ull_rn(u * 0x1p53) << 11; }
__global__ void __launch_bounds__(kTransformThreads) transform_kernel(const double* __restrict__ u, uint64_t n_pairs, double* __restrict__ out,
                                 uint8_t* __restrict__ mask, TParams tp, int method) {
    __shared__ double2 tabs[kTabBytes / 16];
    const Tables tab = load_tables<kTransformThreads>(tabs);
    __syncthreads();
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n_pairs;
         j += (uint64_t)gridDim.x * blockDim.x) {
        double x[1] = {__longlong_as_double(0x7ff8000000000000ULL)}, y[1] = {x[0]};
        if (method == 1 || method == 2) {
            const uint64_t wu[1] = {word_of(u[2 * j])}, wv[1] = {word_of(u[2 * j + 1])};
            if (method == 1)
                b1_pairs<1>(wu, wv, tp, tab, x, y);
            else
                b2_pairs<1>(wu, wv, tp, tab, x, y);
        } else if (method == 3) {
            const uint64_t w1[1] = {word_of(u[3 * j])}, w2[1] = {word_of(u[3 * j + 1])}, w3[1] = {word_of(u[3 * j + 2])};
            b3_pairs<1>(w1, w2, w3, tp, tab, x, y);
        } else if (method == 7) {
            const uint64_t wu[1] = {word_of(u[2 * j])}, wv[1] = {word_of(u[2 * j + 1])};
            double Nu[1], xr[1], a[1];
            int cls[1];
            ratio1_pretest<1>(wu, wv, Nu, xr, a, cls);
            bool ok = cls[0] == 1;
            if (cls[0] == 0) {  // step 3 (the kernel path gathers these; here one per thread)
                double L[1];
                fast_log<1>(Nu, -53, tab, L);
                ok = !(a[0] > __dmul_rn(-4.0, L[0]));
            }
            if (mask) mask[j] = (uint8_t)((ok ? 1 : 0) | (cls[0] << 1));
            if (ok) x[0] = __fma_rn(tp.sigma, xr[0], tp.mu);
            y[0] = xr[0];
        } else if (method == 6) {
            const uint64_t wu[1] = {word_of(u[2 * j])}, wv[1] = {word_of(u[2 * j + 1])};
            double xr[1];
            bool ok[1];
            ratio_candidates<1>(wu, wv, tab, xr, ok);
            if (mask) mask[j] = ok[0] ? 1 : 0;
            if (ok[0]) x[0] = __fma_rn(tp.sigma, xr[0], tp.mu);
            y[0] = xr[0];
        } else {
            PolarCand pc[1];
            const bool ok = polar_candidate(word_of(u[2 * j]), word_of(u[2 * j + 1]), pc[0]);
            if (mask) mask[j] = ok ? 1 : 0;
            if (ok) {
                if (method == 5)
                    p2_transform<1>(pc, tp, tab, x, y);
                else
                    polar_transform<1>(pc, tp, tab, x, y);
            }
        }
        out[2 * j] = x[0];
        out[2 * j + 1] = y[0];
    }
}

// ------------------------------------------------------------------ validation stats
// Block partials of sum (x-c)^k, k = 1..4 (fp64, compensated: each sum carries its running
// rounding error, Neumaier's variant of Kahan summation, through the thread loop, the warp
// and block reductions and the final pass -- the 2^34-deviate runs add ~2^15 terms per
// thread), min, max, and a K-bin histogram (shared-memory int counters -> global u64
// atomics).  A second kernel reduces the block partials in a fixed order (deterministic).
constexpr int kStatsThreads = 256;
constexpr int kStatsCells = 2048;  // uniform cells over [edges[0], edges[K-2]] for the bin lookup
constexpr int kStatsPartial = 10;  // per block: 4 sums, 4 compensations, min, max
// s + v with the rounding error of the addition accumulated into c (Neumaier).
__device__ __forceinline__ void comp_add(double& s, double& c, double v) {
    const double t = __dadd_rn(s, v);
    c = __dadd_rn(c, fabs(s) >= fabs(v) ? __dadd_rn(__dadd_rn(s, -t), v) : __dadd_rn(__dadd_rn(v, -t), s));
    s = t;
}
__global__ void __launch_bounds__(kStatsThreads) stats_partial_kernel(const double* __restrict__ x, uint64_t n,
                                                                      double center, const double* __restrict__ edges,
                                                                      int K, double* __restrict__ partial,
                                                                      unsigned long long* __restrict__ hist) {
    __shared__ double red[kStatsPartial][kStatsThreads / 32];
    __shared__ unsigned int sh[1024];
    __shared__ double se[1023];
    __shared__ unsigned short cell[kStatsCells];  // edges <= the cell's left end (a lower bound)
    for (int b = threadIdx.x; b < K; b += blockDim.x) sh[b] = 0;
    for (int b = threadIdx.x; b < K - 1; b += blockDim.x) se[b] = edges[b];
    __syncthreads();
    // bin(v) = #edges <= v (K-1 edges, bins 0..K-1).  The cell of v gives a starting count that
    // is corrected by short walks in both directions, so the result is exact whatever the
    // rounding of the cell index (a binary search over 1023 edges per element cost 10 dependent
    // shared loads; this costs one table load and one or two edge comparisons).
    const double lo = se[0], hi = se[K - 2];
    const double inv_w = hi > lo ? kStatsCells / (hi - lo) : 0.0;
    for (int c = threadIdx.x; c < kStatsCells; c += blockDim.x) {
        const double v = lo + (hi - lo) * c / kStatsCells;
        int a = 0, b = K - 1;  // count of edges <= v by binary search (once per block)
        while (a < b) {
            const int mid = (a + b) >> 1;
            if (v < se[mid]) b = mid; else a = mid + 1;
        }
        cell[c] = (unsigned short)a;
    }
    __syncthreads();
    double s[4] = {0, 0, 0, 0}, cs[4] = {0, 0, 0, 0};
    double mn = __longlong_as_double(0x7ff0000000000000ULL), mx = -mn;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const double v = x[i];
        const double d = __dadd_rn(v, -center);
        const double d2 = __dmul_rn(d, d);
        comp_add(s[0], cs[0], d);
        comp_add(s[1], cs[1], d2);
        comp_add(s[2], cs[2], __dmul_rn(d2, d));
        comp_add(s[3], cs[3], __dmul_rn(d2, d2));
        mn = fmin(mn, v);
        mx = fmax(mx, v);
        int b;
        if (v < lo) {
            b = 0;
        } else if (!(v < hi)) {  // v >= hi (and NaN, as the binary search placed it)
            b = K - 1;
        } else {
            int c = (int)((v - lo) * inv_w);
            c = c < 0 ? 0 : (c >= kStatsCells ? kStatsCells - 1 : c);
            b = cell[c];
            while (b > 0 && v < se[b - 1]) --b;
            while (b < K - 1 && v >= se[b]) ++b;
        }
        atomicAdd(&sh[b], 1u);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        for (int o = 16; o > 0; o >>= 1) {
            const double ws = __shfl_xor_sync(kFull, s[t], o), wc = __shfl_xor_sync(kFull, cs[t], o);
            comp_add(s[t], cs[t], ws);
            cs[t] = __dadd_rn(cs[t], wc);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(kFull, mn, o));
        mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
    }
    if (lane == 0) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            red[t][warp] = s[t];
            red[4 + t][warp] = cs[t];
        }
        red[8][warp] = mn;
        red[9][warp] = mx;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        const int t = threadIdx.x;
        double v = red[t][0], c = red[4 + t][0];
        for (int w = 1; w < kStatsThreads / 32; ++w) {
            comp_add(v, c, red[t][w]);
            c = __dadd_rn(c, red[4 + t][w]);
        }
        partial[blockIdx.x * kStatsPartial + t] = v;
        partial[blockIdx.x * kStatsPartial + 4 + t] = c;
    } else if (threadIdx.x < 6) {
        const int t = threadIdx.x + 4;  // 8: min, 9: max
        double v = red[t][0];
        for (int w = 1; w < kStatsThreads / 32; ++w) v = t == 8 ? fmin(v, red[t][w]) : fmax(v, red[t][w]);
        partial[blockIdx.x * kStatsPartial + t] = v;
    }
    for (int b = threadIdx.x; b < K; b += blockDim.x)
        if (sh[b]) atomicAdd(&hist[b], (unsigned long long)sh[b]);
}

// sums[0..3] = the compensated power sums (sum + accumulated error), sums[4] = min, [5] = max.
// Warp t reduces quantity t: lane l combines blocks l, l + 32, ... in order, then a fixed
// xor-shuffle tree combines the lanes (a deterministic order for a given block count).
constexpr int kStatsFinalThreads = 6 * 32;
__global__ void __launch_bounds__(kStatsFinalThreads) stats_final_kernel(const double* __restrict__ partial,
                                                                         int nblocks, double* __restrict__ sums) {
    const int t = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (t < 4) {
        double v = 0.0, c = 0.0;
        for (int b = lane; b < nblocks; b += 32) {
            comp_add(v, c, partial[b * kStatsPartial + t]);
            c = __dadd_rn(c, partial[b * kStatsPartial + 4 + t]);
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ws = __shfl_xor_sync(kFull, v, o), wc = __shfl_xor_sync(kFull, c, o);
            comp_add(v, c, ws);
            c = __dadd_rn(c, wc);
        }
        if (lane == 0) sums[t] = __dadd_rn(v, c);
    } else {
        const int q = 4 + t;  // 8: min, 9: max
        double v = t == 4 ? __longlong_as_double(0x7ff0000000000000ULL) : __longlong_as_double(0xfff0000000000000ULL);
        for (int b = lane; b < nblocks; b += 32)
            v = t == 4 ? fmin(v, partial[b * kStatsPartial + q]) : fmax(v, partial[b * kStatsPartial + q]);
        for (int o = 16; o > 0; o >>= 1) {
            const double w = __shfl_xor_sync(kFull, v, o);
            v = t == 4 ? fmin(v, w) : fmax(v, w);
        }
        if (lane == 0) sums[t] = v;
    }
}

// ------------------------------------------------------------------ goodness of fit
// Fine histogram of p = Phi((x - mu)/sigma) over K = 2^log2K equal-probability bins
// (global u32 counters): the input of the KS and Anderson-Darling gates computed on the
// host from the (all-reduced) histogram.  Validation only -- never in the timed region.
__global__ void gof_hist_kernel(const double* __restrict__ x, uint64_t n, double mu, double inv_sigma, int log2K,
                                unsigned int* __restrict__ hist) {
    const double K = (double)(1u << log2K);
    const unsigned kmax = (1u << log2K) - 1;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const double p = normcdf((x[i] - mu) * inv_sigma);
        unsigned b = (unsigned)(p * K);
        b = b > kmax ? kmax : b;
        atomicAdd(&hist[b], 1u);
    }
}

// ------------------------------------------------------------------ serial correlation
// Lagged products for the serial-correlation gate:
// S_k = sum_i d_i d_{i+k}, d_i = x_i - center, k = 0..127 (K <= 127 are written).  Tile t
// covers x[t T, t T + T + 136) staged in shared memory (zero past n); blocks stride over the
// tiles (a fixed grid of min(#tiles, kCorrGrid) blocks, independent of the device, so the
// summation order is deterministic) and write partial[b][k]; the host sums the blocks.
// Register blocking: thread (half h, i-phase r = 0..7, lag phase g = 0..7) owns the 16 lags
// k = g + 8 j and the i = r (mod 8) of its half-tile, keeping the 16 values d_{i+g+8j} in a
// register ring: each step (i += 8) is one broadcast load of d_i, one load of the new
// d_{i+g+128} and 16 FMAs -- FP64-bound instead of two shared loads per FMA.
constexpr int kCorrTile = 4096;
constexpr int kCorrMaxLag = 127;
constexpr int kCorrPad = 136;  // 128 lags + one 8-step stride of lookahead
constexpr unsigned kCorrGrid = 2048;
__global__ void __launch_bounds__(128) serial_corr_kernel(const double* __restrict__ x, uint64_t n, double center,
                                                          int K, double* __restrict__ partial) {
    __shared__ double d[kCorrTile + kCorrPad];
    static_assert(16 * 129 <= kCorrTile + kCorrPad, "the reduction reuses the tile");
    const int t = threadIdx.x, h = t >> 6, r = t & 7, g = (t >> 3) & 7;
    const uint64_t tiles = (n + kCorrTile - 1) / kCorrTile;
    double acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.0;
    for (uint64_t tt = blockIdx.x; tt < tiles; tt += gridDim.x) {
        const uint64_t base = tt * kCorrTile;
        __syncthreads();
        for (int j = t; j < kCorrTile + kCorrPad; j += blockDim.x) {
            const uint64_t i = base + j;
            d[j] = i < n ? x[i] - center : 0.0;  // zero padding past n contributes nothing
        }
        __syncthreads();
        const int i0 = h * (kCorrTile / 2) + r;  // this thread's first i in the tile
        double w[16];                            // ring: slot (j + s) & 15 holds d[i + g + 8 j] at step s
#pragma unroll
        for (int j = 0; j < 16; ++j) w[j] = d[i0 + g + 8 * j];
        for (int m = 0; m < kCorrTile / 2 / 8; m += 16) {
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                const int i = i0 + 8 * (m + s);
                const double di = d[i];
#pragma unroll
                for (int j = 0; j < 16; ++j) acc[j] = __fma_rn(di, w[(j + s) & 15], acc[j]);
                w[s & 15] = d[i + g + 128];
            }
        }
    }
    __syncthreads();
    double (*red)[129] = reinterpret_cast<double (*)[129]>(d);  // [j][thread], padded
#pragma unroll
    for (int j = 0; j < 16; ++j) red[j][t] = acc[j];
    __syncthreads();
    // lag k = g + 8 j collects the 16 threads (h, r) with that (g, j), in a fixed order
    const int k = t, kg = k & 7, kj = k >> 3;
    double sum = 0.0;
    for (int hh = 0; hh < 2; ++hh)
        for (int rr = 0; rr < 8; ++rr) sum += red[kj][hh * 64 + kg * 8 + rr];
    if (k <= K) partial[(uint64_t)blockIdx.x * (K + 1) + k] = sum;
}

}  // namespace nrng
