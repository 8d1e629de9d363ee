// nrng_kernels.cuh -- the sm_100a kernels of the hot path.
//
// One warp owns one LFG stream at a time (607 x u64 of state is too large for a
// thread; the lag structure gives 256 independent words per refill).  Warps stride
// over streams, persistent grid sized to the SM count x resident blocks.
#pragma once
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
    uint32_t s_begin, s_end;
    TParams tp;
    int aligned;
};

// Per-block shared memory: [NW x kWinAlloc u64 windows][tables][per-kernel extras].
// The bulk kernels come in two block shapes: NW = 4 warps (small stream counts: spread
// over all SMs) and NW = kBigBlock warps, one block per SM (the tables are stored once per
// SM instead of once per 4 warps, which is what lets 20 windows fit in 227 KB).
constexpr size_t win_bytes(int nw) { return (size_t)nw * kWinAlloc * sizeof(uint64_t); }
constexpr int kBigBlock = 20;
constexpr int kBigBlockPolar = 20;

// ------------------------------------------------------------------ seeding + warm-up
// Word j of global stream g = splitmix64 output #(607 g + j) of seed (R2); all-even fix
// (R4); 10 rounds of the round update (3 dependency phases 273/273/61) discarded (R3).
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
            buf[j] = x;
            odd |= x & 1;
        }
        const bool any_odd = __any_sync(kFull, odd != 0);
        __syncwarp();
        if (!any_odd && lane == 0) buf[0] |= 1;
        __syncwarp();
        for (int r = 0; r < 10; ++r) {
            for (int i = lane; i < kLagS; i += 32) buf[i] += buf[i + (kLagR - kLagS)];
            __syncwarp();
            for (int i = kLagS + lane; i < 2 * kLagS; i += 32) buf[i] += buf[i - kLagS];
            __syncwarp();
            for (int i = 2 * kLagS + lane; i < kLagR; i += 32) buf[i] += buf[i - kLagS];
            __syncwarp();
        }
        uint64_t* rk = ring + (uint64_t)k * kPitch;
        for (int j = lane; j < kPitch; j += 32) rk[j] = j < kLagR ? buf[j] : 0;
        if (lane == 0) count[k] = 0;
        __syncwarp();
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
            w1[u] = src[32 * per * u];
            w2[u] = src[32 * per * u + 1];
            w3[u] = src[32 * per * u + 2];
        }
        b3_pairs<U>(w1, w2, w3, tp, tab, x, y);
    } else {
        uint64_t wu[U], wv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const ulonglong2 xw = *reinterpret_cast<const ulonglong2*>(src + 32 * per * u);
            wu[u] = xw.x;
            wv[u] = xw.y;
        }
        if (V == 1)
            b1_pairs<U>(wu, wv, tp, tab, x, y);
        else
            b2_pairs<U>(wu, wv, tp, tab, x, y);
    }
}

// B3 tail compaction (fast path only).  A pair with u > tau (prob. 1/9) needs ln + sqrt
// instead of the Moebius/Horner bulk path; evaluating both for every lane would cost the
// tail's ~33 instructions on every pair.  Instead the bulk pass leaves (c, s) in the tail
// pair's output slot and appends the local index of its first word to a per-warp list;
// every kTailEvery iterations (before those words can leave the window: the window keeps
// >= 1024 - 319 words of history) the list is drained 32 entries per warp step: re-read
// u1, u2 from the window, compute the radius, read back (c, s), write the final pair.
constexpr int kTailEvery = 3;
constexpr int kTailCap = kTailEvery * 64;  // entries per drain (U = 2: <= 64 per iteration)
constexpr int kTailAlloc = kTailCap + 32;   // + one scratch slot per lane (branch-free append)
constexpr size_t tailq_bytes(int nw) { return (size_t)nw * kTailAlloc * sizeof(uint32_t); }

__device__ __forceinline__ void b3_tail_drain(const uint32_t* tq, uint32_t tn, const uint64_t* buf, double2* o0,
                                              int lane, const TParams& tp, const Tables& tab) {
    for (uint32_t base = 0; base < tn; base += 32) {
        const bool act = base + lane < tn;
        const uint32_t wl = act ? tq[base + lane] : kW0;
        const uint64_t* src = buf + (wl & kWinMask);
        const uint64_t k1 = ukey(src[0]), k2 = ukey(src[1]);
        const uint64_t Mk[1] = {k1 > k2 ? k1 : k2};
        const uint32_t j = (wl - kW0) / 3;
        const double2 cs = act ? o0[j] : make_double2(0.0, 0.0);
        const double c[1] = {cs.x}, s[1] = {cs.y};
        double x[1], y[1];
        b3_tail_finish<1>(Mk, c, s, tp, tab, x, y);
        if (act) __stcs(o0 + j, make_double2(x[0], y[0]));
    }
}

template <int V, int NW>
__global__ void __launch_bounds__(NW * 32, NW == kBigBlock ? 1 : 5) bm_kernel(BulkParams p) {
    extern __shared__ __align__(16) uint64_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr uint32_t per = (V == 3) ? 3 : 2;
    constexpr int kU = (V == 3) ? 2 : 4;               // pairs per lane per main-loop iteration
    constexpr int kB = 128;                            // refill batch
    constexpr uint32_t kNeedU = 32 * kU * per;         // words per main-loop iteration
    static_assert(kNeedU - 1 + kB <= kWin - kLagR, "lookahead would clobber the write-back words");
    static_assert(kNeedU <= kMirror, "unmasked reads must stay inside the mirror");
    const Tables tab = load_tables(reinterpret_cast<double2*>(smem + NW * kWinAlloc));
    __syncthreads();
    WarpLFG L;
    L.buf = smem + warp * kWinAlloc;
    uint32_t* tq = reinterpret_cast<uint32_t*>(smem + NW * kWinAlloc + kTabBytes / 8) + warp * kTailAlloc;
    for (uint32_t k = p.s_begin + blockIdx.x * NW + warp; k < p.s_end; k += gridDim.x * NW) {
        const Quota qk = quota(p.q, p.rem, k);
        if (qk.cnt == 0) continue;
        const uint64_t C = p.count[k];
        uint64_t* rk = p.ring + (uint64_t)k * kPitch;
        lfg_load(L, rk, C, lane, qk.cnt * per < (uint64_t)kLagR ? (uint32_t)(qk.cnt * per) : (uint32_t)kLagR);
        uint64_t j0 = 0;
        if (p.aligned && 2 * (qk.off + qk.cnt) <= p.n && (V != 3 || qk.cnt * per < (1ull << 31))) {
            double2* o0 = reinterpret_cast<double2*>(p.out + (2 * qk.off - p.shift));
            double2* o = o0 + lane;
            const uint64_t full = qk.cnt - qk.cnt % (32 * kU);
            uint32_t tn = 0, it = 0;  // B3: queued tail pairs, iterations since the last drain
            for (; j0 < full; j0 += 32 * kU, o += 32 * kU) {
                lfg_ensure<kB>(L, lane, kNeedU);
                const uint64_t* src = L.at(per * lane);
                double x[kU], y[kU];
                if (V == 3) {
                    uint64_t w1[kU], w2[kU], w3[kU], Mk[kU];
                    bool tail[kU];
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        w1[u] = src[32 * per * u];
                        w2[u] = src[32 * per * u + 1];
                        w3[u] = src[32 * per * u + 2];
                    }
                    b3_bulk<kU>(w1, w2, w3, p.tp, x, y, tail, Mk);
#pragma unroll
                    for (int u = 0; u < kU; ++u) __stcs(o + 32 * u, make_double2(x[u], y[u]));
                    // branch-free append of the tail pairs' first-word local indices
                    const uint32_t wl = L.wc + per * lane;
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        const unsigned m = __ballot_sync(kFull, tail[u]);
                        const uint32_t slot = tail[u] ? tn + __popc(m & lanemask_lt(lane)) : kTailCap + lane;
                        tq[slot] = wl + 32 * per * u;
                        tn += __popc(m);
                    }
                    if (++it == kTailEvery) {
                        __syncwarp();
                        b3_tail_drain(tq, tn, L.buf, o0, lane, p.tp, tab);
                        tn = 0;
                        it = 0;
                    }
                } else {
                    bm_pairs<V, kU>(src, p.tp, tab, x, y);
#pragma unroll
                    for (int u = 0; u < kU; ++u) __stcs(o + 32 * u, make_double2(x[u], y[u]));
                }
                L.wc += kNeedU;
                __syncwarp();
            }
            if (V == 3 && tn > 0) {
                __syncwarp();
                b3_tail_drain(tq, tn, L.buf, o0, lane, p.tp, tab);
                __syncwarp();
            }
        }
        for (; j0 < qk.cnt; j0 += 32) {
            lfg_ensure<kB>(L, lane, 32 * per);
            const uint64_t left = qk.cnt - j0;
            const uint32_t active = left < 32 ? (uint32_t)left : 32u;
            if ((uint32_t)lane < active) {
                double x[1], y[1];
                bm_pairs<V, 1>(L.at(per * lane), p.tp, tab, x, y);
                store_pair(p.out, 2 * (qk.off + j0 + lane), p.shift, p.n, x[0], y[0], p.aligned);
            }
            L.wc += per * active;
            __syncwarp();
        }
        lfg_store(L, rk, C, lane);
        if (lane == 0) p.count[k] = C + (L.wc - kW0);
        __syncwarp();
    }
}

// ------------------------------------------------------------------ Polar P
// Candidate phase: 64 candidates (128 uniforms) per warp step, two per lane: candidate i
// of the step is lane i%32's (i < 32: words wc + 2i, i >= 32: wc + 64 + 2(i-32)).  Accepts
// are ranked with __ballot_sync/__popc in candidate order, trimmed at the stream's
// remaining quota (exact stop, R5: the last step consumes candidates only up to the
// p_k-th accept), and the window position of each survivor is appended to a per-warp
// shared-memory queue (4 bytes per entry: the words stay in the window, which keeps >= 600
// words of history behind wc).  Transform phase: whenever >= 64 survivors are queued the
// warp re-reads their words, recomputes (X, Y, S) and transforms 64 of them densely (two
// per lane; no lane idles on a rejected candidate), storing 64 consecutive pairs.
constexpr int kQueue = 128;
constexpr int kQueueAlloc = kQueue + 32;  // ring + one scratch slot per lane
constexpr size_t queue_bytes(int nw) { return (size_t)nw * kQueueAlloc * sizeof(uint32_t); }

template <int U, int M>
__device__ __forceinline__ void polar_from_queue(const uint64_t* buf, const uint32_t* q, uint32_t first, int lane,
                                                 const TParams& tp, const Tables& tab, double (&ox)[U],
                                                 double (&oy)[U]) {
    PolarCand c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(buf + q[(first + 32 * u + lane) & (kQueue - 1)]);
        polar_candidate(w.x, w.y, c[u]);
    }
    if (M == 2)
        p2_transform<U>(c, tp, tab, ox, oy);
    else
        polar_transform<U>(c, tp, tab, ox, oy);
}

// M = 1: Algorithm P (= the paper's P1); M = 2: method P2, same candidates.
template <int NW, int M>
__global__ void __launch_bounds__(NW * 32, NW == kBigBlockPolar ? 1 : 4) polar_kernel(BulkParams p) {
    extern __shared__ __align__(16) uint64_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const Tables tab = load_tables(reinterpret_cast<double2*>(smem + NW * kWinAlloc));
    __syncthreads();
    WarpLFG L;
    L.buf = smem + warp * kWinAlloc;
    uint32_t* q = reinterpret_cast<uint32_t*>(smem + NW * kWinAlloc + kTabBytes / 8) + warp * kQueueAlloc;
    const unsigned lt = lanemask_lt(lane);
    for (uint32_t k = p.s_begin + blockIdx.x * NW + warp; k < p.s_end; k += gridDim.x * NW) {
        const Quota qk = quota(p.q, p.rem, k);
        if (qk.cnt == 0) continue;
        const uint64_t C = p.count[k];
        uint64_t* rk = p.ring + (uint64_t)k * kPitch;
        lfg_load(L, rk, C, lane);
        const bool fast = p.aligned && 2 * (qk.off + qk.cnt) <= p.n;
        // the stream's quota in chunks of < 2^31 pairs: 32-bit counters in the loops
        for (uint64_t base = 0; base < qk.cnt;) {
            const uint32_t cnt = (uint32_t)(qk.cnt - base < (1ull << 31) ? qk.cnt - base : (1ull << 31));
            double2* o = reinterpret_cast<double2*>(p.out + (2 * (qk.off + base) - p.shift)) + lane;
            uint32_t acc = 0;   // accepted (queued) pairs of this chunk
            uint32_t done = 0;  // pairs transformed and stored
            while (acc < cnt) {
                lfg_ensure(L, lane, 128);
                const uint32_t pos0 = (L.wc & kWinMask) + 2 * lane, pos1 = pos0 + 64;
                const ulonglong2 w0 = *reinterpret_cast<const ulonglong2*>(L.buf + pos0);
                const ulonglong2 w1 = *reinterpret_cast<const ulonglong2*>(L.buf + pos1);
                PolarCand c0, c1;
                const bool ok0 = polar_candidate(w0.x, w0.y, c0);
                const bool ok1 = polar_candidate(w1.x, w1.y, c1);
                unsigned m0 = __ballot_sync(kFull, ok0), m1 = __ballot_sync(kFull, ok1);
                const uint32_t need = cnt - acc;
                uint32_t used = 64;
                if ((uint32_t)(__popc(m0) + __popc(m1)) >= need) {
                    // exact stop: keep the first `need` accepts in candidate order
                    if ((uint32_t)__popc(m0) >= need) {
                        const unsigned last = __ballot_sync(kFull, ok0 && (uint32_t)__popc(m0 & lt) == need - 1);
                        const int l = __ffs(last) - 1;
                        m0 &= (l == 31) ? kFull : ((2u << l) - 1u);
                        m1 = 0;
                        used = l + 1;
                    } else {
                        const uint32_t need1 = need - __popc(m0);
                        const unsigned last = __ballot_sync(kFull, ok1 && (uint32_t)__popc(m1 & lt) == need1 - 1);
                        const int l = __ffs(last) - 1;
                        m1 &= (l == 31) ? kFull : ((2u << l) - 1u);
                        used = 32 + l + 1;
                    }
                }
                // branch-free append: rejected lanes write their position to a per-lane
                // scratch slot past the ring (q[kQueue + lane]) instead of skipping the store
                const uint32_t n0 = __popc(m0);
                const uint32_t s0 = ((m0 >> lane) & 1u) ? ((acc + __popc(m0 & lt)) & (kQueue - 1)) : kQueue + lane;
                const uint32_t s1 =
                    ((m1 >> lane) & 1u) ? ((acc + n0 + __popc(m1 & lt)) & (kQueue - 1)) : kQueue + lane;
                q[s0] = pos0;
                q[s1] = pos1;
                acc += n0 + __popc(m1);
                L.wc += 2 * used;
                __syncwarp();
                if (fast && acc - done >= 64) {
                    double ox[2], oy[2];
                    polar_from_queue<2, M>(L.buf, q, done, lane, p.tp, tab, ox, oy);
                    __stcs(o + done, make_double2(ox[0], oy[0]));
                    __stcs(o + done + 32, make_double2(ox[1], oy[1]));
                    done += 64;
                    __syncwarp();
                }
                while (!fast && acc - done >= 32) {
                    double ox[1], oy[1];
                    polar_from_queue<1, M>(L.buf, q, done, lane, p.tp, tab, ox, oy);
                    store_pair(p.out, 2 * (qk.off + base + done + lane), p.shift, p.n, ox[0], oy[0], p.aligned);
                    done += 32;
                    __syncwarp();
                }
            }
            for (; done < acc; done += 32) {
                if ((uint32_t)lane < acc - done) {
                    double ox[1], oy[1];
                    polar_from_queue<1, M>(L.buf, q, done, lane, p.tp, tab, ox, oy);
                    store_pair(p.out, 2 * (qk.off + base + done + lane), p.shift, p.n, ox[0], oy[0], p.aligned);
                }
                __syncwarp();
            }
            base += cnt;
        }
        lfg_store(L, rk, C, lane);
        if (lane == 0) p.count[k] = C + (L.wc - kW0);
        __syncwarp();
    }
}

// Direct variant: the survivors are compacted only in the OUTPUT -- each accepted
// candidate's pair index is its __ballot_sync/__popc rank in candidate order -- and the
// warp transforms all 64 candidates of a step, rejected lanes predicated off at the
// store.  On the VP2200 the compress made vector lengths full; on a GPU the
// 21.5% of lanes that do wasted work cost less than a queue's per-candidate bookkeeping.
template <int NW, int M>
__global__ void __launch_bounds__(NW * 32, NW == kBigBlockPolar ? 1 : 4) polar_direct_kernel(BulkParams p) {
    extern __shared__ __align__(16) uint64_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const Tables tab = load_tables(reinterpret_cast<double2*>(smem + NW * kWinAlloc));
    __syncthreads();
    WarpLFG L;
    L.buf = smem + warp * kWinAlloc;
    const unsigned lt = lanemask_lt(lane);
    for (uint32_t k = p.s_begin + blockIdx.x * NW + warp; k < p.s_end; k += gridDim.x * NW) {
        const Quota qk = quota(p.q, p.rem, k);
        if (qk.cnt == 0) continue;
        const uint64_t C = p.count[k];
        uint64_t* rk = p.ring + (uint64_t)k * kPitch;
        lfg_load(L, rk, C, lane);
        const bool fast = p.aligned && 2 * (qk.off + qk.cnt) <= p.n;
        for (uint64_t base = 0; base < qk.cnt;) {
            const uint32_t cnt = (uint32_t)(qk.cnt - base < (1ull << 31) ? qk.cnt - base : (1ull << 31));
            double2* o = reinterpret_cast<double2*>(p.out + (2 * (qk.off + base) - p.shift));
            uint32_t acc = 0;  // accepted pairs of this chunk
            while (acc < cnt) {
                lfg_ensure(L, lane, 128);
                const ulonglong2 w0 = *reinterpret_cast<const ulonglong2*>(L.at(2 * lane));
                const ulonglong2 w1 = *reinterpret_cast<const ulonglong2*>(L.at(64 + 2 * lane));
                PolarCand c[2];
                const bool ok0 = polar_candidate(w0.x, w0.y, c[0]);
                const bool ok1 = polar_candidate(w1.x, w1.y, c[1]);
                unsigned m0 = __ballot_sync(kFull, ok0), m1 = __ballot_sync(kFull, ok1);
                const uint32_t need = cnt - acc;
                uint32_t used = 64;
                if ((uint32_t)(__popc(m0) + __popc(m1)) >= need) {
                    if ((uint32_t)__popc(m0) >= need) {
                        const unsigned last = __ballot_sync(kFull, ok0 && (uint32_t)__popc(m0 & lt) == need - 1);
                        const int l = __ffs(last) - 1;
                        m0 &= (l == 31) ? kFull : ((2u << l) - 1u);
                        m1 = 0;
                        used = l + 1;
                    } else {
                        const uint32_t need1 = need - __popc(m0);
                        const unsigned last = __ballot_sync(kFull, ok1 && (uint32_t)__popc(m1 & lt) == need1 - 1);
                        const int l = __ffs(last) - 1;
                        m1 &= (l == 31) ? kFull : ((2u << l) - 1u);
                        used = 32 + l + 1;
                    }
                }
                const uint32_t n0 = __popc(m0);
                const uint32_t j0 = acc + __popc(m0 & lt), j1 = acc + n0 + __popc(m1 & lt);
                double ox[2], oy[2];
                if (M == 2)
                    p2_transform<2>(c, p.tp, tab, ox, oy);
                else
                    polar_transform<2>(c, p.tp, tab, ox, oy);
                const bool k0 = (m0 >> lane) & 1u, k1 = (m1 >> lane) & 1u;
                if (fast) {
                    if (k0) __stcs(o + j0, make_double2(ox[0], oy[0]));
                    if (k1) __stcs(o + j1, make_double2(ox[1], oy[1]));
                } else {
                    if (k0) store_pair(p.out, 2 * (qk.off + base + j0), p.shift, p.n, ox[0], oy[0], p.aligned);
                    if (k1) store_pair(p.out, 2 * (qk.off + base + j1), p.shift, p.n, ox[1], oy[1], p.aligned);
                }
                acc += n0 + __popc(m1);
                L.wc += 2 * used;
                __syncwarp();
            }
            base += cnt;
        }
        lfg_store(L, rk, C, lane);
        if (lane == 0) p.count[k] = C + (L.wc - kW0);
        __syncwarp();
    }
}

// ------------------------------------------------------------------ tiny quotas
// Calls that give every stream only a few pairs (the C4 sweep: n <= 2^18 over 2^16
// streams) are bound by per-stream latency and state traffic, not arithmetic: one THREAD
// per stream generates its words straight through the HBM ring (x_{C+i} = ring[(C+i) mod
// 607] + ring[(C+i+334) mod 607], written back in place -- exactly the recurrence, in the
// canonical layout), transforms and stores.  Only the words actually used are touched.
constexpr int kTinyThreads = 128;
constexpr uint64_t kTinyMaxPairs = 4;  // per-stream quota routed here (8 words for B1)

struct RingCursor {
    uint64_t* r;
    uint32_t a, b;  // positions of x_{n-607} (= slot of x_n) and x_{n-273}
    __device__ __forceinline__ RingCursor(uint64_t* ring_k, uint64_t C) : r(ring_k) {
        a = (uint32_t)(C % kLagR);
        b = a + (kLagR - kLagS);
        b = b >= (uint32_t)kLagR ? b - kLagR : b;
    }
    __device__ __forceinline__ uint64_t next() {
        const uint64_t x = r[a] + r[b];
        r[a] = x;
        a = a + 1 == (uint32_t)kLagR ? 0 : a + 1;
        b = b + 1 == (uint32_t)kLagR ? 0 : b + 1;
        return x;
    }
};

template <int V>  // 1, 2, 3 = B1, B2, B3; 4 = Polar; 5 = P2
__global__ void __launch_bounds__(kTinyThreads) tiny_kernel(BulkParams p) {
    __shared__ double2 tabs[kTabBytes / 16];
    const Tables tab = load_tables(tabs);
    __syncthreads();
    const uint32_t k = p.s_begin + blockIdx.x * kTinyThreads + threadIdx.x;
    if (k >= p.s_end) return;
    const Quota qk = quota(p.q, p.rem, k);
    if (qk.cnt == 0) return;
    const uint64_t C = p.count[k];
    RingCursor rc(p.ring + (uint64_t)k * kPitch, C);
    uint64_t used = 0;
    for (uint64_t j = 0; j < qk.cnt; ++j) {
        double x[1], y[1];
        if (V >= 4) {
            PolarCand c[1];
            bool ok;
            do {
                const uint64_t wa = rc.next(), wb = rc.next();
                used += 2;
                ok = polar_candidate(wa, wb, c[0]);
            } while (!ok);
            if (V == 5)
                p2_transform<1>(c, p.tp, tab, x, y);
            else
                polar_transform<1>(c, p.tp, tab, x, y);
        } else if (V == 3) {
            const uint64_t w1[1] = {rc.next()}, w2[1] = {rc.next()}, w3[1] = {rc.next()};
            used += 3;
            b3_pairs<1>(w1, w2, w3, p.tp, tab, x, y);
        } else {
            const uint64_t wu[1] = {rc.next()}, wv[1] = {rc.next()};
            used += 2;
            if (V == 1)
                b1_pairs<1>(wu, wv, p.tp, tab, x, y);
            else
                b2_pairs<1>(wu, wv, p.tp, tab, x, y);
        }
        store_pair(p.out, 2 * (qk.off + j), p.shift, p.n, x[0], y[0], p.aligned);
    }
    p.count[k] = C + used;
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
        const Quota qk = quota(p.q, p.rem, k);
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
                p.out[g - p.shift] = (double)ukey(L.buf[(L.wc + lane) & kWinMask]) * 0x1p-53;  // exact
            }
            L.wc += active;
            __syncwarp();
        }
        lfg_store(L, rk, C, lane);
        if (lane == 0) p.count[k] = C + (L.wc - kW0);
        __syncwarp();
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
                const ulonglong2 xw = *reinterpret_cast<const ulonglong2*>(&L.buf[(L.wc + 2 * lane) & kWinMask]);
                PolarCand pc;
                mask[(uint64_t)k * cand + j0 + lane] = polar_candidate(xw.x, xw.y, pc) ? 1 : 0;
            }
            L.wc += 2 * active;
            __syncwarp();
        }
        lfg_store(L, rk, C, lane);
        if (lane == 0) p.count[k] = C + (L.wc - kW0);
        __syncwarp();
    }
}

// nrng_transform_from_uniforms: one thread per pair; the given uniforms (multiples of
// 2^-53 in [0,1)) are turned back into the words the stream would hold, so this runs
// exactly the device code of the bulk kernels.
__device__ __forceinline__ uint64_t word_of(double u) { return __double2ull_rn(u * 0x1p53) << 11; }
__global__ void transform_kernel(const double* __restrict__ u, uint64_t n_pairs, double* __restrict__ out,
                                 uint8_t* __restrict__ mask, TParams tp, int method) {
    __shared__ double2 tabs[kTabBytes / 16];
    const Tables tab = load_tables(tabs);
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
// Block partials of sum (x-c)^k, k = 1..4, min, max (fp64), and a K-bin histogram
// (shared-memory int counters -> global u64 atomics).  A second kernel reduces the
// block partials in a fixed order (deterministic sums).
constexpr int kStatsThreads = 256;
__global__ void __launch_bounds__(kStatsThreads) stats_partial_kernel(const double* __restrict__ x, uint64_t n,
                                                                      double center, const double* __restrict__ edges,
                                                                      int K, double* __restrict__ partial,
                                                                      unsigned long long* __restrict__ hist) {
    __shared__ double red[6][kStatsThreads / 32];
    __shared__ unsigned int sh[1024];
    __shared__ double se[1023];
    for (int b = threadIdx.x; b < K; b += blockDim.x) sh[b] = 0;
    for (int b = threadIdx.x; b < K - 1; b += blockDim.x) se[b] = edges[b];
    __syncthreads();
    double s1 = 0, s2 = 0, s3 = 0, s4 = 0, mn = __longlong_as_double(0x7ff0000000000000ULL), mx = -mn;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const double v = x[i];
        const double d = v - center;
        const double d2 = d * d;
        s1 += d;
        s2 += d2;
        s3 += d2 * d;
        s4 += d2 * d2;
        mn = fmin(mn, v);
        mx = fmax(mx, v);
        int lo = 0, hi = K - 1;  // first edge index with v < edge, in [0, K-1]
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (v < se[mid]) hi = mid; else lo = mid + 1;
        }
        atomicAdd(&sh[lo], 1u);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double vals[6] = {s1, s2, s3, s4, mn, mx};
#pragma unroll
    for (int t = 0; t < 6; ++t) {
        double v = vals[t];
        for (int o = 16; o > 0; o >>= 1) {
            const double w = __shfl_xor_sync(kFull, v, o);
            v = t < 4 ? v + w : (t == 4 ? fmin(v, w) : fmax(v, w));
        }
        if (lane == 0) red[t][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        const int t = threadIdx.x;
        double v = red[t][0];
        for (int w = 1; w < kStatsThreads / 32; ++w)
            v = t < 4 ? v + red[t][w] : (t == 4 ? fmin(v, red[t][w]) : fmax(v, red[t][w]));
        partial[blockIdx.x * 6 + t] = v;
    }
    for (int b = threadIdx.x; b < K; b += blockDim.x)
        if (sh[b]) atomicAdd(&hist[b], (unsigned long long)sh[b]);
}

__global__ void stats_final_kernel(const double* __restrict__ partial, int nblocks, double* __restrict__ sums) {
    const int t = threadIdx.x;
    if (t < 6) {
        double v = partial[t];
        for (int b = 1; b < nblocks; ++b) {
            const double w = partial[b * 6 + t];
            v = t < 4 ? v + w : (t == 4 ? fmin(v, w) : fmax(v, w));
        }
        sums[t] = v;
    }
}

}  // namespace nrng
