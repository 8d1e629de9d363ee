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
    double mu, sigma;
    int aligned;
};

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
// Per warp iteration: 32 pairs of stream k, lane l takes pair j0+l (uniforms 2(j0+l),
// 2(j0+l)+1, or 3 for B3), one 16-byte streaming store per pair, 512 contiguous bytes
// per warp store instruction.
template <int V>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) bm_kernel(BulkParams p) {
    extern __shared__ __align__(16) uint64_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr uint32_t per = (V == 3) ? 3 : 2;
    WarpLFG L;
    L.buf = smem + warp * kWin;
    for (uint32_t k = p.s_begin + blockIdx.x * kWarpsPerBlock + warp; k < p.s_end;
         k += gridDim.x * kWarpsPerBlock) {
        const Quota qk = quota(p.units, p.q, p.rem, k);
        if (qk.cnt == 0) continue;
        const uint64_t C = p.count[k];
        uint64_t* rk = p.ring + (uint64_t)k * kPitch;
        lfg_load(L, rk, C, lane);
        for (uint64_t j0 = 0; j0 < qk.cnt; j0 += 32) {
            lfg_ensure(L, lane, 32 * per);
            const uint64_t left = qk.cnt - j0;
            const uint32_t active = left < 32 ? (uint32_t)left : 32u;
            if ((uint32_t)lane < active) {
                const uint32_t w = L.wc + per * lane;
                double x, y;
                if (V == 3) {
                    double u1 = word_to_uniform(L.buf[w & kWinMask]);
                    double u2 = word_to_uniform(L.buf[(w + 1) & kWinMask]);
                    double u3 = word_to_uniform(L.buf[(w + 2) & kWinMask]);
                    b3_pair(u1, u2, u3, p.mu, p.sigma, x, y);
                } else {
                    const ulonglong2 xw = *reinterpret_cast<const ulonglong2*>(&L.buf[w & kWinMask]);
                    double u = word_to_uniform(xw.x);
                    double v = word_to_uniform(xw.y);
                    if (V == 1)
                        b1_pair(u, v, p.mu, p.sigma, x, y);
                    else
                        b2_pair(u, v, p.mu, p.sigma, x, y);
                }
                store_pair(p.out, 2 * (qk.off + j0 + lane), p.shift, p.n, x, y, p.aligned);
            }
            L.wc += per * active;
            __syncwarp();
        }
        lfg_store(L, rk, C, lane);
        if (lane == 0) p.count[k] = C + (L.wc - (kLagR + 1));
        __syncwarp();
    }
}

// ------------------------------------------------------------------ Polar P
// Per warp iteration: 32 candidates (64 uniforms).  Accepts are ranked with
// __ballot_sync/__popc, trimmed at the stream's remaining quota (exact stop, R5),
// appended to a per-warp shared-memory queue in candidate order; every time the queue
// holds 32 survivors the warp transforms them densely (no lane idles on a rejected
// candidate) and stores 32 consecutive pairs.
constexpr int kQueue = 64;
__global__ void __launch_bounds__(kWarpsPerBlock * 32) polar_kernel(BulkParams p) {
    extern __shared__ __align__(16) uint64_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpLFG L;
    L.buf = smem + warp * kWin;
    double* qx = reinterpret_cast<double*>(smem + kWarpsPerBlock * kWin) + warp * 3 * kQueue;
    double* qy = qx + kQueue;
    double* qs = qy + kQueue;
    for (uint32_t k = p.s_begin + blockIdx.x * kWarpsPerBlock + warp; k < p.s_end;
         k += gridDim.x * kWarpsPerBlock) {
        const Quota qk = quota(p.units, p.q, p.rem, k);
        if (qk.cnt == 0) continue;
        const uint64_t C = p.count[k];
        uint64_t* rk = p.ring + (uint64_t)k * kPitch;
        lfg_load(L, rk, C, lane);
        uint64_t acc = 0;    // accepted (queued) pairs of this stream
        uint64_t done = 0;   // pairs transformed and stored
        while (acc < qk.cnt) {
            lfg_ensure(L, lane, 64);
            const ulonglong2 xw = *reinterpret_cast<const ulonglong2*>(&L.buf[(L.wc + 2 * lane) & kWinMask]);
            double x, y, s;
            const bool ok = polar_candidate(word_to_uniform(xw.x), word_to_uniform(xw.y), x, y, s);
            unsigned m = __ballot_sync(kFull, ok);
            const uint64_t need = qk.cnt - acc;
            uint32_t used = 32;
            if ((uint64_t)__popc(m) >= need) {  // exact stop inside this group of 32
                const int rank = __popc(m & (unsigned)lanemask_lt(lane));
                const unsigned last = __ballot_sync(kFull, ok && (uint64_t)rank == need - 1);
                const int lastlane = __ffs(last) - 1;
                used = lastlane + 1;
                m &= (lastlane == 31) ? kFull : ((2u << lastlane) - 1u);
            }
            if ((m >> lane) & 1u) {
                const uint32_t slot = (uint32_t)(acc + __popc(m & (unsigned)lanemask_lt(lane))) & (kQueue - 1);
                qx[slot] = x;
                qy[slot] = y;
                qs[slot] = s;
            }
            acc += __popc(m);
            L.wc += 2 * used;
            __syncwarp();
            if (acc - done >= 32) {
                const uint32_t slot = (uint32_t)(done + lane) & (kQueue - 1);
                double ox, oy;
                polar_transform(qx[slot], qy[slot], qs[slot], p.mu, p.sigma, ox, oy);
                store_pair(p.out, 2 * (qk.off + done + lane), p.shift, p.n, ox, oy, p.aligned);
                done += 32;
                __syncwarp();
            }
        }
        if ((uint64_t)lane < acc - done) {
            const uint32_t slot = (uint32_t)(done + lane) & (kQueue - 1);
            double ox, oy;
            polar_transform(qx[slot], qy[slot], qs[slot], p.mu, p.sigma, ox, oy);
            store_pair(p.out, 2 * (qk.off + done + lane), p.shift, p.n, ox, oy, p.aligned);
        }
        __syncwarp();
        lfg_store(L, rk, C, lane);
        if (lane == 0) p.count[k] = C + (L.wc - (kLagR + 1));
        __syncwarp();
    }
}

// ------------------------------------------------------------------ test hooks
// nrng_uniform: one uniform per slot, stream-major (units = uniforms).
__global__ void __launch_bounds__(kWarpsPerBlock * 32) uniform_kernel(BulkParams p) {
    extern __shared__ __align__(16) uint64_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpLFG L;
    L.buf = smem + warp * kWin;
    for (uint32_t k = p.s_begin + blockIdx.x * kWarpsPerBlock + warp; k < p.s_end;
         k += gridDim.x * kWarpsPerBlock) {
        const Quota qk = quota(p.units, p.q, p.rem, k);
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
                p.out[g - p.shift] = word_to_uniform(L.buf[(L.wc + lane) & kWinMask]);
            }
            L.wc += active;
            __syncwarp();
        }
        lfg_store(L, rk, C, lane);
        if (lane == 0) p.count[k] = C + (L.wc - (kLagR + 1));
        __syncwarp();
    }
}

// nrng_polar_mask: every stream advances exactly `cand` candidates.
__global__ void __launch_bounds__(kWarpsPerBlock * 32) polar_mask_kernel(BulkParams p, uint8_t* __restrict__ mask,
                                                                         uint64_t cand) {
    extern __shared__ __align__(16) uint64_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpLFG L;
    L.buf = smem + warp * kWin;
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
                double x, y, s;
                mask[(uint64_t)k * cand + j0 + lane] =
                    polar_candidate(word_to_uniform(xw.x), word_to_uniform(xw.y), x, y, s) ? 1 : 0;
            }
            L.wc += 2 * active;
            __syncwarp();
        }
        lfg_store(L, rk, C, lane);
        if (lane == 0) p.count[k] = C + (L.wc - (kLagR + 1));
        __syncwarp();
    }
}

// nrng_transform_from_uniforms: one thread per pair.
__global__ void transform_kernel(const double* __restrict__ u, uint64_t n_pairs, double* __restrict__ out,
                                 uint8_t* __restrict__ mask, double mu, double sigma, int method) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n_pairs;
         j += (uint64_t)gridDim.x * blockDim.x) {
        double x = __longlong_as_double(0x7ff8000000000000ULL), y = x;
        if (method == 1) {
            b1_pair(u[2 * j], u[2 * j + 1], mu, sigma, x, y);
        } else if (method == 2) {
            b2_pair(u[2 * j], u[2 * j + 1], mu, sigma, x, y);
        } else if (method == 3) {
            b3_pair(u[3 * j], u[3 * j + 1], u[3 * j + 2], mu, sigma, x, y);
        } else {
            double cx, cy, s;
            const bool ok = polar_candidate(u[2 * j], u[2 * j + 1], cx, cy, s);
            if (mask) mask[j] = ok ? 1 : 0;
            if (ok) polar_transform(cx, cy, s, mu, sigma, x, y);
        }
        out[2 * j] = x;
        out[2 * j + 1] = y;
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
