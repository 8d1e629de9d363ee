// nrng.cu -- host side of libnrng.so: the C ABI declared in include/nrng.h.
//
// Argument marshalling, validation, launch geometry and the host-buffer (chunked,
// overlapped D2H) path.  Every step of the method runs in the kernels of
// nrng_kernels.cuh; there is no CPU fallback: without a usable CUDA device every
// entry point fails with NRNG_ENODEV / NRNG_ECUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

#include "../../include/nrng.h"
#include "nrng_kernels.cuh"

using namespace nrng;

namespace {

thread_local int g_last = NRNG_OK;

int set_err(int code) {
    g_last = code;
    return code;
}

int cuda_err(cudaError_t e) {
    if (e == cudaSuccess) return set_err(NRNG_OK);
    fprintf(stderr, "[nrng] CUDA error: %s\n", cudaGetErrorString(e));
    return set_err(NRNG_ECUDA);
}

constexpr size_t bm_smem(int nw) { return win_bytes(nw) + kTabBytes; }
constexpr size_t r1_smem(int nw) { return bm_smem(nw) + (size_t)nw * 32 * sizeof(double); }  // + R1 scratch
constexpr size_t polar_smem(int nw) { return win_bytes(nw) + kTabBytes + (size_t)nw * 32 * sizeof(double); }  // + P2 tail scratch
constexpr size_t kMaxSmem = 227 * 1024;  // per block, sm_100a opt-in maximum
static_assert(bm_smem(kPwWarps) <= kMaxSmem && pw_smem(5, false, kPwWarps) <= kMaxSmem && pw_smem(7, false, kPwWarps) <= kMaxSmem && r1_smem(kPwWarps) <= kMaxSmem && tri_smem(kTriWarps) <= kMaxSmem &&
                  bm_smem(kBigBlock) <= kMaxSmem && polar_smem(kBigBlockPolar) <= kMaxSmem,
              "one-block-per-SM kernels must fit the shared memory of an SM");
constexpr size_t kUniSmem = win_bytes(kWarpsPerBlock);
constexpr size_t kInitSmem = kWarpsPerBlock * kPitch * sizeof(uint64_t);
constexpr size_t kStageDoubles = size_t(1) << 24;  // 128 MB per staging buffer (host-output path)

#if NRNG_RACECHECK
// Debug build only (nrng_racecheck.cuh): the shadow arrays, allocated once, cleared before every
// instrumented launch; races accumulate until read by nrng_racecheck_result.
RcState g_rc_host{};
bool rc_ready() {
    if (g_rc_host.w) return true;
    const size_t words = (size_t)kRcMaxBlocks * kRcShadowWords;
    if (cudaMalloc(&g_rc_host.w, words * 8) != cudaSuccess || cudaMalloc(&g_rc_host.r, words * 8) != cudaSuccess ||
        cudaMalloc(&g_rc_host.epoch, (size_t)kRcMaxThreads * 4) != cudaSuccess ||
        cudaMalloc(&g_rc_host.races, 16) != cudaSuccess || cudaMalloc(&g_rc_host.checks, 8) != cudaSuccess)
        return false;
    cudaMemset(g_rc_host.races, 0, 16);
    cudaMemset(g_rc_host.checks, 0, 8);
    return cudaMemcpyToSymbol(g_rc, &g_rc_host, sizeof(g_rc_host)) == cudaSuccess;
}
void rc_reset(cudaStream_t st) {
    if (!rc_ready()) return;
    const size_t words = (size_t)kRcMaxBlocks * kRcShadowWords;
    cudaMemsetAsync(g_rc_host.w, 0, words * 8, st);
    cudaMemsetAsync(g_rc_host.r, 0, words * 8, st);
    cudaMemsetAsync(g_rc_host.epoch, 0, (size_t)kRcMaxThreads * 4, st);
}
#else
void rc_reset(cudaStream_t) {}
#endif

struct Occ {
    int bm[4] = {0, 0, 0, 0}, pw[3] = {0, 0, 0}, tri = 0, polar = 0, ratio = 0, ratio1 = 0, uni = 0, mask = 0, init = 0;  // 4-warp-block kernels
};

}  // namespace

struct nrng_gen {
    int device = 0;
    int num_sms = 148;
    uint64_t seed = 0, first = 0;
    uint32_t S = 0;
    int variant = 1;
    uint64_t* ring = nullptr;   // S x kPitch
    uint64_t* count = nullptr;  // S
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;
    double* stage[2] = {nullptr, nullptr};
    cudaEvent_t ev_ready[2] = {nullptr, nullptr};
    cudaEvent_t ev_free[2] = {nullptr, nullptr};
    uint64_t launches = 0;
    Occ occ;
    // sequential (RANN3-style) mode: the partially consumed last epoch
    struct {
        double* buf = nullptr;
        uint32_t log2E = 7;  // E = 128 pairs per stream per epoch
        uint64_t len = 0, pos = 0;
        int method = 0;
        double mu = 0, sigma = 0;
    } seq;
};

namespace {

template <typename K>
int occupancy(K kernel, int nw, size_t smem) {
    int b = 0;
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (smem > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, nw * 32, smem) != cudaSuccess) b = 1;
    return std::max(b, 1);
}

bool check_device(nrng_handle h) {
    int d = -1;
    if (cudaGetDevice(&d) != cudaSuccess) return false;
    return d == h->device;
}

unsigned grid_for(uint32_t nstreams, int nw, int per_sm, int num_sms) {
    uint64_t want = (nstreams + nw - 1) / nw;
    uint64_t cap = (uint64_t)per_sm * num_sms;
    return (unsigned)std::max<uint64_t>(1, std::min(want, cap));
}

// Launch one bulk kernel over streams [b, e) of the handle.  Stream counts that fill every
// SM with kBigBlock-warp blocks use those (one block per SM); smaller ones use 4-warp
// blocks spread over all SMs.
enum class Kind { BM1, BM2, BM3, POLAR, POLAR2, RATIO, RATIO1, UNIFORM };

// The sequential mode's whole-epoch launches (equal quotas of whole 128-pair blocks, every
// slot in range) run the same one-block-per-SM kernels with the epoch-layout store (EP).
bool epoch_fast(const BulkParams& p) {
    return p.aligned && p.log2E >= 7 && p.rem == 0 && p.q % 128 == 0 && p.n == 2 * p.units && p.shift == 0;
}

// Largest per-stream unit count of one launch (a piece's, if the call is split).
uint64_t eff_qmax(const BulkParams& p) {
    const uint64_t qmax = p.q + (p.rem ? 1 : 0);
    if (!p.jcap) return qmax;
    return std::min(qmax > p.jb ? qmax - p.jb : 0, p.jcap);
}

#ifndef NRNG_PW_SMALL
#define NRNG_PW_SMALL 1
#endif
template <int V>
void launch_bm(nrng_handle h, const BulkParams& p, uint32_t ns, cudaStream_t st) {
    const bool plain = p.aligned && p.log2E == 0;
    if (epoch_fast(p) && ns >= (uint32_t)((V == 3 ? kTriWarps : kPwWarps) * h->num_sms)) {
        if constexpr (V == 3)
            b3_kernel<kTriWarps, true><<<h->num_sms, kTriWarps * 32, tri_smem(kTriWarps), st>>>(p);
        else
            pw_kernel<V, kPwWarps, true><<<h->num_sms, kPwWarps * 32, bm_smem(kPwWarps), st>>>(p);
        return;
    }
    if constexpr (V == 3) {
        if (plain && ns >= (uint32_t)(kTriWarps * h->num_sms)) {
            b3_kernel<kTriWarps><<<h->num_sms, kTriWarps * 32, tri_smem(kTriWarps), st>>>(p);
            return;
        }
        if (NRNG_PW_SMALL && plain) {  // fewer streams than one-block-per-SM slots: 4-warp blocks
            b3_kernel<kWarpsPerBlock><<<grid_for(ns, kWarpsPerBlock, h->occ.tri, h->num_sms), kWarpsPerBlock * 32,
                                        tri_smem(kWarpsPerBlock), st>>>(p);
            return;
        }
    } else {
        if (plain && ns >= (uint32_t)(kPwWarps * h->num_sms)) {
            pw_kernel<V, kPwWarps><<<h->num_sms, kPwWarps * 32, pw_smem(V, false, kPwWarps), st>>>(p);
            return;
        }
        if (NRNG_PW_SMALL && plain) {  // fewer streams than one-block-per-SM slots: 4-warp blocks
            pw_kernel<V, kWarpsPerBlock><<<grid_for(ns, kWarpsPerBlock, h->occ.pw[V], h->num_sms),
                                           kWarpsPerBlock * 32, pw_smem(V, false, kWarpsPerBlock), st>>>(p);
            return;
        }
    }
    if (ns >= (uint32_t)(kBigBlock * h->num_sms))
        bm_kernel<V, kBigBlock><<<h->num_sms, kBigBlock * 32, bm_smem(kBigBlock), st>>>(p);
    else
        bm_kernel<V, kWarpsPerBlock><<<grid_for(ns, kWarpsPerBlock, h->occ.bm[V], h->num_sms), kWarpsPerBlock * 32,
                                       bm_smem(kWarpsPerBlock), st>>>(p);
}

#ifndef NRNG_P2_PW  // P2 on pw_kernel<5> (compacted tails, 104 registers, no mirror): 6.21 vs 6.20 ms burst,
#define NRNG_P2_PW 1  // 6.24 vs 6.39 ms sustained against polar_kernel
#endif
template <int M>
void launch_polar(nrng_handle h, const BulkParams& p, uint32_t ns, cudaStream_t st) {
    constexpr int kPw = M == 1 ? 4 : 5;  // pw_kernel's P and P2 transforms
    if (M == 1 && epoch_fast(p) && eff_qmax(p) < (1ull << 31) && ns >= (uint32_t)(kPwWarps * h->num_sms)) {
        pw_kernel<4, kPwWarps, true><<<h->num_sms, kPwWarps * 32, bm_smem(kPwWarps), st>>>(p);
        return;
    }
    if (M == 2 && NRNG_P2_PW && epoch_fast(p) && eff_qmax(p) < (1ull << 31) && ns >= (uint32_t)(kPwWarps * h->num_sms)) {
        pw_kernel<5, kPwWarps, true><<<h->num_sms, kPwWarps * 32, pw_smem(5, true, kPwWarps), st>>>(p);
        return;
    }
    if (M == 2 && epoch_fast(p) && eff_qmax(p) < (1ull << 31) && ns >= (uint32_t)(kBigBlockPolar * h->num_sms)) {
        polar_kernel<kBigBlockPolar, 2, true><<<h->num_sms, kBigBlockPolar * 32, polar_smem(kBigBlockPolar), st>>>(p);
        return;
    }
    if ((M == 1 || NRNG_P2_PW) && p.aligned && p.log2E == 0 && eff_qmax(p) < (1ull << 31) &&
        ns >= (uint32_t)(kPwWarps * h->num_sms))
        pw_kernel<kPw, kPwWarps><<<h->num_sms, kPwWarps * 32, pw_smem(kPw, false, kPwWarps), st>>>(p);
    else if (ns >= (uint32_t)(kBigBlockPolar * h->num_sms))
        polar_kernel<kBigBlockPolar, M><<<h->num_sms, kBigBlockPolar * 32, polar_smem(kBigBlockPolar), st>>>(p);
    else if (M == 1 && NRNG_PW_SMALL && p.aligned && p.log2E == 0 && eff_qmax(p) < (1ull << 31))
        pw_kernel<4, kWarpsPerBlock><<<grid_for(ns, kWarpsPerBlock, h->occ.pw[0], h->num_sms), kWarpsPerBlock * 32,
                                       pw_smem(4, false, kWarpsPerBlock), st>>>(p);
    else
        polar_kernel<kWarpsPerBlock, M><<<grid_for(ns, kWarpsPerBlock, h->occ.polar, h->num_sms),
                                          kWarpsPerBlock * 32, polar_smem(kWarpsPerBlock), st>>>(p);
}

cudaError_t launch_bulk(nrng_handle h, Kind kind, BulkParams p, cudaStream_t st) {
    rc_reset(st);
    uint32_t ns = p.s_end - p.s_begin;
    const uint64_t qmax = eff_qmax(p);
    if (kind != Kind::UNIFORM && qmax >= kMidMinPairs && qmax <= kMidMaxPairs && NRNG_MID_MAX > 0) {
        const unsigned grid = (unsigned)std::min<uint64_t>((ns + kMidWarps - 1) / kMidWarps, (uint64_t)h->num_sms * 16);
        switch (kind) {
            case Kind::BM1: mid_kernel<1><<<grid, kMidWarps * 32, 0, st>>>(p); break;
            case Kind::BM2: mid_kernel<2><<<grid, kMidWarps * 32, 0, st>>>(p); break;
            case Kind::BM3: mid_kernel<3><<<grid, kMidWarps * 32, 0, st>>>(p); break;
            case Kind::POLAR2: mid_kernel<5><<<grid, kMidWarps * 32, 0, st>>>(p); break;
            case Kind::RATIO:   // R1's pretests change no output: its mid-size calls are R's
            case Kind::RATIO1: mid_kernel<6><<<grid, kMidWarps * 32, 0, st>>>(p); break;
            default: mid_kernel<4><<<grid, kMidWarps * 32, 0, st>>>(p); break;
        }
        h->launches += 1;
        return cudaGetLastError();
    }
    if (kind != Kind::UNIFORM && qmax <= kTinyMaxPairs) {
        const unsigned grid = (ns + kTinyThreads - 1) / kTinyThreads;
        switch (kind) {
            case Kind::BM1: tiny_kernel<1><<<grid, kTinyThreads, 0, st>>>(p); break;
            case Kind::BM2: tiny_kernel<2><<<grid, kTinyThreads, 0, st>>>(p); break;
            case Kind::BM3: tiny_kernel<3><<<grid, kTinyThreads, 0, st>>>(p); break;
            case Kind::POLAR2: tiny_kernel<5><<<grid, kTinyThreads, 0, st>>>(p); break;
            case Kind::RATIO:   // R1's pretests change no output: its short calls are R's
            case Kind::RATIO1: tiny_kernel<6><<<grid, kTinyThreads, 0, st>>>(p); break;
            default: tiny_kernel<4><<<grid, kTinyThreads, 0, st>>>(p); break;
        }
        h->launches += 1;
        return cudaGetLastError();
    }
    switch (kind) {
        case Kind::BM1: launch_bm<1>(h, p, ns, st); break;
        case Kind::BM2: launch_bm<2>(h, p, ns, st); break;
        case Kind::BM3: launch_bm<3>(h, p, ns, st); break;
        case Kind::POLAR: launch_polar<1>(h, p, ns, st); break;
        case Kind::POLAR2: launch_polar<2>(h, p, ns, st); break;
        case Kind::RATIO:
            if (ns >= (uint32_t)(kPwWarps * h->num_sms))
                pw_kernel<6, kPwWarps><<<h->num_sms, kPwWarps * 32, pw_smem(6, false, kPwWarps), st>>>(p);
            else
                pw_kernel<6, kWarpsPerBlock><<<grid_for(ns, kWarpsPerBlock, h->occ.ratio, h->num_sms),
                                                kWarpsPerBlock * 32, pw_smem(6, false, kWarpsPerBlock), st>>>(p);
            break;
        case Kind::RATIO1:
            if (ns >= (uint32_t)(kPwWarps * h->num_sms))
                pw_kernel<7, kPwWarps><<<h->num_sms, kPwWarps * 32, pw_smem(7, false, kPwWarps), st>>>(p);
            else
                pw_kernel<7, kWarpsPerBlock><<<grid_for(ns, kWarpsPerBlock, h->occ.ratio1, h->num_sms),
                                                kWarpsPerBlock * 32, pw_smem(7, false, kWarpsPerBlock), st>>>(p);
            break;
        case Kind::UNIFORM:
            uniform_kernel<<<grid_for(ns, kWarpsPerBlock, h->occ.uni, h->num_sms), kWarpsPerBlock * 32, kUniSmem,
                             st>>>(p);
            break;
    }
    h->launches += 1;
    return cudaGetLastError();
}

bool is_device_pointer(const void* ptr) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int ensure_staging(nrng_handle h) {
    if (h->stage[0]) return NRNG_OK;
    if (cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking) != cudaSuccess) return NRNG_ECUDA;
    for (int i = 0; i < 2; ++i) {
        if (cudaMalloc(&h->stage[i], kStageDoubles * sizeof(double)) != cudaSuccess) return NRNG_ENOMEM;
        if (cudaEventCreateWithFlags(&h->ev_ready[i], cudaEventDisableTiming) != cudaSuccess) return NRNG_ECUDA;
        if (cudaEventCreateWithFlags(&h->ev_free[i], cudaEventDisableTiming) != cudaSuccess) return NRNG_ECUDA;
    }
    return NRNG_OK;
}

// Per-stream quotas above this many units run as pieces of at most this many units per
// stream (BulkParams::jb/jcap): every kernel then counts a stream's units and words of one
// launch in 32 bits, and host outputs never need more than one staging buffer per stream.
constexpr uint64_t kPieceUnits = uint64_t(1) << 28;

// Fill `n` slots (units = pairs for normals, per_unit = 2; or uniforms / R's normals,
// per_unit = 1) into `out` (device or host).
//  * device output: one launch over all streams; quotas above kPieceUnits per stream run
//    as consecutive pieces (per-stream partition invariance makes that exact).
//  * host output: generated into two alternating device staging buffers of kStageDoubles
//    slots, each chunk's D2H copy on the copy stream overlapping the next chunk's kernel.
//    A chunk is a range of whole streams; a stream whose slots exceed a staging buffer is
//    produced alone, in pieces of kStageDoubles / per_unit units.
int run_bulk(nrng_handle h, Kind kind, double* out, size_t n, uint64_t units, int per_unit, double mu,
             double sigma) {
    BulkParams p{};
    p.ring = h->ring;
    p.count = h->count;
    p.units = units;
    p.q = units / h->S;
    p.rem = units % h->S;
    p.n = n;
    p.tp = TParams{mu, sigma, sigma * 0x1.6a09e667f3bcdp+0};
    const uint32_t active = p.q == 0 ? (uint32_t)p.rem : h->S;  // streams with work
    const uint64_t qmax = p.q + (p.rem ? 1 : 0);
    if (is_device_pointer(out)) {
        p.out = out;
        p.shift = 0;
        p.aligned = ((uintptr_t)out & 15) == 0;
        p.s_begin = 0;
        p.s_end = active;
        if (qmax <= kPieceUnits) return cuda_err(launch_bulk(h, kind, p, h->stream));
        p.jcap = kPieceUnits;
        cudaError_t e = cudaSuccess;
        for (p.jb = 0; p.jb < qmax && e == cudaSuccess; p.jb += kPieceUnits) e = launch_bulk(h, kind, p, h->stream);
        return cuda_err(e);
    }
    int rc = ensure_staging(h);
    if (rc != NRNG_OK) return set_err(rc);
    auto slot_off = [&](uint64_t k) { return (k * p.q + std::min<uint64_t>(k, p.rem)) * per_unit; };
    int buf = 0;
    cudaError_t e = cudaSuccess;
    // one chunk: streams [b, en), units [jb, jb + jcap) of each (jcap = 0: all), slots [lo, hi)
    auto chunk = [&](uint64_t b, uint64_t en, uint64_t jb, uint64_t jcap, uint64_t lo, uint64_t hi) {
        if (hi <= lo) return;
        if (hi - lo > kStageDoubles) {  // cannot happen by construction; never write past a stage
            e = cudaErrorInvalidValue;
            return;
        }
        e = cudaStreamWaitEvent(h->stream, h->ev_free[buf], 0);  // previous copy out of this buffer done
        if (e != cudaSuccess) return;
        p.out = h->stage[buf];
        p.shift = lo;
        p.aligned = 1;
        p.s_begin = (uint32_t)b;
        p.s_end = (uint32_t)en;
        p.jb = jb;
        p.jcap = jcap;
        e = launch_bulk(h, kind, p, h->stream);
        if (e != cudaSuccess) return;
        e = cudaEventRecord(h->ev_ready[buf], h->stream);
        if (e != cudaSuccess) return;
        e = cudaStreamWaitEvent(h->copy_stream, h->ev_ready[buf], 0);
        if (e != cudaSuccess) return;
        e = cudaMemcpyAsync(out + lo, h->stage[buf], (hi - lo) * sizeof(double), cudaMemcpyDeviceToHost,
                            h->copy_stream);
        if (e != cudaSuccess) return;
        e = cudaEventRecord(h->ev_free[buf], h->copy_stream);
        buf ^= 1;
    };
    const uint64_t slots_per_stream = qmax * per_unit;
    if (slots_per_stream <= kStageDoubles) {
        // whole streams per chunk, as many as fit a staging buffer
        const uint64_t g = kStageDoubles / slots_per_stream;
        for (uint64_t b = 0; b < active && e == cudaSuccess; b += g) {
            const uint64_t en = std::min<uint64_t>(active, b + g);
            chunk(b, en, 0, 0, slot_off(b), std::min<uint64_t>(slot_off(en), n));
        }
    } else {
        // few streams with long quotas: one stream per chunk, in pieces that fit a stage
        const uint64_t piece = kStageDoubles / per_unit;
        for (uint64_t k = 0; k < active && e == cudaSuccess; ++k) {
            const uint64_t cnt = p.q + (k < p.rem ? 1 : 0);
            for (uint64_t jb = 0; jb < cnt && e == cudaSuccess; jb += piece) {
                const uint64_t lo = slot_off(k) + jb * per_unit;
                const uint64_t hi = std::min<uint64_t>(lo + std::min(piece, cnt - jb) * per_unit, n);
                chunk(k, k + 1, jb, piece, lo, hi);
            }
        }
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->copy_stream);
    return cuda_err(e);
}

bool bad_params(double mu, double sigma) { return !std::isfinite(mu) || !std::isfinite(sigma) || sigma < 0; }

nrng_handle create_impl(uint64_t seed, uint64_t first, uint32_t S, int variant) {
    if (S == 0 || variant < 0 || variant > 3) {
        set_err(NRNG_EINVAL);
        return nullptr;
    }
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        set_err(NRNG_ENODEV);
        return nullptr;
    }
    nrng_gen* h = new (std::nothrow) nrng_gen();
    if (!h) {
        set_err(NRNG_ENOMEM);
        return nullptr;
    }
    h->device = dev;
    h->seed = seed;
    h->first = first;
    h->S = S;
    h->variant = variant == 0 ? 1 : variant;
    cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, dev);
    h->occ.bm[1] = occupancy(bm_kernel<1, kWarpsPerBlock>, kWarpsPerBlock, bm_smem(kWarpsPerBlock));
    h->occ.bm[2] = occupancy(bm_kernel<2, kWarpsPerBlock>, kWarpsPerBlock, bm_smem(kWarpsPerBlock));
    h->occ.bm[3] = occupancy(bm_kernel<3, kWarpsPerBlock>, kWarpsPerBlock, bm_smem(kWarpsPerBlock));
    h->occ.polar = occupancy(polar_kernel<kWarpsPerBlock, 1>, kWarpsPerBlock, polar_smem(kWarpsPerBlock));
    occupancy(polar_kernel<kWarpsPerBlock, 2>, kWarpsPerBlock, polar_smem(kWarpsPerBlock));
    occupancy(bm_kernel<1, kBigBlock>, kBigBlock, bm_smem(kBigBlock));
    occupancy(bm_kernel<2, kBigBlock>, kBigBlock, bm_smem(kBigBlock));
    occupancy(bm_kernel<3, kBigBlock>, kBigBlock, bm_smem(kBigBlock));
    occupancy(b3_kernel<kTriWarps>, kTriWarps, tri_smem(kTriWarps));
    occupancy(pw_kernel<1, kPwWarps>, kPwWarps, pw_smem(1, false, kPwWarps));
    occupancy(pw_kernel<2, kPwWarps>, kPwWarps, pw_smem(2, false, kPwWarps));
    occupancy(pw_kernel<4, kPwWarps>, kPwWarps, pw_smem(4, false, kPwWarps));
    occupancy(pw_kernel<5, kPwWarps>, kPwWarps, pw_smem(5, false, kPwWarps));
    occupancy(pw_kernel<6, kPwWarps>, kPwWarps, pw_smem(6, false, kPwWarps));
    occupancy(pw_kernel<1, kPwWarps, true>, kPwWarps, bm_smem(kPwWarps));
    occupancy(pw_kernel<2, kPwWarps, true>, kPwWarps, bm_smem(kPwWarps));
    occupancy(pw_kernel<4, kPwWarps, true>, kPwWarps, bm_smem(kPwWarps));
    occupancy(pw_kernel<5, kPwWarps, true>, kPwWarps, pw_smem(5, true, kPwWarps));
    occupancy(b3_kernel<kTriWarps, true>, kTriWarps, tri_smem(kTriWarps));
    h->occ.ratio = occupancy(pw_kernel<6, kWarpsPerBlock>, kWarpsPerBlock, pw_smem(6, false, kWarpsPerBlock));
    h->occ.pw[0] = occupancy(pw_kernel<4, kWarpsPerBlock>, kWarpsPerBlock, pw_smem(4, false, kWarpsPerBlock));
    h->occ.tri = occupancy(b3_kernel<kWarpsPerBlock>, kWarpsPerBlock, tri_smem(kWarpsPerBlock));
    h->occ.pw[1] = occupancy(pw_kernel<1, kWarpsPerBlock>, kWarpsPerBlock, pw_smem(1, false, kWarpsPerBlock));
    h->occ.pw[2] = occupancy(pw_kernel<2, kWarpsPerBlock>, kWarpsPerBlock, pw_smem(2, false, kWarpsPerBlock));
    occupancy(pw_kernel<7, kPwWarps>, kPwWarps, pw_smem(7, false, kPwWarps));
    h->occ.ratio1 = occupancy(pw_kernel<7, kWarpsPerBlock>, kWarpsPerBlock, pw_smem(7, false, kWarpsPerBlock));
    occupancy(polar_kernel<kBigBlockPolar, 1>, kBigBlockPolar, polar_smem(kBigBlockPolar));
    occupancy(polar_kernel<kBigBlockPolar, 2>, kBigBlockPolar, polar_smem(kBigBlockPolar));
    occupancy(polar_kernel<kBigBlockPolar, 2, true>, kBigBlockPolar, polar_smem(kBigBlockPolar));
    h->occ.uni = occupancy(uniform_kernel, kWarpsPerBlock, kUniSmem);
    h->occ.mask = occupancy(polar_mask_kernel, kWarpsPerBlock, kUniSmem);
    h->occ.init = occupancy(init_kernel, kWarpsPerBlock, kInitSmem);
    if (cudaMalloc(&h->ring, (size_t)S * kPitch * sizeof(uint64_t)) != cudaSuccess ||
        cudaMalloc(&h->count, (size_t)S * sizeof(uint64_t)) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(h->ring);
        delete h;
        set_err(NRNG_ENOMEM);
        return nullptr;
    }
    rc_reset(h->stream);
    init_kernel<<<grid_for(S, kWarpsPerBlock, h->occ.init, h->num_sms), kWarpsPerBlock * 32, kInitSmem, h->stream>>>(
        h->ring, h->count, seed, first, S);
    h->launches += 1;
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) {
        cuda_err(e);
        cudaFree(h->ring);
        cudaFree(h->count);
        delete h;
        return nullptr;
    }
    set_err(NRNG_OK);
    return h;
}

}  // namespace

extern "C" {

nrng_handle nrng_create(uint64_t seed, uint32_t n_streams, int variant) {
    return create_impl(seed, 0, n_streams, variant);
}

nrng_handle nrng_create_range(uint64_t seed, uint64_t first_stream, uint32_t n_streams, int variant) {
    return create_impl(seed, first_stream, n_streams, variant);
}

void nrng_destroy(nrng_handle h) {
    if (!h) return;
    cudaStreamSynchronize(h->stream);
    if (h->copy_stream) {
        cudaStreamSynchronize(h->copy_stream);
        cudaStreamDestroy(h->copy_stream);
    }
    for (int i = 0; i < 2; ++i) {
        cudaFree(h->stage[i]);
        if (h->ev_ready[i]) cudaEventDestroy(h->ev_ready[i]);
        if (h->ev_free[i]) cudaEventDestroy(h->ev_free[i]);
    }
    cudaFree(h->seq.buf);
    cudaFree(h->ring);
    cudaFree(h->count);
    delete h;
    set_err(NRNG_OK);
}

int nrng_set_stream(nrng_handle h, void* cuda_stream) {
    if (!h) return set_err(NRNG_EINVAL);
    h->stream = (cudaStream_t)cuda_stream;
    return set_err(NRNG_OK);
}

int nrng_normal_boxmuller(nrng_handle h, double* out, size_t n, double mu, double sigma, int variant) {
    if (!h || (n > 0 && !out) || bad_params(mu, sigma) || variant < 0 || variant > 3) return set_err(NRNG_EINVAL);
    if (!check_device(h)) return set_err(NRNG_EINVAL);
    if (n == 0) return set_err(NRNG_OK);
    const int v = variant == 0 ? h->variant : variant;
    const Kind k = v == 1 ? Kind::BM1 : (v == 2 ? Kind::BM2 : Kind::BM3);
    return run_bulk(h, k, out, n, (n + 1) / 2, 2, mu, sigma);
}

int nrng_normal_polar(nrng_handle h, double* out, size_t n, double mu, double sigma) {
    if (!h || (n > 0 && !out) || bad_params(mu, sigma)) return set_err(NRNG_EINVAL);
    if (!check_device(h)) return set_err(NRNG_EINVAL);
    if (n == 0) return set_err(NRNG_OK);
    return run_bulk(h, Kind::POLAR, out, n, (n + 1) / 2, 2, mu, sigma);
}

int nrng_normal_polar2(nrng_handle h, double* out, size_t n, double mu, double sigma) {
    if (!h || (n > 0 && !out) || bad_params(mu, sigma)) return set_err(NRNG_EINVAL);
    if (!check_device(h)) return set_err(NRNG_EINVAL);
    if (n == 0) return set_err(NRNG_OK);
    return run_bulk(h, Kind::POLAR2, out, n, (n + 1) / 2, 2, mu, sigma);
}

int nrng_normal_ratio(nrng_handle h, double* out, size_t n, double mu, double sigma) {
    if (!h || (n > 0 && !out) || bad_params(mu, sigma)) return set_err(NRNG_EINVAL);
    if (!check_device(h)) return set_err(NRNG_EINVAL);
    if (n == 0) return set_err(NRNG_OK);
    return run_bulk(h, Kind::RATIO, out, n, n, 1, mu, sigma);  // units: normals (R26)
}

int nrng_normal_ratio1(nrng_handle h, double* out, size_t n, double mu, double sigma) {
    if (!h || (n > 0 && !out) || bad_params(mu, sigma)) return set_err(NRNG_EINVAL);
    if (!check_device(h)) return set_err(NRNG_EINVAL);
    if (n == 0) return set_err(NRNG_OK);
    return run_bulk(h, Kind::RATIO1, out, n, n, 1, mu, sigma);  // units: normals (R26)
}

// ---------------------------------------------------------------- sequential mode
namespace {
Kind kind_of(int method) {
    return method == 1 ? Kind::BM1 : method == 2 ? Kind::BM2 : method == 3 ? Kind::BM3
         : method == 4 ? Kind::POLAR : Kind::POLAR2;
}
// `epochs` whole epochs into device memory dst (epoch layout).
int seq_epochs(nrng_handle h, int method, double* dst, uint64_t epochs, double mu, double sigma) {
    // whole epochs are contiguous blocks of the epoch-major output, so a long run goes as
    // consecutive launches of at most kPieceUnits pairs per stream (the kernels count a
    // launch's units and words per stream in 32 bits), exact by partition invariance
    const uint64_t max_epochs = std::max<uint64_t>(1, kPieceUnits >> h->seq.log2E);
    const uint64_t epoch_deviates = 2ull * h->S << h->seq.log2E;
    cudaError_t e = cudaSuccess;
    for (uint64_t e0 = 0; e0 < epochs && e == cudaSuccess; e0 += max_epochs) {
        BulkParams p{};
        p.ring = h->ring;
        p.count = h->count;
        p.q = std::min(max_epochs, epochs - e0) << h->seq.log2E;
        p.rem = 0;
        p.units = p.q * h->S;
        p.n = 2 * p.units;
        p.tp = TParams{mu, sigma, sigma * 0x1.6a09e667f3bcdp+0};
        p.out = dst + e0 * epoch_deviates;
        p.shift = 0;
        p.aligned = ((uintptr_t)p.out & 15) == 0;
        p.s_begin = 0;
        p.s_end = h->S;
        p.log2E = h->seq.log2E;
        p.S = h->S;
        e = launch_bulk(h, kind_of(method), p, h->stream);
    }
    return cuda_err(e);
}
}  // namespace

int nrng_seq_configure(nrng_handle h, uint32_t epoch_pairs) {
    if (!h || epoch_pairs < 128 || epoch_pairs > (1u << 20) || (epoch_pairs & (epoch_pairs - 1)))
        return set_err(NRNG_EINVAL);
    cudaStreamSynchronize(h->stream);
    cudaFree(h->seq.buf);
    h->seq.buf = nullptr;
    h->seq.log2E = 31 - __builtin_clz(epoch_pairs);
    h->seq.len = h->seq.pos = 0;
    return set_err(NRNG_OK);
}

int nrng_seq_reset(nrng_handle h) {
    if (!h) return set_err(NRNG_EINVAL);
    h->seq.len = h->seq.pos = 0;
    return set_err(NRNG_OK);
}

size_t nrng_seq_buffered(nrng_handle h) { return h ? (size_t)(h->seq.len - h->seq.pos) : 0; }

int nrng_normal_seq(nrng_handle h, double* out, size_t n, double mu, double sigma, int method) {
    if (!h || (n > 0 && !out) || bad_params(mu, sigma) || method < 1 || method > 5) return set_err(NRNG_EINVAL);
    if (!check_device(h)) return set_err(NRNG_EINVAL);
    auto& q = h->seq;
    if (q.pos < q.len && (q.method != method || q.mu != mu || q.sigma != sigma)) return set_err(NRNG_EINVAL);
    if (n == 0) return set_err(NRNG_OK);
    const uint64_t epoch = 2ull * h->S << q.log2E;  // deviates per epoch
    if (!q.buf && cudaMalloc(&q.buf, epoch * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        return set_err(NRNG_ENOMEM);
    }
    cudaError_t e = cudaSuccess;
    uint64_t done = std::min<uint64_t>(n, q.len - q.pos);
    // whole epochs go straight into device outputs that are 16-byte aligned where they start
    const bool dev = is_device_pointer(out) && (((uintptr_t)(out + done)) & 15) == 0;
    if (done) e = cudaMemcpyAsync(out, q.buf + q.pos, done * sizeof(double), cudaMemcpyDefault, h->stream);
    q.pos += done;
    if (e != cudaSuccess) return cuda_err(e);
    const uint64_t whole = (n - done) / epoch;
    if (whole) {
        if (dev) {
            const int rc = seq_epochs(h, method, out + done, whole, mu, sigma);
            if (rc != NRNG_OK) return rc;
            done += whole * epoch;
        } else {
            for (uint64_t i = 0; i < whole; ++i, done += epoch) {
                int rc = seq_epochs(h, method, q.buf, 1, mu, sigma);
                if (rc != NRNG_OK) return rc;
                e = cudaMemcpyAsync(out + done, q.buf, epoch * sizeof(double), cudaMemcpyDefault, h->stream);
                if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
                if (e != cudaSuccess) return cuda_err(e);
            }
        }
    }
    if (done < n) {
        const int rc = seq_epochs(h, method, q.buf, 1, mu, sigma);
        if (rc != NRNG_OK) return rc;
        q.len = epoch;
        q.pos = n - done;
        q.method = method;
        q.mu = mu;
        q.sigma = sigma;
        e = cudaMemcpyAsync(out + done, q.buf, q.pos * sizeof(double), cudaMemcpyDefault, h->stream);
        if (e != cudaSuccess) return cuda_err(e);
    }
    if (!dev) e = cudaStreamSynchronize(h->stream);
    return cuda_err(e);
}

int nrng_uniform(nrng_handle h, double* out, size_t n) {
    if (!h || (n > 0 && !out)) return set_err(NRNG_EINVAL);
    if (!check_device(h)) return set_err(NRNG_EINVAL);
    if (n == 0) return set_err(NRNG_OK);
    return run_bulk(h, Kind::UNIFORM, out, n, n, 1, 0.0, 1.0);
}

int nrng_polar_mask(nrng_handle h, uint8_t* dev_mask, size_t cand_per_stream) {
    if (!h || (cand_per_stream > 0 && !dev_mask)) return set_err(NRNG_EINVAL);
    if (!check_device(h)) return set_err(NRNG_EINVAL);
    if (cand_per_stream == 0) return set_err(NRNG_OK);
    BulkParams p{};
    p.ring = h->ring;
    p.count = h->count;
    p.s_begin = 0;
    p.s_end = h->S;
    rc_reset(h->stream);
    polar_mask_kernel<<<grid_for(h->S, kWarpsPerBlock, h->occ.mask, h->num_sms), kWarpsPerBlock * 32, kUniSmem,
                        h->stream>>>(
        p, dev_mask, cand_per_stream);
    h->launches += 1;
    return cuda_err(cudaGetLastError());
}

int nrng_transform_from_uniforms(const double* dev_u, size_t n_pairs, double* dev_out, uint8_t* dev_mask, double mu,
                                 double sigma, int method, void* cuda_stream) {
    if ((n_pairs > 0 && (!dev_u || !dev_out)) || bad_params(mu, sigma) || method < 1 || method > 7)
        return set_err(NRNG_EINVAL);
    if (n_pairs == 0) return set_err(NRNG_OK);
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) != cudaSuccess) return set_err(NRNG_ENODEV);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)std::min<uint64_t>((n_pairs + kTransformThreads - 1) / kTransformThreads, (uint64_t)sms * 8);
    transform_kernel<<<grid, kTransformThreads, 0, (cudaStream_t)cuda_stream>>>(dev_u, n_pairs, dev_out, dev_mask,
                                                                  TParams{mu, sigma, sigma * 0x1.6a09e667f3bcdp+0}, method);
    return cuda_err(cudaGetLastError());
}

int nrng_stats(const double* dev_x, size_t n, double center, const double* dev_edges, int K, double* dev_sums,
               int64_t* dev_hist, void* cuda_stream) {
    if (K < 2 || K > 1024 || !dev_edges || !dev_sums || !dev_hist || (n > 0 && !dev_x) || !std::isfinite(center))
        return set_err(NRNG_EINVAL);
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) != cudaSuccess) return set_err(NRNG_ENODEV);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const int nblocks = (int)std::max<uint64_t>(1, std::min<uint64_t>((n + kStatsThreads - 1) / kStatsThreads,
                                                                      (uint64_t)sms * 8));
    double* partial = nullptr;
    cudaError_t e = cudaMallocAsync(&partial, (size_t)nblocks * kStatsPartial * sizeof(double), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(dev_hist, 0, (size_t)K * sizeof(int64_t), st);
    if (e == cudaSuccess) {
        stats_partial_kernel<<<nblocks, kStatsThreads, 0, st>>>(dev_x, n, center, dev_edges, K, partial,
                                                               reinterpret_cast<unsigned long long*>(dev_hist));
        stats_final_kernel<<<1, kStatsFinalThreads, 0, st>>>(partial, nblocks, dev_sums);
        e = cudaGetLastError();
    }
    if (partial) cudaFreeAsync(partial, st);
    return cuda_err(e);
}

int nrng_gof_hist(const double* dev_x, size_t n, double mu, double sigma, int log2K, uint32_t* dev_hist,
                  void* cuda_stream) {
    if (log2K < 4 || log2K > 24 || !dev_hist || (n > 0 && !dev_x) || bad_params(mu, sigma) || !(sigma > 0))
        return set_err(NRNG_EINVAL);
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) != cudaSuccess) return set_err(NRNG_ENODEV);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaStream_t st = (cudaStream_t)cuda_stream;
    cudaError_t e = cudaMemsetAsync(dev_hist, 0, sizeof(uint32_t) << log2K, st);
    if (e == cudaSuccess && n > 0) {
        const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)sms * 16));
        gof_hist_kernel<<<grid, 256, 0, st>>>(dev_x, n, mu, 1.0 / sigma, log2K, dev_hist);
        e = cudaGetLastError();
    }
    return cuda_err(e);
}

int nrng_serial_corr(const double* dev_x, size_t n, double center, int K, double* dev_partial, void* cuda_stream) {
    if (K < 1 || K > kCorrMaxLag || (n > 0 && (!dev_x || !dev_partial)) || !std::isfinite(center))
        return set_err(NRNG_EINVAL);
    if (n == 0) return set_err(NRNG_OK);
    const unsigned blocks = (unsigned)nrng_serial_corr_blocks(n);
    serial_corr_kernel<<<blocks, 128, 0, (cudaStream_t)cuda_stream>>>(dev_x, n, center, K, dev_partial);
    return cuda_err(cudaGetLastError());
}

size_t nrng_serial_corr_blocks(size_t n) {
    const uint64_t tiles = (n + kCorrTile - 1) / kCorrTile;
    return (size_t)std::min<uint64_t>(tiles, kCorrGrid);
}

int nrng_racecheck_result(uint64_t* host_out3) {
    if (!host_out3) return set_err(NRNG_EINVAL);
    host_out3[0] = host_out3[1] = host_out3[2] = 0;
#if NRNG_RACECHECK
    if (!rc_ready()) return set_err(NRNG_ENOMEM);
    cudaDeviceSynchronize();
    cudaError_t e = cudaMemcpy(host_out3, g_rc_host.races, 16, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(host_out3 + 2, g_rc_host.checks, 8, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemset(g_rc_host.races, 0, 16);
    if (e == cudaSuccess) e = cudaMemset(g_rc_host.checks, 0, 8);
    return cuda_err(e);
#else
    return set_err(NRNG_EINVAL);  // not a NRNG_RACECHECK build
#endif
}

int nrng_last_error(void) { return g_last; }

const char* nrng_error_string(int code) {
    switch (code) {
        case NRNG_OK: return "ok";
        case NRNG_EINVAL: return "invalid argument";
        case NRNG_ENOMEM: return "out of device memory";
        case NRNG_ECUDA: return "CUDA error";
        case NRNG_ENODEV: return "no CUDA device";
        default: return "unknown error";
    }
}

uint32_t nrng_num_streams(nrng_handle h) { return h ? h->S : 0; }
uint64_t nrng_first_stream(nrng_handle h) { return h ? h->first : 0; }
uint64_t nrng_kernel_launches(nrng_handle h) { return h ? h->launches : 0; }

int nrng_synchronize(nrng_handle h) {
    if (!h) return set_err(NRNG_EINVAL);
    cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e == cudaSuccess && h->copy_stream) e = cudaStreamSynchronize(h->copy_stream);
    return cuda_err(e);
}

int nrng_stream_counts(nrng_handle h, uint64_t* host_counts) {
    if (!h || !host_counts) return set_err(NRNG_EINVAL);
    cudaError_t e = cudaMemcpyAsync(host_counts, h->count, (size_t)h->S * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                    h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    return cuda_err(e);
}

int nrng_get_state(nrng_handle h, uint64_t* host_ring, uint64_t* host_counts) {
    if (!h) return set_err(NRNG_EINVAL);
    cudaError_t e = cudaSuccess;
    if (host_ring)
        e = cudaMemcpy2DAsync(host_ring, kLagR * sizeof(uint64_t), h->ring, kPitch * sizeof(uint64_t),
                              kLagR * sizeof(uint64_t), h->S, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess && host_counts)
        e = cudaMemcpyAsync(host_counts, h->count, (size_t)h->S * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                            h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    return cuda_err(e);
}

int nrng_set_state(nrng_handle h, const uint64_t* host_ring, const uint64_t* host_counts) {
    if (!h) return set_err(NRNG_EINVAL);
    h->seq.len = h->seq.pos = 0;  // deviates buffered by the sequential mode came from the old state
    cudaError_t e = cudaSuccess;
    if (host_ring)
        e = cudaMemcpy2DAsync(h->ring, kPitch * sizeof(uint64_t), host_ring, kLagR * sizeof(uint64_t),
                              kLagR * sizeof(uint64_t), h->S, cudaMemcpyHostToDevice, h->stream);
    if (e == cudaSuccess && host_counts)
        e = cudaMemcpyAsync(h->count, host_counts, (size_t)h->S * sizeof(uint64_t), cudaMemcpyHostToDevice,
                            h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    return cuda_err(e);
}

}  // extern "C"
