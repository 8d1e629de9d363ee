// nrng_racecheck.cuh -- an intra-warp shared-memory race detector for a DEBUG build of the
// library (-DNRNG_RACECHECK=1, tools/racecheck.sh); in the product build every macro here is
// the plain access.
//
// Why: each warp owns its stream's window (and a 32-slot scratch) in shared memory; lanes read
// words other lanes wrote, ordered only by __syncwarp().  compute-sanitizer (racecheck /
// synccheck) is closed on this GPU pool, so the debug build checks the same property itself.
//
// Model: every thread counts the barriers it has passed -- __syncwarp() (NRNG_SYNCWARP) and
// __syncthreads() (NRNG_SYNCTHREADS) -- its epoch.  The warps of a block pass the same
// __syncthreads(), the lanes of a warp the same __syncwarp(), and a word is shared either within
// one warp (the windows and scratch of the warp-per-stream kernels) or by a block with only
// __syncthreads() ordering it (NRNG_SYNCTHREADS), so the accessors of one word always have
// comparable epochs.  Two accesses to one 8-byte shared word by different threads, at least one
// a write, race unless a barrier separates them, i.e. unless their epochs differ.  Every
// instrumented access checks and records, in global shadow arrays indexed by (block, shared word):
//   W[word] = (epoch + 1) << 32 | writer thread                       (last write)
//   R[word] = (epoch + 1) << 32 | several-readers flag << 16 | reader (reads in that epoch)
//   load  by thread t in epoch e: RAW race if W's epoch is e and its writer is not t;
//   store by thread t in epoch e: WAW race if W's epoch is e and its writer is not t,
//                                 WAR race if R's epoch is e and a thread other than t read.
// Races are counted; the first one's source line, kind and threads are kept
// (nrng_racecheck_result).  The shadows and epochs are cleared before every launch.
#pragma once
#include <cstdint>

#ifndef NRNG_RACECHECK
#define NRNG_RACECHECK 0
#endif

namespace nrng {

#if NRNG_RACECHECK
constexpr uint32_t kRcShadowWords = 232448 / 8;  // one per 8 bytes of a block's shared memory
constexpr uint32_t kRcMaxBlocks = 2368;          // blocks shadowed (larger grids: blocks beyond share)
constexpr uint32_t kRcMaxThreads = kRcMaxBlocks * 640;
struct RcState {
    unsigned long long* w;      // kRcMaxBlocks x kRcShadowWords
    unsigned long long* r;      // kRcMaxBlocks x kRcShadowWords
    uint32_t* epoch;            // per thread (block-major)
    unsigned long long* races;  // [0] count, [1] first race: line << 32 | kind << 24 | thread << 12 | other
    unsigned long long* checks; // accesses checked
};
__device__ RcState g_rc;

__device__ __forceinline__ uint32_t rc_tid() {
    return (blockIdx.x % kRcMaxBlocks) * blockDim.x + threadIdx.x;
}
__device__ __forceinline__ void rc_report(uint32_t line, uint32_t kind, uint32_t me, uint32_t other) {
    const unsigned long long n = atomicAdd(&g_rc.races[0], 1ull);
    if (n == 0)
        atomicExch(&g_rc.races[1], ((unsigned long long)line << 32) | (kind << 24) | ((me & 0xfff) << 12) |
                                       (other & 0xfff));
}
// kind: 1 RAW, 2 WAW, 3 WAR; threads are threadIdx.x (lane + 32 warp)
__device__ __forceinline__ void rc_access(const void* p, bool store, uint32_t line) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
    const uint64_t slot = (uint64_t)(blockIdx.x % kRcMaxBlocks) * kRcShadowWords + (a >> 3);
    const uint32_t me = threadIdx.x;
    const unsigned long long e = (unsigned long long)g_rc.epoch[rc_tid()] + 1;
    atomicAdd(&g_rc.checks[0], 1ull);
    if (store) {
        const unsigned long long w = atomicExch(&g_rc.w[slot], (e << 32) | me);
        if ((w >> 32) == e && (uint32_t)(w & 0xffff) != me) rc_report(line, 2, me, (uint32_t)(w & 0xffff));
        const unsigned long long r = atomicAdd(&g_rc.r[slot], 0ull);
        if ((r >> 32) == e && (((r >> 16) & 1) || (uint32_t)(r & 0xffff) != me))
            rc_report(line, 3, me, (uint32_t)(r & 0xffff));
    } else {
        const unsigned long long w = atomicAdd(&g_rc.w[slot], 0ull);
        if ((w >> 32) == e && (uint32_t)(w & 0xffff) != me) rc_report(line, 1, me, (uint32_t)(w & 0xffff));
        unsigned long long old = atomicAdd(&g_rc.r[slot], 0ull);
        for (;;) {  // this epoch's first reader, or mark the word read by several threads
            const unsigned long long nw = ((old >> 32) != e) ? ((e << 32) | me)
                                          : ((uint32_t)(old & 0xffff) == me ? old : (old | (1ull << 16)));
            if (nw == old) break;
            const unsigned long long prev = atomicCAS(&g_rc.r[slot], old, nw);
            if (prev == old) break;
            old = prev;
        }
    }
}
template <typename T>
__device__ __forceinline__ T rc_ld(const T* p, uint32_t line) {
    for (uint32_t b = 0; b < sizeof(T); b += 8) rc_access(reinterpret_cast<const char*>(p) + b, false, line);
    return *p;
}
template <typename T>
__device__ __forceinline__ void rc_st(T* p, const T& v, uint32_t line) {
    for (uint32_t b = 0; b < sizeof(T); b += 8) rc_access(reinterpret_cast<const char*>(p) + b, true, line);
    *p = v;
}
__device__ __forceinline__ void rc_sync() {
    __syncwarp();
    g_rc.epoch[rc_tid()] += 1;
}
__device__ __forceinline__ void rc_syncthreads() {
    __syncthreads();
    g_rc.epoch[rc_tid()] += 1;
}
#define NRNG_LD(p) ::nrng::rc_ld((p), __LINE__)
#define NRNG_ST(p, v) ::nrng::rc_st((p), (v), __LINE__)
#define NRNG_SYNCWARP() ::nrng::rc_sync()
#define NRNG_SYNCTHREADS() ::nrng::rc_syncthreads()
#else
#define NRNG_LD(p) (*(p))
#define NRNG_ST(p, v) (*(p) = (v))
#define NRNG_SYNCWARP() __syncwarp()
#define NRNG_SYNCTHREADS() __syncthreads()
#endif

}  // namespace nrng
