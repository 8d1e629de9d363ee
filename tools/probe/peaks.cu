// Peak probe for the roofline denominators that MEASURED_PEAKS.json does not carry (SURVEY
// §8(d)): the FP64 DFMA instruction rate and the HBM write-only bandwidth on this B200, each
// as a burst (a short run from idle) and sustained (back-to-back launches for >= 2.5 s, the
// median launch of the last second: the regime of bench.py's long step, where the board sits
// at its 1000 W power cap).  Prints one JSON object.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe/peaks tools/probe/peaks.cu
//   tools/probe/peaks > profiles/<tag>_peaks.json   (clocks sampled beside it: tools/probe/peaks.sh)
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e = (x);                                                               \
        if (e != cudaSuccess) {                                                            \
            fprintf(stderr, "CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);           \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

// 8 independent DFMA chains per thread, 16 x 8 DFMA per loop trip: FP64-pipe bound.
__global__ void dfma_loop(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
           x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 1234.5) out[0] = s;
}

// 16-byte streaming stores over the buffer (the output path of the generators).
__global__ void store_kernel(double2* out, size_t n2) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t st = (size_t)gridDim.x * blockDim.x;
    for (; i < n2; i += st) __stcs(out + i, make_double2((double)i, 1.0));
}

template <typename F>
static int time_series(F launch, double seconds, std::vector<float>& ms_out) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        CK(cudaEventRecord(a));
        launch();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        ms_out.push_back(ms);
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (el >= seconds) break;
    }
    return 0;
}

static double median_of_last(const std::vector<float>& v, double total_s, double last_s) {
    // launches of the last `last_s` seconds (equal-length launches: a suffix of the series)
    const size_t n = v.size();
    size_t k = (size_t)std::max<double>(1.0, n * last_s / total_s);
    std::vector<float> t(v.end() - std::min(k, n), v.end());
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

int main() {
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, 0));
    double* d;
    CK(cudaMalloc(&d, 1 << 20));
    const int grid = p.multiProcessorCount * 16, threads = 128, iters = 2000;
    const double dfma_per_launch = (double)grid * threads * iters * 16 * 8;
    auto dl = [&] { dfma_loop<<<grid, threads>>>(d, iters, 1.0000001, 1e-9); };
    // burst: from idle, best of 3 short launches
    CK(cudaDeviceSynchronize());
    std::vector<float> burst;
    for (int r = 0; r < 3; ++r) {
        std::vector<float> one;
        if (time_series(dl, 0.0, one)) return 1;
        burst.push_back(one[0]);
    }
    const double f_burst = dfma_per_launch / (*std::min_element(burst.begin(), burst.end()) * 1e-3);
    std::vector<float> sus;
    if (time_series(dl, 3.0, sus)) return 1;
    const double f_sus = dfma_per_launch / (median_of_last(sus, 3.0, 1.0) * 1e-3);

    const size_t bytes = (size_t)16 << 30;  // 16 GiB: the generators' per-launch output
    double2* o;
    CK(cudaMalloc(&o, bytes));
    auto sl = [&] { store_kernel<<<p.multiProcessorCount * 16, 256>>>(o, bytes / 16); };
    CK(cudaDeviceSynchronize());
    std::vector<float> wb;
    if (time_series(sl, 0.0, wb)) return 1;  // first touch
    wb.clear();
    for (int r = 0; r < 3; ++r) {
        std::vector<float> one;
        if (time_series(sl, 0.0, one)) return 1;
        wb.push_back(one[0]);
    }
    const double w_burst = bytes / (*std::min_element(wb.begin(), wb.end()) * 1e-3);
    std::vector<float> ws;
    if (time_series(sl, 3.0, ws)) return 1;
    const double w_sus = bytes / (median_of_last(ws, 3.0, 1.0) * 1e-3);
    printf("{\"device\": \"%s\", \"sms\": %d, \"fp64_dfma_per_s_burst\": %.6e, \"fp64_dfma_per_s_sustained\": %.6e, "
           "\"hbm_write_gbs_burst\": %.1f, \"hbm_write_gbs_sustained\": %.1f, \"dfma_launches\": %zu, "
           "\"store_launches\": %zu, \"how\": \"dfma_loop: %d blocks x %d threads x 8 chains, %.0f DFMA per launch; "
           "store_kernel: 16-byte st.global.cs over 16 GiB; burst = best of 3 launches from idle, sustained = median "
           "launch of the last 1 s of 3 s back to back\"}\n",
           p.name, p.multiProcessorCount, f_burst, f_sus, w_burst * 1e-9, w_sus * 1e-9, sus.size(), ws.size(), grid,
           threads, dfma_per_launch);
    return 0;
}
