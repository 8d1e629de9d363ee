// Sustained write bandwidth and board power of two 16 GiB store patterns on B200:
//  linear : grid-stride 16-byte streaming stores (what a memset does)
//  streams: 2960 warps, each writing its own contiguous 256 KB region 2 KB per step
//           (the generator kernels' stream-major output pattern)
// usage: ./write_pattern  (prints ms per pass; sample nvidia-smi alongside)
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <unistd.h>
template <int CS>
__global__ void linear(double2* out, uint64_t n2, double v) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n2; i += (uint64_t)gridDim.x * blockDim.x) {
        if (CS) __stcs(out + i, make_double2(v, v + 1));
        else out[i] = make_double2(v, v + 1);
    }
}
template <int CS>
__global__ void streams(double2* out, uint32_t nstreams, uint32_t per_stream2, double v, int warps_per_block) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint32_t k = blockIdx.x * warps_per_block + warp; k < nstreams; k += gridDim.x * warps_per_block) {
        double2* o = out + (uint64_t)k * per_stream2 + lane;
        for (uint32_t j = 0; j < per_stream2; j += 128, o += 128) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (CS) __stcs(o + 32 * u, make_double2(v + j, v - j));
                else o[32 * u] = make_double2(v + j, v - j);
            }
        }
    }
}
int main(int argc, char** argv) {
    const uint64_t n2 = 1ull << 30;  // double2 = 16 GiB
    double2* d;
    cudaMalloc(&d, n2 * 16);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 4; ++mode) {
        float best = 1e9, total = 0;
        int reps = 0;
        cudaEventRecord(a);
        while (total < 1000) {
            cudaEvent_t x, y;
            cudaEventCreate(&x);
            cudaEventCreate(&y);
            cudaEventRecord(x);
            if (mode == 0)
                linear<1><<<148 * 8, 256>>>(d, n2, 1.0 + reps);
            else if (mode == 1)
                streams<1><<<148, 640>>>(d, 65536, 1 << 14, 1.0 + reps, 20);
            else if (mode == 2)
                linear<0><<<148 * 8, 256>>>(d, n2, 1.0 + reps);
            else
                streams<0><<<148, 640>>>(d, 65536, 1 << 14, 1.0 + reps, 20);
            cudaEventRecord(y);
            cudaEventSynchronize(y);
            float ms;
            cudaEventElapsedTime(&ms, x, y);
            best = ms < best ? ms : best;
            total += ms;
            ++reps;
        }
        const char* names[4] = {"linear .cs", "streams .cs", "linear wb", "streams wb"};
        printf("%s: best %.3f ms, mean %.3f ms over %d passes (%.1f GB/s mean)\n", names[mode], best,
               total / reps, reps, n2 * 16 / (total / reps) / 1e6);
        fflush(stdout);
        sleep(1);
    }
    return 0;
}
