// Probe: sustained FP64 DFMA rate and HBM write bandwidth on this B200.
// Used to derive the ALU roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void dfma_loop(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3,
           x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 1234.5) out[0] = s;
}
__global__ void store_kernel(double2* out, size_t n2) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
    for (; i < n2; i += st) __stcs(out + i, make_double2((double)i, 1.0));
}
__global__ void libm_loop(double* out, int iters) {
    double acc = 0, u = (threadIdx.x + 1) * 1e-4;
    for (int i = 0; i < iters; ++i) { double s, c; sincospi(u, &s, &c); acc += sqrt(-2.0 * log(u)) * s + c; u += 1e-7; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
    printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
    double* d; CK(cudaMalloc(&d, 1 << 26));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int blocksPerSM : {4, 8, 16}) {
        int grid = p.multiProcessorCount * blocksPerSM, iters = 4000;
        dfma_loop<<<grid, 128>>>(d, 10, 1.0000001, 1e-9);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        dfma_loop<<<grid, 128>>>(d, iters, 1.0000001, 1e-9);
        cudaEventRecord(b); CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b);
        double dfma = (double)grid * 128 * iters * 16 * 8;
        printf("DFMA blocks/SM=%d: %.4e DFMA/s = %.2f TFLOP/s (%.3f ms)\n", blocksPerSM, dfma / ms * 1e3, 2 * dfma / ms * 1e-9, ms);
    }
    size_t bytes = (size_t)8 << 30; double2* o; CK(cudaMalloc(&o, bytes));
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a);
        store_kernel<<<p.multiProcessorCount * 16, 256>>>(o, bytes / 16);
        cudaEventRecord(b); CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("write-only store: %.1f GB/s\n", bytes / ms * 1e-6);
    }
    for (int r = 0; r < 2; ++r) {
        int grid = p.multiProcessorCount * 8, iters = 2000;
        cudaEventRecord(a);
        libm_loop<<<grid, 128>>>(d, iters);
        cudaEventRecord(b); CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("libdevice log+sqrt+sincospi: %.4e evals/s\n", (double)grid * 128 * iters / ms * 1e3);
    }
    return 0;
}
