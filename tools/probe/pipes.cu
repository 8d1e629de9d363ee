// Probe: throughput of the instructions the hot path leans on (per SM per clock).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, long long seed, int iters) {
    long long a0 = seed + threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7;
    double d0 = a0 * 1e-3, d1 = d0 + 1, d2 = d0 + 2, d3 = d0 + 3, acc = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (OP == 0) {  // I2F.F64.S64
                acc += 0;  d0 = (double)a0; d1 = (double)a1; d2 = (double)a2; d3 = (double)a3;
                a0 += 1; a1 += 1; a2 += 1; a3 += 1;
            } else if (OP == 1) {  // DADD
                d0 = d0 + 1.5; d1 = d1 + 1.5; d2 = d2 + 1.5; d3 = d3 + 1.5;
            } else if (OP == 2) {  // MUFU.RSQ64H
                double r0, r1, r2, r3;
                asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(d0));
                asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r1) : "d"(d1));
                asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r2) : "d"(d2));
                asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r3) : "d"(d3));
                d0 = r0 + 1.0; d1 = r1 + 1.0; d2 = r2 + 1.0; d3 = r3 + 1.0;
            } else if (OP == 3) {  // I2F.F64.U32
                d0 = (double)(unsigned)a0; d1 = (double)(unsigned)a1; d2 = (double)(unsigned)a2; d3 = (double)(unsigned)a3;
                a0 += 1; a1 += 1; a2 += 1; a3 += 1;
            } else if (OP == 4) {  // F2I.S64.F64 (round)
                a0 += __double2ll_rn(d0); a1 += __double2ll_rn(d1); a2 += __double2ll_rn(d2); a3 += __double2ll_rn(d3);
                d0 += 1; d1 += 1; d2 += 1; d3 += 1;
            } else if (OP == 5) {  // DMUL + DFMA mix
                d0 = fma(d0, 1.0000001, 0.5); d1 = fma(d1, 1.0000001, 0.5); d2 = d2 * 1.0000001; d3 = d3 * 0.9999999;
            }
            if (OP == 0 || OP == 3) acc += d0 + d1 + d2 + d3;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + d0 + d1 + d2 + d3 + (double)(a0 + a1 + a2 + a3);
}
template <int OP>
void run(const char* name, int sms, double per_iter_ops) {
    double* d; cudaMalloc(&d, sizeof(double) * sms * 16 * 256);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int iters = 2000;
    k<OP><<<sms * 8, 256>>>(d, 1, 10);
    cudaEventRecord(a);
    k<OP><<<sms * 8, 256>>>(d, 1, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double thr = (double)sms * 8 * 256 * iters * 8 * per_iter_ops;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-22s %.3e thread-ops/s  = %.1f per SM per clk@1.9GHz\n", name, thr / ms * 1e3, thr / ms * 1e3 / sms / 1.9e9);
    cudaFree(d);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>("I2F.F64.S64 (+4 DADD)", sms, 4);
    run<3>("I2F.F64.U32 (+4 DADD)", sms, 4);
    run<1>("DADD", sms, 4);
    run<2>("MUFU.RSQ64H (+DADD)", sms, 4);
    run<4>("F2I.S64.F64 (+DADD)", sms, 4);
    run<5>("DFMA/DMUL", sms, 4);
    return 0;
}
