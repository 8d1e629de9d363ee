/* A plain-C user of the C ABI (include/nrng.h) -- no Python, no CUDA headers: the library
 * stages host outputs itself.  Generates 2^24 normals over 2^14 streams by B3 and by Polar into
 * host memory, checks (1) the per-stream partition invariance of two half-size calls against
 * one full call, bit for bit, (2) the sample mean and variance, (3) an argument error.
 *
 *   gcc -std=c11 -O2 -Iinclude examples/c_api_demo.c -Lpaper_1004_3105_b200 -lnrng \
 *       -Wl,-rpath,$PWD/paper_1004_3105_b200 -lm -o c_api_demo && ./c_api_demo
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "nrng.h"

#define S (1u << 14)
#define N ((size_t)1 << 24) /* normals per call: 512 pairs per stream */

static int check(int rc, const char* what) {
    if (rc != NRNG_OK) {
        fprintf(stderr, "%s failed: %s\n", what, nrng_error_string(rc));
        exit(1);
    }
    return rc;
}

typedef int (*gen_fn)(nrng_handle, double*, size_t, double, double, int);
static int polar(nrng_handle h, double* o, size_t n, double mu, double sg, int v) {
    (void)v;
    return nrng_normal_polar(h, o, n, mu, sg);
}

static int run(const char* name, gen_fn f, int variant) {
    double* a = malloc(N * sizeof(double));
    double* b = malloc(N * sizeof(double));
    nrng_handle h1 = nrng_create(11, S, 0), h2 = nrng_create(11, S, 0);
    if (!a || !b || !h1 || !h2) {
        fprintf(stderr, "setup failed: %s\n", nrng_error_string(nrng_last_error()));
        return 1;
    }
    check(f(h1, a, N, 0.0, 1.0, variant), name);          /* stream k: pairs [0, 512) at 1024 k */
    check(f(h2, b, N / 2, 0.0, 1.0, variant), name);      /* stream k: pairs [0, 256) at 512 k */
    check(f(h2, b + N / 2, N / 2, 0.0, 1.0, variant), name); /* then pairs [256, 512) */
    const size_t per = N / S, half = per / 2;
    for (size_t k = 0; k < S; ++k) {
        if (memcmp(a + k * per, b + k * half, half * sizeof(double)) ||
            memcmp(a + k * per + half, b + N / 2 + k * half, half * sizeof(double))) {
            fprintf(stderr, "%s: stream %zu differs between one call and two half calls\n", name, k);
            return 1;
        }
    }
    double s1 = 0, s2 = 0;
    for (size_t i = 0; i < N; ++i) s1 += a[i], s2 += a[i] * a[i];
    const double mean = s1 / N, var = s2 / N - mean * mean;
    const int ok = fabs(mean) < 5.0 / sqrt((double)N) && fabs(var - 1.0) < 5.0 * sqrt(2.0 / N);
    printf("%s: n=%zu mean=%.3e var-1=%.3e partition-invariant=yes moments=%s\n", name, N, mean, var - 1.0,
           ok ? "ok" : "FAIL");
    nrng_destroy(h1);
    nrng_destroy(h2);
    free(a);
    free(b);
    return ok ? 0 : 1;
}

int main(void) {
    int bad = run("B3", nrng_normal_boxmuller, NRNG_B3) | run("P", polar, 0);
    nrng_handle h = nrng_create(1, 8, 0);
    double x[4];
    const int rc = nrng_normal_boxmuller(h, x, 4, 0.0, -1.0, NRNG_B1); /* sigma < 0 */
    printf("sigma<0 -> %s\n", nrng_error_string(rc));
    bad |= rc != NRNG_EINVAL;
    nrng_destroy(h);
    puts(bad ? "FAIL" : "ok");
    return bad;
}
