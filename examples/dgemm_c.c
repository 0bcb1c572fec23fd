/* examples/dgemm_c.c -- calling liboz2 from plain C (no Python, no torch): an emulated
 * DGEMM C = A B on host buffers (the library stages them through device memory), checked
 * against a naive triple loop in long double.
 *
 *   gcc -O2 -std=c11 -I include examples/dgemm_c.c -L paper_2603_10634_b200 -loz2 \
 *       -Wl,-rpath,$PWD/paper_2603_10634_b200 -o /tmp/dgemm_c && /tmp/dgemm_c 300 200 250 13
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "oz2.h"

static double urand(uint64_t* s) {            /* xorshift64*, uniform in [-1, 1) */
    *s ^= *s >> 12; *s ^= *s << 25; *s ^= *s >> 27;
    return (double)((*s * 2685821657736338717ull) >> 11) / 4503599627370496.0 - 1.0;
}

int main(int argc, char** argv) {
    const int64_t m = argc > 1 ? atoll(argv[1]) : 300, k = argc > 2 ? atoll(argv[2]) : 200;
    const int64_t n = argc > 3 ? atoll(argv[3]) : 250;
    const int N = argc > 4 ? atoi(argv[4]) : 13;
    double *A = malloc(sizeof(double) * m * k), *B = malloc(sizeof(double) * k * n);
    double *C = malloc(sizeof(double) * m * n);
    if (!A || !B || !C) return 2;
    uint64_t s = 88172645463325252ull;
    for (int64_t x = 0; x < m * k; ++x) A[x] = urand(&s) * exp(3.0 * urand(&s));
    for (int64_t x = 0; x < k * n; ++x) B[x] = urand(&s) * exp(3.0 * urand(&s));
    printf("%s\n", oz2_version());
    /* column-major, op = 'N': C (m x n) <- 1.0 * A (m x k) B (k x n) + 0.0 * C */
    const int rc = oz2_dgemm('N', 'N', m, n, k, 1.0, A, m, B, k, 0.0, C, m, N);
    if (rc != OZ2_SUCCESS) { fprintf(stderr, "oz2_dgemm returned %d\n", rc); return 1; }
    int32_t status = 0;
    oz2_get_status(&status);
    long double num = 0.0L, den = 0.0L;
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) {
            long double ref = 0.0L;
            for (int64_t h = 0; h < k; ++h) ref += (long double)A[i + h * m] * (long double)B[h + j * k];
            const long double d = (long double)C[i + j * m] - ref;
            num += d * d;
            den += ref * ref;
        }
    const double rel = (double)sqrtl(num / den);
    printf("m=%lld n=%lld k=%lld N=%d status=%d |C - AB|/|AB| = %.3e\n", (long long)m, (long long)n,
           (long long)k, N, status, rel);
    oz2_finalize();
    free(A); free(B); free(C);
    return (status == OZ2_SUCCESS && rel < 1e-15) ? 0 : 1;
}
