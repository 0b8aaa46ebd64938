/* A plain C99 consumer of the C ABI (include/la.h): no CUDA headers, no
 * Python.  It multiplies small integer-valued matrices through la_gemm_host
 * and checks every element against the exact integer product (unique fp32
 * result, la.h "Numerics"), then checks a few error paths.
 *
 *   gcc -std=c99 -I include tests/c/abi_host.c -L paper_1306_6192_b200 -lla ...
 *
 * Exit codes: 0 pass, 1 mismatch or unexpected status, 77 no usable GPU. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "la.h"

static int check(la_status s, la_status want, const char *what) {
    if (s != want) {
        fprintf(stderr, "%s: got %s, want %s (%s)\n", what, la_status_string(s), la_status_string(want),
                la_last_error());
        return 1;
    }
    return 0;
}

int main(void) {
    const int64_t n = 300, m = 517, p = 258; /* ragged in every dimension */
    la_status s = la_init(0);
    if (s != LA_OK) {
        fprintf(stderr, "la_init: %s (%s)\n", la_status_string(s), la_last_error());
        return 77;
    }
    float *A = malloc(sizeof(float) * n * m), *B = malloc(sizeof(float) * m * p), *C = malloc(sizeof(float) * n * p);
    if (!A || !B || !C) return 1;
    for (int64_t i = 0; i < n * m; i++) A[i] = (float)((i * 7 + 3) % 17 - 8);
    for (int64_t i = 0; i < m * p; i++) B[i] = (float)((i * 5 + 1) % 17 - 8);
    int bad = check(la_gemm_host(n, m, p, A, B, C, NULL), LA_OK, "la_gemm_host");
    for (int64_t i = 0; i < n && !bad; i++)
        for (int64_t j = 0; j < p; j++) {
            int64_t e = 0; /* exact: |e| <= 64 * m < 2^24 */
            for (int64_t r = 0; r < m; r++) e += (int64_t)A[i * m + r] * (int64_t)B[r * p + j];
            if (C[i * p + j] != (float)e) {
                fprintf(stderr, "C[%lld,%lld] = %.1f, exact %lld\n", (long long)i, (long long)j, C[i * p + j],
                        (long long)e);
                bad = 1;
                break;
            }
        }
    /* two products through the pipelined batch entry point: C2 = A . B2, C3 = A . B */
    float *B2 = malloc(sizeof(float) * m * p), *C2 = malloc(sizeof(float) * n * p), *C3 = malloc(sizeof(float) * n * p);
    if (!B2 || !C2 || !C3) return 1;
    for (int64_t i = 0; i < m * p; i++) B2[i] = -B[i];
    {
        const float *as[2] = {A, A}, *bs[2] = {B2, B};
        float *cs[2] = {C2, C3};
        bad |= check(la_gemm_host_batch(2, n, m, p, as, bs, cs, NULL), LA_OK, "la_gemm_host_batch");
    }
    for (int64_t i = 0; i < n * p && !bad; i++)
        if (C2[i] != -C[i] || C3[i] != C[i]) {
            fprintf(stderr, "batch product mismatch at %lld\n", (long long)i);
            bad = 1;
        }
    free(B2);
    free(C2);
    free(C3);
    bad |= check(la_gemm_host(0, m, p, A, B, C, NULL), LA_ERR_INVALID_VALUE, "zero dimension");
    bad |= check(la_gemm_host(n, m, p, NULL, B, C, NULL), LA_ERR_INVALID_VALUE, "NULL A");
    bad |= check(la_set_mode((la_mode)7), LA_ERR_INVALID_VALUE, "bad mode");
    bad |= check(la_finalize(), LA_OK, "la_finalize");
    free(A);
    free(B);
    free(C);
    if (!bad) printf("abi_host: %lldx%lldx%lld exact (single and batch), error paths ok\n", (long long)n, (long long)m, (long long)p);
    return bad;
}
