/* Plain C99 use of the device-pointer entry points (la_gemm, la_dgemm, la_add)
 * with the CUDA runtime's C API: cudaMalloc'd operands, a user stream, errors
 * checked through la_status / la_last_error.  Integer-valued inputs, so every
 * result element is checked exactly against an int64 loop.
 *
 * Exit codes: 0 pass, 1 mismatch or unexpected status, 77 no usable GPU. */
#include <cuda_runtime_api.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "la.h"

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) {                                                \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));            \
            return 1;                                                           \
        }                                                                       \
    } while (0)

static int expect(la_status s, la_status want, const char *what) {
    if (s == want) return 0;
    fprintf(stderr, "%s: got %s, want %s (%s)\n", what, la_status_string(s), la_status_string(want), la_last_error());
    return 1;
}

int main(void) {
    const int64_t n = 257, m = 300, p = 130;
    if (la_init(0) != LA_OK) {
        fprintf(stderr, "la_init: %s\n", la_last_error());
        return 77;
    }
    float *A = malloc(sizeof(float) * n * m), *B = malloc(sizeof(float) * m * p), *C = malloc(sizeof(float) * n * p);
    double *Ad = malloc(sizeof(double) * n * m), *Bd = malloc(sizeof(double) * m * p),
           *Cd = malloc(sizeof(double) * n * p);
    if (!A || !B || !C || !Ad || !Bd || !Cd) return 1;
    for (int64_t i = 0; i < n * m; i++) Ad[i] = A[i] = (float)((i * 11 + 5) % 17 - 8);
    for (int64_t i = 0; i < m * p; i++) Bd[i] = B[i] = (float)((i * 13 + 2) % 17 - 8);
    float *dA, *dB, *dC, *dS;
    double *dAd, *dBd, *dCd;
    CK(cudaMalloc((void **)&dA, sizeof(float) * n * m));
    CK(cudaMalloc((void **)&dB, sizeof(float) * m * p));
    CK(cudaMalloc((void **)&dC, sizeof(float) * n * p));
    CK(cudaMalloc((void **)&dS, sizeof(float) * n * m));
    CK(cudaMalloc((void **)&dAd, sizeof(double) * n * m));
    CK(cudaMalloc((void **)&dBd, sizeof(double) * m * p));
    CK(cudaMalloc((void **)&dCd, sizeof(double) * n * p));
    CK(cudaMemcpy(dA, A, sizeof(float) * n * m, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B, sizeof(float) * m * p, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dAd, Ad, sizeof(double) * n * m, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dBd, Bd, sizeof(double) * m * p, cudaMemcpyHostToDevice));
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    int bad = 0;
    bad |= expect(la_gemm(n, m, p, dA, dB, dC, (void *)st), LA_OK, "la_gemm");
    bad |= expect(la_dgemm(n, m, p, dAd, dBd, dCd, (void *)st), LA_OK, "la_dgemm");
    bad |= expect(la_add(n, m, dA, dA, dS, 1, (void *)st), LA_OK, "la_add (A - A)");
    bad |= expect(la_gemm(n, m, p, dA, dB, dA, (void *)st), LA_ERR_INVALID_VALUE, "la_gemm with C aliasing A");
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(C, dC, sizeof(float) * n * p, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(Cd, dCd, sizeof(double) * n * p, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n && !bad; i++)
        for (int64_t j = 0; j < p; j++) {
            int64_t e = 0;
            for (int64_t r = 0; r < m; r++) e += (int64_t)A[i * m + r] * (int64_t)B[r * p + j];
            if (C[i * p + j] != (float)e || Cd[i * p + j] != (double)e) {
                fprintf(stderr, "C[%lld,%lld]: gemm %.1f dgemm %.1f exact %lld\n", (long long)i, (long long)j,
                        C[i * p + j], Cd[i * p + j], (long long)e);
                bad = 1;
                break;
            }
        }
    CK(cudaMemcpy(A, dS, sizeof(float) * n * m, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n * m && !bad; i++)
        if (A[i] != 0.0f) {
            fprintf(stderr, "A - A at %lld = %f\n", (long long)i, A[i]);
            bad = 1;
        }
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dC);
    cudaFree(dS);
    cudaFree(dAd);
    cudaFree(dBd);
    cudaFree(dCd);
    cudaStreamDestroy(st);
    bad |= expect(la_finalize(), LA_OK, "la_finalize");
    free(A);
    free(B);
    free(C);
    free(Ad);
    free(Bd);
    free(Cd);
    if (!bad) printf("abi_device: gemm, dgemm exact; add ok; aliasing rejected\n");
    return bad;
}
