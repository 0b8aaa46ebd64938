/*
 * oracle.c -- CPU oracle for C = A.B (TEST INFRASTRUCTURE ONLY).
 *
 * This file is test infrastructure.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load it.  It shares no
 * code, header, table or helper with the CUDA path under
 * paper_1306_6192_b200/; neither side includes or links the other.
 *
 * What it computes (PAPER.md, section "Implementacje algorytmow"):
 *   P:47   c_ij = sum_{r=1..m} a_ir * b_rj,  1 <= i <= n, 1 <= j <= p
 *   P:53-69 (Listing 1) the sequential C triple loop: i over rows of A,
 *          j over columns of B, k innermost and ascending, C zeroed first
 *          (P:56), row-major indexing A[k + i*m], B[k*p + j].
 * Readings taken where the paper is silent:
 *   C1  float arrays, float accumulator (Table 2 "Float" column).
 *   C2  every product and every sum is one IEEE-754 binary32 operation,
 *       round-to-nearest-even, no fused multiply-add.  Built with
 *       -ffp-contract=off -fno-fast-math (load-bearing: with contraction
 *       3706/4096 elements differ at K=4096).
 *   C3  accumulator starts at +0.0f.
 *   C4  the strength-reduced indices of Listing 1 are the plain row-major
 *       offsets i*m+k and k*p+j.
 * Splitting rows across threads changes no per-element arithmetic.
 *
 * Pins: tests/test_oracle.py (worked examples, identity/permutation/diagonal
 * closed forms, (AB)^T = B^T A^T, integer brute force vs int64, 2^-k grid
 * inputs vs exact Python integers within Higham's gamma_m bound).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#if defined(__FP_FAST_FMAF) && !defined(ORACLE_ALLOW_FMA)
/* Not an error by itself (the target may have FMA), but the build flags
 * -ffp-contract=off must be in force; checked at run time by the FMA witness
 * test.  Nothing to do here. */
#endif

/* ------------------------------------------------------------------------- */
/* Listing 1, rows [i0, i1) of C.                                    */
/* ------------------------------------------------------------------------- */
static void listing1_rows(int64_t i0, int64_t i1, int64_t m, int64_t p,
                          const float *A, const float *B, float *C)
{
    for (int64_t i = i0; i < i1; i++) {              /* rows_size_A           */
        for (int64_t j = 0; j < p; j++) {            /* columns_size_B        */
            float s = 0.0f;                          /* matrix_C[..] = 0 P:56 */
            for (int64_t k = 0; k < m; k++) {        /* columns_size_A, asc.  */
                float t = A[i * m + k] * B[k * p + j];   /* fl32(a_ik * b_kj) */
                s = s + t;                               /* fl32(s + t)       */
            }
            C[i * p + j] = s;
        }
    }
}

typedef struct {
    int64_t i0, i1, m, p;
    const float *A, *B;
    float *C;
} stripe_t;

static void *stripe_main(void *arg)
{
    stripe_t *s = (stripe_t *)arg;
    listing1_rows(s->i0, s->i1, s->m, s->p, s->A, s->B, s->C);
    return NULL;
}

/* C (n x p) = A (n x m) . B (m x p), all row-major float32, Listing 1 per
 * element, rows split in contiguous stripes over `threads` POSIX threads.
 * Returns 0 on success, -1 on bad arguments, -2 if a thread could not start. */
int oracle_gemm(int64_t n, int64_t m, int64_t p, const float *A, const float *B,
                float *C, int threads)
{
    if (n < 0 || m < 0 || p < 0 || (n * p > 0 && (!C || (m > 0 && (!A || !B)))))
        return -1;
    if (threads < 1) threads = 1;
    if (threads > n) threads = (int)(n > 0 ? n : 1);
    if (threads == 1) {
        listing1_rows(0, n, m, p, A, B, C);
        return 0;
    }
    pthread_t *tid = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    stripe_t *st = (stripe_t *)calloc((size_t)threads, sizeof(stripe_t));
    if (!tid || !st) { free(tid); free(st); return -2; }
    int started = 0, rc = 0;
    for (int t = 0; t < threads; t++) {
        st[t].i0 = n * t / threads;
        st[t].i1 = n * (t + 1) / threads;
        st[t].m = m; st[t].p = p; st[t].A = A; st[t].B = B; st[t].C = C;
        if (pthread_create(&tid[t], NULL, stripe_main, &st[t]) != 0) { rc = -2; break; }
        started++;
    }
    for (int t = 0; t < started; t++) pthread_join(tid[t], NULL);
    if (rc != 0)   /* finish the stripes that never started, sequentially */
        for (int t = started; t < threads; t++)
            listing1_rows(st[t].i0, st[t].i1, m, p, A, B, C);
    free(tid); free(st);
    return 0;
}

/* The same Listing 1 inner loop but with an explicit fmaf accumulation.  It is
 * NOT the oracle: it exists only so the "not gpu" tests can prove that the
 * oracle build really keeps multiply and add separate (FMA witness, SURVEY
 * App. A).  */
int oracle_gemm_fma_witness(int64_t n, int64_t m, int64_t p, const float *A,
                            const float *B, float *C)
{
    for (int64_t i = 0; i < n; i++)
        for (int64_t j = 0; j < p; j++) {
            float s = 0.0f;
            for (int64_t k = 0; k < m; k++) s = fmaf(A[i * m + k], B[k * p + j], s);
            C[i * p + j] = s;
        }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Tolerance scale and exact references (used to judge the GPU within the    */
/* north_star bound |C - C_ref| <= 2^-20 * sum_r |a_ir||b_rj|).               */
/* ------------------------------------------------------------------------- */

/* S_ij = sum_r |a_ir| * |b_rj| accumulated in binary64 (each |a||b| product of
 * two floats is exact in binary64; the sum carries relative error <= m*2^-53,
 * irrelevant at the 2^-20 scale it multiplies).  */
int oracle_abs_scale(int64_t n, int64_t m, int64_t p, const float *A,
                     const float *B, double *S)
{
    for (int64_t i = 0; i < n; i++)
        for (int64_t j = 0; j < p; j++) {
            double s = 0.0;
            for (int64_t k = 0; k < m; k++)
                s += fabs((double)A[i * m + k]) * fabs((double)B[k * p + j]);
            S[i * p + j] = s;
        }
    return 0;
}

/* Exact c_ij for inputs that are integers times 2^-shift (|integer| < 2^25):
 * c_ij * 2^(2*shift) = sum_r ka_ir * kb_rj evaluated exactly in __int128, then
 * converted to binary64 (one rounding, relative 2^-53).  Returns -1 if an input
 * is not on the grid.  */
int oracle_exact_grid(int64_t n, int64_t m, int64_t p, const float *A,
                      const float *B, int shift, double *E)
{
    const double scale_in = ldexp(1.0, shift);
    for (int64_t i = 0; i < n; i++)
        for (int64_t j = 0; j < p; j++) {
            __int128 acc = 0;
            for (int64_t k = 0; k < m; k++) {
                double da = (double)A[i * m + k] * scale_in;
                double db = (double)B[k * p + j] * scale_in;
                int64_t ka = (int64_t)da, kb = (int64_t)db;
                if ((double)ka != da || (double)kb != db) return -1;
                acc += (__int128)ka * (__int128)kb;
            }
            /* split the int128 into two doubles and recombine exactly enough */
            int neg = acc < 0;
            unsigned __int128 u = neg ? (unsigned __int128)(-acc) : (unsigned __int128)acc;
            double hi = ldexp((double)(uint64_t)(u >> 64), 64);
            double lo = (double)(uint64_t)u;
            double v = ldexp(hi + lo, -2 * shift);
            E[i * p + j] = neg ? -v : v;
        }
    return 0;
}

/* Freivalds' check for integer-valued products: with x a vector
 * of small integers, C.x must equal A.(B.x) exactly in int64.  C, A, B hold
 * integer-valued floats with |values| small enough that every partial sum
 * fits in int64 (|a|,|b| <= 8, |x| <= 8, m, p <= 2^20 gives < 2^41).
 * Returns the number of rows i where (C.x)_i != (A.(B.x))_i, or -1 if an input
 * is not an integer.  rows_bad[] (optional, length >= 1) receives the first
 * mismatching row.  */
int64_t oracle_freivalds_i64(int64_t n, int64_t m, int64_t p, const float *A,
                             const float *B, const float *C, const int64_t *x,
                             int64_t *first_bad)
{
    int64_t *bx = (int64_t *)calloc((size_t)(m > 0 ? m : 1), sizeof(int64_t));
    if (!bx) return -2;
    for (int64_t r = 0; r < m; r++) {
        int64_t s = 0;
        for (int64_t j = 0; j < p; j++) {
            float b = B[r * p + j];
            int64_t kb = (int64_t)b;
            if ((float)kb != b) { free(bx); return -1; }
            s += kb * x[j];
        }
        bx[r] = s;
    }
    int64_t bad = 0;
    if (first_bad) *first_bad = -1;
    for (int64_t i = 0; i < n; i++) {
        int64_t lhs = 0, rhs = 0;
        for (int64_t j = 0; j < p; j++) {
            float c = C[i * p + j];
            int64_t kc = (int64_t)c;
            if ((float)kc != c || isnan(c)) { free(bx); return -1; }
            lhs += kc * x[j];
        }
        for (int64_t r = 0; r < m; r++) {
            float a = A[i * m + r];
            int64_t ka = (int64_t)a;
            if ((float)ka != a) { free(bx); return -1; }
            rhs += ka * bx[r];
        }
        if (lhs != rhs) {
            if (bad == 0 && first_bad) *first_bad = i;
            bad++;
        }
    }
    free(bx);
    return bad;
}

/* ------------------------------------------------------------------------- */
/* Matrix addition / subtraction (PAPER.md section "Rezultaty i wnioski",     */
/* C = A +/- B, rows x cols elementary operations, 16,777,216 at       */
/* 4096 x 4096).  One binary32 add or subtract per element, RN-even.          */
/* ------------------------------------------------------------------------- */
int oracle_elementwise(int64_t rows, int64_t cols, const float *A, const float *B, float *C,
                       int subtract)
{
    const int64_t count = rows * cols;
    if (subtract)
        for (int64_t i = 0; i < count; i++) C[i] = A[i] - B[i];
    else
        for (int64_t i = 0; i < count; i++) C[i] = A[i] + B[i];
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Complex single-precision product (Table 2 "Complex Float";      */
/* SPEC S:85-93 complex_mul).  Listing 1 over complex64 elements stored as    */
/* interleaved (re, im) float pairs: for each (i, j), s = 0 + 0i, then for r  */
/* ascending  t = a_ir * b_rj  with                                            */
/*     t.re = fl(fl(ar*br) - fl(ai*bi)),  t.im = fl(fl(ar*bi) + fl(ai*br)),    */
/* and s = s + t componentwise, every operation one binary32 RN operation.    */
/* ------------------------------------------------------------------------- */
int oracle_cgemm(int64_t n, int64_t m, int64_t p, const float *A, const float *B, float *C)
{
    for (int64_t i = 0; i < n; i++)
        for (int64_t j = 0; j < p; j++) {
            float sr = 0.0f, si = 0.0f;
            for (int64_t k = 0; k < m; k++) {
                const float ar = A[2 * (i * m + k)], ai = A[2 * (i * m + k) + 1];
                const float br = B[2 * (k * p + j)], bi = B[2 * (k * p + j) + 1];
                const float p1 = ar * br, p2 = ai * bi, p3 = ar * bi, p4 = ai * br;
                const float tr = p1 - p2, ti = p3 + p4;
                sr = sr + tr;
                si = si + ti;
            }
            C[2 * (i * p + j)] = sr;
            C[2 * (i * p + j) + 1] = si;
        }
    return 0;
}

/* Tolerance scales for the complex product, binary64:
 *   Sr_ij = sum_r |ar||br| + |ai||bi|,   Si_ij = sum_r |ar||bi| + |ai||br|. */
int oracle_cabs_scale(int64_t n, int64_t m, int64_t p, const float *A, const float *B, double *S)
{
    for (int64_t i = 0; i < n; i++)
        for (int64_t j = 0; j < p; j++) {
            double sr = 0.0, si = 0.0;
            for (int64_t k = 0; k < m; k++) {
                const double ar = fabs((double)A[2 * (i * m + k)]), ai = fabs((double)A[2 * (i * m + k) + 1]);
                const double br = fabs((double)B[2 * (k * p + j)]), bi = fabs((double)B[2 * (k * p + j) + 1]);
                sr += ar * br + ai * bi;
                si += ar * bi + ai * br;
            }
            S[2 * (i * p + j)] = sr;
            S[2 * (i * p + j) + 1] = si;
        }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Double-precision Listing 1 (Table 2 "Double" column): binary64  */
/* arrays and accumulator, product then sum each RN-even, no FMA, ascending r. */
/* ------------------------------------------------------------------------- */
int oracle_dgemm(int64_t n, int64_t m, int64_t p, const double *A, const double *B, double *C)
{
    for (int64_t i = 0; i < n; i++)
        for (int64_t j = 0; j < p; j++) {
            double s = 0.0;
            for (int64_t k = 0; k < m; k++) {
                double t = A[i * m + k] * B[k * p + j];
                s = s + t;
            }
            C[i * p + j] = s;
        }
    return 0;
}

/* S_ij = sum_r |a_ir||b_rj| for binary64 inputs, accumulated in binary64. */
int oracle_dabs_scale(int64_t n, int64_t m, int64_t p, const double *A, const double *B, double *S)
{
    for (int64_t i = 0; i < n; i++)
        for (int64_t j = 0; j < p; j++) {
            double s = 0.0;
            for (int64_t k = 0; k < m; k++) s += fabs(A[i * m + k]) * fabs(B[k * p + j]);
            S[i * p + j] = s;
        }
    return 0;
}
