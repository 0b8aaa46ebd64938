/*
 * la.h -- C ABI of the B200-native fp32-accurate GEMM (after arXiv 1306.6192).
 *
 * The one operation is the Cauchy product of PAPER.md P:47 (section
 * "Implementacje algorytmow"):
 *
 *     c_ij = sum_{r=1..m} a_ir * b_rj,   1 <= i <= n, 1 <= j <= p,
 *
 * for dense ROW-MAJOR single-precision matrices: A is n x m (element (i,r) at
 * A[i*m + r]), B is m x p (B[r*p + j]), C is n x p (C[i*p + j]) -- the
 * indexing of Listing 1 and of Listing 4's write-back.
 * There is no alpha/beta and no accumulate-into-C: C is overwritten.
 *
 * Conventions for every function:
 *  - Returns la_status; never throws or aborts across the ABI.  On failure a
 *    thread-local detail string is available from la_last_error().
 *  - Pointers named d_* are DEVICE pointers on the device given to la_init()
 *    (e.g. torch tensor data_ptr()); pointers named h_* are HOST pointers.
 *    Device operands are caller-owned; the library owns only its workspace
 *    (stream-ordered, from a CUDA memory pool), its TMA descriptors and, after
 *    la_comm_init, one NCCL communicator.  C must not overlap A or B.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Device work is enqueued on it and the call returns without a host sync;
 *    asynchronous kernel faults surface at the caller's next synchronisation
 *    (or as LA_ERR_CUDA from a later la_* call).  la_gemm does no host
 *    synchronisation and allocates with cudaMallocAsync, so it may be captured
 *    into a CUDA graph.
 *  - Library state is process-wide (one device per process, set by la_init).
 *    Every entry point serialises its host-side work on one library lock, so
 *    calls from several host threads are safe; their device work on different
 *    streams may overlap.  la_gemm_host holds the lock until its copies finish.
 *  - Sizes are int64_t; all index arithmetic on the device is 64-bit
 *    (n*p = 2^32 at n = 65536 overflows Listing 4's 32-bit `int c`).
 *
 * Numerics (BASELINE.json north_star):
 *  - LA_MODE_3XTF32 (default): a = hi + lo with hi = tf32 round-to-nearest
 *    (ties away) of a and lo = a - hi; c = sum(hi*hi' + hi*lo' + lo*hi') on
 *    the tcgen05 tensor pipe with fp32 accumulation.  Contract:
 *    |c - c_ref| <= 2^-20 * sum_r |a_ir||b_rj| per element (c_ref = the fp32
 *    Listing 1 loop; for same-sign inputs, where that loop's own error grows
 *    toward gamma_m * sum|a||b|, c is at least as close to the exact product
 *    as c_ref, within 2^-20 * sum -- DESIGN.md reading C14'), and value-exact
 *    (==) on integer-valued inputs whose partial sums stay below 2^24.
 *    Measured envelope against the EXACT product (DESIGN.md section 4,
 *    units of 2^-20 * sum|a||b|, automatic promotion interval): random signs
 *    <= 0.7 at every K tested; same-sign and other structured inputs
 *    (scripts/fuzz_structured.py, ~1900 random shapes) <= 1.23 once K spans >= 8
 *    promotion chunks (K >= 1024: sign-centred chunks; <= 0.85 for 256-wide
 *    outputs) where Listing 1 itself is up to 7.6 off, and up to 1.6 for
 *    shorter K where Listing 1 is up to 1.4 off -- always within the oracle's
 *    own error + 2^-20 * sum (reading C14').
 *  - Deterministic: the same call on the same inputs gives the same bits
 *    (split-K partials are reduced in piece order).
 *  - LA_MODE_TF32: one pass on hi only; contract 2^-9 * sum_r |a_ir||b_rj|.
 *  - Inputs must be finite; non-finite inputs are out of contract.
 */
#ifndef LA_H_
#define LA_H_

#include <stdint.h>

#if defined(__GNUC__)
#define LA_API __attribute__((visibility("default")))
#else
#define LA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    LA_OK = 0,
    LA_ERR_INVALID_VALUE = 1,   /* bad dimension (<= 0), NULL or aliased pointer, bad mode/option */
    LA_ERR_NOT_INITIALIZED = 2, /* la_init (or la_comm_init for *_multi) has not been called */
    LA_ERR_UNSUPPORTED = 3,     /* device is not sm_100 (B200), or a shape the multi-GPU path rejects */
    LA_ERR_OUT_OF_MEMORY = 4,   /* workspace / host staging allocation failed */
    LA_ERR_CUDA = 5,            /* a CUDA runtime/driver call failed (detail in la_last_error) */
    LA_ERR_NCCL = 6             /* an NCCL call failed (detail in la_last_error) */
} la_status;

typedef enum {
    LA_MODE_3XTF32 = 0, /* fp32-accurate: three TF32 tensor-core passes (default) */
    LA_MODE_TF32 = 1    /* one TF32 pass, ~2^-10 relative per product */
} la_mode;

typedef enum {
    /* 3xTF32 only: K elements accumulated in tensor memory before the partial
     * sum is added into an fp32 register running sum (round-to-nearest).  0 =
     * never (the whole K range accumulates in TMEM); > 0: that many, rounded up
     * to a multiple of 32.  Default -1 (automatic): 32 for K <= 64, 64 for
     * K <= 192, 128 beyond -- the tcgen05 tf32 accumulator truncates at every
     * MMA, and one long chunk breaks the 2^-20 bound; chunks are sign-centred
     * when K spans >= 8 of them. */
    LA_OPT_PROMOTE_K = 0,
    /* Upper bound on the number of SMs the GEMM kernel occupies (0 = all).  The
     * multi-GPU path uses it to leave SMs for NCCL. */
    LA_OPT_MAX_SMS = 1,
    /* N-panels B is broadcast in by la_gemm_multi: 0 (default) = the plan of
     * la_panel_plan's timeline model, >= 1 = that many equal panels. */
    LA_OPT_PANELS = 2,
    /* 1: record CUDA events around every split and GEMM launch so that
     * la_kernel_times() can report their device durations (bench.py's
     * roofline).  0 (default): no events. */
    LA_OPT_KERNEL_TIMING = 3,
    /* SMs left to NCCL while la_gemm_multi's B panels are in flight (0..64,
     * default 8): the communicator is created with ncclConfig_t.maxCTAs = this
     * value (read by la_comm_init) and every GEMM launch but the last panel's
     * runs on the remaining SMs.  Takes effect at the next la_comm_init. */
    LA_OPT_NCCL_SMS = 4
} la_option;

/* Bind the (process-wide) library state to CUDA device `device`, check that it
 * is compute capability 10.0 (sm_100, B200) and set up the workspace pool.
 * Idempotent for the same device.  Errors: INVALID_VALUE (no such device),
 * UNSUPPORTED (not sm_100), CUDA. */
LA_API la_status la_init(int device);

/* Process-wide arithmetic mode for subsequent calls (default LA_MODE_3XTF32).
 * Errors: INVALID_VALUE (unknown mode). */
LA_API la_status la_set_mode(la_mode mode);

/* Set / get a tuning option (see la_option).  Errors: INVALID_VALUE. */
LA_API la_status la_set_option(la_option option, int64_t value);
LA_API la_status la_get_option(la_option option, int64_t *value);

/* C = A . B on one GPU, enqueued on `stream` (Listing 4's role).
 *   n, m, p   : dimensions, each >= 1;
 *   d_A       : n x m row-major fp32, device;  d_B : m x p row-major fp32, device;
 *   d_C       : n x p row-major fp32, device, written exactly once per element.
 * Work: one split pass over A and B into a library workspace (one launch when
 * both take the vectorised kernels), then one persistent tcgen05 GEMM kernel
 * (programmatic dependent launch); problems with few output tiles and a long K
 * split K across clusters and add one in-order reduction kernel (deterministic,
 * integer inputs still exact).  Errors: NOT_INITIALIZED, INVALID_VALUE
 * (dims, NULL, C overlapping A or B), OUT_OF_MEMORY, CUDA. */
LA_API la_status la_gemm(int64_t n, int64_t m, int64_t p, const float *d_A, const float *d_B,
                  float *d_C, void *stream);

/* End-to-end variant on HOST buffers (the paper's host flow):
 * copies h_A and h_B to the device, computes, copies C back into h_C and
 * returns after everything completed.  The copies are pipelined with the
 * compute (2-D schedule): A row panels and B column panels alternate on a
 * copy-in stream; each panel, as it lands, is split and unlocks one rectangle
 * of C (that panel against every panel of the other operand already present),
 * computed by one GEMM launch on `stream` and copied back on a copy-out stream
 * while later panels are in flight.  Every element accumulates in
 * la_gemm's order (bitwise identical to la_gemm whenever la_gemm does not split
 * K).  Host buffers may be pageable or pinned (only pinned buffers overlap).
 * Device staging is library-owned and reused.  Errors: as la_gemm. */
LA_API la_status la_gemm_host(int64_t n, int64_t m, int64_t p, const float *h_A, const float *h_B,
                       float *h_C, void *stream);

/* `count` independent products of one shape from HOST buffers, returning after
 * all of them completed: C_i = A_i . B_i for h_A[i], h_B[i], h_C[i] (arrays of
 * `count` host pointers; each as in la_gemm_host).  Two device staging slots
 * alternate, so the copy-in of product i + 1 overlaps the compute and copy-out
 * of product i: with pinned buffers the PCIe copy engines stay busy across
 * products (the serving-pipeline form of la_gemm_host).  Each product is
 * bitwise equal to la_gemm_host on the same inputs.  The h_C[i] must not
 * overlap each other or any input.  Errors: as la_gemm_host; INVALID_VALUE
 * also for count < 1 or a NULL array. */
LA_API la_status la_gemm_host_batch(int64_t count, int64_t n, int64_t m, int64_t p, const float *const *h_A,
                                    const float *const *h_B, float *const *h_C, void *stream);

/* Complex single-precision product (Table 2 "Complex Float" column, P:222-228;
 * complex multiply as in SPEC S:85-93):
 *   d_A : n x m complex64, row-major, interleaved (re, im) float pairs, device;
 *   d_B : m x p complex64;  d_C : n x p complex64, overwritten.
 * Computed on the same tcgen05 path as la_gemm through the real embedding
 * [[Ar, -Ai], [Ai, Ar]] . [Br; Bi] = [Cr; Ci] (four real GEMMs of work, one
 * launch).  Numerics as la_gemm per component, with the scales
 * sum_r |ar||br| + |ai||bi| (real part) and sum_r |ar||bi| + |ai||br|
 * (imaginary part).  Pointers 8-byte aligned.  Errors: as la_gemm. */
LA_API la_status la_cgemm(int64_t n, int64_t m, int64_t p, const float *d_A, const float *d_B,
                          float *d_C, void *stream);

/* Double-precision product (Table 2 "Double" column; 8-byte tiles,
 * P:130): d_A n x m, d_B m x p, d_C n x p, row-major binary64, device, 8-byte
 * aligned.  FP64 tensor path (DMMA, mma.sync f64): every product and sum is a
 * binary64 operation (fused multiply-add), so |C - C_ref| <= 2 gamma_m S with
 * S = sum_r |a_ir||b_rj|, gamma_m = m 2^-53 / (1 - m 2^-53), against the binary64
 * Listing 1; integer-valued inputs with partial sums below 2^53 are exact.
 * Errors: NOT_INITIALIZED, INVALID_VALUE, UNSUPPORTED, CUDA. */
LA_API la_status la_dgemm(int64_t n, int64_t m, int64_t p, const double *d_A, const double *d_B,
                          double *d_C, void *stream);

/* Matrix addition / subtraction (PAPER.md section "Rezultaty i wnioski", P:203:
 * "Dodawanie macierzy ... 16 777 216 operacji elementarnych" at 4096 x 4096):
 * C = A + B (subtract = 0) or C = A - B (subtract != 0), rows x cols row-major
 * fp32, one IEEE binary32 operation per element (bitwise reproducible).  C may
 * be A or B (in place) but must not partially overlap them.  HBM-bound
 * (12 bytes per element).  Errors: NOT_INITIALIZED, INVALID_VALUE, CUDA. */
LA_API la_status la_add(int64_t rows, int64_t cols, const float *d_A, const float *d_B, float *d_C,
                        int subtract, void *stream);

/* ---- multi-GPU (one process per GPU, SPMD) ------------------ */

/* Rank 0 writes a 128-byte NCCL unique id into out128; the caller distributes
 * it (e.g. torch.distributed broadcast).  Errors: INVALID_VALUE, NCCL. */
LA_API la_status la_get_unique_id(void *out128);

/* Create this rank's communicator (rank in [0, ngpu)).  Requires la_init.
 * Errors: NOT_INITIALIZED, INVALID_VALUE, NCCL. */
LA_API la_status la_comm_init(const void *uid128, int rank, int ngpu);

/* Ranks in this process's communicator as NCCL reports them (ncclCommCount)
 * and this process's rank (ncclCommUserRank).  Errors: NOT_INITIALIZED (no
 * la_comm_init), INVALID_VALUE (NULL), NCCL. */
LA_API la_status la_comm_size(int *nranks, int *rank);

/* Row-sharded product over the communicator:
 *   rank r owns rows [r*n/g, (r+1)*n/g) of A and C (g = ngpu);
 *   d_A_local : (rows_r x m) row-major fp32;
 *   d_B       : m x p on rank `root` (ignored, may be NULL, elsewhere) --
 *               broadcast with ncclBroadcast in N-panels overlapped with the
 *               GEMM on the panels already received;
 *   d_C_local : (rows_r x p) row-major fp32;
 *   d_C_full  : NULL, or n x p: if given, C is all-gathered (ncclAllGather)
 *               into it on every rank (requires n % g == 0).  Reads of d_C_full
 *               from a previous call must be ordered before this call on
 *               `stream` (the fused gather of la_gather_alloc writes peers'
 *               buffers; a cross-rank barrier at the start of the call waits
 *               for every rank's earlier work on its stream).
 * All ranks pass identical n, m, p, root, ngpu.  Every output element is
 * accumulated in the same order as la_gemm (which never splits K here), so
 * results are bitwise identical to the single-GPU path without split-K.
 * Errors: NOT_INITIALIZED, INVALID_VALUE (ngpu != communicator size, dims),
 * UNSUPPORTED (C_full with n % g != 0), NCCL, CUDA. */
LA_API la_status la_gemm_multi(int64_t n, int64_t m, int64_t p, const float *d_A_local,
                        const float *d_B, float *d_C_local, float *d_C_full, int root,
                        int ngpu, void *stream);

/* Collective over the communicator (every rank, same `bytes`): allocate a
 * symmetric device buffer (ncclMemAlloc) registered as an NCCL window
 * (NCCL_WIN_COLL_SYMMETRIC) and return it in *d_out.  Passing it as
 * la_gemm_multi's d_C_full selects the FUSED all-gather: the GEMM epilogue
 * stores this rank's rows straight into every rank's buffer over NVLink
 * (load/store-accessible peers, up to 8) while later tiles compute, followed by
 * one tiny cross-rank barrier instead of an ncclAllGather (NEXT item #1 of
 * SURVEY 8(f)).  Freed by the next call, la_comm_init or la_finalize.
 * Errors: NOT_INITIALIZED, INVALID_VALUE, NCCL. */
LA_API la_status la_gather_alloc(int64_t bytes, void **d_out);

/* Column panels la_gemm_multi broadcasts B in (pure host arithmetic, no
 * device needed): widths[0 .. *count) sum to p, multiples of 256 except the
 * last.  panels > 0: that many equal panels; panels == 0: the plan a timeline
 * model of one rank (broadcast of panel c overlapping the GEMM of panel c-1,
 * replicated split, wave quantisation on sms - reserved SMs) scores best among
 * equal and geometric (narrow first panel) plans.  Errors: INVALID_VALUE (bad
 * sizes, more than max_panels panels). */
LA_API la_status la_panel_plan(int64_t n, int64_t m, int64_t p, int ngpu, int sms, int reserved, int64_t panels,
                               int64_t *widths, int max_panels, int *count);

/* Rows owned by `rank` of g: [*row0, *row0 + *rows).  Pure host arithmetic. */
LA_API la_status la_shard_rows(int64_t n, int rank, int ngpu, int64_t *row0, int64_t *rows);

/* Release workspace pools, staging buffers and the communicator.  The library
 * may be re-initialised afterwards. */
LA_API la_status la_finalize(void);

/* Static description of a status code. */
LA_API const char *la_status_string(la_status s);

/* Thread-local detail message of the last failing call on this thread ("" if none). */
LA_API const char *la_last_error(void);

/* Number of kernels the last la_gemm / la_gemm_multi call launched. */
LA_API int la_last_launch_count(void);

/* With LA_OPT_KERNEL_TIMING = 1: synchronise on the recorded events and return
 * the summed device time (ms) of the split kernels and of the GEMM kernels of
 * every call since the previous la_kernel_times(), and how many GEMM launches
 * that covers; then forget them.  Events are recorded on the caller's stream,
 * the stream the kernels run on.  Errors: INVALID_VALUE (NULL), CUDA. */
LA_API la_status la_kernel_times(double *split_ms, double *gemm_ms, int *gemm_launches);

#ifdef __cplusplus
}
#endif

#endif /* LA_H_ */
