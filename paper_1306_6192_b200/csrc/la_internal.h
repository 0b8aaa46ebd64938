// la_internal.h -- state and helpers shared by la.cu (single GPU) and multi.cu (NCCL).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "la.h"

namespace la {

struct State {
    bool initialized = false;
    int device = -1;
    int sms = 0;
    uint64_t generation = 0;  // bumped by every la_init: per-device setup cached in statics is redone
    cudaMemPool_t pool = nullptr;
    la_mode mode = LA_MODE_3XTF32;
    // Accumulator promotion interval in K elements (0 = whole K in TMEM): the
    // tcgen05 kind::tf32 accumulator truncates (probes in tests/test_probe.py).
    int64_t promote_k = -1;  // -1: automatic by K (launch_gemm)
    int64_t max_sms = 0;
    int64_t panels = 0;      // la_gemm_multi N-panels: 0 = la_panel_plan's model
    int64_t nccl_sms = 8;    // SMs left to NCCL (ncclConfig_t.maxCTAs) while B panels are in flight
    int last_launches = 0;
    void *staging = nullptr;  // la_gemm_host device staging
    size_t staging_bytes = 0;
    bool kernel_timing = false;
    cudaStream_t h2d = nullptr, d2h = nullptr;  // la_gemm_host copy streams
    std::vector<cudaEvent_t> host_events;
    std::vector<cudaEvent_t> slot_events;  // la_gemm_host(_batch): start + per-slot completion
};

// Event pairs bracketing split and GEMM launches (LA_OPT_KERNEL_TIMING).
enum TimedKind { TIMED_SPLIT = 0, TIMED_GEMM = 1 };
la_status timing_begin(cudaStream_t st, cudaEvent_t *ev);
la_status timing_end(cudaStream_t st, cudaEvent_t ev, TimedKind kind);

extern State g_state;
extern std::recursive_mutex g_mutex;  // serialises every entry point's host-side work
extern thread_local std::string g_last_error;

la_status fail(la_status s, const char *fmt, ...);

// Environment hooks, all read through these two functions.
// Test hooks force one of several CORRECT dispatch paths, so that the tests can
// compare the paths bitwise (always compiled; each is set by a test):
//   LA_SPLIT_K=0|S         split-K off / forced to S pieces (tests/test_parity.py, test_multi.py)
//   LA_TAIL_SPLIT=0        no half-width tail items            (tests/test_fuzz.py)
//   LA_SPLIT_SEPARATE=1    two split launches instead of one   (tests/test_parity.py)
//   LA_TMA_STORE=0         per-thread epilogue stores          (tests/test_parity.py)
//   LA_CTA_GROUP=1|2       single-CTA or CTA-pair kernel       (tests/test_fuzz.py)
//   LA_TF32_KB=32|64       plain-TF32 K-block width            (tests/test_parity.py)
//   LA_HOST_PANELS=q       host transfer panels                (tests/test_parity.py)
//   LA_DGEMM_CPASYNC=1     cp.async DGEMM instead of TMA       (tests/test_parity_ext.py)
//   LA_TEST_GATHER_ROW0=r  fused-gather destination row, 1 rank (tests/test_multi.py)
//   LA_TEST_PLAN_NGPU=g    panel plan of g ranks, 1 rank         (tests/test_multi.py)
//   LA_TEST_GATHER_PEERS=g, LA_TEST_GATHER_STRIDE=s  one rank emulating g ranks'
//                          C_full copies at float offsets 0, s, 2s.. of its own
//                          window (tests/test_multi.py)
// Experiment knobs (LA_SPLIT_T32, LA_GROUP_M, LA_WAVE_SYNC, LA_HOST_TAIL_SPLIT,
// LA_HOST_TRACE, LA_DIAG_CLUSTERS, LA_DIAG_TRACE, LA_DEBUG_KERNEL,
// LA_SPLITK_MIN_PIECE1) are read only
// in the diagnostics build (LA_BUILD_DIAGNOSTICS=1); elsewhere diag_knob
// returns the default.
int64_t test_hook(const char *name, int64_t dflt);
int64_t diag_knob(const char *name, int64_t dflt);
la_status cuda_fail(cudaError_t e, const char *what, const char *file, int line);
la_status validate_gemm(int64_t n, int64_t m, int64_t p, const float *A, const float *B, const float *C);

// Split operands of one product (layouts in split.cuh).  b rows are the
// columns of B (Bt is p x mp); a panel of B's columns is a contiguous row range.
struct Operands {
    float *a_hi = nullptr, *a_lo = nullptr;  // n x mp
    float *b_hi = nullptr, *b_lo = nullptr;  // p x mp
    int64_t mp = 0;
    int passes = 3;
};

inline int64_t pad_k(int64_t m) { return (m + 3) / 4 * 4; }
size_t operands_bytes(int64_t n, int64_t m, int64_t p, int passes);
Operands operands_carve(void *ws, int64_t n, int64_t m, int64_t p, int passes);

// A (n x m, row stride m) -> ops.a_hi/a_lo
la_status split_a(int64_t n, int64_t m, const float *A, const Operands &ops, cudaStream_t st, int *launches);
// B -> rows [j0, j0+pc) of ops.b_hi/b_lo, where B points at column j0 of an
// m x (>= pc) row-major matrix with row stride ldb
la_status split_b(int64_t m, int64_t j0, int64_t pc, const float *B, int64_t ldb, const Operands &ops,
                  cudaStream_t st, int *launches);
// Output addressing beyond plain row-major (see GemmArgs in gemm_sm100.cuh).
struct OutSpec {
    int64_t cstride = 1, half_rows = 0, half_off = 0;
    // fused all-gather into a registered symmetric window (see GemmArgs)
    const void *gather_win = nullptr;
    int gather_peers = 0;
    int64_t gather_row0 = 0, gather_col0 = 0, gather_ld = 0;
    int64_t gather_emul_stride = 0;  // test hook: emulated peers inside one window (GemmArgs)
    // la_gemm may split K across clusters when there are few output tiles (the
    // multi-GPU path never does, so its result stays bitwise equal to la_gemm
    // without split-K)
    bool splitk_ok = false;
    // K length the automatic promotion interval is chosen for (0: the GEMM's
    // own K).  la_cgemm passes m for its 2m-long embedding, so zero-imaginary
    // products stay bitwise equal to la_gemm (zero products do not change a
    // truncating or a rounding sum).
    int64_t policy_k = 0;
};

// C[:, j0:j0+pc] (n x pc block of a row-major matrix with row stride ldc) =
// A . B[:, j0:j0+pc] from split operands; at most max_sms SMs (0 = all).
la_status gemm_run(int64_t n, int64_t m, int64_t j0, int64_t pc, const Operands &ops, float *C, int64_t ldc,
                   int max_sms, cudaStream_t st, int *launches, OutSpec out = OutSpec());

la_status comm_destroy();

}  // namespace la
