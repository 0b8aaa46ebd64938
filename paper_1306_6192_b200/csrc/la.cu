// la.cu -- host side of the C ABI declared in include/la.h (single-GPU path).
//
// la_gemm(n, m, p, A, B, C, stream) enqueues, on the caller's stream:
//   1. K1 split of A  -> A_hi, A_lo   (n x mp, row-major, K-major for UMMA) and
//      split of B  -> Bt_hi, Bt_lo (p x mp, B transposed to K-major), one launch
//      when both take the vectorised kernels (split_ab_kernel), else two
//   2. K2 persistent tcgen05 GEMM reading the four operands through TMA
// with the workspace taken from (and returned to) a CUDA memory pool in stream
// order, so the call never synchronises the host and can be graph-captured.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "dgemm_sm100.cuh"
#include "gemm_sm100.cuh"
#include "la.h"
#include "la_internal.h"
#include "split.cuh"

namespace la {

thread_local std::string g_last_error;
State g_state;
std::recursive_mutex g_mutex;  // serialises every entry point's host-side work

la_status fail(la_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return s;
}

int64_t test_hook(const char *name, int64_t dflt) {
    const char *e = getenv(name);
    return e && *e ? atoll(e) : dflt;
}

int64_t diag_knob(const char *name, int64_t dflt) {
#ifdef LA_DIAGNOSTICS
    return test_hook(name, dflt);
#else
    (void)name;
    return dflt;
#endif
}

la_status cuda_fail(cudaError_t e, const char *what, const char *file, int line) {
    return fail(LA_ERR_CUDA, "%s failed: %s (%s) at %s:%d", what, cudaGetErrorName(e),
                cudaGetErrorString(e), file, line);
}

// Tuned kernel configurations.
constexpr int kStages3 = 3;  // 3 x 64 KB stages for 3xTF32
constexpr int kStages1 = 6;  // 6 x 32 KB stages for plain TF32

static PFN_cuTensorMapEncodeTiled_v12000 get_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 2-D fp32 tensor map over a rows x cols row-major buffer (cols % 4 == 0),
// box = box_rows x 32 columns, 128-byte swizzle, OOB elements read as zero.
// L2 promotion of 128 B (one swizzle row): n = 4096 0.552 vs 0.555 ms with
// 256 B, equal at 16384 (scripts/ab_raw.py).
static la_status make_tmap(CUtensorMap *map, const float *ptr, int64_t rows, int64_t cols,
                           int box_rows, int box_k = BK) {
    auto enc = get_encoder();
    if (!enc) return fail(LA_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * sizeof(float)};
    cuuint32_t box[2] = {(cuuint32_t)box_k, (cuuint32_t)box_rows};  // box_rows <= 256
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(ptr), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     box_k == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(LA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) rows=%lld cols=%lld", (int)r,
                    (long long)rows, (long long)cols);
    return LA_OK;
}

// Row-major fp64 matrix (rows x cols) for the DGEMM's TMA boxes of 16 doubles x
// box_rows, 128-byte swizzle.  cols must be even (16-byte row stride).
static la_status make_tmap_f64(CUtensorMap *map, const double *ptr, int64_t rows, int64_t cols, int box_rows) {
    auto enc = get_encoder();
    if (!enc) return fail(LA_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * sizeof(double)};
    cuuint32_t box[2] = {16, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(LA_ERR_CUDA, "cuTensorMapEncodeTiled (f64) failed (%d) rows=%lld cols=%lld", (int)r,
                    (long long)rows, (long long)cols);
    return LA_OK;
}

// Output map for the GEMM's TMA-store epilogue: fp32 {cols, rows, slices}, row
// stride ldc floats (ldc % 4 == 0), slice stride rows * ldc, 32 x 32 boxes,
// 128-byte swizzle (the epilogue's smem layout).
static la_status make_tmap_c(CUtensorMap *map, float *ptr, int64_t rows, int64_t cols, int64_t ldc, int64_t slices) {
    auto enc = get_encoder();
    if (!enc) return fail(LA_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)slices};
    cuuint64_t strides[2] = {(cuuint64_t)ldc * sizeof(float), (cuuint64_t)(rows * ldc) * sizeof(float)};
    cuuint32_t box[3] = {32, 32, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ptr, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(LA_ERR_CUDA, "cuTensorMapEncodeTiled (C) failed (%d) rows=%lld cols=%lld ldc=%lld", (int)r,
                    (long long)rows, (long long)cols, (long long)ldc);
    return LA_OK;
}

// ---- optional per-kernel device timing (bench.py roofline) ----------------
struct TimedSpan {
    cudaEvent_t a, b;
    TimedKind kind;
};
static std::vector<TimedSpan> g_spans;     // recorded, not yet read
static std::vector<cudaEvent_t> g_free_ev;  // reusable events

static cudaEvent_t take_event() {
    if (!g_free_ev.empty()) {
        cudaEvent_t e = g_free_ev.back();
        g_free_ev.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

la_status timing_begin(cudaStream_t st, cudaEvent_t *ev) {
    *ev = nullptr;
    if (!g_state.kernel_timing) return LA_OK;
    *ev = take_event();
    cudaError_t e = cudaEventRecord(*ev, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord", __FILE__, __LINE__);
    return LA_OK;
}

la_status timing_end(cudaStream_t st, cudaEvent_t ev, TimedKind kind) {
    if (!ev) return LA_OK;
    cudaEvent_t b = take_event();
    cudaError_t e = cudaEventRecord(b, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord", __FILE__, __LINE__);
    g_spans.push_back({ev, b, kind});
    return LA_OK;
}

size_t operands_bytes(int64_t n, int64_t m, int64_t p, int passes) {
    const int64_t mp = pad_k(m);
    return (size_t)((n + p) * mp) * sizeof(float) * (passes == 3 ? 2 : 1) + 1024;
}

Operands operands_carve(void *ws, int64_t n, int64_t m, int64_t p, int passes) {
    Operands o;
    o.mp = pad_k(m);
    o.passes = passes;
    float *base = static_cast<float *>(ws);
    // every buffer 16-byte aligned (n*mp and p*mp are multiples of 4 floats)
    o.a_hi = base;
    o.b_hi = o.a_hi + n * o.mp;
    o.a_lo = passes == 3 ? o.b_hi + p * o.mp : o.a_hi;
    o.b_lo = passes == 3 ? o.a_lo + n * o.mp : o.b_hi;
    return o;
}

la_status split_a(int64_t n, int64_t m, const float *A, const Operands &ops, cudaStream_t st, int *launches) {
    cudaEvent_t t0;
    la_status ts = timing_begin(st, &t0);
    if (ts != LA_OK) return ts;
    if (m % 4 == 0) {
        const int64_t count4 = n * m / 4;
        const int64_t per_block = 256 * SPLIT_UNROLL;
        const int blocks =
            (int)std::max<int64_t>(1, std::min<int64_t>((count4 + per_block - 1) / per_block, (int64_t)g_state.sms * 8));
        if (ops.passes == 3)
            split_rows_vec4_kernel<3><<<blocks, 256, 0, st>>>(reinterpret_cast<const float4 *>(A),
                                                              reinterpret_cast<float4 *>(ops.a_hi),
                                                              reinterpret_cast<float4 *>(ops.a_lo), count4);
        else
            split_rows_vec4_kernel<1><<<blocks, 256, 0, st>>>(reinterpret_cast<const float4 *>(A),
                                                              reinterpret_cast<float4 *>(ops.a_hi),
                                                              reinterpret_cast<float4 *>(ops.a_lo), count4);
    } else {
        dim3 grid((unsigned)std::min<int64_t>((ops.mp + 255) / 256, 64), (unsigned)std::min<int64_t>(n, 65535));
        if (ops.passes == 3)
            split_rows_kernel<3><<<grid, 256, 0, st>>>(A, ops.a_hi, ops.a_lo, n, m, ops.mp);
        else
            split_rows_kernel<1><<<grid, 256, 0, st>>>(A, ops.a_hi, ops.a_lo, n, m, ops.mp);
    }
    (*launches)++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "split_a launch", __FILE__, __LINE__);
    return timing_end(st, t0, TIMED_SPLIT);
}

la_status split_b(int64_t m, int64_t j0, int64_t pc, const float *B, int64_t ldb, const Operands &ops,
                  cudaStream_t st, int *launches) {
    dim3 grid((unsigned)((pc + 31) / 32), (unsigned)((ops.mp + 31) / 32));
    if (grid.y > 65535) return fail(LA_ERR_UNSUPPORTED, "m = %lld too large for the split grid", (long long)m);
    const float *b = B;  // B points at column j0 of the source matrix
    cudaEvent_t t0;
    la_status ts = timing_begin(st, &t0);
    if (ts != LA_OK) return ts;
    float *hi = ops.b_hi + j0 * ops.mp, *lo = ops.b_lo + j0 * ops.mp;
    const bool vec = pc % 4 == 0 && ldb % 4 == 0 && (reinterpret_cast<uintptr_t>(b) & 15) == 0;
    const bool T64 = vec && diag_knob("LA_SPLIT_T32", 0) == 0;
    if (T64) {
        dim3 g64((unsigned)((pc + 63) / 64), (unsigned)((ops.mp + 63) / 64));
        if (ops.passes == 3)
            split_transpose64_kernel<3><<<g64, 256, 0, st>>>(b, hi, lo, m, pc, ldb, ops.mp);
        else
            split_transpose64_kernel<1><<<g64, 256, 0, st>>>(b, hi, lo, m, pc, ldb, ops.mp);
    } else if (ops.passes == 3)
        split_transpose_kernel<3><<<grid, dim3(32, 8), 0, st>>>(b, hi, lo, m, pc, ldb, ops.mp);
    else
        split_transpose_kernel<1><<<grid, dim3(32, 8), 0, st>>>(b, hi, lo, m, pc, ldb, ops.mp);
    (*launches)++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "split_b launch", __FILE__, __LINE__);
    return timing_end(st, t0, TIMED_SPLIT);
}

// Both splits in one launch when A takes the float4 pass and B the 64 x 64
// vectorised transpose; returns false (nothing launched) otherwise.
static bool split_ab(int64_t n, int64_t m, int64_t p, const float *A, const float *B, const Operands &ops,
                     cudaStream_t st, int *launches, la_status *status) {
    const bool t32 = diag_knob("LA_SPLIT_T32", 0) != 0;
    if (m % 4 || p % 4 || ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) || t32 ||
        test_hook("LA_SPLIT_SEPARATE", 0) != 0)
        return false;
    const int64_t count4 = n * m / 4;
    const int64_t per_block = 256 * SPLIT_UNROLL;
    const int64_t na =
        std::max<int64_t>(1, std::min<int64_t>((count4 + per_block - 1) / per_block, (int64_t)g_state.sms * 8));
    const int64_t nbx = (p + 63) / 64, nby = (ops.mp + 63) / 64;
    if (na + nbx * nby > INT32_MAX) return false;
    cudaEvent_t t0;
    if ((*status = timing_begin(st, &t0)) != LA_OK) return true;
    const unsigned grid = (unsigned)(na + nbx * nby);
    const float4 *a4 = reinterpret_cast<const float4 *>(A);
    float4 *ah = reinterpret_cast<float4 *>(ops.a_hi), *al = reinterpret_cast<float4 *>(ops.a_lo);
    if (ops.passes == 3)
        split_ab_kernel<3><<<grid, 256, 0, st>>>(a4, ah, al, count4, na, B, ops.b_hi, ops.b_lo, m, p, ops.mp, nbx);
    else
        split_ab_kernel<1><<<grid, 256, 0, st>>>(a4, ah, al, count4, na, B, ops.b_hi, ops.b_lo, m, p, ops.mp, nbx);
    (*launches)++;
    cudaError_t e = cudaGetLastError();
    *status = e != cudaSuccess ? cuda_fail(e, "split_ab launch", __FILE__, __LINE__) : timing_end(st, t0, TIMED_SPLIT);
    return true;
}

// Split-K factor for a launch of `tiles` output tiles over `slots` concurrent
// clusters: only with few tiles (at most half the slots) and a long K, at least
// `min_piece` K-blocks per piece, at most 64 pieces (S * tiles <= slots bounds
// the partial workspace by slots x one tile, whatever S is).
static int splitk_pieces(int64_t tiles, int64_t slots, int num_kb, int min_piece) {
    if (2 * tiles > slots || num_kb < 2 * min_piece) return 1;
    int S = (int)std::min<int64_t>(std::min<int64_t>(slots / tiles, num_kb / min_piece), 64);
    if (S <= 1) return 1;
    const int per = (num_kb + S - 1) / S;
    return (num_kb + per - 1) / per;
}

// Pieces of at least 8 K-blocks; single-CTA launches (cg == 1, whose K-blocks
// take half the time, so the fixed prologue / epilogue / reduce cost weighs
// more) go down to 4 while the pieces fill at most 3/4 of the SMs: 512^3 14.7
// -> 12.2 us per call in a graph, 256x2048x256 16.6 -> 14.3, 128x4096x128
// 17.1 -> 15.4, 384x1536x384 16.4 -> 14.1, 300x500x200 15.2 -> 12.5; filling
// the machine with short pieces lost (777x1236x260 19.1 -> 20.8, 147 pieces;
// 2000x700x300 20.3 -> 21.4, 144), and so did 4 on CTA pairs
// (scripts/splitk_piece_sweep.py).  The kernel choice (for_choice) prices both
// kernels with 8.
static int splitk_factor(int64_t tiles, int64_t slots, int num_kb, int cg, bool for_choice = false) {
    const int64_t forced = test_hook("LA_SPLIT_K", -1);
    if (forced >= 0) return forced <= 1 ? 1 : (int)std::min<int64_t>(forced, 1024);
    const int S8 = splitk_pieces(tiles, slots, num_kb, 8);
    if (for_choice || cg != 1) return S8;
    const int S4 = splitk_pieces(tiles, slots, num_kb, (int)std::max<int64_t>(1, diag_knob("LA_SPLITK_MIN_PIECE1", 4)));
    return 4 * tiles * S4 <= 3 * slots ? S4 : S8;
}

template <int CG, int BN, int STAGES, int PASSES, int KB = BK>
static la_status launch_gemm(int64_t n, int64_t m, int64_t j0, int64_t pc, const Operands &ops, float *C,
                             int64_t ldc, int max_sms, cudaStream_t st, int *launches, const OutSpec &out) {
    using Cfg = GemmCfg<CG, BN, STAGES, PASSES, KB>;
    CUtensorMap ta_hi, ta_lo, tb_hi, tb_lo;
    la_status s;
    const float *bh = ops.b_hi + j0 * ops.mp, *bl = ops.b_lo + j0 * ops.mp;
    if ((s = make_tmap(&ta_hi, ops.a_hi, n, ops.mp, ROWS_PER_CTA, Cfg::ATOM_K)) != LA_OK) return s;
    if ((s = make_tmap(&tb_hi, bh, pc, ops.mp, Cfg::B_ROWS, Cfg::ATOM_K)) != LA_OK) return s;
    if (PASSES == 3) {
        if ((s = make_tmap(&ta_lo, ops.a_lo, n, ops.mp, ROWS_PER_CTA, Cfg::ATOM_K)) != LA_OK) return s;
        if ((s = make_tmap(&tb_lo, bl, pc, ops.mp, Cfg::B_ROWS, Cfg::ATOM_K)) != LA_OK) return s;
    } else {
        ta_lo = ta_hi;
        tb_lo = tb_hi;
    }
    GemmArgs args;
    args.C = C + j0 * out.cstride;
    args.n = n;
    args.p = pc;
    args.ldc = ldc;
    args.cstride = out.cstride;
    args.half_rows = out.half_rows;
    args.half_off = out.half_off;
    args.gather_win = out.gather_win;
    args.gather_peers = out.gather_peers;
    args.gather_row0 = out.gather_row0;
    args.gather_col0 = out.gather_col0 + j0;
    args.gather_ld = out.gather_ld;
    args.gather_emul_stride = out.gather_emul_stride;
    args.num_kb = (int32_t)((m + KB - 1) / KB);
    // Promotion only in 3xTF32: plain TF32's 2^-9 bound is 2^11 times looser than
    // the truncation bias of whole-K accumulation (~3 x 2^-20 S at K = 16384).
    // Automatic interval (promote_k < 0, the default): the TMEM accumulator
    // truncates at every MMA, so one chunk of K_c elements carries 3 K_c / 8
    // truncations at the chunk's own magnitude; long K averages them out over
    // many chunks (RN running sum), short K does not.  Measured worst case on
    // random-sign inputs vs the exact product (scripts/positive_check.py):
    // K = 256 in one chunk 0.79 x 2^-20 S, in two of 128 0.39, in four of 64
    // 0.19; so chunks of 32 up to K = 64 (24-bit inputs at K = 61: 0.58 in one
    // chunk, 0.27 in two), 64 up to K = 192, 128 beyond (256 halves the drain
    // work but doubles the same-sign truncation bias: 2.94 vs 1.68 x 2^-20 S
    // at K = 16384 before sign-centring, and costs nothing measurable at 128
    // for n >= 4096).  Chunks of 64 cost ~18% at K = 256, of 32 ~12% at K = 64
    // on 4096-wide outputs (scripts/promote_cost.py).
    int64_t pk = PASSES == 3 ? g_state.promote_k : 0;
    const int64_t km = out.policy_k > 0 ? out.policy_k : m;
    if (pk < 0) pk = km <= 64 ? 32 : (km <= 192 ? 64 : 128);
    args.kc = pk <= 0 ? args.num_kb : (int32_t)std::max<int64_t>(1, (pk + KB - 1) / KB);
    if (args.kc > args.num_kb) args.kc = args.num_kb;
    // Sign-centred promotion chunks (gemm_sm100.cuh ChunkPlan) end within the
    // policy K (la_cgemm: the real half of its 2m-long embedding, so
    // zero-imaginary products keep la_gemm's bits), and only when K spans at
    // least 8 chunks: an offset is extrapolated from the chunk two before, so a
    // sign change along K can enlarge one chunk's partial sums -- diluted over
    // >= 8 chunks, not over 2 or 3 (K = 256 with sign-flipped halves: 0.70 ->
    // 1.71 x 2^-20 S against the exact product when centred).
    const int64_t policy_kb = (km + KB - 1) / KB;
    auto set_center = [&]() {
        args.center_kb = args.kc >= 2 && policy_kb >= 8 * (int64_t)args.kc
                             ? (int32_t)std::min<int64_t>(args.num_kb, policy_kb) : 0;
    };
    set_center();
    args.tiles_m = (int32_t)((n + Cfg::TILE_M - 1) / Cfg::TILE_M);
    args.tiles_n = (int32_t)((pc + BN - 1) / BN);
    args.group_m = (int32_t)std::max<int64_t>(1, diag_knob("LA_GROUP_M", 8));
    const int64_t tiles = (int64_t)args.tiles_m * args.tiles_n;

    auto kern = gemm_tf32_sm100_kernel<CG, BN, STAGES, PASSES, KB>;
    // per-device setup, redone after la_finalize + la_init (possibly another device)
    static int max_clusters = 0;
    static uint64_t setup_gen = 0;
    if (setup_gen != g_state.generation) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(smem)", __FILE__, __LINE__);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(CG * g_state.sms / CG);
        cfg.blockDim = dim3(NUM_THREADS);
        cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
        cudaLaunchAttribute attr;
        attr.id = cudaLaunchAttributeClusterDimension;
        attr.val.clusterDim.x = CG;
        attr.val.clusterDim.y = 1;
        attr.val.clusterDim.z = 1;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        int nc = 0;
        e = cudaOccupancyMaxActiveClusters(&nc, kern, &cfg);
        if (e != cudaSuccess || nc <= 0) {
            cudaGetLastError();
            nc = g_state.sms / CG;
        }
        max_clusters = nc;
        setup_gen = g_state.generation;
    }
    // A static persistent grid: one cluster per SM pair, tiles strided in
    // grouped raster order.  (A dynamic schedule through cluster launch control
    // was measured worse -- 129 vs 105-113 GB of DRAM reads per n = 16384
    // launch, profiles/ncu_r01_sched_ab.md -- and removed.)
    int clusters = max_clusters;
    if (max_sms > 0) clusters = std::min(clusters, std::max(1, max_sms / CG));
#ifdef LA_DIAGNOSTICS
    clusters = std::min<int>(clusters, (int)std::max<int64_t>(1, diag_knob("LA_DIAG_CLUSTERS", clusters)));
#endif
    clusters = (int)std::min<int64_t>(tiles, clusters);
    // Split-K: fewer tiles than half the clusters and a long K -> each tile's K
    // range is cut into S pieces (at least 8 K-blocks each) computed by
    // different clusters; partial tiles go to a workspace and are summed in
    // order by splitk_reduce_kernel, launched as a programmatic dependent of the
    // GEMM on the whole GPU.  (An in-kernel fix-up -- the last piece to finish a
    // region of a tile sums the S slices -- was measured 2.8x slower at C2: one
    // warp per region reads S x 16 KB latency-bound, ~50 GB/s per SM, on the few
    // SMs that hold the tiles.)  Plain real outputs from la_gemm only
    // (OutSpec::splitk_ok).  LA_SPLIT_K=0 disables, =S forces S.
    args.ksplit = 1;
    args.kb_per = args.num_kb;
    args.partial = nullptr;
    void *part_buf = nullptr;
    {
        const int kb32 = (int)((m + 31) / 32);
        const int S = out.splitk_ok ? splitk_factor(tiles, max_clusters, kb32, CG) : 1;
        if (S > 1) {
            // pieces of kb_per K-blocks; recount S from the piece size so every
            // piece is non-empty ((S - 1) * kb_per < num_kb)
            args.kb_per = (args.num_kb + S - 1) / S;
            const int S2 = (args.num_kb + args.kb_per - 1) / args.kb_per;
            args.ksplit = S2;
            // promotion inside short pieces: at least two chunks per piece, so
            // the sign-centred plan (leading chunks of kc/2, then kc) still
            // centres part of every piece (pieces of 4 K-blocks at kc = 4
            // would be single chunks)
            if (args.kc < args.num_kb && args.kc > 1 && args.kb_per < 2 * args.kc) {
                args.kc = std::max(1, args.kb_per / 2);
                set_center();
            }
        }
        if (args.ksplit > 1) {
            const int S = args.ksplit;
            const size_t pbytes = (size_t)S * (size_t)(n * pc) * sizeof(float);
            cudaError_t e = cudaMallocFromPoolAsync(&part_buf, pbytes, g_state.pool, st);
            if (e != cudaSuccess) {
                cudaGetLastError();
                return fail(LA_ERR_OUT_OF_MEMORY, "split-K partials of %zu bytes", pbytes);
            }
            args.partial = static_cast<float *>(part_buf);
            clusters = (int)std::min<int64_t>((int64_t)tiles * S, max_clusters);
        }
    }
    // Tail split: if the last wave is at most half full, its tiles run as two
    // half-width items each, so it takes half a tile time (n = 4096: 3.46 waves
    // of 256x256 tiles -> 3.5 instead of 4).  Per-element accumulation order is
    // unchanged (same K blocks, same promotion chunks), so results are bitwise
    // identical with or without it.  LA_TAIL_SPLIT=0 disables.
    args.full_items = args.num_items = (int32_t)(tiles * args.ksplit);
    {
        const bool tail_split = args.ksplit == 1 && test_hook("LA_TAIL_SPLIT", 1) != 0;
        const int64_t W = clusters, R = tiles % W;
        if (tail_split && R > 0 && 2 * R <= W && tiles > W) {
            args.full_items = (int32_t)(tiles - R);
            args.num_items = (int32_t)(tiles + R);
        }
    }
    // TMA-store epilogue for plain row-major outputs (C or the split-K partial
    // slices); LA_TMA_STORE=0 selects the per-thread stores (A/B knob).
    CUtensorMap tm_c;
    memset(&tm_c, 0, sizeof tm_c);
    {
        float *base = args.ksplit > 1 ? args.partial : args.C;
        const bool env_off = test_hook("LA_TMA_STORE", 1) == 0;
        args.tma_store = !env_off && out.cstride == 1 && out.half_rows == 0 && out.gather_win == nullptr &&
                         ldc % 4 == 0 && (reinterpret_cast<uintptr_t>(base) & 15) == 0 && n < ((int64_t)1 << 31) &&
                         pc < ((int64_t)1 << 31);
        if (args.tma_store && (s = make_tmap_c(&tm_c, base, n, pc, ldc, args.ksplit)) != LA_OK) return s;
    }
    args.trace = nullptr;
#ifdef LA_DIAGNOSTICS
    // Energy diagnostics only (results are garbage): 1 = skip TMA loads, 2 = skip
    // MMAs.  Compiled in only with LA_BUILD_DIAGNOSTICS=1 at build time.
    args.debug = (int32_t)diag_knob("LA_DEBUG_KERNEL", 0);
    // LA_DIAG_TRACE=1: per-CTA globaltimer stamps, printed after the launch
    // (host-synchronising; diagnostics only)
    static int64_t *trace_buf = nullptr;
    const bool trace_on = diag_knob("LA_DIAG_TRACE", 0) != 0;
    if (trace_on) {
        if (!trace_buf) cudaMalloc(&trace_buf, TRACE_SLOTS * sizeof(int64_t) * 1024);
        cudaMemsetAsync(trace_buf, 0, TRACE_SLOTS * sizeof(int64_t) * 1024, st);
        args.trace = trace_buf;
    }
#else
    args.debug = 0;
#endif
    args.wave_sync = nullptr;
    args.wave_slots = 0;
    args.sync_kb = args.num_kb;
    void *sync_buf = nullptr;
    // K-phase alignment of the static schedule (gemm_sm100.cuh wave_barrier):
    // every 16 K-blocks the producers of a wave meet at a counter, so clusters
    // that share A rows / B columns stream K together and hit each other's
    // slabs in L2.  Measured at n = 16384: DRAM reads 105-129 GB -> 42 GB per
    // launch, 13% less energy and +14% sustained throughput under the power cap
    // (profiles/energy_r01.md).  On by default for multi-wave problems with a
    // long K; LA_WAVE_SYNC=0 disables, =N sets the interval in K-blocks.
    const int64_t ws_env = diag_knob("LA_WAVE_SYNC", -1);
    // Never with an SM cap: the capped launch runs beside other kernels (NCCL in
    // la_gemm_multi) and every participant of a wave must be resident.
    // Default only for 3xTF32: with one TF32 pass each K phase is 3x shorter and
    // the barrier costs more than it saves (n = 8192 TF32: 660 vs 628 TFLOP/s off/on).
    int wave_sync = ws_env >= 0 ? (int)ws_env * BK / KB
                           : (PASSES == 3 && args.num_kb * KB >= 64 * BK ? 16 * BK / KB : 0);
    if (max_sms > 0 || args.ksplit > 1) wave_sync = 0;
    if (wave_sync > 0) {
        args.sync_kb = std::max(1, std::min(args.num_kb, wave_sync));
        const int64_t phases = (args.num_kb + args.sync_kb - 1) / args.sync_kb;
        const size_t nw = (size_t)((args.num_items + clusters - 1) / clusters * phases);
        args.wave_slots = (int32_t)nw;
        cudaError_t e = cudaMallocFromPoolAsync(&sync_buf, (nw + 1) * sizeof(int32_t), g_state.pool, st);
        if (e != cudaSuccess) return cuda_fail(e, "wave sync buffer", __FILE__, __LINE__);
        e = cudaMemsetAsync(sync_buf, 0, (nw + 1) * sizeof(int32_t), st);
        if (e != cudaSuccess) return cuda_fail(e, "wave sync memset", __FILE__, __LINE__);
        args.wave_sync = static_cast<int32_t *>(sync_buf);
    }
    cudaEvent_t t0;
    if ((s = timing_begin(st, &t0)) != LA_OK) return s;
    // launched with programmatic stream serialization: the kernel's prologue may
    // overlap the preceding split kernels; it waits (griddepcontrol.wait) before
    // reading their output
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)(clusters * CG));
    lc.blockDim = dim3(NUM_THREADS);
    lc.dynamicSmemBytes = Cfg::SMEM_BYTES;
    lc.stream = st;
    cudaLaunchAttribute la_attr[1];
    la_attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la_attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = la_attr;
    lc.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&lc, kern, ta_hi, ta_lo, tb_hi, tb_lo, tm_c, args);
    if (e != cudaSuccess) return cuda_fail(e, "gemm kernel launch", __FILE__, __LINE__);
    (*launches)++;
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "gemm kernel launch", __FILE__, __LINE__);
    if (sync_buf) cudaFreeAsync(sync_buf, st);
#ifdef LA_DIAGNOSTICS
    if (args.trace) {
        const int nb = clusters * CG;
        std::vector<int64_t> h((size_t)nb * TRACE_SLOTS);
        cudaStreamSynchronize(st);
        cudaMemcpy(h.data(), args.trace, h.size() * sizeof(int64_t), cudaMemcpyDeviceToHost);
        int64_t t0s = INT64_MAX;
        for (int b = 0; b < nb; b++) if (h[b * TRACE_SLOTS]) t0s = std::min(t0s, h[b * TRACE_SLOTS]);
        static const char *names[8] = {"entry", "setup done", "producer past griddepcontrol.wait",
                                       "MMA: first stage full", "MMA: last commit", "epilogue: first chunk ready",
                                       "epilogue: stores done", "exit sync done"};
        fprintf(stderr, "la_diag_trace grid=%d n=%lld p=%lld num_kb=%d kc=%d ksplit=%d (us after first entry)\n", nb,
                (long long)n, (long long)pc, args.num_kb, args.kc, args.ksplit);
        for (int k = 0; k < 8; k++) {
            std::vector<double> v;
            for (int b = 0; b < nb; b++) if (h[b * TRACE_SLOTS + k]) v.push_back((h[b * TRACE_SLOTS + k] - t0s) * 1e-3);
            if (v.empty()) continue;
            std::sort(v.begin(), v.end());
            fprintf(stderr, "la_diag_trace %-36s min %9.2f med %9.2f max %9.2f (%zu CTAs)\n", names[k], v.front(),
                    v[v.size() / 2], v.back(), v.size());
        }
        for (int k = 8; k < 10; k++) {
            std::vector<double> v;
            for (int b = 0; b < nb; b += CG) v.push_back((double)h[b * TRACE_SLOTS + k]);
            std::sort(v.begin(), v.end());
            fprintf(stderr, "la_diag_trace MMA warp waited on %-8s cycles: min %.0f med %.0f max %.0f (%zu CTAs)\n",
                    k == 8 ? "tempty" : "full", v.front(), v[v.size() / 2], v.back(), v.size());
        }
    }
#endif
    la_status rs = timing_end(st, t0, TIMED_GEMM);
    if (rs != LA_OK) return rs;
    if (args.ksplit > 1) {
        const int64_t count = n * pc;
        const bool vec = count % 4 == 0 && (reinterpret_cast<uintptr_t>(args.C) & 15) == 0;
        const int64_t work = vec ? count / 4 : count;
        const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, (int64_t)g_state.sms * 8));
        cudaEvent_t t1;
        if ((rs = timing_begin(st, &t1)) != LA_OK) return rs;
        // programmatic dependent launch: scheduled while the GEMM drains, the
        // kernel's griddepcontrol.wait holds it until the partials are complete
        cudaLaunchConfig_t rc = {};
        rc.gridDim = dim3((unsigned)blocks);
        rc.blockDim = dim3(256);
        rc.stream = st;
        cudaLaunchAttribute ra[1];
        ra[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        ra[0].val.programmaticStreamSerializationAllowed = 1;
        rc.attrs = ra;
        rc.numAttrs = 1;
        if (vec)
            e = cudaLaunchKernelEx(&rc, splitk_reduce_vec4_kernel, reinterpret_cast<const float4 *>(args.partial),
                                   reinterpret_cast<float4 *>(args.C), work, args.ksplit);
        else
            e = cudaLaunchKernelEx(&rc, splitk_reduce_kernel, static_cast<const float *>(args.partial), args.C,
                                   count, args.ksplit);
        if (e != cudaSuccess) return cuda_fail(e, "split-K reduce launch", __FILE__, __LINE__);
        (*launches)++;
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "split-K reduce launch", __FILE__, __LINE__);
        cudaFreeAsync(part_buf, st);
        return timing_end(st, t1, TIMED_SPLIT);  // counted with the auxiliary passes
    }
    return LA_OK;
}

// Kernel choice by a small cost model: time ~ waves x K-blocks per item x
// cycles per K-block, with the single-CTA 128 x 128 kernel (768 tensor cycles
// per K-block) charged 1.5x for its doubled operand traffic per flop (it is
// L2-bound) against the CTA pair's 256 x 256 tiles (1536 cycles per K-block on
// two SMs), each with its best split-K factor.  Measured checks
// (scripts/cg_choice.py): pair wins from ~40 tiles up without split-K
// (n = 2048: 108 vs 145 us), single-CTA for tiny problems (n = 256).
static int choose_cta_group(int64_t n, int64_t pc, int num_kb, bool splitk_ok) {
    const int64_t forced = test_hook("LA_CTA_GROUP", 0);
    if (forced == 1 || forced == 2) return (int)forced;
    double cost[3] = {0, 0, 0};
    for (int cg = 1; cg <= 2; cg++) {
        const int64_t tm = 128 * cg, tn = cg == 2 ? 256 : 128;
        const int64_t tiles = ((n + tm - 1) / tm) * ((pc + tn - 1) / tn);
        const int64_t slots = g_state.sms / cg;
        const int S = splitk_ok ? splitk_factor(tiles, slots, num_kb, cg, true) : 1;
        const int64_t items = tiles * S;
        const int64_t kb_item = (num_kb + S - 1) / S;
        const double waves = (double)((items + slots - 1) / slots);
        cost[cg] = waves * kb_item * (cg == 2 ? 1536.0 : 768.0 * 1.5);
    }
    return cost[2] <= cost[1] ? 2 : 1;
}

la_status gemm_run(int64_t n, int64_t m, int64_t j0, int64_t pc, const Operands &ops, float *C, int64_t ldc,
                   int max_sms, cudaStream_t st, int *launches, OutSpec out) {
    const int num_kb = (int)((m + 31) / 32);  // cost model in 32-wide K-blocks
    const bool splitk_ok = out.splitk_ok && max_sms <= 0 && out.cstride == 1 && out.half_rows == 0 &&
                           out.gather_win == nullptr && ldc == pc;
    out.splitk_ok = splitk_ok;
    const int cg = choose_cta_group(n, pc, num_kb, splitk_ok);
    // (KB = 16 with a 6-stage ring was measured slower and costlier: 202 vs 244
    // TFLOP/s and 42.9 vs 35.3 J per n = 16384 GEMM -- not dispatched.)
    if (ops.passes == 3) {
        if (cg == 2) return launch_gemm<2, 256, kStages3, 3>(n, m, j0, pc, ops, C, ldc, max_sms, st, launches, out);
        return launch_gemm<1, 128, kStages3, 3>(n, m, j0, pc, ops, C, ldc, max_sms, st, launches, out);
    }
    // plain TF32, long power-capped runs: K-blocks of 64 (two swizzle atoms per
    // stage, 3 x 64 KB) halve the per-stage barrier and issue work of the single
    // pass -- measured +2.6..4.7% at n = 16384, -0.7..1.6% at n = 4096 / 8192
    // (more, smaller stages win when the clock is not capped), hence only from
    // 2^41 multiply-adds up.  LA_TF32_KB=32|64 forces either (A/B knob).
    const int64_t kbe = test_hook("LA_TF32_KB", 0);
    const bool kb64 = kbe ? kbe == 64 : (double)n * (double)pc * (double)m >= 2199023255552.0;
    if (kb64) {
        if (cg == 2) return launch_gemm<2, 256, 3, 1, 64>(n, m, j0, pc, ops, C, ldc, max_sms, st, launches, out);
        return launch_gemm<1, 128, 3, 1, 64>(n, m, j0, pc, ops, C, ldc, max_sms, st, launches, out);
    }
    if (cg == 2) return launch_gemm<2, 256, kStages1, 1>(n, m, j0, pc, ops, C, ldc, max_sms, st, launches, out);
    return launch_gemm<1, 128, kStages1, 1>(n, m, j0, pc, ops, C, ldc, max_sms, st, launches, out);
}

la_status validate_gemm(int64_t n, int64_t m, int64_t p, const float *A, const float *B, const float *C) {
    if (!g_state.initialized) return fail(LA_ERR_NOT_INITIALIZED, "la_init has not been called");
    if (n <= 0 || m <= 0 || p <= 0)
        return fail(LA_ERR_INVALID_VALUE, "dimensions must be >= 1 (n=%lld m=%lld p=%lld)", (long long)n,
                    (long long)m, (long long)p);
    if (n > (int64_t)1 << 31 || m > (int64_t)1 << 31 || p > (int64_t)1 << 31)
        return fail(LA_ERR_UNSUPPORTED, "dimension exceeds 2^31 (TMA coordinates are int32)");
    if (!A || !B || !C) return fail(LA_ERR_INVALID_VALUE, "NULL matrix pointer");
    auto overlap = [](const void *x, int64_t xb, const void *y, int64_t yb) {
        const char *a = (const char *)x, *b = (const char *)y;
        return a < b + yb && b < a + xb;
    };
    const int64_t ab = n * m * 4, bb = m * p * 4, cb = n * p * 4;
    if (overlap(C, cb, A, ab) || overlap(C, cb, B, bb))
        return fail(LA_ERR_INVALID_VALUE, "C overlaps A or B");
    return LA_OK;
}

// C (n x p, row stride ldc) = A (n x m) . B (m x p), one GPU.
static la_status gemm_impl(int64_t n, int64_t m, int64_t p, const float *A, const float *B, float *C, int64_t ldc,
                           cudaStream_t st, int *launches) {
    const int passes = g_state.mode == LA_MODE_TF32 ? 1 : 3;
    const size_t bytes = operands_bytes(n, m, p, passes);
    void *ws = nullptr;
    cudaError_t e = cudaMallocFromPoolAsync(&ws, bytes, g_state.pool, st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(LA_ERR_OUT_OF_MEMORY, "workspace of %zu bytes: %s", bytes, cudaGetErrorString(e));
    }
    const Operands ops = operands_carve(ws, n, m, p, passes);
    la_status s = LA_OK;
    if (!split_ab(n, m, p, A, B, ops, st, launches, &s)) {
        s = split_a(n, m, A, ops, st, launches);
        if (s == LA_OK) s = split_b(m, 0, p, B, p, ops, st, launches);
    }
    OutSpec out;
    out.splitk_ok = true;
    if (s == LA_OK) s = gemm_run(n, m, 0, p, ops, C, ldc, (int)g_state.max_sms, st, launches, out);
    e = cudaFreeAsync(ws, st);
    if (s == LA_OK && e != cudaSuccess) return cuda_fail(e, "cudaFreeAsync", __FILE__, __LINE__);
    return s;
}

}  // namespace la

using namespace la;

#define LA_CK(call)                                                          \
    do {                                                                     \
        cudaError_t e_ = (call);                                             \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call, __FILE__, __LINE__); \
    } while (0)

extern "C" {

la_status la_init(int device) {
    std::lock_guard<std::recursive_mutex> lk(g_mutex);
    g_last_error.clear();
    if (g_state.initialized) {
        if (device == g_state.device) {
            LA_CK(cudaSetDevice(device));
            return LA_OK;
        }
        return fail(LA_ERR_INVALID_VALUE, "already initialised on device %d", g_state.device);
    }
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount", __FILE__, __LINE__);
    if (device < 0 || device >= count) return fail(LA_ERR_INVALID_VALUE, "no CUDA device %d (%d present)", device, count);
    LA_CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    LA_CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0)
        return fail(LA_ERR_UNSUPPORTED, "device %d is sm_%d%d (%s); this library is built for sm_100a (B200)",
                    device, prop.major, prop.minor, prop.name);
    cudaMemPoolProps pp;
    memset(&pp, 0, sizeof pp);
    pp.allocType = cudaMemAllocationTypePinned;
    pp.handleTypes = cudaMemHandleTypeNone;
    pp.location.type = cudaMemLocationTypeDevice;
    pp.location.id = device;
    LA_CK(cudaMemPoolCreate(&g_state.pool, &pp));
    uint64_t thr = UINT64_MAX;
    LA_CK(cudaMemPoolSetAttribute(g_state.pool, cudaMemPoolAttrReleaseThreshold, &thr));
    g_state.device = device;
    g_state.sms = prop.multiProcessorCount;
    static uint64_t generations = 0;
    g_state.generation = ++generations;  // invalidates per-device kernel setup cached by earlier inits
    g_state.initialized = true;
    return LA_OK;
}

la_status la_set_mode(la_mode mode) {
    std::lock_guard<std::recursive_mutex> lk(g_mutex);
    if (mode != LA_MODE_3XTF32 && mode != LA_MODE_TF32) return fail(LA_ERR_INVALID_VALUE, "unknown mode %d", (int)mode);
    g_state.mode = mode;
    return LA_OK;
}

la_status la_set_option(la_option option, int64_t value) {
    std::lock_guard<std::recursive_mutex> lk(g_mutex);
    switch (option) {
        case LA_OPT_PROMOTE_K:
            if (value < -1) return fail(LA_ERR_INVALID_VALUE, "promote_k must be >= -1 (-1: automatic)");
            g_state.promote_k = value;
            return LA_OK;
        case LA_OPT_MAX_SMS:
            if (value < 0) return fail(LA_ERR_INVALID_VALUE, "max_sms must be >= 0");
            g_state.max_sms = value;
            return LA_OK;
        case LA_OPT_PANELS:
            if (value < 0) return fail(LA_ERR_INVALID_VALUE, "panels must be >= 0 (0: automatic)");
            g_state.panels = value;
            return LA_OK;
        case LA_OPT_KERNEL_TIMING:
            if (value != 0 && value != 1) return fail(LA_ERR_INVALID_VALUE, "kernel_timing is 0 or 1");
            g_state.kernel_timing = value == 1;
            return LA_OK;
        case LA_OPT_NCCL_SMS:
            if (value < 0 || value > 64) return fail(LA_ERR_INVALID_VALUE, "nccl_sms must be in [0, 64]");
            g_state.nccl_sms = value;
            return LA_OK;

    }
    return fail(LA_ERR_INVALID_VALUE, "unknown option %d", (int)option);
}

la_status la_get_option(la_option option, int64_t *value) {
    std::lock_guard<std::recursive_mutex> lk(g_mutex);
    if (!value) return fail(LA_ERR_INVALID_VALUE, "NULL value pointer");
    switch (option) {
        case LA_OPT_PROMOTE_K: *value = g_state.promote_k; return LA_OK;
        case LA_OPT_MAX_SMS: *value = g_state.max_sms; return LA_OK;
        case LA_OPT_PANELS: *value = g_state.panels; return LA_OK;
        case LA_OPT_KERNEL_TIMING: *value = g_state.kernel_timing ? 1 : 0; return LA_OK;
        case LA_OPT_NCCL_SMS: *value = g_state.nccl_sms; return LA_OK;
    }
    return fail(LA_ERR_INVALID_VALUE, "unknown option %d", (int)option);
}

la_status la_gemm(int64_t n, int64_t m, int64_t p, const float *d_A, const float *d_B, float *d_C,
                  void *stream) {
    std::lock_guard<std::recursive_mutex> lk(g_mutex);
    la_status s = validate_gemm(n, m, p, d_A, d_B, d_C);
    if (s != LA_OK) return s;
    int launches = 0;
    s = gemm_impl(n, m, p, d_A, d_B, d_C, p, static_cast<cudaStream_t>(stream), &launches);
    g_state.last_launches = launches;
    return s;
}

// End-to-end product on host buffers, pipelined (the paper's host flow, P:23
// and P:144, with the transfer the paper calls the weak point hidden behind
// compute): B goes first (every output row needs all of it), then A in row
// panels on a copy-in stream; the caller's stream splits B once and then, per
// panel, splits the A rows and runs the GEMM on them as soon as they land; a
// copy-out stream returns each C panel while later panels compute.  With
// pinned host buffers the copies overlap compute in both directions.
// Panels per operand for la_gemm_host's 2-D transfer schedule (LA_HOST_PANELS
// overrides; measured in profiles/e2e_r01.md).
// LA_HOST_TRACE=1: print the schedule's timeline (ms after the first copy
// starts) to stderr -- a diagnostic for profiles/e2e_r01.md, off by default.
struct HostTrace {
    bool on = false;
    std::vector<std::pair<std::string, cudaEvent_t>> marks;
    void mark(const std::string &label, cudaStream_t s) {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        marks.push_back({label, e});
    }
    void dump() {
        if (!on || marks.empty()) return;
        cudaDeviceSynchronize();
        for (auto &m : marks) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, marks[0].second, m.second);
            fprintf(stderr, "la_host_trace %8.3f %s\n", ms, m.first.c_str());
        }
        for (auto &m : marks) cudaEventDestroy(m.second);
        marks.clear();
    }
};

static int64_t host_tail_split() {
    const int64_t t = diag_knob("LA_HOST_TAIL_SPLIT", 2);
    return std::max<int64_t>(1, std::min<int64_t>(t, 16));
}

static int64_t host_panels() {
    const int64_t q = test_hook("LA_HOST_PANELS", 12);
    return std::max<int64_t>(1, std::min<int64_t>(q, 64));
}

}  // extern "C"

namespace la {

// One product of a host call on device staging (dA, dB, dC): the 2-D transfer
// schedule.  A travels in row panels and B in column panels (heights and widths
// multiples of the 256-wide tile), interleaved on the copy-in stream so that
// the fraction of A and of B on the device grow together.  Each panel that
// lands unlocks one rectangle of C -- its rows (or columns) against every panel
// of the other operand already present -- computed by one GEMM launch and
// copied out while later panels are still in flight.  Every C element is
// produced by exactly one tile over the whole K range, in la_gemm's order.
// gate_h2d / gate_compute (optional): the staging slot's previous user has
// finished computing from it / copying C out of it.
static la_status host_item(int64_t n, int64_t m, int64_t p, const float *h_A, const float *h_B, float *h_C,
                           float *dA, float *dB, float *dC, const Operands &ops, cudaStream_t st,
                           cudaEvent_t gate_h2d, cudaEvent_t gate_compute, cudaEvent_t done_compute,
                           cudaEvent_t done_d2h, int *launches, HostTrace &tr) {
    const int64_t q = host_panels();
    auto panel = [q](int64_t len) {
        return len >= 2048 ? std::min(len, ((len + q - 1) / q + 255) / 256 * 256) : len;
    };
    const int64_t rh = panel(n), pw = panel(p);
    const int64_t Qr = (n + rh - 1) / rh, Qc = (p + pw - 1) / pw;
    const int64_t tail_split = host_tail_split();
    while ((int64_t)g_state.host_events.size() < 2 * (Qr + Qc) + 2 * tail_split) {
        cudaEvent_t e;
        LA_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        g_state.host_events.push_back(e);
    }
    // (events are re-recorded by later items only after every wait on them
    // has been enqueued, so one set serves all items of a call)
    cudaEvent_t *ev_a = &g_state.host_events[0], *ev_b = ev_a + Qr, *ev_c = ev_b + Qc;
    // arrival order: the operand whose present fraction is smaller goes next (A first)
    std::vector<std::pair<bool, int64_t>> order;  // (is_A, panel index)
    for (int64_t a = 0, bq = 0; a < Qr || bq < Qc;) {
        if (bq >= Qc || (a < Qr && a * Qc <= bq * Qr)) order.push_back({true, a++});
        else order.push_back({false, bq++});
    }
    if (gate_h2d) LA_CK(cudaStreamWaitEvent(g_state.h2d, gate_h2d, 0));
    for (const auto &o : order) {
        if (o.first) {
            const int64_t r0 = o.second * rh, rows = std::min(rh, n - r0);
            LA_CK(cudaMemcpyAsync(dA + r0 * m, h_A + r0 * m, (size_t)(rows * m) * 4, cudaMemcpyHostToDevice,
                                  g_state.h2d));
            LA_CK(cudaEventRecord(ev_a[o.second], g_state.h2d));
            tr.mark("h2d A" + std::to_string(o.second), g_state.h2d);
        } else {
            const int64_t c0 = o.second * pw, w = std::min(pw, p - c0);
            LA_CK(cudaMemcpy2DAsync(dB + c0, (size_t)p * 4, h_B + c0, (size_t)p * 4, (size_t)w * 4, (size_t)m,
                                    cudaMemcpyHostToDevice, g_state.h2d));
            LA_CK(cudaEventRecord(ev_b[o.second], g_state.h2d));
            tr.mark("h2d B" + std::to_string(o.second), g_state.h2d);
        }
    }
    if (gate_compute) LA_CK(cudaStreamWaitEvent(st, gate_compute, 0));
    la_status s = LA_OK;
    int64_t rows_in = 0, cols_in = 0, regions = 0;
    for (const auto &o : order) {
        int64_t r0, r1, c0, c1;
        if (o.first) {
            r0 = o.second * rh;
            r1 = std::min(n, r0 + rh);
            LA_CK(cudaStreamWaitEvent(st, ev_a[o.second], 0));
            Operands pan = ops;
            pan.a_hi = ops.a_hi + r0 * ops.mp;
            pan.a_lo = ops.a_lo + r0 * ops.mp;
            s = split_a(r1 - r0, m, dA + r0 * m, pan, st, launches);
            rows_in = r1;
            c0 = 0;
            c1 = cols_in;
        } else {
            c0 = o.second * pw;
            c1 = std::min(p, c0 + pw);
            LA_CK(cudaStreamWaitEvent(st, ev_b[o.second], 0));
            s = split_b(m, c0, c1 - c0, dB + c0, p, ops, st, launches);
            cols_in = c1;
            r0 = 0;
            r1 = rows_in;
        }
        if (s != LA_OK) return s;
        tr.mark(std::string("split ") + (o.first ? "A" : "B") + std::to_string(o.second), st);
        if (r1 <= r0 || c1 <= c0) continue;
        // the last two rectangles are computed in pieces along their long side
        // so that the copy-out of one piece overlaps the GEMM of the next
        const int64_t pieces = (int64_t)(&o - order.data()) + 2 >= (int64_t)order.size() ? tail_split : 1;
        const bool by_rows = r1 - r0 >= c1 - c0;
        const int64_t len = by_rows ? r1 - r0 : c1 - c0;
        const int64_t step = std::max<int64_t>(256, ((len + pieces - 1) / pieces + 255) / 256 * 256);
        for (int64_t x0 = 0; x0 < len; x0 += step) {
            const int64_t x1 = std::min(len, x0 + step);
            const int64_t q0 = by_rows ? r0 + x0 : r0, q1 = by_rows ? r0 + x1 : r1;
            const int64_t k0 = by_rows ? c0 : c0 + x0, k1 = by_rows ? c1 : c0 + x1;
            Operands pan = ops;
            pan.a_hi = ops.a_hi + q0 * ops.mp;
            pan.a_lo = ops.a_lo + q0 * ops.mp;
            s = gemm_run(q1 - q0, m, k0, k1 - k0, pan, dC + q0 * p, p, (int)g_state.max_sms, st, launches);
            if (s != LA_OK) return s;
            tr.mark("gemm " + std::to_string(q1 - q0) + "x" + std::to_string(k1 - k0), st);
            LA_CK(cudaEventRecord(ev_c[regions], st));
            LA_CK(cudaStreamWaitEvent(g_state.d2h, ev_c[regions], 0));
            LA_CK(cudaMemcpy2DAsync(h_C + q0 * p + k0, (size_t)p * 4, dC + q0 * p + k0, (size_t)p * 4,
                                    (size_t)(k1 - k0) * 4, (size_t)(q1 - q0), cudaMemcpyDeviceToHost,
                                    g_state.d2h));
            tr.mark("d2h " + std::to_string(regions), g_state.d2h);
            regions++;
        }
    }
    LA_CK(cudaEventRecord(done_compute, st));
    LA_CK(cudaEventRecord(done_d2h, g_state.d2h));
    return LA_OK;
}

// `count` independent host products of one shape.  With count > 1 two device
// staging slots alternate, so the copy-in of product i + 1 runs while product i
// still computes and copies out (the copy engines stay busy across products).
static la_status host_run(int64_t count, int64_t n, int64_t m, int64_t p, const float *const *hA,
                          const float *const *hB, float *const *hC, cudaStream_t st) {
    if (!g_state.initialized) return fail(LA_ERR_NOT_INITIALIZED, "la_init has not been called");
    if (count < 1) return fail(LA_ERR_INVALID_VALUE, "count must be >= 1");
    if (n <= 0 || m <= 0 || p <= 0) return fail(LA_ERR_INVALID_VALUE, "dimensions must be >= 1");
    if (n > (int64_t)1 << 31 || m > (int64_t)1 << 31 || p > (int64_t)1 << 31)
        return fail(LA_ERR_UNSUPPORTED, "dimension exceeds 2^31 (TMA coordinates are int32)");
    for (int64_t i = 0; i < count; i++)
        if (!hA[i] || !hB[i] || !hC[i]) return fail(LA_ERR_INVALID_VALUE, "NULL matrix pointer (product %lld)",
                                                    (long long)i);
    const size_t ab = (size_t)(n * m) * 4, bb = (size_t)(m * p) * 4, cb = (size_t)(n * p) * 4;
    const size_t slot_bytes = (ab + 255) / 256 * 256 + (bb + 255) / 256 * 256 + (cb + 255) / 256 * 256;
    const int slots = count > 1 ? 2 : 1;
    const size_t need = slots * slot_bytes;
    if (!g_state.h2d) {
        LA_CK(cudaStreamCreateWithFlags(&g_state.h2d, cudaStreamNonBlocking));
        LA_CK(cudaStreamCreateWithFlags(&g_state.d2h, cudaStreamNonBlocking));
    }
    while (g_state.slot_events.size() < 5) {
        cudaEvent_t e;
        LA_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        g_state.slot_events.push_back(e);
    }
    if (g_state.staging_bytes < need) {
        if (g_state.staging) {
            LA_CK(cudaDeviceSynchronize());
            LA_CK(cudaFree(g_state.staging));
            g_state.staging = nullptr;
            g_state.staging_bytes = 0;
        }
        cudaError_t e = cudaMalloc(&g_state.staging, need);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(LA_ERR_OUT_OF_MEMORY, "device staging of %zu bytes", need);
        }
        g_state.staging_bytes = need;
    }
    const int passes = g_state.mode == LA_MODE_TF32 ? 1 : 3;
    void *ws = nullptr;
    cudaError_t e = cudaMallocFromPoolAsync(&ws, operands_bytes(n, m, p, passes), g_state.pool, st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(LA_ERR_OUT_OF_MEMORY, "workspace");
    }
    // one operand workspace serves every product: their splits and GEMMs are
    // ordered on `st`
    const Operands ops = operands_carve(ws, n, m, p, passes);
    int launches = 0;
    HostTrace tr;
    tr.on = diag_knob("LA_HOST_TRACE", 0) != 0;
    cudaEvent_t ev_start = g_state.slot_events[0];
    cudaEvent_t *done_compute = &g_state.slot_events[1], *done_d2h = &g_state.slot_events[3];
    // the copy streams start after everything already queued on `st`
    LA_CK(cudaEventRecord(ev_start, st));
    LA_CK(cudaStreamWaitEvent(g_state.h2d, ev_start, 0));
    LA_CK(cudaStreamWaitEvent(g_state.d2h, ev_start, 0));
    tr.mark("start", g_state.h2d);
    la_status s = LA_OK;
    for (int64_t i = 0; i < count && s == LA_OK; i++) {
        const int sl = (int)(i % slots);
        char *base = static_cast<char *>(g_state.staging) + sl * slot_bytes;
        float *dA = reinterpret_cast<float *>(base);
        float *dB = reinterpret_cast<float *>(base + (ab + 255) / 256 * 256);
        float *dC = reinterpret_cast<float *>(base + (ab + 255) / 256 * 256 + (bb + 255) / 256 * 256);
        const bool reuse = i >= slots;
        s = host_item(n, m, p, hA[i], hB[i], hC[i], dA, dB, dC, ops, st, reuse ? done_compute[sl] : nullptr,
                      reuse ? done_d2h[sl] : nullptr, done_compute[sl], done_d2h[sl], &launches, tr);
    }
    cudaFreeAsync(ws, st);
    g_state.last_launches = launches;
    if (s != LA_OK) {
        cudaStreamSynchronize(g_state.h2d);
        cudaStreamSynchronize(g_state.d2h);
        return s;
    }
    LA_CK(cudaStreamSynchronize(g_state.d2h));
    LA_CK(cudaStreamSynchronize(st));
    tr.dump();
    return LA_OK;
}

}  // namespace la

extern "C" {

la_status la_gemm_host(int64_t n, int64_t m, int64_t p, const float *h_A, const float *h_B, float *h_C,
                       void *stream) {
    std::lock_guard<std::recursive_mutex> lk(g_mutex);
    return host_run(1, n, m, p, &h_A, &h_B, &h_C, static_cast<cudaStream_t>(stream));
}

la_status la_gemm_host_batch(int64_t count, int64_t n, int64_t m, int64_t p, const float *const *h_A,
                             const float *const *h_B, float *const *h_C, void *stream) {
    std::lock_guard<std::recursive_mutex> lk(g_mutex);
    if (!h_A || !h_B || !h_C) return fail(LA_ERR_INVALID_VALUE, "NULL pointer array");
    return host_run(count, n, m, p, h_A, h_B, h_C, static_cast<cudaStream_t>(stream));
}

// Complex single-precision product (Table 2 "Complex Float") through
// the real embedding [[Ar, -Ai], [Ai, Ar]] . [Br; Bi] = [Cr; Ci] (split.cuh),
// one persistent GEMM launch writing interleaved complex64 C.
la_status la_cgemm(int64_t n, int64_t m, int64_t p, const float *d_A, const float *d_B, float *d_C,
                   void *stream) {
    std::lock_guard<std::recursive_mutex> lk(g_mutex);
    if (!g_state.initialized) return fail(LA_ERR_NOT_INITIALIZED, "la_init has not been called");
    if (n <= 0 || m <= 0 || p <= 0) return fail(LA_ERR_INVALID_VALUE, "dimensions must be >= 1");
    if (2 * n > (int64_t)1 << 31 || 2 * m > (int64_t)1 << 31 || p > (int64_t)1 << 31)
        return fail(LA_ERR_UNSUPPORTED, "dimension exceeds the int32 TMA coordinate range");
    if (!d_A || !d_B || !d_C) return fail(LA_ERR_INVALID_VALUE, "NULL matrix pointer");
    if ((reinterpret_cast<uintptr_t>(d_A) | reinterpret_cast<uintptr_t>(d_B)) & 7)
        return fail(LA_ERR_INVALID_VALUE, "complex operands must be 8-byte aligned");
    auto overlap = [](const void *x, int64_t xb, const void *y, int64_t yb) {
        const char *a = (const char *)x, *b = (const char *)y;
        return a < b + yb && b < a + xb;
    };
    if (overlap(d_C, 8 * n * p, d_A, 8 * n * m) || overlap(d_C, 8 * n * p, d_B, 8 * m * p))
        return fail(LA_ERR_INVALID_VALUE, "C overlaps A or B");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int passes = g_state.mode == LA_MODE_TF32 ? 1 : 3;
    const int64_t n2 = 2 * n, m2 = 2 * m;
    void *ws = nullptr;
    cudaError_t e = cudaMallocFromPoolAsync(&ws, operands_bytes(n2, m2, p, passes), g_state.pool, st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(LA_ERR_OUT_OF_MEMORY, "workspace");
    }
    const Operands ops = operands_carve(ws, n2, m2, p, passes);
    int launches = 0;
    la_status s = LA_OK;
    {
        cudaEvent_t t0;
        if ((s = timing_begin(st, &t0)) != LA_OK) return s;
        const int64_t width = ops.mp - m;
        dim3 ga((unsigned)std::min<int64_t>((width + 255) / 256, 64), (unsigned)std::min<int64_t>(n, 65535));
        dim3 gb((unsigned)((p + 31) / 32), (unsigned)((width + 31) / 32));
        if (gb.y > 65535) return fail(LA_ERR_UNSUPPORTED, "m too large for the split grid");
        const float2 *a2 = reinterpret_cast<const float2 *>(d_A);
        const float2 *b2 = reinterpret_cast<const float2 *>(d_B);
        // even m and a 16-byte aligned A: the vectorised A split (pairs of elements)
        const bool avec = m % 2 == 0 && (reinterpret_cast<uintptr_t>(d_A) & 15) == 0;
        const int blocks_a = (int)std::max<int64_t>(1, std::min<int64_t>((n * (m / 2) + 255) / 256,
                                                                          (int64_t)g_state.sms * 8));
        const float4 *a4 = reinterpret_cast<const float4 *>(d_A);
        if (passes == 3) {
            if (avec) split_complex_a_vec_kernel<3><<<blocks_a, 256, 0, st>>>(a4, ops.a_hi, ops.a_lo, n, m, ops.mp);
            else split_complex_a_kernel<3><<<ga, 256, 0, st>>>(a2, ops.a_hi, ops.a_lo, n, m, ops.mp);
            split_complex_b_kernel<3><<<gb, dim3(32, 8), 0, st>>>(b2, ops.b_hi, ops.b_lo, m, p, ops.mp);
        } else {
            if (avec) split_complex_a_vec_kernel<1><<<blocks_a, 256, 0, st>>>(a4, ops.a_hi, ops.a_lo, n, m, ops.mp);
            else split_complex_a_kernel<1><<<ga, 256, 0, st>>>(a2, ops.a_hi, ops.a_lo, n, m, ops.mp);
            split_complex_b_kernel<1><<<gb, dim3(32, 8), 0, st>>>(b2, ops.b_hi, ops.b_lo, m, p, ops.mp);
        }
        launches += 2;
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "complex split launch", __FILE__, __LINE__);
        if ((s = timing_end(st, t0, TIMED_SPLIT)) != LA_OK) return s;
    }
    OutSpec out;
    out.cstride = 2;
    out.half_rows = n;
    out.half_off = 1;
    out.policy_k = m;
    s = gemm_run(n2, m2, 0, p, ops, d_C, 2 * p, (int)g_state.max_sms, st, &launches, out);
    e = cudaFreeAsync(ws, st);
    g_state.last_launches = launches;
    if (s == LA_OK && e != cudaSuccess) return cuda_fail(e, "cudaFreeAsync", __FILE__, __LINE__);
    return s;
}

// Double-precision product (Table 2 "Double" column) on the DMMA path.
la_status la_dgemm(int64_t n, int64_t m, int64_t p, const double *d_A, const double *d_B, double *d_C,
                   void *stream) {
    std::lock_guard<std::recursive_mutex> lk(g_mutex);
    if (!g_state.initialized) return fail(LA_ERR_NOT_INITIALIZED, "la_init has not been called");
    if (n <= 0 || m <= 0 || p <= 0) return fail(LA_ERR_INVALID_VALUE, "dimensions must be >= 1");
    if (!d_A || !d_B || !d_C) return fail(LA_ERR_INVALID_VALUE, "NULL matrix pointer");
    if ((reinterpret_cast<uintptr_t>(d_A) | reinterpret_cast<uintptr_t>(d_B) | reinterpret_cast<uintptr_t>(d_C)) & 7)
        return fail(LA_ERR_INVALID_VALUE, "double operands must be 8-byte aligned");
    auto overlap = [](const void *x, int64_t xb, const void *y, int64_t yb) {
        const char *a = (const char *)x, *b = (const char *)y;
        return a < b + yb && b < a + xb;
    };
    if (overlap(d_C, 8 * n * p, d_A, 8 * n * m) || overlap(d_C, 8 * n * p, d_B, 8 * m * p))
        return fail(LA_ERR_INVALID_VALUE, "C overlaps A or B");
    const int64_t gy = (n + DBM - 1) / DBM, gx = (p + DBN - 1) / DBN;
    if (gy > 65535 || gx > INT32_MAX) return fail(LA_ERR_UNSUPPORTED, "matrix too large for the DGEMM grid");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    static uint64_t attr_gen = 0;
    if (attr_gen != g_state.generation) {
        cudaError_t e = cudaFuncSetAttribute(dgemm_sm100_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             DSMEM_BYTES);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(dgemm_sm100_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     DSMEM_BYTES);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(dgemm)", __FILE__, __LINE__);
        attr_gen = g_state.generation;
    }
    const bool vec16 = m % 2 == 0 && p % 2 == 0 &&
                       ((reinterpret_cast<uintptr_t>(d_A) | reinterpret_cast<uintptr_t>(d_B)) & 15) == 0;
    // TMA path (int32 box coordinates); LA_DGEMM_CPASYNC=1 selects the cp.async kernel (A/B knob)
    const bool tma = vec16 && n < ((int64_t)1 << 31) && m < ((int64_t)1 << 31) && p < ((int64_t)1 << 31) &&
                     test_hook("LA_DGEMM_CPASYNC", 0) == 0;
    CUtensorMap tA, tB;
    if (tma) {
        static uint64_t attr_tma_gen = 0;
        if (attr_tma_gen != g_state.generation) {
            cudaError_t e = cudaFuncSetAttribute(dgemm_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 DT_SMEM_BYTES);
            if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(dgemm_tma)", __FILE__, __LINE__);
            attr_tma_gen = g_state.generation;
        }
        la_status ms;
        if ((ms = make_tmap_f64(&tA, d_A, n, m, DBM)) != LA_OK) return ms;
        if ((ms = make_tmap_f64(&tB, d_B, m, p, DBK)) != LA_OK) return ms;
    }
    cudaEvent_t t0;
    la_status s = timing_begin(st, &t0);
    if (s != LA_OK) return s;
    const dim3 grid((unsigned)gx, (unsigned)gy);
    if (tma) dgemm_tma_kernel<<<grid, DT_THREADS, DT_SMEM_BYTES, st>>>(tA, tB, d_C, n, m, p);
    else if (vec16) dgemm_sm100_kernel<true><<<grid, DTHREADS, DSMEM_BYTES, st>>>(d_A, d_B, d_C, n, m, p);
    else dgemm_sm100_kernel<false><<<grid, DTHREADS, DSMEM_BYTES, st>>>(d_A, d_B, d_C, n, m, p);
    g_state.last_launches = 1;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "dgemm launch", __FILE__, __LINE__);
    return timing_end(st, t0, TIMED_GEMM);
}

// Matrix addition / subtraction: C = A + B (subtract = 0) or A - B.
// C may be exactly A or B (in place) but must not partially overlap them.
la_status la_add(int64_t rows, int64_t cols, const float *d_A, const float *d_B, float *d_C, int subtract,
                 void *stream) {
    std::lock_guard<std::recursive_mutex> lk(g_mutex);
    if (!g_state.initialized) return fail(LA_ERR_NOT_INITIALIZED, "la_init has not been called");
    if (rows <= 0 || cols <= 0) return fail(LA_ERR_INVALID_VALUE, "dimensions must be >= 1");
    if (!d_A || !d_B || !d_C) return fail(LA_ERR_INVALID_VALUE, "NULL matrix pointer");
    const int64_t count = rows * cols, bytes = 4 * count;
    auto partial = [&](const void *x) {
        const char *a = (const char *)d_C, *b = (const char *)x;
        return a != b && a < b + bytes && b < a + bytes;
    };
    if (partial(d_A) || partial(d_B)) return fail(LA_ERR_INVALID_VALUE, "C partially overlaps A or B");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const bool vec = count % 4 == 0 &&
                     ((reinterpret_cast<uintptr_t>(d_A) | reinterpret_cast<uintptr_t>(d_B) |
                       reinterpret_cast<uintptr_t>(d_C)) & 15) == 0;
    const int64_t items = vec ? count / 4 : count;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, (int64_t)g_state.sms * 8));
    cudaEvent_t t0;
    la_status s = timing_begin(st, &t0);
    if (s != LA_OK) return s;
    if (vec) {
        const float4 *a = reinterpret_cast<const float4 *>(d_A), *b = reinterpret_cast<const float4 *>(d_B);
        float4 *c = reinterpret_cast<float4 *>(d_C);
        if (subtract) elementwise_vec4_kernel<true><<<blocks, 256, 0, st>>>(a, b, c, items);
        else elementwise_vec4_kernel<false><<<blocks, 256, 0, st>>>(a, b, c, items);
    } else {
        if (subtract) elementwise_kernel<true><<<blocks, 256, 0, st>>>(d_A, d_B, d_C, items);
        else elementwise_kernel<false><<<blocks, 256, 0, st>>>(d_A, d_B, d_C, items);
    }
    g_state.last_launches = 1;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "elementwise launch", __FILE__, __LINE__);
    return timing_end(st, t0, TIMED_SPLIT);
}

la_status la_shard_rows(int64_t n, int rank, int ngpu, int64_t *row0, int64_t *rows) {
    if (n < 0 || ngpu < 1 || rank < 0 || rank >= ngpu || !row0 || !rows)
        return fail(LA_ERR_INVALID_VALUE, "bad shard query n=%lld rank=%d ngpu=%d", (long long)n, rank, ngpu);
    const int64_t a = n * rank / ngpu, b = n * (rank + 1) / ngpu;
    *row0 = a;
    *rows = b - a;
    return LA_OK;
}

la_status la_finalize(void) {
    std::lock_guard<std::recursive_mutex> lk(g_mutex);
    if (!g_state.initialized) return LA_OK;
    cudaDeviceSynchronize();
    la_status s = comm_destroy();
    if (g_state.staging) cudaFree(g_state.staging);
    g_state.staging = nullptr;
    for (auto e : g_state.host_events) cudaEventDestroy(e);
    g_state.host_events.clear();
    for (auto e : g_state.slot_events) cudaEventDestroy(e);
    g_state.slot_events.clear();
    if (g_state.h2d) cudaStreamDestroy(g_state.h2d);
    if (g_state.d2h) cudaStreamDestroy(g_state.d2h);
    g_state.h2d = g_state.d2h = nullptr;
    g_state.staging_bytes = 0;
    if (g_state.pool) cudaMemPoolDestroy(g_state.pool);
    g_state.pool = nullptr;
    g_state.initialized = false;
    g_state.device = -1;
    return s;
}

const char *la_status_string(la_status s) {
    switch (s) {
        case LA_OK: return "LA_OK";
        case LA_ERR_INVALID_VALUE: return "LA_ERR_INVALID_VALUE";
        case LA_ERR_NOT_INITIALIZED: return "LA_ERR_NOT_INITIALIZED";
        case LA_ERR_UNSUPPORTED: return "LA_ERR_UNSUPPORTED";
        case LA_ERR_OUT_OF_MEMORY: return "LA_ERR_OUT_OF_MEMORY";
        case LA_ERR_CUDA: return "LA_ERR_CUDA";
        case LA_ERR_NCCL: return "LA_ERR_NCCL";
    }
    return "LA_ERR_UNKNOWN";
}

const char *la_last_error(void) { return g_last_error.c_str(); }

int la_last_launch_count(void) { return g_state.last_launches; }

la_status la_kernel_times(double *split_ms, double *gemm_ms, int *gemm_launches) {
    std::lock_guard<std::recursive_mutex> lk(g_mutex);
    if (!split_ms || !gemm_ms || !gemm_launches) return fail(LA_ERR_INVALID_VALUE, "NULL output pointer");
    double t[2] = {0.0, 0.0};
    int ng = 0;
    la_status s = LA_OK;
    for (auto &sp : g_spans) {
        float ms = 0.f;
        cudaError_t e = cudaEventSynchronize(sp.b);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, sp.a, sp.b);
        if (e != cudaSuccess && s == LA_OK) s = cuda_fail(e, "cudaEventElapsedTime", __FILE__, __LINE__);
        t[sp.kind] += ms;
        ng += sp.kind == TIMED_GEMM;
        g_free_ev.push_back(sp.a);
        g_free_ev.push_back(sp.b);
    }
    g_spans.clear();
    *split_ms = t[0];
    *gemm_ms = t[1];
    *gemm_launches = ng;
    return s;
}

}  // extern "C"
