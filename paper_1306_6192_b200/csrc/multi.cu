// multi.cu -- the multi-GPU partition.
//
// One process per GPU.  Rank r owns rows [r*n/g, (r+1)*n/g) of A and C.  B is
// replicated with ncclBroadcast from `root` in N-panels (column blocks of B,
// packed contiguously) on a library-owned communication stream; the caller's
// stream waits for panel c, splits it and runs the GEMM on
// A_r . B[:, panel c] while panels c+1.. are still in flight.  There is no K
// split, so no reduction: C row blocks are complete where they are computed and
// are optionally all-gathered (ncclAllGather) into the full n x p matrix.
// Every output element accumulates in exactly the order la_gemm uses, so the
// multi-GPU C is bitwise identical to the single-GPU C.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "gemm_sm100.cuh"
#include "la.h"
#include "la_internal.h"

namespace la {

struct Comm {
    ncclComm_t comm = nullptr;
    int rank = -1, size = 0;
    cudaStream_t stream = nullptr;  // communication stream
    cudaEvent_t start = nullptr;
    std::vector<cudaEvent_t> panel_ready;
    void *bstage = nullptr;  // packed B panels (m x p floats), every rank
    size_t bstage_bytes = 0;
    // fused all-gather target: symmetric memory registered as an NCCL window
    void *gather = nullptr;
    size_t gather_bytes = 0;
    ncclWindow_t gather_win = nullptr;
    int lsa_size = 0;
    int *barrier_buf = nullptr;  // 1 int for the post-GEMM cross-rank barrier
};
static Comm g_comm;

static la_status nccl_fail(ncclResult_t r, const char *what) {
    return fail(LA_ERR_NCCL, "%s failed: %s", what, ncclGetErrorString(r));
}

#define LA_NCCL(call)                                      \
    do {                                                   \
        ncclResult_t r_ = (call);                          \
        if (r_ != ncclSuccess) return nccl_fail(r_, #call); \
    } while (0)
#define LA_CK(call)                                                             \
    do {                                                                        \
        cudaError_t e_ = (call);                                                \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call, __FILE__, __LINE__); \
    } while (0)

static la_status gather_release() {
    la_status s = LA_OK;
    if (g_comm.gather_win) {
        ncclResult_t r = ncclCommWindowDeregister(g_comm.comm, g_comm.gather_win);
        if (r != ncclSuccess) s = nccl_fail(r, "ncclCommWindowDeregister");
    }
    if (g_comm.gather) {
        ncclResult_t r = ncclMemFree(g_comm.gather);
        if (r != ncclSuccess && s == LA_OK) s = nccl_fail(r, "ncclMemFree");
    }
    g_comm.gather = nullptr;
    g_comm.gather_win = nullptr;
    g_comm.gather_bytes = 0;
    return s;
}

la_status comm_destroy() {
    la_status s = LA_OK;
    if (g_comm.comm) gather_release();
    if (g_comm.barrier_buf) cudaFree(g_comm.barrier_buf);
    if (g_comm.comm) {
        ncclResult_t r = ncclCommDestroy(g_comm.comm);
        if (r != ncclSuccess) s = nccl_fail(r, "ncclCommDestroy");
    }
    for (auto e : g_comm.panel_ready) cudaEventDestroy(e);
    if (g_comm.start) cudaEventDestroy(g_comm.start);
    if (g_comm.stream) cudaStreamDestroy(g_comm.stream);
    if (g_comm.bstage) cudaFree(g_comm.bstage);
    g_comm = Comm();
    return s;
}

// SMs left free for NCCL's kernels while broadcasts are in flight
// (LA_OPT_NCCL_SMS, default 8; read by la_comm_init for ncclConfig_t.maxCTAs).
static int reserved_sms() { return (int)std::max<int64_t>(0, g_state.nccl_sms); }

// ---- panel plan (la_panel_plan) -------------------------------------------
// B travels in column panels; panel c's GEMM starts when panel c has arrived
// and panel c-1's GEMM is done.  A timeline model scores candidate plans:
//   broadcast  4 m w / link + 25 us per call (+ the root's pack copy),
//   split      12 m w bytes of HBM traffic per panel (replicated on every rank),
//   GEMM       waves x one 256 x 256 tile's time, waves counted on the clusters
//              the launch gets (SMs - reserved for all but the last panel), with
//              the half-width tail items of launch_gemm (a last wave at most
//              half full costs half a wave).
// Rates: tile time from the measured single-GPU kernel (793 TFLOP/s issued
// over 74 clusters, 3xTF32), link 700 GB/s (B200_PROFILING: 770 GB/s peer copy),
// HBM 6 TB/s.  Candidates: 1, 2, 4, 8, 16 equal panels and geometric plans
// (first panel 256 .. 2048 columns, each next one 2x or 3x wider) -- a narrow
// first panel shortens the broadcast nothing can overlap.  Widths are
// multiples of 256 (the CTA pair's N tile) except the last.
namespace {
struct PlanModel {
    double rows, m, t_tile, link, hbm;
    int clusters_all, clusters_capped;
    double waves(double tiles, int W) const {
        const double full = std::floor(tiles / W), r = tiles - full * W;
        if (r <= 0) return full;
        return full + ((2 * r <= W && tiles > W) ? 0.5 : 1.0);
    }
    double time(const std::vector<int64_t> &ws) const {
        double comm = 0, comp = 12.0 * rows * m / hbm;  // split of A_r
        for (size_t c = 0; c < ws.size(); c++) {
            const double w = (double)ws[c];
            comm += 4.0 * m * w / link + 25e-6 + 8.0 * m * w / (3 * hbm);
            const double tiles = std::ceil(rows / 256.0) * std::ceil(w / 256.0);
            const int W = c + 1 < ws.size() ? clusters_capped : clusters_all;
            comp = std::max(comp, comm) + 12.0 * m * w / hbm + 5e-6 + waves(tiles, W) * t_tile;
        }
        return comp;
    }
};
std::vector<int64_t> equal_plan(int64_t p, int64_t P) {
    int64_t w = (p + P - 1) / P;
    w = (w + 255) / 256 * 256;
    std::vector<int64_t> ws;
    for (int64_t j = 0; j < p; j += w) ws.push_back(std::min(w, p - j));
    return ws;
}
std::vector<int64_t> geometric_plan(int64_t p, int64_t first, int64_t grow) {
    std::vector<int64_t> ws;
    int64_t j = 0, w = first;
    while (j < p) {
        int64_t ww = std::min(w, p - j);
        if (p - j - ww < first) ww = p - j;  // no sliver at the end
        ws.push_back(ww);
        j += ww;
        w = (w * grow + 255) / 256 * 256;
    }
    return ws;
}
}  // namespace

}  // namespace la

using namespace la;

extern "C" {

la_status la_get_unique_id(void *out128) {
    std::lock_guard<std::recursive_mutex> lk(g_mutex);
    if (!out128) return fail(LA_ERR_INVALID_VALUE, "NULL unique-id buffer");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    LA_NCCL(ncclGetUniqueId(&id));
    memcpy(out128, &id, sizeof id);
    return LA_OK;
}

la_status la_comm_init(const void *uid128, int rank, int ngpu) {
    std::lock_guard<std::recursive_mutex> lk(g_mutex);
    if (!g_state.initialized) return fail(LA_ERR_NOT_INITIALIZED, "la_init has not been called");
    if (!uid128 || ngpu < 1 || rank < 0 || rank >= ngpu)
        return fail(LA_ERR_INVALID_VALUE, "bad communicator arguments rank=%d ngpu=%d", rank, ngpu);
    if (g_comm.comm) {
        la_status s = comm_destroy();
        if (s != LA_OK) return s;
    }
    ncclUniqueId id;
    memcpy(&id, uid128, sizeof id);
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 1;
    // NCCL's kernels must fit in the SMs the GEMM leaves free while panels are
    // in flight (la_gemm_multi launches the GEMM on sms - reserved SMs).
    cfg.maxCTAs = reserved_sms() > 0 ? reserved_sms() : 8;
    cfg.minCTAs = 1;
    ncclResult_t r = ncclCommInitRankConfig(&g_comm.comm, ngpu, id, rank, &cfg);
    if (r == ncclInvalidArgument) {  // an NCCL that rejects the CTA bounds: default config
        ncclConfig_t dflt = NCCL_CONFIG_INITIALIZER;
        dflt.blocking = 1;
        r = ncclCommInitRankConfig(&g_comm.comm, ngpu, id, rank, &dflt);
    }
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRankConfig");
    g_comm.rank = rank;
    g_comm.size = ngpu;
    LA_CK(cudaStreamCreateWithFlags(&g_comm.stream, cudaStreamNonBlocking));
    LA_CK(cudaEventCreateWithFlags(&g_comm.start, cudaEventDisableTiming));
    return LA_OK;
}

la_status la_comm_size(int *nranks, int *rank) {
    std::lock_guard<std::recursive_mutex> lk(g_mutex);
    if (!nranks || !rank) return fail(LA_ERR_INVALID_VALUE, "NULL output pointer");
    if (!g_comm.comm) return fail(LA_ERR_NOT_INITIALIZED, "la_comm_init has not been called");
    LA_NCCL(ncclCommCount(g_comm.comm, nranks));
    LA_NCCL(ncclCommUserRank(g_comm.comm, rank));
    return LA_OK;
}

la_status la_panel_plan(int64_t n, int64_t m, int64_t p, int ngpu, int sms, int reserved, int64_t panels,
                        int64_t *widths, int max_panels, int *count) {
    if (n <= 0 || m <= 0 || p <= 0 || ngpu < 1 || sms < 2 || reserved < 0 || panels < 0 || !widths || !count ||
        max_panels < 1)
        return fail(LA_ERR_INVALID_VALUE, "bad panel-plan arguments");
    std::vector<int64_t> best;
    if (panels > 0) {
        best = equal_plan(p, panels);
    } else if (ngpu == 1) {
        best = {p};  // nothing to overlap: one panel
    } else {
        PlanModel pm;
        pm.rows = (double)((n + ngpu - 1) / ngpu);
        pm.m = (double)m;
        pm.clusters_all = std::max(1, sms / 2);
        pm.clusters_capped = std::max(1, (sms - reserved) / 2);
        pm.t_tile = 6.0 * 256.0 * 256.0 * (double)m / (793e12 / 74.0);
        pm.link = 700e9;
        pm.hbm = 6e12;
        double bt = 0;
        auto consider = [&](const std::vector<int64_t> &ws) {
            if ((int)ws.size() > max_panels) return;
            const double t = pm.time(ws);
            if (best.empty() || t < bt) {
                best = ws;
                bt = t;
            }
        };
        for (int64_t P : {1, 2, 4, 8, 16}) consider(equal_plan(p, P));
        for (int64_t first : {256, 512, 1024, 2048})
            for (int64_t grow : {2, 3})
                if (first < p) consider(geometric_plan(p, first, grow));
    }
    if ((int)best.size() > max_panels)
        return fail(LA_ERR_INVALID_VALUE, "%zu panels exceed the caller's %d", best.size(), max_panels);
    for (size_t c = 0; c < best.size(); c++) widths[c] = best[c];
    *count = (int)best.size();
    return LA_OK;
}

la_status la_gather_alloc(int64_t bytes, void **d_out) {
    std::lock_guard<std::recursive_mutex> lk(g_mutex);
    if (!g_state.initialized) return fail(LA_ERR_NOT_INITIALIZED, "la_init has not been called");
    if (!g_comm.comm) return fail(LA_ERR_NOT_INITIALIZED, "la_comm_init has not been called");
    if (bytes <= 0 || !d_out) return fail(LA_ERR_INVALID_VALUE, "bad gather buffer request");
    la_status s = gather_release();
    if (s != LA_OK) return s;
    const size_t sz = ((size_t)bytes + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT *
                      NCCL_WIN_REQUIRED_ALIGNMENT;
    LA_NCCL(ncclMemAlloc(&g_comm.gather, sz));
    ncclResult_t r = ncclCommWindowRegister(g_comm.comm, g_comm.gather, sz, &g_comm.gather_win,
                                            NCCL_WIN_COLL_SYMMETRIC);
    if (r != ncclSuccess) {
        ncclMemFree(g_comm.gather);
        g_comm.gather = nullptr;
        g_comm.gather_win = nullptr;
        return nccl_fail(r, "ncclCommWindowRegister");
    }
    g_comm.gather_bytes = sz;
    g_comm.lsa_size = ncclTeamLsa(g_comm.comm).nRanks;
    if (!g_comm.barrier_buf) {
        LA_CK(cudaMalloc(&g_comm.barrier_buf, sizeof(int)));
        LA_CK(cudaMemset(g_comm.barrier_buf, 0, sizeof(int)));
    }
    *d_out = g_comm.gather;
    return LA_OK;
}

la_status la_gemm_multi(int64_t n, int64_t m, int64_t p, const float *d_A_local, const float *d_B,
                        float *d_C_local, float *d_C_full, int root, int ngpu, void *stream) {
    std::lock_guard<std::recursive_mutex> lk(g_mutex);
    if (!g_state.initialized) return fail(LA_ERR_NOT_INITIALIZED, "la_init has not been called");
    if (!g_comm.comm) return fail(LA_ERR_NOT_INITIALIZED, "la_comm_init has not been called");
    if (ngpu != g_comm.size)
        return fail(LA_ERR_INVALID_VALUE, "ngpu=%d but the communicator has %d ranks", ngpu, g_comm.size);
    if (root < 0 || root >= ngpu) return fail(LA_ERR_INVALID_VALUE, "root %d out of range", root);
    if (n <= 0 || m <= 0 || p <= 0) return fail(LA_ERR_INVALID_VALUE, "dimensions must be >= 1");
    if (n < ngpu) return fail(LA_ERR_UNSUPPORTED, "n=%lld < ngpu=%d leaves a rank without rows", (long long)n, ngpu);
    if (d_C_full && n % ngpu != 0)
        return fail(LA_ERR_UNSUPPORTED, "all-gather of C needs n %% ngpu == 0 (n=%lld, ngpu=%d)", (long long)n, ngpu);
    const int rank = g_comm.rank;
    if (rank == root && !d_B) return fail(LA_ERR_INVALID_VALUE, "B is NULL on the root rank");
    if (!d_A_local || !d_C_local) return fail(LA_ERR_INVALID_VALUE, "NULL A_local or C_local");
    int64_t row0 = 0, rows = 0;
    la_shard_rows(n, rank, ngpu, &row0, &rows);
    cudaStream_t st = static_cast<cudaStream_t>(stream);

    // N-panels (la_panel_plan): LA_OPT_PANELS = 0 (default) lets the timeline
    // model choose, > 0 forces that many equal panels.
    std::vector<int64_t> widths(64);
    int P32 = 0;
    {
        // test hook (one rank): plan the panels as for LA_TEST_PLAN_NGPU ranks
        const int plan_g = ngpu == 1 ? (int)std::max<int64_t>(1, test_hook("LA_TEST_PLAN_NGPU", 1)) : ngpu;
        la_status ps = la_panel_plan(n, m, p, plan_g, g_state.sms, reserved_sms(), g_state.panels, widths.data(),
                                     (int)widths.size(), &P32);
        if (ps != LA_OK) return ps;
    }
    const int64_t P = P32;
    std::vector<int64_t> col0(P + 1, 0);
    for (int64_t c = 0; c < P; c++) col0[c + 1] = col0[c] + widths[c];
    while ((int64_t)g_comm.panel_ready.size() < P) {
        cudaEvent_t e;
        LA_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        g_comm.panel_ready.push_back(e);
    }
    const size_t bbytes = (size_t)(m * p) * sizeof(float);
    if (g_comm.bstage_bytes < bbytes) {
        LA_CK(cudaDeviceSynchronize());
        if (g_comm.bstage) LA_CK(cudaFree(g_comm.bstage));
        g_comm.bstage = nullptr;
        g_comm.bstage_bytes = 0;
        cudaError_t e = cudaMalloc(&g_comm.bstage, bbytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(LA_ERR_OUT_OF_MEMORY, "B staging of %zu bytes", bbytes);
        }
        g_comm.bstage_bytes = bbytes;
    }
    float *bstage = static_cast<float *>(g_comm.bstage);

    const int passes = g_state.mode == LA_MODE_TF32 ? 1 : 3;
    const size_t wbytes = operands_bytes(rows, m, p, passes);
    void *ws = nullptr;
    cudaError_t e = cudaMallocFromPoolAsync(&ws, wbytes, g_state.pool, st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(LA_ERR_OUT_OF_MEMORY, "workspace of %zu bytes", wbytes);
    }
    const Operands ops = operands_carve(ws, rows, m, p, passes);
    int launches = 0;

    // Fused all-gather: C_full is the registered symmetric window and every
    // rank is load/store reachable (one NVLink domain) -> the epilogue writes
    // this rank's rows into every rank's C_full while the GEMM runs, instead of
    // a separate ncclAllGather afterwards.
    OutSpec out;
    const bool fused = d_C_full != nullptr && d_C_full == g_comm.gather && g_comm.gather_win != nullptr &&
                       g_comm.lsa_size == ngpu && ngpu <= MAX_GATHER_PEERS &&
                       (size_t)(n * p) * sizeof(float) <= g_comm.gather_bytes;
    if (fused) {
        out.gather_win = g_comm.gather_win;
        out.gather_peers = g_comm.lsa_size;
        out.gather_row0 = row0;
        out.gather_ld = p;
        // test hooks (one rank): a non-zero destination row, and g emulated
        // peers whose C_full copies sit at offsets 0, s, 2s.. of this window
        const int64_t hook_row0 = ngpu == 1 ? test_hook("LA_TEST_GATHER_ROW0", -1) : -1;
        const int64_t hook_peers = ngpu == 1 ? test_hook("LA_TEST_GATHER_PEERS", 1) : 1;
        const int64_t hook_stride = ngpu == 1 ? test_hook("LA_TEST_GATHER_STRIDE", 0) : 0;
        if (hook_row0 >= 0) out.gather_row0 = hook_row0;
        if (hook_peers > 1) {
            if (hook_peers > MAX_GATHER_PEERS || hook_stride < (out.gather_row0 + rows) * p)
                return fail(LA_ERR_INVALID_VALUE, "bad LA_TEST_GATHER_PEERS / LA_TEST_GATHER_STRIDE");
            out.gather_peers = (int)hook_peers;
            out.gather_emul_stride = hook_stride;
        }
        const int64_t span = (out.gather_peers - 1) * out.gather_emul_stride + (out.gather_row0 + rows) * p;
        if ((size_t)span * sizeof(float) > g_comm.gather_bytes)
            return fail(LA_ERR_INVALID_VALUE, "fused gather test hooks reach past the gather buffer");
    }
    // comm stream starts after everything already queued on the caller's stream
    LA_CK(cudaEventRecord(g_comm.start, st));
    LA_CK(cudaStreamWaitEvent(g_comm.stream, g_comm.start, 0));
    if (fused && ngpu > 1) {
        // Write-after-read guard for the fused gather: this call's epilogues store
        // into every rank's C_full, which a rank may still be reading from the
        // previous call (work queued on its `stream` before this call).  A 1-int
        // all-reduce on the comm stream, which starts only after that work,
        // holds every rank's broadcasts -- and so every GEMM, which waits for
        // panel 0 -- until all ranks have reached this call.
        LA_NCCL(ncclAllReduce(g_comm.barrier_buf, g_comm.barrier_buf, 1, ncclInt, ncclSum, g_comm.comm,
                              g_comm.stream));
    }
    for (int64_t c = 0; c < P; c++) {
        const int64_t j0 = col0[c], w = widths[c];
        float *panel = bstage + m * j0;  // packed m x w panel
        if (rank == root) {
            if (P == 1) {
                LA_NCCL(ncclBroadcast(d_B, panel, (size_t)(m * w), ncclFloat, root, g_comm.comm, g_comm.stream));
            } else {
                LA_CK(cudaMemcpy2DAsync(panel, w * sizeof(float), d_B + j0, p * sizeof(float), w * sizeof(float),
                                        m, cudaMemcpyDeviceToDevice, g_comm.stream));
                LA_NCCL(ncclBroadcast(panel, panel, (size_t)(m * w), ncclFloat, root, g_comm.comm, g_comm.stream));
            }
        } else {
            LA_NCCL(ncclBroadcast(nullptr, panel, (size_t)(m * w), ncclFloat, root, g_comm.comm, g_comm.stream));
        }
        LA_CK(cudaEventRecord(g_comm.panel_ready[c], g_comm.stream));
    }

    la_status s = split_a(rows, m, d_A_local, ops, st, &launches);
    const int reserve = ngpu > 1 ? reserved_sms() : 0;
    for (int64_t c = 0; c < P && s == LA_OK; c++) {
        const int64_t j0 = col0[c], w = widths[c];
        LA_CK(cudaStreamWaitEvent(st, g_comm.panel_ready[c], 0));
        s = split_b(m, j0, w, bstage + m * j0, w, ops, st, &launches);
        if (s != LA_OK) break;
        const int max_sms = (c < P - 1 && reserve > 0) ? std::max(1, g_state.sms - reserve) : (int)g_state.max_sms;
        s = gemm_run(rows, m, j0, w, ops, d_C_local, p, max_sms, st, &launches, out);
    }
    e = cudaFreeAsync(ws, st);
    if (s != LA_OK) return s;
    if (e != cudaSuccess) return cuda_fail(e, "cudaFreeAsync", __FILE__, __LINE__);
    if (fused) {
        // cross-rank barrier: every rank's GEMM (and its fenced peer stores) is
        // complete before any rank's stream moves past this point
        LA_NCCL(ncclAllReduce(g_comm.barrier_buf, g_comm.barrier_buf, 1, ncclInt, ncclSum, g_comm.comm, st));
    } else if (d_C_full) {
        LA_NCCL(ncclAllGather(d_C_local, d_C_full, (size_t)(rows * p), ncclFloat, g_comm.comm, st));
    }
    g_state.last_launches = launches;
    return LA_OK;
}

}  // extern "C"
