// gemm_sm100.cuh -- K2: persistent warp-specialised tcgen05 GEMM, C = A . B.
//
// The paper's optimised kernel (Listing 4) stages a 16x16
// tile of A and of B in shared memory per K step, synchronises
// (P:178), does 16 FMAs per thread, synchronises again and
// writes one C element per thread.  The same structure, re-built
// for sm_100a:
//   * staging      : TMA (cp.async.bulk.tensor) fills a STAGES-deep ring of
//                    128B-swizzled K-major tiles; mbarrier full[s] replaces the
//                    first __syncthreads;
//   * inner product: the MMA warp, converged, with one lane elected inside each
//                    asm statement and every descriptor on the uniform
//                    datapath, issues tcgen05.mma.kind::tf32 into a TMEM
//                    accumulator (3 passes hi.lo', lo.hi', hi.hi' per K=8 step
//                    for 3xTF32); tcgen05.commit -> empty[s] replaces the
//                    second __syncthreads;
//   * write-back   : epilogue warps tcgen05.ld the accumulator and store C
//                    exactly once per element: 32x32 pieces laid out
//                    in swizzled smem and written by TMA bulk tensor stores
//                    (ragged edges clipped by the hardware), or per-thread
//                    coalesced stores for non-plain layouts (complex interleave,
//                    fused gather); 64-bit offsets.
// Accumulator promotion: the tcgen05 tf32 path sums each K=8 group exactly and
// then TRUNCATES into the fp32 accumulator (measured, tests/test_probe.py), a
// bias that grows with the number of MMAs per accumulator (3.1 x 2^-20 S at
// K=16384).  So the MMA warp accumulates `kc` K-blocks per TMEM chunk and the
// epilogue adds every chunk into an fp32 round-to-nearest register running
// sum (0.06 x 2^-20 S at chunks of 256 on random signs; the host picks 32 /
// 64 / 128 by K, because one long chunk's truncations do not average out).
// Two TMEM accumulator buffers let the epilogue of chunk c overlap the MMAs of
// c+1.  Same-sign sums would still drift toward zero chunk by chunk, so chunks
// are sign-centred (ChunkPlan; the epilogue preloads an offset of the other
// sign into the buffer of chunk c+2).
//
// CG == 1: one CTA computes a 128 x BN tile (UMMA M=128).
// CG == 2: a cluster of two CTAs (a CTA pair on one TPC) computes a 256 x BN
//          tile with tcgen05.mma.cta_group::2 (UMMA M=256): each CTA stages its
//          128 rows of A and BN/2 rows of B^T, the leader CTA issues the MMAs,
//          and each CTA's TMEM holds its 128 rows of the accumulator.  Operand
//          traffic per FLOP is half that of CG == 1 at the same BN.
// Persistent: one CTA (pair) per SM (pair), tiles in grouped raster order.
#pragma once
#include <cstdint>

#include <nccl.h>
#include <nccl_device.h>

#include "ptx.cuh"

namespace la {

constexpr int BK = 32;            // default K per stage: 32 fp32 = one 128-byte swizzle row
                                  // (KB = 16: 64-byte rows, SWIZZLE_64B, twice the stages)
constexpr int ROWS_PER_CTA = 128; // UMMA M per CTA
constexpr int NUM_CTRL_WARPS = 4; // warp0 TMA, warp1 MMA, warp2 TMEM alloc, warp3 idle
constexpr int NUM_EPI_WARPS = 8;  // two per TMEM lane quarter (column halves)
constexpr int NUM_THREADS = 32 * (NUM_CTRL_WARPS + NUM_EPI_WARPS);
// setmaxnreg budgets.  A CTA's register pool is what it was launched with:
// __launch_bounds__(384, 1) gives 168 registers x 384 threads = 64512; the
// control warpgroup shrinks to CTRL_REGS and the two epilogue warpgroups grow
// to EPI_REGS, and the sum must stay inside that pool or setmaxnreg.inc
// blocks forever.  (ptxas still allocates every region within the launch
// bound's 168, so the promotion loop's 128 running sums + two 32-column loads
// spill a few registers.)
constexpr int LAUNCH_REGS = 168;
constexpr int CTRL_REGS = 56;
constexpr int EPI_REGS = 216;
constexpr bool SIGN_CENTRE = true;  // sign-centred promotion chunks (epilogue, below)
static_assert(32 * NUM_CTRL_WARPS * CTRL_REGS + 32 * NUM_EPI_WARPS * EPI_REGS <= NUM_THREADS * LAUNCH_REGS,
              "setmaxnreg budget exceeds the CTA's register pool");

struct GemmArgs {
    float *C;
    int64_t n, p, ldc;  // C is n x p with row stride ldc
    // Output addressing: element (r, c) of the n x p product goes to
    //   C + r * ldc + c * cstride                      (r <  half_rows or half_rows == 0)
    //   C + (r - half_rows) * ldc + half_off + c * cstride   (r >= half_rows)
    // Real products use cstride 1, half_rows 0.  The complex embedding writes
    // [Cr; Ci] into interleaved complex64 C: ldc = 2p, cstride 2, half_rows = n,
    // half_off = 1.
    int64_t cstride, half_rows, half_off;
    int32_t num_kb;     // K-blocks of BK
    int32_t kc;         // K-blocks per TMEM chunk (promotion interval); >= num_kb: no promotion
    int32_t center_kb;  // sign-centred chunks only end at or before this K-block; 0: off (ChunkPlan)
    int32_t tiles_m, tiles_n, group_m;
    // Work items: items [0, full_items) are whole tiles in raster order; the
    // remaining tiles (the last, partial wave) are split into two half-width
    // (BN/2 column) items each, so the tail wave takes half a tile time.
    int32_t full_items, num_items;
    // Split-K (few output tiles, long K): item w is K range w % ksplit of tile
    // w / ksplit, K-blocks [s * kb_per, min(num_kb, (s + 1) * kb_per)); its
    // promoted partial tile goes to partial + s * n * ldc (same layout as C),
    // and a reduction kernel sums the ksplit partials in order.  ksplit == 1: off.
    int32_t ksplit, kb_per;
    float *partial;
    int32_t *wave_sync; // optional: arrival counters (zeroed per launch), one per
                        // (wave, K phase of sync_kb K-blocks)
    int32_t sync_kb;    // K-blocks between arrival barriers (>= num_kb: once per tile)
    int32_t wave_slots; // counters in wave_sync; wave_sync[wave_slots] is the give-up flag
    int32_t debug;      // diagnostics only (results are garbage): 1 = skip TMA loads, 2 = skip MMAs
    int64_t *trace;     // diagnostics only: per-CTA globaltimer stamps + MMA wait cycles (TRACE_SLOTS), or nullptr
    // 1: plain row-major output (cstride 1, no half rows, no gather) stored by
    // TMA through the kernel's tm_c map {p, n, ksplit} (C, or the split-K
    // partial slices); 0: per-thread stores (store_piece)
    int32_t tma_store;
    // Fused all-gather (la_gemm_multi into a registered symmetric C_full): every
    // output element (r, c) is also stored at row gather_row0 + r, column
    // gather_col0 + c (row stride gather_ld) of each LSA peer's window, i.e.
    // straight into every rank's C_full over NVLink, while the GEMM runs.
    const void *gather_win;  // ncclWindow_t (device-resident struct) or nullptr
    int32_t gather_peers;    // LSA team size (<= MAX_GATHER_PEERS)
    int64_t gather_row0, gather_col0, gather_ld;
    // test hook (one rank emulating gather_peers ranks): 0, or the float
    // offset between the emulated peers' C_full copies inside this rank's own
    // window (peer pe's copy at pe * gather_emul_stride)
    int64_t gather_emul_stride;
};

constexpr int MAX_GATHER_PEERS = 8;  // one NVLink / NVSwitch domain of 8 GPUs

// Split-K reduction: C = ((P_0 + P_1) + P_2) + ... elementwise, in split order
// (deterministic).  HBM-bound, 4 (ksplit + 1) bytes per element.
static __global__ void __launch_bounds__(256) splitk_reduce_kernel(const float *__restrict__ part, float *__restrict__ C,
                                                            int64_t count, int ksplit) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // launched early (PDL): the GEMM's partials first
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        float acc = part[i];
        for (int s = 1; s < ksplit; s++) acc += part[(int64_t)s * count + i];
        C[i] = acc;
    }
}

constexpr int TRACE_SLOTS = 10;  // 8 timestamps + the MMA warp's wait cycles (tempty, full)
__device__ __forceinline__ void trace_stamp(int64_t *trace, int k) {
    if (trace == nullptr) return;
    int64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    trace[blockIdx.x * TRACE_SLOTS + k] = t;
}

// Same, four elements per thread (count % 4 == 0, 16-byte aligned buffers).
static __global__ void __launch_bounds__(256) splitk_reduce_vec4_kernel(const float4 *__restrict__ part,
                                                                 float4 *__restrict__ C, int64_t count4,
                                                                 int ksplit) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count4;
         i += (int64_t)gridDim.x * blockDim.x) {
        float4 acc = __ldcs(part + i);
        for (int s = 1; s < ksplit; s++) {
            const float4 v = __ldcs(part + (int64_t)s * count4 + i);
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
        C[i] = acc;
    }
}

// Optional K-phase alignment of the static persistent schedule: at every K
// phase of sync_kb K-blocks each producer of a wave arrives on that (wave,
// phase) counter and waits (bounded, 200 us) until all producers of the wave
// have arrived, so the clusters that share A rows / B columns stream through K
// together and reuse each other's slabs in L2 instead of re-reading them from
// HBM.
__device__ __forceinline__ void wave_barrier(int32_t *ctr, int target, int32_t *give_up) {
    atomicAdd(ctr, 1);
    // a wave that cannot be co-resident (other kernels hold SMs) would pay the
    // full timeout at every phase: after the first timeout every producer of
    // this launch stops waiting
    if (*reinterpret_cast<volatile int32_t *>(give_up)) return;
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        int v;
        asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        if (v >= target) break;
        uint64_t t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t0 > 200000) {
            atomicExch(give_up, 1);
            break;
        }
        __nanosleep(128);
    }
}

template <int CG, int BN, int STAGES, int PASSES, int KB = BK>
struct GemmCfg {
    static constexpr int TILE_M = CG * ROWS_PER_CTA;        // rows of C per tile
    static constexpr int B_ROWS = BN / CG;                  // rows of B^T staged per CTA
    static constexpr int NOPS = PASSES == 3 ? 2 : 1;        // hi (+ lo) tiles per operand
    static constexpr int A_TILE = ROWS_PER_CTA * KB * 4;    // 16 KB at KB = 32
    static constexpr int B_TILE = B_ROWS * KB * 4;
    // A stage of KB = 64 holds two 128-byte swizzle atoms (K 0-31, 32-63) per
    // operand, each loaded by its own TMA box; KB <= 32 is one atom.
    static constexpr int ATOM_K = KB < 32 ? KB : 32;
    static constexpr int ATOMS = KB / ATOM_K;
    static constexpr int A_ATOM = ROWS_PER_CTA * ATOM_K * 4;
    static constexpr int B_ATOM = B_ROWS * ATOM_K * 4;
    static constexpr int STAGE_BYTES = NOPS * (A_TILE + B_TILE);  // per CTA
    static constexpr int EPI_BYTES = NUM_EPI_WARPS * 32 * 32 * 4; // per-warp transpose buffers
    static constexpr int BAR_BYTES = 512;  // mbarriers, TMEM address, tile ids; gather peer bases at +320
    static constexpr int SMEM_BYTES = 1024 /*align slack*/ + STAGES * STAGE_BYTES + EPI_BYTES + BAR_BYTES;
    static constexpr uint32_t TMEM_COLS = 2 * BN;  // two accumulator buffers
    static constexpr int COLS_PER_WARP = BN / 2;   // epilogue column half
    static constexpr int PIECES = COLS_PER_WARP / 32;
    static_assert(CG == 1 || CG == 2, "cta_group");
    static_assert(BN % 64 == 0 && BN <= 256, "UMMA N: multiple of 16 (32 per epilogue piece), <= 256");
    static_assert(TMEM_COLS == 128 || TMEM_COLS == 256 || TMEM_COLS == 512, "TMEM alloc is a power of 2");
    static_assert(SMEM_BYTES <= 232448, "exceeds 227 KB of shared memory per CTA");
};

__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int group, int &tm, int &tn) {
    const int per_group = group * tiles_n;
    const int g = t / per_group;
    const int first = g * group;
    const int gsz = min(group, tiles_m - first);
    const int r = t - g * per_group;
    tm = first + r % gsz;
    tn = r / gsz;
}

// Promotion chunks of one work item (nkb K-blocks, interval kc).  Without
// promotion (kc >= nkb) one chunk.  With sign-centring (kc >= 2) the first two
// chunks are f = kc/2 K-blocks (they carry no offset: nothing is known about
// the sums yet, and a short chunk's truncation bias is small), then chunks of
// kc; the offset for chunk j >= 2 comes from chunk j-2, scaled by kc / len.
// Both the MMA warp and the epilogue walk the item with this plan.
struct ChunkPlan {
    int nkb, kc, f;
    bool sc;  // sign-centred: chunks >= 2 accumulate onto a preloaded offset
    __device__ __forceinline__ ChunkPlan(int nkb_, int kc_, bool center) : nkb(nkb_), kc(kc_) {
        sc = SIGN_CENTRE && center && kc >= 2 && kc < nkb;
        f = sc ? kc / 2 : kc;
    }
    __device__ __forceinline__ int count() const {
        if (kc >= nkb) return 1;
        return sc ? 2 + (nkb - 2 * f + kc - 1) / kc : (nkb + kc - 1) / kc;
    }
    __device__ __forceinline__ int start(int j) const { return j < 2 ? j * f : 2 * f + (j - 2) * kc; }
    __device__ __forceinline__ int len(int j) const {
        const int s0 = start(j);
        return min(j < 2 ? f : kc, nkb - s0);
    }
};

// Work item w -> tile (tm, tn), part (-1 = whole tile, 0/1 = column half) and
// its K-block range [kb0, kb1) and split index ks.
__device__ __forceinline__ void decode_item(int w, const GemmArgs &a, int &tm, int &tn, int &part, int &kb0,
                                            int &kb1, int &ks) {
    if (a.ksplit > 1) {
        ks = w % a.ksplit;
        tile_coords(w / a.ksplit, a.tiles_m, a.tiles_n, a.group_m, tm, tn);
        part = -1;
        kb0 = ks * a.kb_per;
        kb1 = min(a.num_kb, kb0 + a.kb_per);
        return;
    }
    ks = 0;
    kb0 = 0;
    kb1 = a.num_kb;
    if (w < a.full_items) {
        tile_coords(w, a.tiles_m, a.tiles_n, a.group_m, tm, tn);
        part = -1;
    } else {
        const int h = w - a.full_items;
        tile_coords(a.full_items + (h >> 1), a.tiles_m, a.tiles_n, a.group_m, tm, tn);
        part = h & 1;
    }
}

// Write one 32 x 32 piece of C held as (thread = row, v[i] = column i) through
// a per-warp XOR-swizzled smem transpose (conflict-free both ways), so each
// store instruction writes one contiguous run of a C row (128 B for real
// products).  Rows >= n and columns >= p are skipped (ragged edges); offsets
// are 64-bit.
__device__ __forceinline__ float *row_ptr(const GemmArgs &args, int64_t r) {
    if (args.half_rows > 0 && r >= args.half_rows) return args.C + (r - args.half_rows) * args.ldc + args.half_off;
    return args.C + r * args.ldc;
}

// The same 32 x 32 piece (row lane of the piece in v[0..31]) written by TMA:
// the warp lays it out in its 4 KB smem buffer in the 128-byte-swizzle pattern
// of tm_c (16-byte chunk j of row r at chunk j ^ (r % 8)), one lane issues the
// bulk tensor store at (col0, row0, slice) and rows / columns past the map's
// extent are clipped by the hardware.  The buffer is reused only after the
// previous store has read it.
__device__ __forceinline__ void store_piece_tma(const CUtensorMap *tm_c, float *tbuf, uint32_t lane, int64_t row0,
                                                int64_t col0, int32_t slice, const uint32_t (&v)[32]) {
    if (lane == 0) ptx::bulk_wait_read();
    __syncwarp();
    uint8_t *rowp = reinterpret_cast<uint8_t *>(tbuf) + lane * 128;
#pragma unroll
    for (int j = 0; j < 8; j++) {
        const uint4 w = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        *reinterpret_cast<uint4 *>(rowp + ((j ^ (lane & 7)) << 4)) = w;
    }
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
        ptx::tma_store_3d(tm_c, tbuf, (int32_t)col0, (int32_t)row0, slice);
        ptx::bulk_commit();
    }
}

__device__ __forceinline__ void store_piece(const GemmArgs &args, float *tbuf, uint32_t lane, int64_t row0,
                                            int64_t col0, const uint32_t (&v)[32],
                                            float *const *gbase = nullptr, float *cbase = nullptr) {
#pragma unroll
    for (int i = 0; i < 32; i++) tbuf[lane * 32 + (i ^ lane)] = __uint_as_float(v[i]);
    __syncwarp();
    const int64_t col = col0 + lane;
    const int64_t rem = args.n - row0;
    if (col < args.p && rem > 0) {
        const int rows = rem < 32 ? (int)rem : 32;
        if (args.half_rows == 0 && args.cstride == 1) {
            float *cp = (cbase ? cbase : args.C) + row0 * args.ldc + col;
            if (rows == 32) {
#pragma unroll 4
                for (int rr = 0; rr < 32; rr++) cp[rr * args.ldc] = tbuf[rr * 32 + (lane ^ rr)];
            } else {
                for (int rr = 0; rr < rows; rr++) cp[rr * args.ldc] = tbuf[rr * 32 + (lane ^ rr)];
            }
        } else {
            for (int rr = 0; rr < rows; rr++)
                row_ptr(args, row0 + rr)[col * args.cstride] = tbuf[rr * 32 + (lane ^ rr)];
        }
        if (gbase != nullptr) {
            // the same 32 x 32 piece into every rank's C_full (128-B row segments over NVLink)
            const int64_t goff = (args.gather_row0 + row0) * args.gather_ld + args.gather_col0 + col;
            for (int pe = 0; pe < args.gather_peers; pe++) {
                float *gp = gbase[pe] + goff;
                for (int rr = 0; rr < rows; rr++) gp[rr * args.gather_ld] = tbuf[rr * 32 + (lane ^ rr)];
            }
        }
    }
    __syncwarp();
}

template <int CG, int BN, int STAGES, int PASSES, int KB = BK>
__global__ void __cluster_dims__(CG, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    gemm_tf32_sm100_kernel(const __grid_constant__ CUtensorMap tm_a_hi, const __grid_constant__ CUtensorMap tm_a_lo,
                           const __grid_constant__ CUtensorMap tm_b_hi, const __grid_constant__ CUtensorMap tm_b_lo,
                           const __grid_constant__ CUtensorMap tm_c, const GemmArgs args) {
    using Cfg = GemmCfg<CG, BN, STAGES, PASSES, KB>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // stage s: [A_hi | A_lo | B_hi | B_lo]   (identical offsets in both CTAs of a pair)
    auto a_tile = [&](int s, int op) { return smem + s * Cfg::STAGE_BYTES + op * Cfg::A_TILE; };
    auto b_tile = [&](int s, int op) {
        return smem + s * Cfg::STAGE_BYTES + Cfg::NOPS * Cfg::A_TILE + op * Cfg::B_TILE;
    };
    float *epi = reinterpret_cast<float *>(smem + STAGES * Cfg::STAGE_BYTES);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * Cfg::STAGE_BYTES + Cfg::EPI_BYTES);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(tempty + 2);
    float **gbase = reinterpret_cast<float **>(reinterpret_cast<uint8_t *>(full) + 320);  // [MAX_GATHER_PEERS]

    const uint32_t warp = ptx::warp_id();
    const uint32_t lane = threadIdx.x & 31;
    if (threadIdx.x == 0) trace_stamp(args.trace, 0);
    // a dependent launched with programmatic serialization (the split-K
    // reduction) may be scheduled now; it waits for this grid's completion
    asm volatile("griddepcontrol.launch_dependents;");
    const uint32_t rank = CG == 2 ? ptx::cluster_ctarank() : 0;  // CTA rank in the pair
    const int cluster_id = blockIdx.x / CG;
    const int num_clusters = gridDim.x / CG;

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tm_a_hi);
        ptx::prefetch_tmap(&tm_b_hi);
        if constexpr (PASSES == 3) {
            ptx::prefetch_tmap(&tm_a_lo);
            ptx::prefetch_tmap(&tm_b_lo);
        }
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < STAGES; s++) {
            ptx::mbar_init(&full[s], 1);   // leader producer's arrive.expect_tx (+ tx bytes of both CTAs)
            ptx::mbar_init(&empty[s], 1);  // one tcgen05.commit (multicast to both CTAs)
        }
        for (int b = 0; b < 2; b++) {
            ptx::mbar_init(&tfull[b], 1);                      // one tcgen05.commit
            ptx::mbar_init(&tempty[b], CG * NUM_EPI_WARPS);    // one arrive per epilogue warp of the pair
        }
        if (args.gather_win != nullptr)
            for (int pe = 0; pe < args.gather_peers; pe++)
                gbase[pe] = static_cast<float *>(ncclGetLsaPointer(
                    reinterpret_cast<ncclWindow_t>(const_cast<void *>(args.gather_win)),
                    args.gather_emul_stride > 0 ? (size_t)(pe * args.gather_emul_stride) * sizeof(float) : 0,
                    args.gather_emul_stride > 0 ? 0 : pe));
        ptx::fence_mbar_init();
    }
    if (warp == 2) ptx::tmem_alloc<CG>(tmem_holder, Cfg::TMEM_COLS);
    ptx::tc_fence_before();
    if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
    if (threadIdx.x == 0) trace_stamp(args.trace, 1);
    ptx::tc_fence_after();
    const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_holder, 0);  // uniform

    const int num_items = args.num_items;
    const int num_kb = args.num_kb;
    const int kc = args.kc;

    // Register budget per warpgroup role (setmaxnreg must dominate the role's
    // code, so it is the first statement of each warpgroup branch).
    if (warp < NUM_CTRL_WARPS) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(CTRL_REGS));
    if (warp == 0) {
        // ======================= TMA producer (both CTAs) =======================
        // Programmatic dependent launch: everything above (barrier init, TMEM
        // allocation, tensor-map prefetch, cluster sync) overlapped the split
        // kernels' tail; the operands they write are read only after this.
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (lane == 0) trace_stamp(args.trace, 2);
        const uint64_t pol = ptx::policy_evict_normal();
        int s = 0;
        uint32_t ph = 0;
        for (int t = cluster_id; t < num_items; t += num_clusters) {
            int tm, tn, part, kb0, kb1, ks;
            decode_item(t, args, tm, tn, part, kb0, kb1, ks);
            const int32_t m0 = tm * Cfg::TILE_M + rank * ROWS_PER_CTA;
            // half items need B_ROWS/2 rows per CTA; the full box is loaded (the
            // extra rows are never read by the N = BN/2 MMA)
            const int32_t n0 = part < 0 ? tn * BN + rank * Cfg::B_ROWS
                                        : tn * BN + part * (BN / 2) + rank * (Cfg::B_ROWS / 2);
            const int wave = t / num_clusters;
            const int wave_target = CG * min(num_clusters, num_items - wave * num_clusters);
            const int phases = (num_kb + args.sync_kb - 1) / args.sync_kb;
            for (int kb = kb0; kb < kb1; kb++) {
                if (args.wave_sync != nullptr && kb % args.sync_kb == 0) {
                    if (lane == 0)
                        wave_barrier(args.wave_sync + wave * phases + kb / args.sync_kb, wave_target,
                                     args.wave_sync + args.wave_slots);
                    __syncwarp();
                }
                ptx::mbar_wait(&empty[s], ph ^ 1);
                if (lane == 0 && (args.debug & 1)) {
                    if (rank == 0) ptx::mbar_arrive(&full[s]);
                } else if (lane == 0) {
                    const int32_t k0 = kb * KB;
                    if (rank == 0) ptx::mbar_arrive_expect_tx(&full[s], CG * Cfg::STAGE_BYTES);
                    auto load = [&](uint8_t *dst, const CUtensorMap *map, int32_t kc0, int32_t row) {
                        if constexpr (CG == 1) ptx::tma_load_2d(dst, map, &full[s], kc0, row, pol);
                        else ptx::tma_load_2d_pair(dst, map, &full[s], kc0, row, pol);
                    };
#pragma unroll
                    for (int at = 0; at < Cfg::ATOMS; at++) {
                        const int32_t ka = k0 + at * Cfg::ATOM_K;
                        load(a_tile(s, 0) + at * Cfg::A_ATOM, &tm_a_hi, ka, m0);
                        load(b_tile(s, 0) + at * Cfg::B_ATOM, &tm_b_hi, ka, n0);
                        if constexpr (PASSES == 3) {
                            load(a_tile(s, 1) + at * Cfg::A_ATOM, &tm_a_lo, ka, m0);
                            load(b_tile(s, 1) + at * Cfg::B_ATOM, &tm_b_lo, ka, n0);
                        }
                    }
                }
                __syncwarp();
                if (++s == STAGES) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1 && rank == 0) {
        // ======================= MMA issuer (leader CTA) =======================
        constexpr uint32_t idesc_full = ptx::idesc_tf32(Cfg::TILE_M, BN);
        constexpr uint32_t idesc_half = ptx::idesc_tf32(Cfg::TILE_M, BN / 2);
        int s = 0;
        uint32_t ph = 0, buf = 0, aph = 0;
        bool traced_mma = false;
#ifdef LA_DIAGNOSTICS
        int64_t wait_tempty = 0, wait_full = 0;  // cycles the MMA warp waited (LA_DIAG_TRACE)
#endif
        for (int t = cluster_id; t < num_items; t += num_clusters) {
            const uint32_t idesc = t < args.full_items ? idesc_full : idesc_half;
            int tm_, tn_, part_, kb0, kb1, ks_;
            decode_item(t, args, tm_, tn_, part_, kb0, kb1, ks_);
            const ChunkPlan plan(kb1 - kb0, kc, args.center_kb > 0);
            // walk the chunk plan incrementally (no division in the issue loop:
            // with one TF32 pass a K-block is only 4 MMAs of 128 cycles)
            int ci = 0, left = plan.len(0);  // current chunk, K-blocks left in it
            bool chunk_first = true;
            for (int kb = kb0; kb < kb1; kb++) {
                const bool chunk_last = left == 1;
                // sign-centred chunks accumulate onto the offset the epilogue
                // preloaded into the buffer
                const bool preloaded = plan.sc && ci >= 2;
#ifdef LA_DIAGNOSTICS
                const int64_t w0 = args.trace ? clock64() : 0;
#endif
                if (chunk_first) {
                    if constexpr (CG == 2) ptx::mbar_wait_cluster(&tempty[buf], aph ^ 1);
                    else ptx::mbar_wait(&tempty[buf], aph ^ 1);
                    ptx::tc_fence_after();
                }
#ifdef LA_DIAGNOSTICS
                const int64_t w1 = args.trace ? clock64() : 0;
#endif
                ptx::mbar_wait(&full[s], ph);
#ifdef LA_DIAGNOSTICS
                if (args.trace) {
                    wait_tempty += w1 - w0;
                    wait_full += clock64() - w1;
                }
#endif
                if (lane == 0 && kb == kb0 && !traced_mma) { trace_stamp(args.trace, 3); traced_mma = true; }
                ptx::tc_fence_after();
                {
                    // whole warp, converged: descriptors are warp-uniform; one
                    // elected lane issues each MMA / commit (ptx::*_elect)
                    const uint32_t d = tmem_base + buf * BN;
                    if (!(args.debug & 2)) {
                    const uint32_t ah = ptx::smem_u32(a_tile(s, 0)), bh = ptx::smem_u32(b_tile(s, 0));
                    const uint32_t al = ptx::smem_u32(a_tile(s, PASSES == 3 ? 1 : 0));
                    const uint32_t bl = ptx::smem_u32(b_tile(s, PASSES == 3 ? 1 : 0));
#pragma unroll
                    for (int j = 0; j < KB / 8; j++) {  // K = 8 per tf32 MMA = 32 bytes of a swizzled row
                        constexpr int JA = Cfg::ATOM_K / 8;  // MMA K steps per swizzle atom
                        const uint32_t oa = (j / JA) * Cfg::A_ATOM + 32 * (j % JA);
                        const uint32_t ob = (j / JA) * Cfg::B_ATOM + 32 * (j % JA);
                        const uint64_t dah = ptx::sdesc_kmajor<Cfg::ATOM_K>(ah + oa);
                        const uint64_t dbh = ptx::sdesc_kmajor<Cfg::ATOM_K>(bh + ob);
                        const uint32_t acc = (chunk_first && j == 0 && !preloaded) ? 0u : 1u;
                        if constexpr (PASSES == 3) {
                            const uint64_t dal = ptx::sdesc_kmajor<Cfg::ATOM_K>(al + oa);
                            const uint64_t dbl = ptx::sdesc_kmajor<Cfg::ATOM_K>(bl + ob);
                            ptx::mma_tf32_elect<CG>(d, dah, dbl, idesc, acc);  // hi . lo'
                            ptx::mma_tf32_elect<CG>(d, dal, dbh, idesc, 1u);   // lo . hi'
                            ptx::mma_tf32_elect<CG>(d, dah, dbh, idesc, 1u);   // hi . hi'
                        } else {
                            ptx::mma_tf32_elect<CG>(d, dah, dbh, idesc, acc);
                        }
                    }
                    }
                    ptx::mma_commit_elect<CG>(&empty[s]);
                    if (chunk_last) ptx::mma_commit_elect<CG>(&tfull[buf]);
                }
                __syncwarp();
                chunk_first = chunk_last;
                if (chunk_last) {
                    buf ^= 1;
                    if (buf == 0) aph ^= 1;
                    ++ci;
                    left = kb + 1 < kb1 ? plan.len(ci) : 0;
                } else {
                    --left;
                }
                if (++s == STAGES) { s = 0; ph ^= 1; }
            }
        }
        if (lane == 0) trace_stamp(args.trace, 4);
#ifdef LA_DIAGNOSTICS
        if (args.trace && lane == 0) {
            args.trace[blockIdx.x * TRACE_SLOTS + 8] = wait_tempty;
            args.trace[blockIdx.x * TRACE_SLOTS + 9] = wait_full;
        }
#endif
    }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(EPI_REGS));
        // ======================= epilogue (both CTAs) =======================
        const uint32_t e = warp - NUM_CTRL_WARPS;
        const uint32_t q = warp & 3;        // TMEM lane quarter this warp may access
        const uint32_t half = e >> 2;       // column half of the accumulator
        float *tbuf = epi + e * (32 * 32);
        const uint32_t tq0 = tmem_base + ((32u * q) << 16);
        float *const *epi_gbase = args.gather_win != nullptr ? gbase : nullptr;
        uint32_t buf = 0, aph = 0;
        bool traced_epi = false;
        for (int t = cluster_id; t < num_items; t += num_clusters) {
            int tm, tn, part, kb0, kb1, ks;
            decode_item(t, args, tm, tn, part, kb0, kb1, ks);
            const ChunkPlan plan(kb1 - kb0, kc, args.center_kb > 0);
            const int nchunks = kb1 > kb0 ? plan.count() : 0;
            float *cbase = args.ksplit > 1 ? args.partial + (int64_t)ks * args.n * args.ldc : nullptr;
            // whole tile: this warp owns columns [half*BN/2, +BN/2); half item: [half*BN/4, +BN/4)
            const int cpw = part < 0 ? Cfg::COLS_PER_WARP : Cfg::COLS_PER_WARP / 2;
            const int pieces = cpw / 32;
            const uint32_t tq = tq0 + half * cpw;
            const int64_t row0 = (int64_t)tm * Cfg::TILE_M + rank * ROWS_PER_CTA + 32 * q;
            const int64_t col0 = (int64_t)tn * BN + (part < 0 ? 0 : part * (BN / 2)) + half * cpw;
            auto put = [&](int64_t col, const uint32_t(&v)[32]) {
                if (args.tma_store) store_piece_tma(&tm_c, tbuf, lane, row0, col, args.ksplit > 1 ? ks : 0, v);
                else store_piece(args, tbuf, lane, row0, col, v, epi_gbase, cbase);
            };
            if (nchunks <= 0) {
                // empty K range (never produced by the host's split-K plan): the
                // partial contribution is zero; the MMA warp issues nothing for it
                uint32_t v[32];
#pragma unroll
                for (int i = 0; i < 32; i++) v[i] = 0u;
                for (int qq = 0; qq < pieces; qq++)
                    put(col0 + qq * 32, v);
            } else if (nchunks == 1) {
                // whole K accumulated in TMEM: stream 32-column pieces to C
                ptx::mbar_wait(&tfull[buf], aph);
                if (e == 0 && lane == 0 && !traced_epi) { trace_stamp(args.trace, 5); traced_epi = true; }
                ptx::tc_fence_after();
#pragma unroll 1
                for (int qq = 0; qq < pieces; qq++) {
                    uint32_t v[32];
                    ptx::tmem_ld_32x32b_x32(tq + buf * BN + qq * 32, v);
                    ptx::tmem_ld_wait();
                    if (qq == pieces - 1) {  // accumulator buffer free for the next tile
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive_cta0<CG>(&tempty[buf]);
                    }
                    put(col0 + qq * 32, v);
                }
                buf ^= 1;
                if (buf == 0) aph ^= 1;
            } else {
                // accumulator promotion: fp32 (RN) running sum of TMEM chunks.
                // Sign-centred chunks: the accumulator truncates toward zero, so
                // a chunk whose partial sums keep one sign is biased toward zero
                // (same-sign data: 1.68 x 2^-20 S at K = 16384).  After draining
                // chunk c, if this thread's chunk values x (its row, BN/2
                // columns) all share one sign, the offset -x_min/2 (x_min: the
                // value of smallest magnitude, so no partial sum exceeds |x|) is
                // written into the buffer for chunk c+2, which the MMA then
                // accumulates onto: the partial sums start on the other side of
                // zero and cross it, and truncations up and down cancel (0.96 x
                // 2^-20 S at K = 16384).  Chunk values are x = R - off; mixed
                // signs give off = 0 and the same bits as plain promotion.  Exact
                // on integer data: off is half an integer chunk sum and |R| <= |x|.
                float acc[Cfg::PIECES][32];
                float off_cur = 0.0f, off_oth = 0.0f;  // offsets preloaded in this / the other buffer
                // the drained values R = off + x are summed as they are and the
                // offsets (one per row) subtracted once at the end: one FADD per
                // element per chunk instead of two (off_sum = 0 on mixed signs)
                float off_sum = 0.0f;
#pragma unroll 1
                for (int c = 0; c < nchunks; c++) {
                    ptx::mbar_wait(&tfull[buf], aph);
                    if (e == 0 && lane == 0 && !traced_epi) { trace_stamp(args.trace, 5); traced_epi = true; }
                    ptx::tc_fence_after();
                    const uint32_t taddr = tq + buf * BN;
                    const bool refill = plan.sc && c + 2 < nchunks;  // this buffer holds chunk c+2 next
                    float lo = __uint_as_float(0x7f800000u), hi = -lo;   // chunk values' range (this row)
                    // two 32-column loads in flight per wait (the drain's latency
                    // bounds how short a chunk can be without stalling the MMAs)
#pragma unroll
                    for (int qq = 0; qq < Cfg::PIECES; qq += 2) {
                        if (qq < pieces) {
                            uint32_t v0[32], v1[32];
                            const bool two = qq + 1 < pieces;
                            ptx::tmem_ld_32x32b_x32(taddr + qq * 32, v0);
                            if (two) ptx::tmem_ld_32x32b_x32(taddr + (qq + 1) * 32, v1);
                            ptx::tmem_ld_wait();
                            if (c == 0) {
#pragma unroll
                                for (int i = 0; i < 32; i++) acc[qq][i] = __uint_as_float(v0[i]);
                                if (two) {
#pragma unroll
                                    for (int i = 0; i < 32; i++) acc[qq + 1][i] = __uint_as_float(v1[i]);
                                }
                            } else {
#pragma unroll
                                for (int i = 0; i < 32; i++) acc[qq][i] += __uint_as_float(v0[i]);
                                if (two) {
#pragma unroll
                                    for (int i = 0; i < 32; i++) acc[qq + 1][i] += __uint_as_float(v1[i]);
                                }
                            }
                            // (once this row's values have shown both signs the offset
                            // is 0 whatever follows: skip the rest of the scan)
                            if (refill && !(lo < off_cur && hi > off_cur)) {
#pragma unroll
                                for (int i = 0; i < 32; i++) {
                                    lo = fminf(lo, __uint_as_float(v0[i]));
                                    hi = fmaxf(hi, __uint_as_float(v0[i]));
                                }
                                if (two) {
#pragma unroll
                                    for (int i = 0; i < 32; i++) {
                                        lo = fminf(lo, __uint_as_float(v1[i]));
                                        hi = fmaxf(hi, __uint_as_float(v1[i]));
                                    }
                                }
                            }
                        }
                    }
                    // the range of x = v - off_cur is [lo - off_cur, hi - off_cur]
                    float off_new = 0.0f;
                    if (refill) {
                        lo -= off_cur;
                        hi -= off_cur;
                        // chunk c+2 is a full chunk of kc inside the centring range:
                        // half the smallest-magnitude value, scaled from this chunk's
                        // length (f or kc) to kc
                        const int c2 = c + 2;
                        if (plan.len(c2) == kc && kb0 + plan.start(c2) + kc <= args.center_kb) {
                            const float scale = -0.5f * (float)kc / (float)plan.len(c);
                            off_new = lo > 0.0f ? scale * lo : (hi < 0.0f ? scale * hi : 0.0f);
                        }
#pragma unroll
                        for (int qq = 0; qq < Cfg::PIECES; qq++)
                            if (qq < pieces) ptx::tmem_st_32x32b_x32_bcast(taddr + qq * 32, __float_as_uint(off_new));
                        ptx::tmem_st_wait();
                    }
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive_cta0<CG>(&tempty[buf]);
                    buf ^= 1;
                    if (buf == 0) aph ^= 1;
                    off_sum += off_cur;
                    off_cur = off_oth;
                    off_oth = off_new;
                }
#pragma unroll
                for (int qq = 0; qq < Cfg::PIECES; qq++) {
                    if (qq < pieces) {
                        uint32_t v[32];
#pragma unroll
                        for (int i = 0; i < 32; i++) v[i] = __float_as_uint(acc[qq][i] - off_sum);
                        put(col0 + qq * 32, v);
                    }
                }
            }
        }
        // fused gather: make this thread's peer stores visible system-wide before
        // the kernel completes (the host orders a cross-rank barrier after it)
        if (epi_gbase != nullptr) __threadfence_system();
        if (args.tma_store && lane == 0) ptx::bulk_wait_all();  // this warp's TMA stores complete
        if (e == 0 && lane == 0) trace_stamp(args.trace, 6);
    }

    ptx::tc_fence_before();
    if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x == 0) trace_stamp(args.trace, 7);
    if (warp == 2) ptx::tmem_dealloc<CG>(tmem_base, Cfg::TMEM_COLS);
}

}  // namespace la
