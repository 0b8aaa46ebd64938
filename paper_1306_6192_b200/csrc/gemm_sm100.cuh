// gemm_sm100.cuh -- K2: persistent warp-specialised tcgen05 GEMM, C = A . B.
//
// The paper's optimised kernel (Listing 4) stages a 16x16
// tile of A and of B in shared memory per K step, synchronises
// (P:178), does 16 FMAs per thread, synchronises again and
// writes one C element per thread.  The same structure, re-built
// for sm_100a:
//   * staging     : TMA (cp.async.bulk.tensor) fills a STAGES-deep ring of
//                   128B-swizzled K-major tiles; mbarrier full[s] replaces the
//                   first __syncthreads;
//   * inner product: one elected thread issues tcgen05.mma.kind::tf32 into a
//                   TMEM accumulator (3 passes hi.lo', lo.hi', hi.hi' per K=8
//                   step for 3xTF32); tcgen05.commit -> empty[s] replaces the
//                   second __syncthreads;
//   * write-back  : epilogue warps tcgen05.ld the accumulator, optionally add it
//                   into an fp32 register running sum every `kc` K-blocks
//                   (accumulator promotion), and store C exactly once per
//                   element, coalesced through a per-warp smem transpose, with
//                   64-bit offsets and ragged-edge predication.
// Two TMEM accumulator buffers let the epilogue of one tile (or chunk) overlap
// the MMAs of the next.  One CTA per SM, persistent over output tiles in a
// grouped raster order (tiles sharing A rows run concurrently -> L2 reuse).
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace la {

constexpr int BM = 128;  // rows of C per CTA (UMMA M, cta_group::1)
constexpr int BK = 32;   // K per stage: 32 fp32 = one 128-byte swizzle row
constexpr int EPI_WARP0 = 4;
constexpr int NUM_THREADS = 256;  // warp0 TMA, warp1 MMA, warp2 TMEM alloc, warp3 idle, warps4-7 epilogue

struct GemmArgs {
    float *C;
    int64_t n, p, ldc;  // C is n x p with row stride ldc
    int32_t num_kb;     // K-blocks of BK
    int32_t kc;         // K-blocks per TMEM chunk (promotion interval); >= num_kb: no promotion
    int32_t tiles_m, tiles_n, group_m;
};

template <int BN, int STAGES, int PASSES>
struct GemmCfg {
    static constexpr int NOPS = PASSES == 3 ? 2 : 1;  // hi (+ lo) tiles per operand
    static constexpr int A_TILE = BM * BK * 4;        // 16 KB
    static constexpr int B_TILE = BN * BK * 4;
    static constexpr int STAGE_BYTES = NOPS * (A_TILE + B_TILE);
    static constexpr int EPI_BYTES = 4 * 32 * 33 * 4;  // per-warp 32x33 transpose buffers
    static constexpr int BAR_BYTES = 256;
    static constexpr int SMEM_BYTES = 1024 /*align slack*/ + STAGES * STAGE_BYTES + EPI_BYTES + BAR_BYTES;
    static constexpr uint32_t TMEM_COLS = 2 * BN;  // two accumulator buffers
    static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "UMMA N for M=128 must be a multiple of 16 <= 256");
    static_assert(TMEM_COLS == 64 || TMEM_COLS == 128 || TMEM_COLS == 256 || TMEM_COLS == 512, "TMEM alloc");
    static_assert(SMEM_BYTES <= 232448, "exceeds 227 KB of shared memory per CTA");
};

__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int group, int &tm,
                                            int &tn) {
    const int per_group = group * tiles_n;
    const int g = t / per_group;
    const int first = g * group;
    const int gsz = min(group, tiles_m - first);
    const int r = t - g * per_group;
    tm = first + r % gsz;
    tn = r / gsz;
}

// Write one 32 x 32 piece of C held as (thread = row, v[i] = column i) through
// a per-warp padded smem transpose, so each store instruction writes 128
// contiguous bytes of one C row.  Rows >= n and columns >= p are skipped
// (ragged edges); offsets are 64-bit.
__device__ __forceinline__ void store_piece(const GemmArgs &args, float *tbuf, uint32_t lane, int64_t row0,
                                            int64_t col0, const uint32_t (&v)[32]) {
#pragma unroll
    for (int i = 0; i < 32; i++) tbuf[lane * 33 + i] = __uint_as_float(v[i]);
    __syncwarp();
    const int64_t col = col0 + lane;
    if (col < args.p) {
        float *cp = args.C + row0 * args.ldc + col;
        const int64_t rem = args.n - row0;
        const int rows = rem < 32 ? (int)rem : 32;
#pragma unroll 8
        for (int rr = 0; rr < 32; rr++)
            if (rr < rows) cp[rr * args.ldc] = tbuf[rr * 33 + lane];
    }
    __syncwarp();
}

template <int BN, int STAGES, int PASSES>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_tf32_sm100_kernel(const __grid_constant__ CUtensorMap tm_a_hi,
                           const __grid_constant__ CUtensorMap tm_a_lo,
                           const __grid_constant__ CUtensorMap tm_b_hi,
                           const __grid_constant__ CUtensorMap tm_b_lo, const GemmArgs args) {
    using Cfg = GemmCfg<BN, STAGES, PASSES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // stage s: [A_hi | A_lo | B_hi | B_lo]
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

    const uint32_t warp = ptx::warp_id();
    const uint32_t lane = threadIdx.x & 31;

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
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; b++) {
            ptx::mbar_init(&tfull[b], 1);
            ptx::mbar_init(&tempty[b], 128);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 2) ptx::tmem_alloc<1>(tmem_holder, Cfg::TMEM_COLS);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;

    const int num_tiles = args.tiles_m * args.tiles_n;
    const int num_kb = args.num_kb;
    const int kc = args.kc;

    if (warp == 0) {
        // ======================= TMA producer =======================
        const uint64_t pol = ptx::policy_evict_normal();
        int s = 0;
        uint32_t ph = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            int tm, tn;
            tile_coords(t, args.tiles_m, args.tiles_n, args.group_m, tm, tn);
            const int32_t m0 = tm * BM, n0 = tn * BN;
            for (int kb = 0; kb < num_kb; kb++) {
                ptx::mbar_wait(&empty[s], ph ^ 1);
                if (lane == 0) {
                    const int32_t k0 = kb * BK;
                    ptx::mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
                    ptx::tma_load_2d(a_tile(s, 0), &tm_a_hi, &full[s], k0, m0, pol);
                    ptx::tma_load_2d(b_tile(s, 0), &tm_b_hi, &full[s], k0, n0, pol);
                    if constexpr (PASSES == 3) {
                        ptx::tma_load_2d(a_tile(s, 1), &tm_a_lo, &full[s], k0, m0, pol);
                        ptx::tma_load_2d(b_tile(s, 1), &tm_b_lo, &full[s], k0, n0, pol);
                    }
                }
                __syncwarp();
                if (++s == STAGES) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1) {
        // ======================= MMA issuer =======================
        constexpr uint32_t idesc = ptx::idesc_tf32(BM, BN);
        int s = 0;
        uint32_t ph = 0, buf = 0, aph = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            for (int kb = 0; kb < num_kb; kb++) {
                const bool chunk_first = (kb % kc) == 0;
                const bool chunk_last = (kb % kc) == kc - 1 || kb == num_kb - 1;
                if (chunk_first) {
                    ptx::mbar_wait(&tempty[buf], aph ^ 1);
                    ptx::tc_fence_after();
                }
                ptx::mbar_wait(&full[s], ph);
                ptx::tc_fence_after();
                if (lane == 0) {
                    const uint32_t d = tmem_base + buf * BN;
                    const uint32_t ah = ptx::smem_u32(a_tile(s, 0)), bh = ptx::smem_u32(b_tile(s, 0));
                    const uint32_t al = ptx::smem_u32(a_tile(s, PASSES == 3 ? 1 : 0));
                    const uint32_t bl = ptx::smem_u32(b_tile(s, PASSES == 3 ? 1 : 0));
#pragma unroll
                    for (int j = 0; j < BK / 8; j++) {  // K = 8 per tf32 MMA = 32 bytes
                        const uint64_t dah = ptx::sdesc_kmajor_sw128(ah + 32 * j);
                        const uint64_t dbh = ptx::sdesc_kmajor_sw128(bh + 32 * j);
                        const uint32_t acc = (chunk_first && j == 0) ? 0u : 1u;
                        if constexpr (PASSES == 3) {
                            const uint64_t dal = ptx::sdesc_kmajor_sw128(al + 32 * j);
                            const uint64_t dbl = ptx::sdesc_kmajor_sw128(bl + 32 * j);
                            ptx::mma_tf32<1>(d, dah, dbl, idesc, acc);  // hi . lo'
                            ptx::mma_tf32<1>(d, dal, dbh, idesc, 1u);   // lo . hi'
                            ptx::mma_tf32<1>(d, dah, dbh, idesc, 1u);   // hi . hi'
                        } else {
                            ptx::mma_tf32<1>(d, dah, dbh, idesc, acc);
                        }
                    }
                    ptx::mma_commit<1>(&empty[s]);
                    if (chunk_last) ptx::mma_commit<1>(&tfull[buf]);
                }
                __syncwarp();
                if (chunk_last) {
                    buf ^= 1;
                    if (buf == 0) aph ^= 1;
                }
                if (++s == STAGES) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp >= EPI_WARP0) {
        // ======================= epilogue =======================
        const uint32_t q = warp & 3;  // TMEM lane quarter this warp may access
        float *tbuf = epi + (warp - EPI_WARP0) * (32 * 33);
        const uint32_t lane_off = (32u * q) << 16;
        uint32_t buf = 0, aph = 0;
        const int nchunks = (num_kb + kc - 1) / kc;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            int tm, tn;
            tile_coords(t, args.tiles_m, args.tiles_n, args.group_m, tm, tn);
            const int64_t row0 = (int64_t)tm * BM + 32 * q;
            if (nchunks == 1) {
                // whole K accumulated in TMEM: stream 32-column pieces to C
                ptx::mbar_wait(&tfull[buf], aph);
                ptx::tc_fence_after();
#pragma unroll 1
                for (int qq = 0; qq < BN / 32; qq++) {
                    uint32_t v[32];
                    ptx::tmem_ld_32x32b_x32(tmem_base + lane_off + buf * BN + qq * 32, v);
                    ptx::tmem_ld_wait();
                    if (qq == BN / 32 - 1) {  // accumulator buffer free for the next tile
                        ptx::tc_fence_before();
                        ptx::mbar_arrive(&tempty[buf]);
                    }
                    store_piece(args, tbuf, lane, row0, (int64_t)tn * BN + qq * 32, v);
                }
                buf ^= 1;
                if (buf == 0) aph ^= 1;
            } else {
                // accumulator promotion: fp32 (RN) running sum of TMEM chunks
                float acc[BN / 32][32];
#pragma unroll 1
                for (int c = 0; c < nchunks; c++) {
                    ptx::mbar_wait(&tfull[buf], aph);
                    ptx::tc_fence_after();
                    const uint32_t taddr = tmem_base + lane_off + buf * BN;
                    if (c == 0) {
#pragma unroll
                        for (int qq = 0; qq < BN / 32; qq++) {
                            uint32_t v[32];
                            ptx::tmem_ld_32x32b_x32(taddr + qq * 32, v);
                            ptx::tmem_ld_wait();
#pragma unroll
                            for (int i = 0; i < 32; i++) acc[qq][i] = __uint_as_float(v[i]);
                        }
                    } else {
#pragma unroll
                        for (int qq = 0; qq < BN / 32; qq++) {
                            uint32_t v[32];
                            ptx::tmem_ld_32x32b_x32(taddr + qq * 32, v);
                            ptx::tmem_ld_wait();
#pragma unroll
                            for (int i = 0; i < 32; i++) acc[qq][i] += __uint_as_float(v[i]);
                        }
                    }
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(&tempty[buf]);
                    buf ^= 1;
                    if (buf == 0) aph ^= 1;
                }
#pragma unroll
                for (int qq = 0; qq < BN / 32; qq++) {
                    uint32_t v[32];
#pragma unroll
                    for (int i = 0; i < 32; i++) v[i] = __float_as_uint(acc[qq][i]);
                    store_piece(args, tbuf, lane, row0, (int64_t)tn * BN + qq * 32, v);
                }
            }
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 2) ptx::tmem_dealloc<1>(tmem_base, Cfg::TMEM_COLS);
}

}  // namespace la
