// dgemm_sm100.cuh -- double-precision C = A . B (Table 2 "Double" column,
// PAPER.md P:222-228; 8-byte shared-memory tiles).
//
// tcgen05 has no f64 kind; the B200's FP64 tensor path is DMMA (SASS
// DMMA.8x8x4, reached through mma.sync m16n8k8 f64, which ptxas splits into four
// DMMA.8x8x4).  The kernel is Listing 4's structure widened:
//   * 128 x 128 block tiles, 8 warps of 64 x 32 (4 x 4 m16n8 fragments each);
//   * K staged 32 doubles at a time in a 3-stage cp.async ring (16-byte copies
//     when m, p are even and A, B 16-byte aligned, else 8-byte; zero-filled
//     outside the matrix, so any n, m, p >= 1 works), padded rows (A: 36
//     doubles, B: 132) so every fragment load is bank-conflict free;
//   * fp64 FMA accumulation in registers (64 doubles per thread), each C element
//     written once, 64-bit offsets.
// Numerics: every product and sum is an IEEE binary64 operation (fused
// multiply-add), so |C - C_ref| <= 2 gamma_m(2^-53) sum|a||b| against the
// binary64 oracle, and integer inputs are exact.
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace la {

constexpr int DBM = 128, DBN = 128, DBK = 32, DSTAGES = 3;
constexpr int DLDA = DBK + 4;  // doubles per A row in smem (288 B: conflict-free fragment loads)
constexpr int DLDB = DBN + 4;  // doubles per B row in smem (1056 B)
constexpr int DTHREADS = 256;
constexpr int DSMEM_BYTES = DSTAGES * (DBM * DLDA + DBK * DLDB) * 8;

__device__ __forceinline__ void cp_async_f64(void *dst, const double *src, bool valid) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    const int sz = valid ? 8 : 0;  // src-size 0: zero-fill, no global read
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_f64x2(void *dst, const double *src, bool valid) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    const int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma_16x8x8(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

// VEC16: m and p even and A, B 16-byte aligned -> 16-byte copies (two doubles).
template <bool VEC16>
__global__ void __launch_bounds__(DTHREADS, 1)
    dgemm_sm100_kernel(const double *__restrict__ A, const double *__restrict__ B, double *__restrict__ C,
                       int64_t n, int64_t m, int64_t p) {
    extern __shared__ __align__(16) double dsm[];
    double *As = dsm;                              // [DSTAGES][DBM][DLDA]
    double *Bs = dsm + DSTAGES * DBM * DLDA;       // [DSTAGES][DBK][DLDB]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;         // fragment row group / thread in group
    const int wm = warp >> 2, wn = warp & 3;       // warp tile origin: rows wm*64, cols wn*32
    const int64_t m0 = (int64_t)blockIdx.y * DBM, n0 = (int64_t)blockIdx.x * DBN;
    const int kt_count = (int)((m + DBK - 1) / DBK);

    auto load_stage = [&](int stage, int kt) {
        const int64_t k0 = (int64_t)kt * DBK;
        double *as = As + stage * DBM * DLDA;
        double *bs = Bs + stage * DBK * DLDB;
        if constexpr (VEC16) {
#pragma unroll
            for (int i = 0; i < DBM * DBK / 2 / DTHREADS; i++) {  // A: 128 rows x 16 pairs
                const int idx = tid + i * DTHREADS, r = idx / (DBK / 2), c = 2 * (idx % (DBK / 2));
                const int64_t gr = m0 + r, gc = k0 + c;
                const bool ok = gr < n && gc < m;
                cp_async_f64x2(as + r * DLDA + c, ok ? A + gr * m + gc : A, ok);
            }
#pragma unroll
            for (int i = 0; i < DBK * DBN / 2 / DTHREADS; i++) {  // B: 32 rows x 64 pairs
                const int idx = tid + i * DTHREADS, r = idx / (DBN / 2), c = 2 * (idx % (DBN / 2));
                const int64_t gr = k0 + r, gc = n0 + c;
                const bool ok = gr < m && gc < p;
                cp_async_f64x2(bs + r * DLDB + c, ok ? B + gr * p + gc : B, ok);
            }
        } else {
#pragma unroll 4
            for (int i = 0; i < DBM * DBK / DTHREADS; i++) {  // A: 128 rows x 32
                const int idx = tid + i * DTHREADS, r = idx / DBK, c = idx % DBK;
                const int64_t gr = m0 + r, gc = k0 + c;
                const bool ok = gr < n && gc < m;
                cp_async_f64(as + r * DLDA + c, ok ? A + gr * m + gc : A, ok);
            }
#pragma unroll 4
            for (int i = 0; i < DBK * DBN / DTHREADS; i++) {  // B: 32 rows x 128
                const int idx = tid + i * DTHREADS, r = idx / DBN, c = idx % DBN;
                const int64_t gr = k0 + r, gc = n0 + c;
                const bool ok = gr < m && gc < p;
                cp_async_f64(bs + r * DLDB + c, ok ? B + gr * p + gc : B, ok);
            }
        }
    };

    double acc[4][4][4];
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++)
#pragma unroll
            for (int v = 0; v < 4; v++) acc[i][j][v] = 0.0;

#pragma unroll
    for (int s = 0; s < DSTAGES - 1; s++) {
        if (s < kt_count) load_stage(s, s);
        cp_async_commit();
    }
    for (int kt = 0; kt < kt_count; kt++) {
        cp_async_wait<DSTAGES - 2>();
        __syncthreads();  // stage kt landed for everyone; stage kt-1 no longer read
        const int nxt = kt + DSTAGES - 1;
        if (nxt < kt_count) load_stage(nxt % DSTAGES, nxt);
        cp_async_commit();
        const double *as = As + (kt % DSTAGES) * DBM * DLDA + (wm * 64) * DLDA;
        const double *bs = Bs + (kt % DSTAGES) * DBK * DLDB + wn * 32;
#pragma unroll
        for (int kk = 0; kk < DBK; kk += 8) {
            double af[4][4], bf[4][2];
#pragma unroll
            for (int mi = 0; mi < 4; mi++) {
                const double *a = as + (mi * 16 + g) * DLDA + kk + t;
                af[mi][0] = a[0];
                af[mi][1] = a[8 * DLDA];
                af[mi][2] = a[4];
                af[mi][3] = a[8 * DLDA + 4];
            }
#pragma unroll
            for (int ni = 0; ni < 4; ni++) {
                const double *b = bs + (kk + t) * DLDB + ni * 8 + g;
                bf[ni][0] = b[0];
                bf[ni][1] = b[4 * DLDB];
            }
#pragma unroll
            for (int mi = 0; mi < 4; mi++)
#pragma unroll
                for (int ni = 0; ni < 4; ni++) dmma_16x8x8(acc[mi][ni], af[mi], bf[ni]);
        }
    }
    cp_async_wait<0>();

    // write-back: d0 (g, 2t), d1 (g, 2t+1), d2 (g+8, 2t), d3 (g+8, 2t+1)
    const bool pair_ok = (p & 1) == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0;
#pragma unroll
    for (int mi = 0; mi < 4; mi++)
#pragma unroll
        for (int half = 0; half < 2; half++) {
            const int64_t row = m0 + wm * 64 + mi * 16 + g + 8 * half;
            if (row >= n) continue;
            double *crow = C + row * p;
#pragma unroll
            for (int ni = 0; ni < 4; ni++) {
                const int64_t col = n0 + wn * 32 + ni * 8 + 2 * t;
                const double v0 = acc[mi][ni][2 * half], v1 = acc[mi][ni][2 * half + 1];
                if (pair_ok && col + 1 < p) {
                    *reinterpret_cast<double2 *>(crow + col) = make_double2(v0, v1);
                } else {
                    if (col < p) crow[col] = v0;
                    if (col + 1 < p) crow[col + 1] = v1;
                }
            }
        }
}

// ---------------------------------------------------------------------------
// Warp-specialised TMA variant (m, p even; A, B 16-byte aligned).  The
// cp.async kernel above leaves the DMMA pipe idle ~11% of the time (ncu: the
// consumer warps also run the copy address arithmetic and a CTA-wide barrier
// per K-stage).  Here one producer warp feeds a 3-stage ring with TMA
// (SWIZZLE_128B boxes of 16 doubles, zero fill past every edge) and mbarriers;
// the eight consumer warps only load fragments and issue DMMA.
//
// Shared layout per stage: A = 2 boxes (K halves) of 128 rows x 16 doubles,
// B = 8 boxes (16-column groups) of 32 K-rows x 16 doubles; in each 128-byte
// box row the 16-byte chunk c sits at chunk c ^ (row % 8).  Bank conflicts of
// the fragment loads are removed by feeding the MMA's k index t (and t + 4) from
// K-row sigma(t) = (t >> 1) | ((t & 1) << 2) (and sigma(t) + 2) of each 8-wide
// K group -- the same permutation for A and B, so every product a_ik * b_kj is
// still formed exactly once (only the order of the fp64 additions inside one
// K group changes, which the binary64 bound already covers).
__device__ __forceinline__ double lds_f64(uint32_t addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}

constexpr int DT_STAGES = 3;
constexpr int DT_A_BYTES = DBM * DBK * 8;  // 32 KB
constexpr int DT_B_BYTES = DBK * DBN * 8;  // 32 KB
constexpr int DT_STAGE_BYTES = DT_A_BYTES + DT_B_BYTES;
constexpr int DT_THREADS = 384;  // 2 consumer warpgroups + 1 producer warpgroup (one TMA lane)
constexpr int DT_SMEM_BYTES = 1024 + DT_STAGES * DT_STAGE_BYTES + 2 * DT_STAGES * 8;
// setmaxnreg: the pool is 384 x 168; the producer warpgroup shrinks to 40 so the
// consumers (128 fp64 accumulators + fragments each) can grow to 232.
constexpr int DT_LAUNCH_REGS = 168, DT_PROD_REGS = 40, DT_CONS_REGS = 232;
static_assert(128 * DT_PROD_REGS + 256 * DT_CONS_REGS <= DT_THREADS * DT_LAUNCH_REGS, "register pool");

__global__ void __launch_bounds__(DT_THREADS, 1)
    dgemm_tma_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                     double *__restrict__ C, int64_t n, int64_t m, int64_t p) {
    extern __shared__ __align__(1024) uint8_t dt_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(dt_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + DT_STAGES * DT_STAGE_BYTES);
    uint64_t *empty = full + DT_STAGES;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int32_t m0 = (int32_t)blockIdx.y * DBM, n0 = (int32_t)blockIdx.x * DBN;
    const int kt_count = (int)((m + DBK - 1) / DBK);
    if (threadIdx.x == 0) {
        for (int s = 0; s < DT_STAGES; s++) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 8);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();

    if (warp >= 8) {  // producer warpgroup
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(DT_PROD_REGS));
        if (warp == 8 && lane == 0) {
            ptx::prefetch_tmap(&tA);
            ptx::prefetch_tmap(&tB);
            const uint64_t pol = ptx::policy_evict_normal();
            for (int kt = 0; kt < kt_count; kt++) {
                const int s = kt % DT_STAGES;
                ptx::mbar_wait(&empty[s], ((kt / DT_STAGES) & 1) ^ 1);
                ptx::mbar_arrive_expect_tx(&full[s], DT_STAGE_BYTES);
                uint8_t *a = smem + s * DT_STAGE_BYTES, *b = a + DT_A_BYTES;
                const int32_t k0 = kt * DBK;
                ptx::tma_load_2d(a, &tA, &full[s], k0, m0, pol);
                ptx::tma_load_2d(a + DBM * 128, &tA, &full[s], k0 + 16, m0, pol);
#pragma unroll
                for (int j = 0; j < DBN / 16; j++) ptx::tma_load_2d(b + j * DBK * 128, &tB, &full[s], n0 + 16 * j, k0, pol);
            }
        }
        return;
    }

    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(DT_CONS_REGS));
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp >> 2, wn = warp & 3;  // warp tile origin: rows wm*64, cols wn*32
    const uint32_t sbase = ptx::smem_u32(smem);
    const int s0 = (t >> 1) | ((t & 1) << 2), s1 = s0 + 2;  // K rows of MMA k = t, t + 4
    // byte offsets inside a box (row term + swizzled chunk + 8-byte half)
    const uint32_t a_lo = g * 128 + ((((uint32_t)s0 >> 1) ^ g) << 4) + (s0 & 1) * 8;
    const uint32_t a_hi = g * 128 + ((((uint32_t)s1 >> 1) ^ g) << 4) + (s1 & 1) * 8;
    const uint32_t b_lo = s0 * 128 + ((((uint32_t)g >> 1) ^ s0) << 4) + (g & 1) * 8;
    const uint32_t b_hi = s1 * 128 + ((((uint32_t)g >> 1) ^ s1) << 4) + (g & 1) * 8;

    double acc[4][4][4];
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++)
#pragma unroll
            for (int v = 0; v < 4; v++) acc[i][j][v] = 0.0;

    for (int kt = 0; kt < kt_count; kt++) {
        const int s = kt % DT_STAGES;
        ptx::mbar_wait(&full[s], (kt / DT_STAGES) & 1);
        const uint32_t as = sbase + s * DT_STAGE_BYTES + (wm * 64) * 128;
        const uint32_t bs = sbase + s * DT_STAGE_BYTES + DT_A_BYTES + (wn * 2) * DBK * 128;
#pragma unroll
        for (int kk = 0; kk < DBK; kk += 8) {
            const uint32_t xa = ((kk >> 3) & 1) << 6;  // chunk ^ 4 in the upper half of a box
            const uint32_t ak = as + (kk >> 4) * (DBM * 128);
            const uint32_t bk = bs + kk * 128;
            double af[4][4], bf[4][2];
#pragma unroll
            for (int mi = 0; mi < 4; mi++) {
                const uint32_t r = ak + mi * 16 * 128;
                af[mi][0] = lds_f64(r + (a_lo ^ xa));
                af[mi][1] = lds_f64(r + 1024 + (a_lo ^ xa));
                af[mi][2] = lds_f64(r + (a_hi ^ xa));
                af[mi][3] = lds_f64(r + 1024 + (a_hi ^ xa));
            }
#pragma unroll
            for (int ni = 0; ni < 4; ni++) {
                const uint32_t xb = (ni & 1) << 6;
                const uint32_t c = bk + (ni >> 1) * DBK * 128;
                bf[ni][0] = lds_f64(c + (b_lo ^ xb));
                bf[ni][1] = lds_f64(c + (b_hi ^ xb));
            }
#pragma unroll
            for (int mi = 0; mi < 4; mi++)
#pragma unroll
                for (int ni = 0; ni < 4; ni++) dmma_16x8x8(acc[mi][ni], af[mi], bf[ni]);
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&empty[s]);
    }

    const bool pair_ok = (p & 1) == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0;
#pragma unroll
    for (int mi = 0; mi < 4; mi++)
#pragma unroll
        for (int half = 0; half < 2; half++) {
            const int64_t row = (int64_t)m0 + wm * 64 + mi * 16 + g + 8 * half;
            if (row >= n) continue;
            double *crow = C + row * p;
#pragma unroll
            for (int ni = 0; ni < 4; ni++) {
                const int64_t col = (int64_t)n0 + wn * 32 + ni * 8 + 2 * t;
                const double v0 = acc[mi][ni][2 * half], v1 = acc[mi][ni][2 * half + 1];
                if (pair_ok && col + 1 < p) {
                    *reinterpret_cast<double2 *>(crow + col) = make_double2(v0, v1);
                } else {
                    if (col < p) crow[col] = v0;
                    if (col + 1 < p) crow[col + 1] = v1;
                }
            }
        }
}

}  // namespace la
