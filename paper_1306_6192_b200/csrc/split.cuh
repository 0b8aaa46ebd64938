// split.cuh -- K1: operand split for the 3xTF32 product (HBM-bound pass).
//
// a = hi + lo,  hi = tf32_rna(a) (11 significant bits, low 13 mantissa bits 0),
// lo = a - hi   (exact in fp32: the rounding error of rounding to fewer bits).
// The tensor pipe then forms hi*hi' + hi*lo' + lo*hi' (lo*lo' <= 2^-22 |a a'|
// is dropped).  Not in the paper (its kernels multiply fp32 on SIMT cores,
// P:118); it is how fp32 accuracy comes off the TF32 tensor pipe
// (BASELINE.json north_star).
//
// Layouts written (the GEMM's TMA descriptors read them):
//   A (n x m row-major)  -> A_hi, A_lo : n x mp row-major, mp = round_up(m, 4)
//   B (m x p row-major)  -> Bt_hi, Bt_lo: p x mp row-major (B transposed, so both
//                           operands are K-major for the UMMA descriptors)
// Columns [m, mp) are written as 0 so TMA rows are 16-byte aligned and the
// padding contributes exact zeros.  With PASSES == 1 (plain TF32 mode) only hi
// is written.
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace la {

// lo is stored rounded to TF32 as well (cvt.rna): the tensor pipe reads only the
// TF32 bits of its fp32 operands, so this changes lo by at most half a TF32 ulp
// (the per-product bound improves from 2^-21.06 to 2^-21.03 for 24-bit inputs,
// SURVEY App. A) and stops 13 dead low bits from toggling through shared memory
// and the operand path.
__device__ __forceinline__ float lo_part(float x, float h) { return ptx::to_tf32_rna(x - h); }

template <int PASSES>
__device__ __forceinline__ void split_store(float x, float *hi, float *lo, int64_t off) {
    const float h = ptx::to_tf32_rna(x);
    hi[off] = h;
    if constexpr (PASSES == 3) lo[off] = lo_part(x, h);
}

// Row-major A, m % 4 == 0: flat float4 grid-stride loop (mp == m), four
// independent 16-byte loads in flight per thread before any store (a small
// split is latency-bound: the launch sizes the grid so one batch covers it).
constexpr int SPLIT_UNROLL = 4;

template <int PASSES>
__device__ __forceinline__ void split4_store(float4 x, float4 *__restrict__ hi, float4 *__restrict__ lo, int64_t i) {
    float4 h;
    h.x = ptx::to_tf32_rna(x.x);
    h.y = ptx::to_tf32_rna(x.y);
    h.z = ptx::to_tf32_rna(x.z);
    h.w = ptx::to_tf32_rna(x.w);
    __stcg(hi + i, h);
    if constexpr (PASSES == 3) {
        float4 l;
        l.x = lo_part(x.x, h.x);
        l.y = lo_part(x.y, h.y);
        l.z = lo_part(x.z, h.z);
        l.w = lo_part(x.w, h.w);
        __stcg(lo + i, l);
    }
}

template <int PASSES>
__device__ __forceinline__ void split_rows_vec4_body(const float4 *__restrict__ a, float4 *__restrict__ hi,
                                                    float4 *__restrict__ lo, int64_t count4, int64_t block,
                                                    int64_t nblocks) {
    const int64_t stride = nblocks * blockDim.x;
    int64_t i = block * (int64_t)blockDim.x + threadIdx.x;
    for (; i + (SPLIT_UNROLL - 1) * stride < count4; i += SPLIT_UNROLL * stride) {
        float4 x[SPLIT_UNROLL];
#pragma unroll
        for (int u = 0; u < SPLIT_UNROLL; u++) x[u] = __ldcs(a + i + u * stride);
#pragma unroll
        for (int u = 0; u < SPLIT_UNROLL; u++) split4_store<PASSES>(x[u], hi, lo, i + u * stride);
    }
    for (; i < count4; i += stride) split4_store<PASSES>(__ldcs(a + i), hi, lo, i);
}

template <int PASSES>
__global__ void __launch_bounds__(256) split_rows_vec4_kernel(const float4 *__restrict__ a,
                                                              float4 *__restrict__ hi,
                                                              float4 *__restrict__ lo,
                                                              int64_t count4) {
    asm volatile("griddepcontrol.launch_dependents;");  // let the GEMM start its prologue
    split_rows_vec4_body<PASSES>(a, hi, lo, count4, blockIdx.x, gridDim.x);
}

// Row-major A, general m: one block-row per grid.y step, columns padded to mp.
template <int PASSES>
__global__ void __launch_bounds__(256) split_rows_kernel(const float *__restrict__ a,
                                                         float *__restrict__ hi,
                                                         float *__restrict__ lo, int64_t n,
                                                         int64_t m, int64_t mp) {
    asm volatile("griddepcontrol.launch_dependents;");  // let the GEMM start its prologue
    for (int64_t r = blockIdx.y; r < n; r += gridDim.y) {
        for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < mp;
             c += (int64_t)gridDim.x * blockDim.x) {
            const float x = c < m ? a[r * m + c] : 0.0f;
            split_store<PASSES>(x, hi, lo, r * mp + c);
        }
    }
}

// B (m x p block, row stride ldb) -> Bt (p x mp row-major), 32x32 tiles through
// smem so both the read (along j) and the write (along k) are coalesced.
// Block (32, 8).
template <int PASSES>
__global__ void __launch_bounds__(256) split_transpose_kernel(const float *__restrict__ b,
                                                              float *__restrict__ hi,
                                                              float *__restrict__ lo, int64_t m,
                                                              int64_t p, int64_t ldb, int64_t mp) {
    asm volatile("griddepcontrol.launch_dependents;");  // let the GEMM start its prologue
    __shared__ float tile[32][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t j0 = (int64_t)blockIdx.x * 32;  // column of B = row of Bt
    const int64_t k0 = (int64_t)blockIdx.y * 32;  // row of B = column of Bt
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const int64_t k = k0 + ty + 8 * i, j = j0 + tx;
        tile[ty + 8 * i][tx] = (k < m && j < p) ? __ldcs(b + k * ldb + j) : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const int64_t j = j0 + ty + 8 * i, k = k0 + tx;
        if (j < p && k < mp) split_store<PASSES>(tile[tx][ty + 8 * i], hi, lo, j * mp + k);
    }
}

// B (m x p block, row stride ldb, p % 4 == 0, ldb % 4 == 0, 16-B aligned) ->
// Bt (p x mp): 64 x 64 tiles, 16-byte loads along j and 16-byte stores along k
// (each half-warp writes 256 contiguous bytes of one Bt row).  Block 256.
template <int PASSES>
__device__ __forceinline__ void split_transpose64_body(const float *__restrict__ b, float *__restrict__ hi,
                                                      float *__restrict__ lo, int64_t m, int64_t p, int64_t ldb,
                                                      int64_t mp, int64_t bx, int64_t by,
                                                      float (*tile)[65]) {
    const int tid = threadIdx.x;
    const int64_t j0 = bx * 64;  // columns of B = rows of Bt
    const int64_t k0 = by * 64;  // rows of B = columns of Bt
    // load: 64 rows (k) x 16 float4 (j); thread -> (row r = tid / 16 + 16 i, col4 c = tid % 16)
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const int r = tid / 16 + 16 * i, c = (tid % 16) * 4;
        const int64_t k = k0 + r, j = j0 + c;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k < m && j < p) v = __ldcs(reinterpret_cast<const float4 *>(b + k * ldb + j));  // p % 4 == 0
        tile[r][c] = v.x;
        tile[r][c + 1] = v.y;
        tile[r][c + 2] = v.z;
        tile[r][c + 3] = v.w;
    }
    __syncthreads();
    // store: 64 rows (j) x 16 float4 (k); thread -> (row j = tid / 16 + 16 i, k4 = tid % 16)
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const int jr = tid / 16 + 16 * i, kc = (tid % 16) * 4;
        const int64_t j = j0 + jr, k = k0 + kc;
        if (j >= p || k >= mp) continue;  // mp % 4 == 0, so a float4 never straddles mp
        float x[4] = {tile[kc][jr], tile[kc + 1][jr], tile[kc + 2][jr], tile[kc + 3][jr]};
        float4 h, l;
        h.x = ptx::to_tf32_rna(x[0]);
        h.y = ptx::to_tf32_rna(x[1]);
        h.z = ptx::to_tf32_rna(x[2]);
        h.w = ptx::to_tf32_rna(x[3]);
        __stcg(reinterpret_cast<float4 *>(hi + j * mp + k), h);
        if constexpr (PASSES == 3) {
            l.x = lo_part(x[0], h.x);
            l.y = lo_part(x[1], h.y);
            l.z = lo_part(x[2], h.z);
            l.w = lo_part(x[3], h.w);
            __stcg(reinterpret_cast<float4 *>(lo + j * mp + k), l);
        }
    }
}

template <int PASSES>
__global__ void __launch_bounds__(256) split_transpose64_kernel(const float *__restrict__ b,
                                                                float *__restrict__ hi,
                                                                float *__restrict__ lo, int64_t m,
                                                                int64_t p, int64_t ldb, int64_t mp) {
    asm volatile("griddepcontrol.launch_dependents;");  // let the GEMM start its prologue
    __shared__ float tile[64][65];
    split_transpose64_body<PASSES>(b, hi, lo, m, p, ldb, mp, blockIdx.x, blockIdx.y, tile);
}

// Both operand splits of one la_gemm in ONE launch (saves a launch and the
// first kernel's tail on small and mid-size problems): blocks [0, na) run the
// A pass (m % 4 == 0), the rest one 64 x 64 B tile each (the vectorised
// transpose's conditions).  Same per-element arithmetic as the two kernels.
template <int PASSES>
__global__ void __launch_bounds__(256) split_ab_kernel(const float4 *__restrict__ a, float4 *__restrict__ ahi,
                                                       float4 *__restrict__ alo, int64_t count4, int64_t na,
                                                       const float *__restrict__ b, float *__restrict__ bhi,
                                                       float *__restrict__ blo, int64_t m, int64_t p, int64_t mp,
                                                       int64_t nbx) {
    asm volatile("griddepcontrol.launch_dependents;");  // let the GEMM start its prologue
    __shared__ float tile[64][65];
    if ((int64_t)blockIdx.x < na) {
        split_rows_vec4_body<PASSES>(a, ahi, alo, count4, blockIdx.x, na);
    } else {
        const int64_t t = (int64_t)blockIdx.x - na;
        split_transpose64_body<PASSES>(b, bhi, blo, m, p, p, mp, t % nbx, t / nbx, tile);
    }
}

}  // namespace la

namespace la {

// ---- complex64 operands (Table 2 "Complex Float") ----------------
// C = A.B with A (n x m), B (m x p) complex64, interleaved (re, im).  Computed as
// one real product of the embedding
//     [ Ar  -Ai ]   [ Br ]   [ Cr ]
//     [ Ai   Ar ] . [ Bi ] = [ Ci ]        (2n x 2m) . (2m x p) = (2n x p)
// which is four real GEMMs of work; every real and imaginary output component is
// a 2m-term real inner product, so the 3xTF32 bound applies with the scales
// sum |ar||br| + |ai||bi| (real) and sum |ar||bi| + |ai||br| (imaginary).
// The split kernels write the embedding's hi/lo directly (Kp = pad4(2m) columns;
// padding columns hold 0).

// A (n x m complex) -> rows i and n+i of the 2n x Kp embedding.  One thread per
// (row i, column k), k in [0, Kp - m): k < m writes (ar, -ai) into row i and
// (ai, ar) into row n+i at columns k and m+k; k >= m zero-fills column m+k.
template <int PASSES>
__global__ void __launch_bounds__(256) split_complex_a_kernel(const float2 *__restrict__ a, float *__restrict__ hi,
                                                              float *__restrict__ lo, int64_t n, int64_t m,
                                                              int64_t kp) {
    const int64_t width = kp - m;
    for (int64_t r = blockIdx.y; r < n; r += gridDim.y) {
        for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < width;
             k += (int64_t)gridDim.x * blockDim.x) {
            const int64_t top = r * kp, bot = (n + r) * kp;
            if (k < m) {
                const float2 v = a[r * m + k];
                split_store<PASSES>(v.x, hi, lo, top + k);
                split_store<PASSES>(-v.y, hi, lo, top + m + k);
                split_store<PASSES>(v.y, hi, lo, bot + k);
                split_store<PASSES>(v.x, hi, lo, bot + m + k);
            } else {
                split_store<PASSES>(0.0f, hi, lo, top + m + k);
                split_store<PASSES>(0.0f, hi, lo, bot + m + k);
            }
        }
    }
}

// Same for even m: grid-stride over pairs of complex elements (16-byte loads,
// 8-byte stores); the padding columns [2m, Kp) of both rows are zero-filled by
// the first Kp - 2m threads of each row pair's last element.
template <int PASSES>
__device__ __forceinline__ void split_store2(float x0, float x1, float *hi, float *lo, int64_t off) {
    const float h0 = ptx::to_tf32_rna(x0), h1 = ptx::to_tf32_rna(x1);
    *reinterpret_cast<float2 *>(hi + off) = make_float2(h0, h1);
    if constexpr (PASSES == 3)
        *reinterpret_cast<float2 *>(lo + off) = make_float2(lo_part(x0, h0), lo_part(x1, h1));
}
template <int PASSES>
__global__ void __launch_bounds__(256) split_complex_a_vec_kernel(const float4 *__restrict__ a, float *__restrict__ hi,
                                                                  float *__restrict__ lo, int64_t n, int64_t m,
                                                                  int64_t kp) {
    const int64_t half = m / 2, total = n * half;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / half, k = 2 * (i - r * half);
        const float4 v = __ldcs(a + i);  // (ar_k, ai_k, ar_k+1, ai_k+1)
        const int64_t top = r * kp, bot = (n + r) * kp;
        split_store2<PASSES>(v.x, v.z, hi, lo, top + k);
        split_store2<PASSES>(-v.y, -v.w, hi, lo, top + m + k);
        split_store2<PASSES>(v.y, v.w, hi, lo, bot + k);
        split_store2<PASSES>(v.x, v.z, hi, lo, bot + m + k);
        if (k == m - 2)
            for (int64_t c = 2 * m; c < kp; c++) {
                split_store<PASSES>(0.0f, hi, lo, top + c);
                split_store<PASSES>(0.0f, hi, lo, bot + c);
            }
    }
}

// B (m x p complex) -> Bt (p x Kp): Bt[j][k] = Br[k][j], Bt[j][m + k] = Bi[k][j],
// columns [2m, Kp) zero.  32x32 complex tiles through smem; block (32, 8).
template <int PASSES>
__global__ void __launch_bounds__(256) split_complex_b_kernel(const float2 *__restrict__ b, float *__restrict__ hi,
                                                              float *__restrict__ lo, int64_t m, int64_t p,
                                                              int64_t kp) {
    __shared__ float2 tile[32][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t j0 = (int64_t)blockIdx.x * 32;
    const int64_t k0 = (int64_t)blockIdx.y * 32;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const int64_t k = k0 + ty + 8 * i, j = j0 + tx;
        tile[ty + 8 * i][tx] = (k < m && j < p) ? b[k * p + j] : make_float2(0.0f, 0.0f);
    }
    __syncthreads();
    const int64_t width = kp - m;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const int64_t j = j0 + ty + 8 * i, k = k0 + tx;
        if (j >= p || k >= width) continue;
        const float2 v = tile[tx][ty + 8 * i];
        if (k < m) {
            split_store<PASSES>(v.x, hi, lo, j * kp + k);
            split_store<PASSES>(v.y, hi, lo, j * kp + m + k);
        } else {
            split_store<PASSES>(0.0f, hi, lo, j * kp + m + k);
        }
    }
}

// ---- matrix addition / subtraction -----------------------------------
// C = A + B or A - B elementwise, one binary32 operation per element (exact IEEE
// RN: bitwise equal to any correct implementation).  HBM-bound: 12 B/element.
template <bool SUB>
__global__ void __launch_bounds__(256) elementwise_vec4_kernel(const float4 *__restrict__ a,
                                                               const float4 *__restrict__ b,
                                                               float4 *__restrict__ c, int64_t count4) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count4;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float4 x = __ldcs(a + i), y = __ldcs(b + i);
        float4 z;
        z.x = SUB ? x.x - y.x : x.x + y.x;
        z.y = SUB ? x.y - y.y : x.y + y.y;
        z.z = SUB ? x.z - y.z : x.z + y.z;
        z.w = SUB ? x.w - y.w : x.w + y.w;
        __stcs(c + i, z);
    }
}

template <bool SUB>
__global__ void __launch_bounds__(256) elementwise_kernel(const float *__restrict__ a, const float *__restrict__ b,
                                                          float *__restrict__ c, int64_t count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        c[i] = SUB ? a[i] - b[i] : a[i] + b[i];
}

}  // namespace la
