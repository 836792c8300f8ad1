// k_ffma.cu — KN3: FP32 FFMA SGEMM on CUDA cores (EMM_MATH_FFMA).
//
// The paper's L0 idea — "accumulate results in registers for as long as
// possible ... and re-use values in registers as much as possible"
// (§SIMD Parallelisation; 5 dot products, each loaded A
// value reused 5x) — becomes an 8x8 register tile per thread
// (64 accumulators; each loaded A value reused 8x, each B value 8x).  The L1
// block becomes a 128x128x16 SMEM tile, double buffered
// through registers (the paper's alternating xmm1/xmm2 loads),
// fed by 128-bit loads along each operand's contiguous dimension (MOVAPS vs
// MOVUPS, PAPER.md:330-331 -> LDG.128 when 16-byte aligned) and computed with
// FFMA2 (two FP32 FMAs per issue slot on sm_100).
// K/M/N tails are predicated loads (zero fill) and
// predicated stores.  Any trans / leading dimension / alignment is handled by
// the per-thread load mapping, so no packing pass is needed.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "emm_internal.h"

namespace emm {

// K-tile 32 (one CTA per SM leaves the registers for it): the per-tile
// staging, barrier and address work is amortised over 2x the FFMA2s of the
// earlier K-tile 16.
constexpr int FB_M = 128, FB_N = 128, FB_K = 32, FB_THREADS = 256;
constexpr int FB_H = FB_K / 8;   // float4 staged per thread per operand tile
// Promotion: every FB_PROMOTE K-tiles (256 of K) the 64 register partial sums
// are added (round-to-nearest) into a per-thread master copy in SMEM and
// restarted, so sequential FP32 rounding error grows with 256 + K/256 terms
// instead of K (same-sign data at K = 32768 otherwise exceeds 1e-5 * S).
constexpr int FB_PROMOTE = 256 / FB_K;
constexpr int FB_SMEM_BYTES = (2 * FB_K * FB_M + 2 * FB_K * FB_N + 64 * FB_THREADS) * 4;
// SMEM tiles S[k][row] (row-contiguous, unpadded) with the 16-byte groups of
// row k XOR-swizzled by (k / 4) % 8: the transposing scalar stores of a
// K-contiguous operand (8 k x 4 rows per warp instruction) hit 32 distinct
// banks, and every float4 read stays a contiguous float4.
__device__ __forceinline__ int fb_swz(int k, int r) { return r ^ (((k >> 2) & 7) << 2); }

// Global -> register staging of one 128 x 16 (A) or 16 x 128 (B) tile with
// 128-bit loads along the operand's contiguous dimension when the whole
// float4 is in bounds and 16-byte aligned (VEC), scalar loads otherwise.
//   "MN-contiguous" (A !TA, B TB):  4 consecutive rows/cols at one k
//   "K-contiguous"  (A TA,  B !TB): 4 consecutive k at one row/col
struct TileLoad {
    float v[FB_H][4];
};

template <bool KCONT, bool VEC>
__device__ __forceinline__ void load_tile(TileLoad &t, const float *__restrict__ X, int64_t ld, int64_t r_base,
                                          int64_t R, int64_t k0, int64_t K, int tid) {
#pragma unroll
    for (int h = 0; h < FB_H; ++h) {
        int rr, kk;
        if (!KCONT) { rr = (tid & 31) * 4; kk = (tid >> 5) + 8 * h; }      // 32 float4 along rows x 32 k
        else        { kk = (tid & 7) * 4;  rr = (tid >> 3) + 32 * h; }     // 8 float4 along k x 128 rows
        const int64_t r = r_base + rr, p = k0 + kk;
        if (!KCONT) {
            const float *src = X + r + p * ld;
            if (VEC && p < K && r + 3 < R) {
                const float4 q = __ldg(reinterpret_cast<const float4 *>(src));
                t.v[h][0] = q.x; t.v[h][1] = q.y; t.v[h][2] = q.z; t.v[h][3] = q.w;
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) t.v[h][e] = (p < K && r + e < R) ? __ldg(src + e) : 0.0f;
            }
        } else {
            const float *src = X + p + r * ld;
            if (VEC && r < R && p + 3 < K) {
                const float4 q = __ldg(reinterpret_cast<const float4 *>(src));
                t.v[h][0] = q.x; t.v[h][1] = q.y; t.v[h][2] = q.z; t.v[h][3] = q.w;
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) t.v[h][e] = (r < R && p + e < K) ? __ldg(src + e) : 0.0f;
            }
        }
    }
}

// registers -> S[k][row] (row-contiguous smem tile, fb_swz-swizzled)
template <bool KCONT>
__device__ __forceinline__ void store_tile(const TileLoad &t, float (*S)[FB_M], int tid) {
#pragma unroll
    for (int h = 0; h < FB_H; ++h) {
        if (!KCONT) {
            const int rr = (tid & 31) * 4, kk = (tid >> 5) + 8 * h;
            *reinterpret_cast<float4 *>(&S[kk][fb_swz(kk, rr)]) =
                make_float4(t.v[h][0], t.v[h][1], t.v[h][2], t.v[h][3]);
        } else {
            const int kk = (tid & 7) * 4, rr = (tid >> 3) + 32 * h;
#pragma unroll
            for (int e = 0; e < 4; ++e) S[kk + e][fb_swz(kk + e, rr)] = t.v[h][e];
        }
    }
}

template <bool TA, bool TB, bool VEC>
// One CTA per SM: the 128-register cap of two CTAs spilled the prefetch
// registers (up to 332 B); without it: equal at 4096-8192, c3 281 -> 228 us.
__global__ void __launch_bounds__(FB_THREADS, 1) ffma_sgemm_kernel(int64_t M, int64_t N, int64_t K, float alpha,
                                                                const float *__restrict__ A, int64_t lda,
                                                                const float *__restrict__ B, int64_t ldb, float beta,
                                                                float *__restrict__ C, int64_t ldc) {
    extern __shared__ __align__(16) float fb_smem[];
    float(*As)[FB_K][FB_M] = reinterpret_cast<float(*)[FB_K][FB_M]>(fb_smem);
    float(*Bs)[FB_K][FB_N] = reinterpret_cast<float(*)[FB_K][FB_N]>(fb_smem + 2 * FB_K * FB_M);
    float *master = fb_smem + 2 * FB_K * FB_M + 2 * FB_K * FB_N;   // [64][256]
    const int tid = threadIdx.x;
    const int64_t m0 = (int64_t)blockIdx.x * FB_M;
    const int64_t n0 = (int64_t)blockIdx.y * FB_N;
    // op(A)(i, p): !TA -> A[i + p*lda] (MN-contiguous); TA -> A[p + i*lda] (K-contiguous)
    // op(B)(p, j): !TB -> B[p + j*ldb] (K-contiguous);  TB -> B[j + p*ldb] (MN-contiguous)
    constexpr bool A_KC = TA, B_KC = !TB;

    const int tm = tid & 15, tn = tid >> 4;   // thread's 8x8 sub-tile: rows tm*4+{0..3}, 64+tm*4+{0..3}
    // FFMA2: the 8x8 accumulators as 8 x 4 pairs of adjacent columns
    float2 acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int e = 0; e < 64; ++e) master[e * FB_THREADS + tid] = 0.0f;

    TileLoad ta, tb;
    load_tile<A_KC, VEC>(ta, A, lda, m0, M, 0, K, tid);
    load_tile<B_KC, VEC>(tb, B, ldb, n0, N, 0, K, tid);
    store_tile<A_KC>(ta, As[0], tid);
    store_tile<B_KC>(tb, Bs[0], tid);
    __syncthreads();

    const int64_t nk = (K + FB_K - 1) / FB_K;
    for (int64_t kt = 0; kt < nk; ++kt) {
        const int buf = (int)(kt & 1);
        const bool more = kt + 1 < nk;
        if (more) {                      // prefetch the next L1 block into registers
            load_tile<A_KC, VEC>(ta, A, lda, m0, M, (kt + 1) * FB_K, K, tid);
            load_tile<B_KC, VEC>(tb, B, ldb, n0, N, (kt + 1) * FB_K, K, tid);
        }
#pragma unroll
        for (int k = 0; k < FB_K; ++k) {
            const float4 a0 = *reinterpret_cast<const float4 *>(&As[buf][k][fb_swz(k, tm * 4)]);
            const float4 a1 = *reinterpret_cast<const float4 *>(&As[buf][k][fb_swz(k, 64 + tm * 4)]);
            const float4 b0 = *reinterpret_cast<const float4 *>(&Bs[buf][k][fb_swz(k, tn * 4)]);
            const float4 b1 = *reinterpret_cast<const float4 *>(&Bs[buf][k][fb_swz(k, 64 + tn * 4)]);
            const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float2 bv[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                                  make_float2(b1.z, b1.w)};
            // b pair fixed over 8 FFMA2s (operand reuse), scalar a varies
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[i][j] = __ffma2_rn(make_float2(av[i], av[i]), bv[j], acc[i][j]);
        }
        if (more) {
            store_tile<A_KC>(ta, As[buf ^ 1], tid);
            store_tile<B_KC>(tb, Bs[buf ^ 1], tid);
        }
        if ((kt + 1) % FB_PROMOTE == 0 || !more) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    master[(i * 8 + 2 * j) * FB_THREADS + tid] += acc[i][j].x;
                    master[(i * 8 + 2 * j + 1) * FB_THREADS + tid] += acc[i][j].y;
                    acc[i][j] = make_float2(0.0f, 0.0f);
                }
        }
        __syncthreads();
    }

    // epilogue: alpha*acc + beta*C (C not read when beta == 0), predicated;
    // a column's 8 C_in loads are issued before its stores (a store could
    // alias a later load through ldc: one round trip each otherwise)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int64_t col = n0 + (j < 4 ? tn * 4 + j : 64 + tn * 4 + (j - 4));
        if (col >= N) continue;
        float cin[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int64_t row = m0 + (i < 4 ? tm * 4 + i : 64 + tm * 4 + (i - 4));
            cin[i] = (beta != 0.0f && row < M) ? C[row + col * ldc] : 0.0f;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int64_t row = m0 + (i < 4 ? tm * 4 + i : 64 + tm * 4 + (i - 4));
            if (row < M) {
                const float v = master[(i * 8 + j) * FB_THREADS + tid];
                C[row + col * ldc] = beta == 0.0f ? alpha * v : fmaf(beta, cin[i], alpha * v);
            }
        }
    }
}

cudaError_t launch_ffma_sgemm(bool tA, bool tB, int64_t M, int64_t N, int64_t K, float alpha, const float *A,
                              int64_t lda, const float *B, int64_t ldb, float beta, float *C, int64_t ldc,
                              cudaStream_t s, int splits, float *partial) {
    // KN3b (TMA-fed, warp-specialised) whenever it covers the layout, split
    // over K when the caller planned it (sub-wave grids); EMM_FFMA_CLASSIC=1
    // keeps KN3 (A/B comparisons, tests; never split)
    const char *cv = getenv("EMM_FFMA_CLASSIC");
    const bool classic = cv && *cv && *cv != '0';
    if (!classic && ffma_tma_eligible(tA, tB, A, lda, B, ldb))
        return launch_ffma_tma_sgemm(tA, tB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, s, splits, partial);
    const int64_t gx = (M + FB_M - 1) / FB_M, gy = (N + FB_N - 1) / FB_N;
    if (gx > 0x7fffffffLL || gy > 65535) return cudaErrorInvalidConfiguration;
    dim3 grid((unsigned)gx, (unsigned)gy);
    static cudaError_t attr = [] {
        cudaError_t e = cudaSuccess;
        auto set = [&](const void *f) {
            cudaError_t r = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, FB_SMEM_BYTES);
            if (r != cudaSuccess) e = r;
        };
        set((const void *)ffma_sgemm_kernel<false, false, false>);
        set((const void *)ffma_sgemm_kernel<false, true, false>);
        set((const void *)ffma_sgemm_kernel<true, false, false>);
        set((const void *)ffma_sgemm_kernel<true, true, false>);
        set((const void *)ffma_sgemm_kernel<false, false, true>);
        set((const void *)ffma_sgemm_kernel<false, true, true>);
        set((const void *)ffma_sgemm_kernel<true, false, true>);
        set((const void *)ffma_sgemm_kernel<true, true, true>);
        return e;
    }();
    if (attr != cudaSuccess) return attr;
    // 128-bit loads need 16-byte aligned bases and leading dimensions
    const bool vec = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15u) == 0 &&
                     (lda & 3) == 0 && (ldb & 3) == 0;
    cudaEvent_t ev = nullptr;
    prof_begin(s, true, &ev);
#define EMM_FFMA_LAUNCH(TA_, TB_)                                                                                    \
    (vec ? ffma_sgemm_kernel<TA_, TB_, true><<<grid, FB_THREADS, FB_SMEM_BYTES, s>>>(M, N, K, alpha, A, lda, B, ldb, \
                                                                                     beta, C, ldc)                   \
         : ffma_sgemm_kernel<TA_, TB_, false><<<grid, FB_THREADS, FB_SMEM_BYTES, s>>>(M, N, K, alpha, A, lda, B,    \
                                                                                      ldb, beta, C, ldc))
    if (!tA && !tB) EMM_FFMA_LAUNCH(false, false);
    else if (!tA && tB) EMM_FFMA_LAUNCH(false, true);
    else if (tA && !tB) EMM_FFMA_LAUNCH(true, false);
    else EMM_FFMA_LAUNCH(true, true);
#undef EMM_FFMA_LAUNCH
    g_launches.fetch_add(1, std::memory_order_relaxed);
    prof_end(s, true, ev);
    return cudaGetLastError();
}

}  // namespace emm
