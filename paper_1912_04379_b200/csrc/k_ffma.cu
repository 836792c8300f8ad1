// k_ffma.cu — KN3: FP32 FFMA SGEMM on CUDA cores (EMM_MATH_FFMA).
//
// The paper's L0 idea — "accumulate results in registers for as long as
// possible ... and re-use values in registers as much as possible"
// (§SIMD Parallelisation; 5 dot products, each loaded A
// value reused 5x) — becomes an 8x8 register tile per thread
// (64 accumulators; each loaded A value reused 8x, each B value 8x).  The L1
// block becomes a 128x128x16 SMEM tile, double buffered
// through registers (the paper's alternating xmm1/xmm2 loads).
// K/M/N tails are predicated loads (zero fill) and
// predicated stores.  Any trans / leading dimension / alignment is handled by
// the per-thread load mapping, so no packing pass is needed.
#include <cuda_runtime.h>

#include <cstdint>

#include "emm_internal.h"

namespace emm {

constexpr int FB_M = 128, FB_N = 128, FB_K = 16, FB_THREADS = 256;
constexpr int FB_PAD = 4;
// Promotion: every FB_PROMOTE K-tiles (256 of K) the 64 register partial sums
// are added (round-to-nearest) into a per-thread master copy in SMEM and
// restarted, so sequential FP32 rounding error grows with 256 + K/256 terms
// instead of K (same-sign data at K = 32768 otherwise exceeds 1e-5 * S).
constexpr int FB_PROMOTE = 16;
constexpr int FB_SMEM_BYTES = (2 * FB_K * (FB_M + FB_PAD) + 2 * FB_K * (FB_N + FB_PAD) + 64 * FB_THREADS) * 4;

template <bool TA, bool TB>
__global__ void __launch_bounds__(FB_THREADS) ffma_sgemm_kernel(int64_t M, int64_t N, int64_t K, float alpha,
                                                                const float *__restrict__ A, int64_t lda,
                                                                const float *__restrict__ B, int64_t ldb, float beta,
                                                                float *__restrict__ C, int64_t ldc) {
    extern __shared__ __align__(16) float fb_smem[];
    float(*As)[FB_K][FB_M + FB_PAD] = reinterpret_cast<float(*)[FB_K][FB_M + FB_PAD]>(fb_smem);
    float(*Bs)[FB_K][FB_N + FB_PAD] =
        reinterpret_cast<float(*)[FB_K][FB_N + FB_PAD]>(fb_smem + 2 * FB_K * (FB_M + FB_PAD));
    float *master = fb_smem + 2 * FB_K * (FB_M + FB_PAD) + 2 * FB_K * (FB_N + FB_PAD);   // [64][256]
    const int tid = threadIdx.x;
    const int64_t m0 = (int64_t)blockIdx.x * FB_M;
    const int64_t n0 = (int64_t)blockIdx.y * FB_N;

    // Load mapping: consecutive threads read consecutive addresses.
    // A (i, p): !TA -> A[i + p*lda] (i fast); TA -> A[p + i*lda] (p fast)
    // B (p, j): !TB -> B[p + j*ldb] (p fast); TB -> B[j + p*ldb] (j fast)
    auto load_a = [&](int64_t k0, float (&ra)[8]) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            int ii, pp;
            if (!TA) { ii = tid & 127; pp = (tid >> 7) + 2 * r; }
            else     { pp = tid & 15;  ii = (tid >> 4) + 16 * r; }
            const int64_t i = m0 + ii, p = k0 + pp;
            ra[r] = (i < M && p < K) ? __ldg(TA ? A + p + i * lda : A + i + p * lda) : 0.0f;
        }
    };
    auto store_a = [&](int buf, const float (&ra)[8]) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            int ii, pp;
            if (!TA) { ii = tid & 127; pp = (tid >> 7) + 2 * r; }
            else     { pp = tid & 15;  ii = (tid >> 4) + 16 * r; }
            As[buf][pp][ii] = ra[r];
        }
    };
    auto load_b = [&](int64_t k0, float (&rb)[8]) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            int jj, pp;
            if (!TB) { pp = tid & 15;  jj = (tid >> 4) + 16 * r; }
            else     { jj = tid & 127; pp = (tid >> 7) + 2 * r; }
            const int64_t j = n0 + jj, p = k0 + pp;
            rb[r] = (j < N && p < K) ? __ldg(TB ? B + j + p * ldb : B + p + j * ldb) : 0.0f;
        }
    };
    auto store_b = [&](int buf, const float (&rb)[8]) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            int jj, pp;
            if (!TB) { pp = tid & 15;  jj = (tid >> 4) + 16 * r; }
            else     { jj = tid & 127; pp = (tid >> 7) + 2 * r; }
            Bs[buf][pp][jj] = rb[r];
        }
    };

    const int tm = tid & 15, tn = tid >> 4;   // thread's 8x8 sub-tile: rows tm*4+{0..3}, 64+tm*4+{0..3}
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;

#pragma unroll
    for (int e = 0; e < 64; ++e) master[e * FB_THREADS + tid] = 0.0f;

    float ra[8], rb[8];
    load_a(0, ra);
    load_b(0, rb);
    store_a(0, ra);
    store_b(0, rb);
    __syncthreads();

    const int64_t nk = (K + FB_K - 1) / FB_K;
    for (int64_t kt = 0; kt < nk; ++kt) {
        const int buf = (int)(kt & 1);
        const bool more = kt + 1 < nk;
        if (more) {                      // prefetch the next L1 block into registers
            load_a((kt + 1) * FB_K, ra);
            load_b((kt + 1) * FB_K, rb);
        }
#pragma unroll
        for (int k = 0; k < FB_K; ++k) {
            const float4 a0 = *reinterpret_cast<const float4 *>(&As[buf][k][tm * 4]);
            const float4 a1 = *reinterpret_cast<const float4 *>(&As[buf][k][64 + tm * 4]);
            const float4 b0 = *reinterpret_cast<const float4 *>(&Bs[buf][k][tn * 4]);
            const float4 b1 = *reinterpret_cast<const float4 *>(&Bs[buf][k][64 + tn * 4]);
            const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        if (more) {
            store_a(buf ^ 1, ra);
            store_b(buf ^ 1, rb);
        }
        if ((kt + 1) % FB_PROMOTE == 0 || !more) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    master[(i * 8 + j) * FB_THREADS + tid] += acc[i][j];
                    acc[i][j] = 0.0f;
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = master[(i * 8 + j) * FB_THREADS + tid];

    // epilogue: alpha*acc + beta*C (C not read when beta == 0), predicated
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int64_t col = n0 + (j < 4 ? tn * 4 + j : 64 + tn * 4 + (j - 4));
        if (col >= N) continue;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int64_t row = m0 + (i < 4 ? tm * 4 + i : 64 + tm * 4 + (i - 4));
            if (row < M) {
                float *d = C + row + col * ldc;
                *d = beta == 0.0f ? alpha * acc[i][j] : fmaf(beta, *d, alpha * acc[i][j]);
            }
        }
    }
}

cudaError_t launch_ffma_sgemm(bool tA, bool tB, int64_t M, int64_t N, int64_t K, float alpha, const float *A,
                              int64_t lda, const float *B, int64_t ldb, float beta, float *C, int64_t ldc,
                              cudaStream_t s) {
    const int64_t gx = (M + FB_M - 1) / FB_M, gy = (N + FB_N - 1) / FB_N;
    if (gx > 0x7fffffffLL || gy > 65535) return cudaErrorInvalidConfiguration;
    dim3 grid((unsigned)gx, (unsigned)gy);
    static cudaError_t attr = [] {
        cudaError_t e = cudaSuccess;
        auto set = [&](const void *f) {
            cudaError_t r = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, FB_SMEM_BYTES);
            if (r != cudaSuccess) e = r;
        };
        set((const void *)ffma_sgemm_kernel<false, false>);
        set((const void *)ffma_sgemm_kernel<false, true>);
        set((const void *)ffma_sgemm_kernel<true, false>);
        set((const void *)ffma_sgemm_kernel<true, true>);
        return e;
    }();
    if (attr != cudaSuccess) return attr;
    cudaEvent_t ev = nullptr;
    prof_begin(s, true, &ev);
    if (!tA && !tB) ffma_sgemm_kernel<false, false><<<grid, FB_THREADS, FB_SMEM_BYTES, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    else if (!tA && tB) ffma_sgemm_kernel<false, true><<<grid, FB_THREADS, FB_SMEM_BYTES, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    else if (tA && !tB) ffma_sgemm_kernel<true, false><<<grid, FB_THREADS, FB_SMEM_BYTES, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    else ffma_sgemm_kernel<true, true><<<grid, FB_THREADS, FB_SMEM_BYTES, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    prof_end(s, true, ev);
    return cudaGetLastError();
}

}  // namespace emm
