// k_tiny.cu — KN10: latency-bound small SGEMMs (2MNK <= EMM_SMALL_FLOPS).
//
// "Below this size the overhead of setting up buffers is prohibitive"
// (PAPER.md:418-420): for a 64^3 or 100^3 problem the cost is launches and
// DRAM round trips, not flops.  One launch, no workspace, 32x32 output tiles
// (many CTAs even for tiny M, N), each 64-wide K chunk loaded with all of a
// thread's loads in flight at once (16 per operand), FP32 FFMA in increasing
// k with promotion every 256 of K (FP32-accurate for every math mode).
#include <cuda_runtime.h>

#include <cstdint>

#include "emm_internal.h"

namespace emm {

constexpr int TY_T = 32;    // output tile (rows and columns)
constexpr int TY_KC = 64;   // K per chunk

template <bool TA, bool TB>
__global__ void __launch_bounds__(256) tiny_sgemm_kernel(int64_t M, int64_t N, int64_t K, float alpha,
                                                         const float *__restrict__ A, int64_t lda,
                                                         const float *__restrict__ B, int64_t ldb, float beta,
                                                         float *__restrict__ C, int64_t ldc) {
    __shared__ float As[TY_KC][TY_T + 1];   // As[k][row]
    __shared__ float Bs[TY_KC][TY_T + 1];   // Bs[k][col]
    const int tid = threadIdx.x;
    const int64_t m0 = (int64_t)blockIdx.x * TY_T, n0 = (int64_t)blockIdx.y * TY_T;
    const int tx = tid & 15, ty = tid >> 4;   // outputs rows ty*2+{0,1}, cols tx*2+{0,1}
    float acc[2][2] = {{0.f, 0.f}, {0.f, 0.f}}, mas[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
    float ra[8], rb[8];
    // element e of a 32 x 64 chunk: consecutive threads along the contiguous dimension
    auto load = [&](int64_t k0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int e = tid + 256 * i;
            const int r = TA ? e / TY_KC : e % TY_T;
            const int k = TA ? e % TY_KC : e / TY_T;
            const int64_t gr = m0 + r, gk = k0 + k;
            ra[i] = (gr < M && gk < K) ? __ldg(TA ? A + gk + gr * lda : A + gr + gk * lda) : 0.0f;
            const int c = TB ? e % TY_T : e / TY_KC;
            const int kb = TB ? e / TY_T : e % TY_KC;
            const int64_t gc = n0 + c, gkb = k0 + kb;
            rb[i] = (gc < N && gkb < K) ? __ldg(TB ? B + gc + gkb * ldb : B + gkb + gc * ldb) : 0.0f;
        }
    };
    const int64_t nchunks = (K + TY_KC - 1) / TY_KC;
    load(0);
    for (int64_t ch = 0; ch < nchunks; ++ch) {
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int e = tid + 256 * i;
            As[TA ? e % TY_KC : e / TY_T][TA ? e / TY_KC : e % TY_T] = ra[i];
            Bs[TB ? e / TY_T : e % TY_KC][TB ? e % TY_T : e / TY_KC] = rb[i];
        }
        __syncthreads();
        if (ch + 1 < nchunks) load((ch + 1) * TY_KC);
#pragma unroll 16
        for (int k = 0; k < TY_KC; ++k) {
            const float a0 = As[k][ty * 2], a1 = As[k][ty * 2 + 1];
            const float b0 = Bs[k][tx * 2], b1 = Bs[k][tx * 2 + 1];
            acc[0][0] = fmaf(a0, b0, acc[0][0]);
            acc[0][1] = fmaf(a0, b1, acc[0][1]);
            acc[1][0] = fmaf(a1, b0, acc[1][0]);
            acc[1][1] = fmaf(a1, b1, acc[1][1]);
        }
        if ((ch + 1) % (256 / TY_KC) == 0 || ch + 1 == nchunks) {
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    mas[i][j] += acc[i][j];
                    acc[i][j] = 0.0f;
                }
        }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int64_t col = n0 + tx * 2 + j;
        if (col >= N) continue;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int64_t row = m0 + ty * 2 + i;
            if (row < M) {
                float *d = C + row + col * ldc;
                *d = beta == 0.0f ? alpha * mas[i][j] : fmaf(beta, *d, alpha * mas[i][j]);
            }
        }
    }
}

cudaError_t launch_tiny_sgemm(bool tA, bool tB, int64_t M, int64_t N, int64_t K, float alpha, const float *A,
                              int64_t lda, const float *B, int64_t ldb, float beta, float *C, int64_t ldc,
                              cudaStream_t s) {
    const int64_t gx = (M + TY_T - 1) / TY_T, gy = (N + TY_T - 1) / TY_T;
    if (gx > 0x7fffffffLL || gy > 65535) return cudaErrorInvalidConfiguration;
    const dim3 grid((unsigned)gx, (unsigned)gy);
    cudaEvent_t ev = nullptr;
    prof_begin(s, true, &ev);
    if (!tA && !tB) tiny_sgemm_kernel<false, false><<<grid, 256, 0, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    else if (!tA && tB) tiny_sgemm_kernel<false, true><<<grid, 256, 0, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    else if (tA && !tB) tiny_sgemm_kernel<true, false><<<grid, 256, 0, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    else tiny_sgemm_kernel<true, true><<<grid, 256, 0, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    prof_end(s, true, ev);
    return cudaGetLastError();
}

}  // namespace emm
