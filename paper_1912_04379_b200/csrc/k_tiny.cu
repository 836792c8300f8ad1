// k_tiny.cu — KN10: latency-bound small SGEMMs (2MNK <= EMM_SMALL_FLOPS).
//
// "Below this size the overhead of setting up buffers is prohibitive"
// (PAPER.md:418-420): for a 64^3 or 100^3 problem the cost is launches and
// DRAM round trips, not flops.  One launch, no workspace, 32x32 output tiles
// (many CTAs even for tiny M, N), each 64-wide K chunk loaded with all of a
// thread's loads in flight at once (8 per operand), FP32 FFMA with promotion
// every 256 of K (FP32-accurate for every math mode).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "emm_internal.h"

namespace emm {

// Tile geometry (T = 32 or 64 output rows and columns per block): 256
// threads of 4 x 4 outputs each; G = 256 / (T/4)^2 thread groups split every
// 64-wide K chunk (T = 32: four groups of 64 threads, k = 16g .. 16g+15;
// T = 64: one group).  T = 64 (the FFMA mode's mid sizes) quarters the shared
// and L2 traffic per flop against T = 32 at a quarter of the blocks.
constexpr int TY_KC = 64;   // K per chunk
template <int T>
struct TyCfg {
    static constexpr int ST = T == 32 ? 4 : 3;       // chunks in flight (cp.async ring; T = 64: 2 blocks per SM)
    static constexpr int LD = T + 4;                 // shared row pitch: 16-B aligned 4-row / 4-column groups
    static constexpr int TPG = (T / 4) * (T / 4);    // threads per K group
    static constexpr int G = 256 / TPG;              // K groups
    static constexpr int KG = TY_KC / G;             // k per group per chunk
    static constexpr int STAGE = 2 * TY_KC * LD;     // floats per stage: As[k][row] | Bs[k][col]
    static constexpr int SMEM = ST * STAGE * 4;
    static constexpr int EPT = T * TY_KC / 256;      // elements per operand per thread per chunk
};

// 4-byte async copy, zero-filled (nothing read; `base` is a valid dummy
// address) when the element is outside the matrix
__device__ __forceinline__ void ty_cp4(float *dst, const float *src, const float *base, bool ok) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(ok ? src : base), "r"(ok ? 4 : 0)
                 : "memory");
}

// Block = 256 threads on one T x T tile; a thread computes a 4 x 4 sub-tile
// from two 128-bit shared loads per k (16 FMAs per 2 loads; round 1's 2 x 2
// per thread needed one load per FMA and was LDS-bound), promotes into its
// master every 256 of K, and the G groups' masters are added in fixed order
// g = 0..G-1 at the end (deterministic).  Operands reach shared memory by
// cp.async (4-byte, zero-filled outside the matrices, transposed on the fly)
// in a ring of ST K chunks, so up to ST chunks' DRAM latencies overlap
// instead of one per chunk.
template <bool TA, bool TB, int T>
__global__ void __launch_bounds__(256) tiny_sgemm_kernel(int64_t M, int64_t N, int64_t K, float alpha,
                                                         const float *__restrict__ A, int64_t lda,
                                                         const float *__restrict__ B, int64_t ldb, float beta,
                                                         float *__restrict__ C, int64_t ldc) {
    using Cf = TyCfg<T>;
    constexpr int LD = Cf::LD, G = Cf::G, KG = Cf::KG, TY_ST = Cf::ST;
    extern __shared__ __align__(16) float sm[];
    const int tid = threadIdx.x;
    const int64_t m0 = (int64_t)blockIdx.x * T, n0 = (int64_t)blockIdx.y * T;
    const int g = tid / Cf::TPG, lt = tid % Cf::TPG;
    const int ty = lt / (T / 4), tx = lt % (T / 4);   // rows 4ty..4ty+3, cols 4tx..4tx+3
    float acc[4][4], mas[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = mas[i][j] = 0.0f;
    // chunk ch into its ring stage: element e of a T x 64 chunk, consecutive
    // threads along the contiguous dimension of the source
    auto issue = [&](int64_t ch) {
        float *As = sm + (ch % TY_ST) * Cf::STAGE, *Bs = As + TY_KC * LD;
        const int64_t k0 = ch * TY_KC;
#pragma unroll
        for (int i = 0; i < Cf::EPT; ++i) {
            const int e = tid + 256 * i;
            const int r = TA ? e / TY_KC : e % T;
            const int k = TA ? e % TY_KC : e / T;
            const int64_t gr = m0 + r, gk = k0 + k;
            ty_cp4(As + k * LD + r, TA ? A + gk + gr * lda : A + gr + gk * lda, A, gr < M && gk < K);
            const int c = TB ? e % T : e / TY_KC;
            const int kb = TB ? e / T : e % TY_KC;
            const int64_t gc = n0 + c, gkb = k0 + kb;
            ty_cp4(Bs + kb * LD + c, TB ? B + gc + gkb * ldb : B + gkb + gc * ldb, B, gc < N && gkb < K);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const int64_t nchunks = (K + TY_KC - 1) / TY_KC;
#pragma unroll
    for (int c = 0; c < TY_ST - 1; ++c)
        if (c < nchunks) issue(c);
        else asm volatile("cp.async.commit_group;" ::: "memory");   // keep the group count uniform
    for (int64_t ch = 0; ch < nchunks; ++ch) {
        if (ch + TY_ST - 1 < nchunks) issue(ch + TY_ST - 1);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group %0;" ::"n"(TY_ST - 1) : "memory");   // chunk ch (this thread's copies)
        __syncthreads();                                                         // ... and everyone's
        const float *As = sm + (ch % TY_ST) * Cf::STAGE, *Bs = As + TY_KC * LD;
#pragma unroll
        for (int kk = 0; kk < KG; ++kk) {
            const int k = KG * g + kk;
            const float4 a = *reinterpret_cast<const float4 *>(As + k * LD + 4 * ty);
            const float4 b = *reinterpret_cast<const float4 *>(Bs + k * LD + 4 * tx);
            const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        if ((ch + 1) % (256 / TY_KC) == 0 || ch + 1 == nchunks) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    mas[i][j] += acc[i][j];
                    acc[i][j] = 0.0f;
                }
        }
        __syncthreads();   // stage ch % TY_ST is refilled by the next iteration's issue
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    // the G K-groups' partials: red[g][col][row], summed in order g = 0..G-1
    float *red = sm;   // G x T x T floats <= the ring
#pragma unroll
    for (int j = 0; j < 4; ++j)
        *reinterpret_cast<float4 *>(red + g * T * T + (4 * tx + j) * T + 4 * ty) =
            make_float4(mas[0][j], mas[1][j], mas[2][j], mas[3][j]);
    __syncthreads();
    // beta != 0: all of this thread's C_in loads first (a store could alias a
    // later load through ldc, so they would otherwise run one round trip each)
    float cin[T * T / 256];
#pragma unroll
    for (int q = 0; q < T * T / 256; ++q) {
        const int o = tid + 256 * q;
        const int64_t grow = m0 + o % T, gcol = n0 + o / T;
        cin[q] = (beta != 0.0f && grow < M && gcol < N) ? C[grow + gcol * ldc] : 0.0f;
    }
#pragma unroll
    for (int q = 0; q < T * T / 256; ++q) {
        const int o = tid + 256 * q;   // output (row = o % T, col = o / T): coalesced along rows
        const int row = o % T, colo = o / T;
        float v = red[o];
#pragma unroll
        for (int gg = 1; gg < G; ++gg) v += red[gg * T * T + o];
        const int64_t grow = m0 + row, gcol = n0 + colo;
        if (grow < M && gcol < N) C[grow + gcol * ldc] = beta == 0.0f ? alpha * v : fmaf(beta, cin[q], alpha * v);
    }
}

template <int T>
static cudaError_t launch_tiny_t(bool tA, bool tB, int64_t M, int64_t N, int64_t K, float alpha, const float *A,
                                 int64_t lda, const float *B, int64_t ldb, float beta, float *C, int64_t ldc,
                                 cudaStream_t s) {
    constexpr int SMEM = TyCfg<T>::SMEM;
    static const cudaError_t attr = [] {
        cudaError_t e = cudaSuccess;
        const void *fs[4] = {(const void *)tiny_sgemm_kernel<false, false, T>,
                             (const void *)tiny_sgemm_kernel<false, true, T>,
                             (const void *)tiny_sgemm_kernel<true, false, T>,
                             (const void *)tiny_sgemm_kernel<true, true, T>};
        for (int i = 0; i < 4 && e == cudaSuccess; ++i)
            e = cudaFuncSetAttribute(fs[i], cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        return e;
    }();
    if (attr != cudaSuccess) return attr;
    const int64_t gx = (M + T - 1) / T, gy = (N + T - 1) / T;
    if (gx > 0x7fffffffLL || gy > 65535) return cudaErrorInvalidConfiguration;
    const dim3 grid((unsigned)gx, (unsigned)gy);
    cudaEvent_t ev = nullptr;
    prof_begin(s, true, &ev);
    if (!tA && !tB) tiny_sgemm_kernel<false, false, T><<<grid, 256, SMEM, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    else if (!tA && tB) tiny_sgemm_kernel<false, true, T><<<grid, 256, SMEM, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    else if (tA && !tB) tiny_sgemm_kernel<true, false, T><<<grid, 256, SMEM, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    else tiny_sgemm_kernel<true, true, T><<<grid, 256, SMEM, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    prof_end(s, true, ev);
    return cudaGetLastError();
}

// T = 64 once the 32 x 32 grid has more than two blocks per SM (the mid-size
// FFMA-mode problems; measured: 512^3 T32 22.5 vs T64 29.2 us, 700^3 47.1 vs
// 38.9, 1024^3 106.6 vs 88.0 — profiles/r02_small_threshold.md);
// EMM_TINY_T=32 / 64 forces.
cudaError_t launch_tiny_sgemm(bool tA, bool tB, int64_t M, int64_t N, int64_t K, float alpha, const float *A,
                              int64_t lda, const float *B, int64_t ldb, float beta, float *C, int64_t ldc,
                              cudaStream_t s) {
    const double tiles32 = (double)((M + 31) / 32) * (double)((N + 31) / 32);
    bool t64 = tiles32 > 2.0 * tc_num_sms();
    if (const char *e = getenv("EMM_TINY_T")) t64 = atoi(e) == 64;
    return t64 ? launch_tiny_t<64>(tA, tB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, s)
               : launch_tiny_t<32>(tA, tB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, s);
}

}  // namespace emm
