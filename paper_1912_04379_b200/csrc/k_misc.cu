// k_misc.cu — small HBM-bound kernels of the path.
//   KN5 scale_c:      alpha == 0 or K == 0  ->  C <- beta*C  (beta == 0: C <- 0,
//                     C never read) — BLAS semantics, reading R4.
//   KN6 unpack_rows:  after an NCCL all-gather of compact per-rank row blocks
//                     (rank-major), scatter them into the column-major M x N C.
#include <cuda_runtime.h>

#include <cstdint>

#include "emm_internal.h"

namespace emm {

__global__ void scale_c_kernel(int64_t M, int64_t N, float beta, float *__restrict__ C, int64_t ldc) {
    const int64_t total = M * N;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % M, j = e / M;
        float *d = C + i + j * ldc;
        *d = beta == 0.0f ? 0.0f : beta * *d;
    }
}

cudaError_t launch_scale_c(int64_t M, int64_t N, float beta, float *C, int64_t ldc, cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (M * N + 255) / 256;
    const int blocks = (int)(want < (int64_t)sms * 8 ? want : (int64_t)sms * 8);
    cudaEvent_t ev = nullptr;
    prof_begin(s, false, &ev);
    scale_c_kernel<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(M, N, beta, C, ldc);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    prof_end(s, false, ev);
    return cudaGetLastError();
}

struct UnpackArgs {
    int nranks;
    int64_t row0[8];
    int64_t rows[8];
    int64_t off[8];  // element offset of block r in src
};

__global__ void unpack_rows_kernel(const float *__restrict__ src, UnpackArgs a, int64_t Nc, float *__restrict__ dst,
                                   int64_t ld_dst) {
    const int r = blockIdx.y;
    const int64_t rows = a.rows[r];
    const int64_t total = rows * Nc;
    const float *s = src + a.off[r];
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % rows, j = e / rows;
        dst[a.row0[r] + i + j * ld_dst] = s[e];
    }
}

cudaError_t launch_unpack_rows(const float *src, int nranks, const int64_t *row0, const int64_t *rows, int64_t Nc,
                               float *dst, int64_t ld_dst, cudaStream_t s) {
    if (nranks < 1 || nranks > 8) return cudaErrorInvalidValue;
    UnpackArgs a{};
    a.nranks = nranks;
    int64_t off = 0;
    for (int r = 0; r < nranks; ++r) {
        a.row0[r] = row0[r];
        a.rows[r] = rows[r];
        a.off[r] = off;
        off += rows[r] * Nc;
    }
    dim3 grid(1024, (unsigned)nranks);
    unpack_rows_kernel<<<grid, 256, 0, s>>>(src, a, Nc, dst, ld_dst);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

}  // namespace emm
