// k_skinny.cu — KN9: skinny / memory-bound SGEMM.
//
// When one output dimension is tiny (N <= 16, or M <= 16 after an operand-
// role swap C^T = op(B)^T op(A)^T), the GEMM moves 4 bytes of the long
// operand per 2*N flops: arithmetic intensity ~N/2 flop/B, below the FP32 and
// tensor ridge points, so HBM bandwidth is the roofline and every byte of the
// long operand must be read exactly once.  The paper's own observation that
// "performance is better if buffering occurs on the matrix with the largest
// non-common dimension" becomes: keep the SMALL operand
// (B', K x N') resident in shared memory and stream the large one through
// registers, one row of C per thread, coalesced.
//
// Arithmetic: FP32 FFMA in increasing k, with the partial sums promoted into
// a master accumulator every 256 of K (as KN3, R13), so every math
// mode gets the FP32-accurate bound.  Deterministic (no atomics).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>

#include "emm_internal.h"
#include "ptx.cuh"

namespace emm {

// ROWS: rows of C' per CTA (one per thread); KC: K per staged chunk.

// C'(r, c) = alpha * sum_p A'(r, p) B'(p, c) + beta * C'(r, c),  r < Mr, c < Nc <= NC
//   A'(r, p) at Ap[r + p*lda] (!TA) or Ap[p + r*lda] (TA)
//   B'(p, c) at Bp[p + c*ldb] (!TB) or Bp[c + p*ldb] (TB)
//   C'(r, c) at C[r*rs + c*cs]
template <bool TA, bool TB, int NC, int SK_ROWS, int SK_KC>
__global__ void __launch_bounds__(SK_ROWS) skinny_sgemm_kernel(int64_t Mr, int Nc, int64_t K, float alpha,
                                                               const float *__restrict__ Ap, int64_t lda,
                                                               const float *__restrict__ Bp, int64_t ldb, float beta,
                                                               float *__restrict__ C, int64_t rs, int64_t cs) {
    constexpr int SK_WARPS = SK_ROWS / 32;
    constexpr int SK_PROMOTE = 256 / SK_KC;     // chunks per promotion (256 of K)
    constexpr int BPT = SK_KC * NC / SK_ROWS;   // B' elements staged per thread per chunk (>= 1 when NC >= 8)
    constexpr int BPT1 = BPT > 0 ? BPT : 1;
    __shared__ __align__(16) float Bs[2][SK_KC][NC];
    __shared__ float As[TA ? SK_ROWS : 1][TA ? SK_KC + 1 : 1];   // TA: single buffer (34 KB)
    const int tid = threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.x * SK_ROWS;
    const int64_t row = r0 + tid;
    const bool row_ok = row < Mr;
    float acc[NC], master[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = master[c] = 0.0f;

    const int64_t nchunks = (K + SK_KC - 1) / SK_KC;
    float a_next[SK_KC], b_next[BPT1];
    // Chunk ch of A' (this thread's row, or for TA a 32-wide slice of 32 rows)
    // and of B' (BPT elements) into registers: the loads of chunk ch+1 are in
    // flight while chunk ch is computed.
    auto load = [&](int64_t k0) {
        if (!TA) {
#pragma unroll
            for (int p = 0; p < SK_KC; ++p)
                a_next[p] = (row_ok && k0 + p < K) ? __ldcs(Ap + row + (k0 + p) * lda) : 0.0f;
        } else {
#pragma unroll
            for (int i = 0; i < SK_KC; ++i) {
                const int64_t r = r0 + (tid >> 5) + SK_WARPS * i;
                const int64_t p = k0 + (tid & 31);
                a_next[i] = (r < Mr && p < K) ? __ldcs(Ap + p + r * lda) : 0.0f;
            }
        }
#pragma unroll
        for (int i = 0; i < BPT1; ++i) {
            const int e = tid + i * SK_ROWS;
            const int p = TB ? e / NC : e % SK_KC;
            const int c = TB ? e % NC : e / SK_KC;
            const int64_t kk = k0 + p;
            b_next[i] = (e < SK_KC * NC && kk < K && c < Nc)
                            ? __ldg(TB ? Bp + c + kk * ldb : Bp + kk + (int64_t)c * ldb) : 0.0f;
        }
    };
    auto stage = [&](int buf) {   // registers -> shared buffer `buf`
#pragma unroll
        for (int i = 0; i < BPT1; ++i) {
            const int e = tid + i * SK_ROWS;
            if (e < SK_KC * NC) {
                const int p = TB ? e / NC : e % SK_KC;
                const int c = TB ? e % NC : e / SK_KC;
                Bs[buf][p][c] = b_next[i];
            }
        }
        if (TA) {
#pragma unroll
            for (int i = 0; i < SK_KC; ++i) As[(tid >> 5) + SK_WARPS * i][tid & 31] = a_next[i];
        }
    };
    load(0);
    stage(0);
    __syncthreads();
    for (int64_t ch = 0; ch < nchunks; ++ch) {
        const int buf = (int)(ch & 1);
        float a_cur[SK_KC];
        if (!TA) {
#pragma unroll
            for (int p = 0; p < SK_KC; ++p) a_cur[p] = a_next[p];
        }
        const bool more = ch + 1 < nchunks;
        if (more) load((ch + 1) * SK_KC);   // stream the next chunk while computing this one
#pragma unroll
        for (int p = 0; p < SK_KC; ++p) {
            const float a = TA ? As[tid][p] : a_cur[p];
#pragma unroll
            for (int c = 0; c < NC; c += 4) {
                const float4 b = *reinterpret_cast<const float4 *>(&Bs[buf][p][c]);
                acc[c] = fmaf(a, b.x, acc[c]);
                acc[c + 1] = fmaf(a, b.y, acc[c + 1]);
                acc[c + 2] = fmaf(a, b.z, acc[c + 2]);
                acc[c + 3] = fmaf(a, b.w, acc[c + 3]);
            }
        }
        if ((ch + 1) % SK_PROMOTE == 0 || !more) {
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                master[c] += acc[c];
                acc[c] = 0.0f;
            }
        }
        if (TA) __syncthreads();    // single As buffer: everyone done reading chunk ch
        if (more) stage(buf ^ 1);   // Bs: the other buffer (last read in chunk ch-1, before the barrier)
        __syncthreads();
    }
    if (!row_ok) return;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        if (c < Nc) {
            float *d = C + row * rs + (int64_t)c * cs;
            *d = beta == 0.0f ? alpha * master[c] : fmaf(beta, *d, alpha * master[c]);
        }
    }
}

template <bool TA, bool TB, int ROWS, int KC>
static cudaError_t launch_cfg(int64_t Mr, int Nc, int64_t K, float alpha, const float *Ap, int64_t lda,
                             const float *Bp, int64_t ldb, float beta, float *C, int64_t rs, int64_t cs,
                             cudaStream_t s) {
    const dim3 grid((unsigned)((Mr + ROWS - 1) / ROWS));
    if (Nc <= 4)
        skinny_sgemm_kernel<TA, TB, 4, ROWS, KC><<<grid, ROWS, 0, s>>>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C,
                                                                        rs, cs);
    else if (Nc <= 8)
        skinny_sgemm_kernel<TA, TB, 8, ROWS, KC><<<grid, ROWS, 0, s>>>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C,
                                                                        rs, cs);
    else
        skinny_sgemm_kernel<TA, TB, 16, ROWS, KC><<<grid, ROWS, 0, s>>>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C,
                                                                         rs, cs);
    return cudaGetLastError();
}

template <bool TA, bool TB>
static cudaError_t launch_nc(int64_t Mr, int Nc, int64_t K, float alpha, const float *Ap, int64_t lda,
                             const float *Bp, int64_t ldb, float beta, float *C, int64_t rs, int64_t cs,
                             cudaStream_t s) {
    int cfg = TA ? 0 : 2;
    if (const char *e = getenv("EMM_SKINNY_CFG")) cfg = atoi(e);   // experiments
    if (TA) cfg = cfg == 1 ? 1 : 0;   // the TA staging needs KC == 32
    switch (cfg) {
        case 1: return launch_cfg<TA, TB, 128, 32>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C, rs, cs, s);
        case 2: return launch_cfg<TA, TB, 256, 16>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C, rs, cs, s);
        case 3: return launch_cfg<TA, TB, 128, 16>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C, rs, cs, s);
        default: return launch_cfg<TA, TB, 256, 32>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C, rs, cs, s);
    }
}


// ---------------------------------------------------------------------------
// TMA streaming variant (both operands TMA-legal).  Persistent CTAs walk
// 256-row blocks of C'; one producer warp streams 256 x 32 tiles of A' and
// 32 x NC tiles of B' through a 4-stage mbarrier ring; 8 compute warps (one
// row of C' per thread) consume them.  A' tiles: !TA -> [32 p][256 rows]
// (row-contiguous, no swizzle); TA -> [256 rows][32 p] (128B swizzle, read as
// 16-byte chunks).  B' tiles: !TB -> [NC][32 p]; TB -> [32 p][NC].
// ---------------------------------------------------------------------------
namespace {
constexpr int SKT_TPB = 256, SKT_KC = 32;        // compute threads per CTA, K per stage
constexpr int SKT_THREADS = SKT_TPB + 32;        // + one producer warp
}  // namespace

// RPT rows of C' per compute thread (rows tid, tid + 256, ...): the B'
// broadcast loads are shared by RPT rows.
template <bool TA, bool TB, int NC, int RPT>
__global__ void __launch_bounds__(SKT_THREADS, 1)
    skinny_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int64_t Mr,
                      int Nc, int64_t K, float alpha, float beta, float *__restrict__ C, int64_t rs, int64_t cs) {
    using namespace ptx;
    constexpr int SKT_ROWS = SKT_TPB * RPT;
    constexpr int SKT_STAGES = RPT == 1 ? 4 : 3;
    constexpr int SKT_A_BYTES = SKT_ROWS * SKT_KC * 4;
    constexpr int B_BYTES = SKT_KC * NC * 4;
    constexpr int STAGE = SKT_A_BYTES + ((B_BYTES + 1023) / 1024) * 1024;
    extern __shared__ uint8_t skt_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(skt_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + SKT_STAGES * STAGE);
    uint64_t *empty = full + SKT_STAGES;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t nblocks = (Mr + SKT_ROWS - 1) / SKT_ROWS;
    const int64_t nchunks = (K + SKT_KC - 1) / SKT_KC;
    if (tid == 0) {
        for (int s = 0; s < SKT_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], SKT_TPB / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == SKT_TPB / 32) {
        // ===== producer =====
        if (lane == 0) {
            prefetch_tmap(&tmA);
            prefetch_tmap(&tmB);
            const uint64_t pa = policy_evict_first(), pb = policy_evict_last();
            int64_t it = 0;
            for (int64_t rb = blockIdx.x; rb < nblocks; rb += gridDim.x) {
                for (int64_t ch = 0; ch < nchunks; ++ch, ++it) {
                    const int s = (int)(it % SKT_STAGES);
                    mbar_wait(&empty[s], ((uint32_t)(it / SKT_STAGES) & 1u) ^ 1u);
                    mbar_arrive_expect_tx(&full[s], (uint32_t)(SKT_A_BYTES + B_BYTES));
                    const uint32_t st = smem_u32(smem + s * STAGE);
                    const int32_t r0 = (int32_t)(rb * SKT_ROWS), k0 = (int32_t)(ch * SKT_KC);
#pragma unroll
                    for (int h = 0; h < RPT; ++h) {   // 256-row boxes
                        if (!TA) tma_load_2d(st + h * SKT_TPB * SKT_KC * 4, &tmA, &full[s], r0 + h * SKT_TPB, k0, pa);
                        else tma_load_2d(st + h * SKT_TPB * SKT_KC * 4, &tmA, &full[s], k0, r0 + h * SKT_TPB, pa);
                    }
                    if (!TB) tma_load_2d(st + SKT_A_BYTES, &tmB, &full[s], k0, 0, pb);
                    else tma_load_2d(st + SKT_A_BYTES, &tmB, &full[s], 0, k0, pb);
                }
            }
        }
        return;
    }
    // ===== compute warps: RPT rows of C' per thread =====
    int64_t it = 0;
    for (int64_t rb = blockIdx.x; rb < nblocks; rb += gridDim.x) {
        float acc[RPT][NC], master[RPT][NC];
#pragma unroll
        for (int h = 0; h < RPT; ++h)
#pragma unroll
            for (int c = 0; c < NC; ++c) acc[h][c] = master[h][c] = 0.0f;
        for (int64_t ch = 0; ch < nchunks; ++ch, ++it) {
            const int s = (int)(it % SKT_STAGES);
            mbar_wait(&full[s], (uint32_t)(it / SKT_STAGES) & 1u);
            const float *As = reinterpret_cast<const float *>(smem + s * STAGE);
            const float *Bs = reinterpret_cast<const float *>(smem + s * STAGE + SKT_A_BYTES);
#pragma unroll
            for (int j = 0; j < SKT_KC / 4; ++j) {
                float4 a[RPT];
#pragma unroll
                for (int h = 0; h < RPT; ++h) {
                    const float *Ah = As + h * SKT_TPB * SKT_KC;   // box h
                    if (!TA) {
                        a[h].x = Ah[(4 * j + 0) * SKT_TPB + tid];
                        a[h].y = Ah[(4 * j + 1) * SKT_TPB + tid];
                        a[h].z = Ah[(4 * j + 2) * SKT_TPB + tid];
                        a[h].w = Ah[(4 * j + 3) * SKT_TPB + tid];
                    } else {   // 128B swizzle: 16-byte chunk j of row tid sits at chunk j ^ (tid & 7)
                        a[h] = *reinterpret_cast<const float4 *>(Ah + tid * SKT_KC + 4 * (j ^ (tid & 7)));
                    }
                }
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    float4 b;
                    if (!TB) {
                        b = *reinterpret_cast<const float4 *>(Bs + c * SKT_KC + 4 * j);
                    } else {
                        b.x = Bs[(4 * j + 0) * NC + c];
                        b.y = Bs[(4 * j + 1) * NC + c];
                        b.z = Bs[(4 * j + 2) * NC + c];
                        b.w = Bs[(4 * j + 3) * NC + c];
                    }
#pragma unroll
                    for (int h = 0; h < RPT; ++h) {   // increasing k within each entry's sum
                        acc[h][c] = fmaf(a[h].x, b.x, acc[h][c]);
                        acc[h][c] = fmaf(a[h].y, b.y, acc[h][c]);
                        acc[h][c] = fmaf(a[h].z, b.z, acc[h][c]);
                        acc[h][c] = fmaf(a[h].w, b.w, acc[h][c]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if ((ch + 1) % (256 / SKT_KC) == 0 || ch + 1 == nchunks) {
#pragma unroll
                for (int h = 0; h < RPT; ++h)
#pragma unroll
                    for (int c = 0; c < NC; ++c) {
                        master[h][c] += acc[h][c];
                        acc[h][c] = 0.0f;
                    }
            }
        }
#pragma unroll
        for (int h = 0; h < RPT; ++h) {
            const int64_t row = rb * SKT_ROWS + h * SKT_TPB + tid;
            if (row < Mr) {
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    if (c < Nc) {
                        float *d = C + row * rs + (int64_t)c * cs;
                        *d = beta == 0.0f ? alpha * master[h][c] : fmaf(beta, *d, alpha * master[h][c]);
                    }
            }
        }
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 skinny_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    }();
    return fn;
}

static bool skinny_tmap(CUtensorMap *tm, const float *ptr, int64_t ld, uint64_t d0, uint64_t d1, uint32_t b0,
                        uint32_t b1, bool swz) {
    auto enc = skinny_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {d0, d1}, strides[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {b0, b1}, estr[2] = {1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(ptr), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool TA, bool TB, int NC, int RPT>
static cudaError_t launch_tma_nc(int64_t Mr, int Nc, int64_t K, float alpha, const float *Ap, int64_t lda,
                                 const float *Bp, int64_t ldb, float beta, float *C, int64_t rs, int64_t cs,
                                 cudaStream_t s) {
    constexpr int ROWS = SKT_TPB * RPT;
    constexpr int STAGES = RPT == 1 ? 4 : 3;
    constexpr int B_BYTES = SKT_KC * NC * 4;
    constexpr int STAGE = ROWS * SKT_KC * 4 + ((B_BYTES + 1023) / 1024) * 1024;
    constexpr int SMEM = STAGES * STAGE + 1024 + 128;
    static cudaError_t attr = cudaFuncSetAttribute(skinny_tma_kernel<TA, TB, NC, RPT>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (attr != cudaSuccess) return attr;
    CUtensorMap ta, tb;
    const bool ok_a = !TA ? skinny_tmap(&ta, Ap, lda, (uint64_t)Mr, (uint64_t)K, SKT_TPB, SKT_KC, false)
                          : skinny_tmap(&ta, Ap, lda, (uint64_t)K, (uint64_t)Mr, SKT_KC, SKT_TPB, true);
    const bool ok_b = !TB ? skinny_tmap(&tb, Bp, ldb, (uint64_t)K, (uint64_t)Nc, SKT_KC, NC, false)
                          : skinny_tmap(&tb, Bp, ldb, (uint64_t)Nc, (uint64_t)K, NC, SKT_KC, false);
    if (!ok_a || !ok_b) return cudaErrorInvalidValue;
    const int64_t nblocks = (Mr + ROWS - 1) / ROWS;
    const int64_t grid = nblocks < tc_num_sms() ? nblocks : tc_num_sms();
    skinny_tma_kernel<TA, TB, NC, RPT><<<(unsigned)grid, SKT_THREADS, SMEM, s>>>(ta, tb, Mr, Nc, K, alpha, beta, C,
                                                                                  rs, cs);
    return cudaGetLastError();
}

template <bool TA, bool TB>
static cudaError_t launch_tma(int64_t Mr, int Nc, int64_t K, float alpha, const float *Ap, int64_t lda,
                              const float *Bp, int64_t ldb, float beta, float *C, int64_t rs, int64_t cs,
                              cudaStream_t s) {
    int rpt = 2;
    if (const char *e = getenv("EMM_SKINNY_RPT")) rpt = atoi(e);   // experiments
    if (rpt == 1) {
        if (Nc <= 4) return launch_tma_nc<TA, TB, 4, 1>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C, rs, cs, s);
        if (Nc <= 8) return launch_tma_nc<TA, TB, 8, 1>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C, rs, cs, s);
        return launch_tma_nc<TA, TB, 16, 1>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C, rs, cs, s);
    }
    if (Nc <= 4) return launch_tma_nc<TA, TB, 4, 2>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C, rs, cs, s);
    if (Nc <= 8) return launch_tma_nc<TA, TB, 8, 2>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C, rs, cs, s);
    return launch_tma_nc<TA, TB, 16, 2>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C, rs, cs, s);
}

cudaError_t launch_skinny_sgemm(bool tA, bool tB, int64_t M, int64_t N, int64_t K, float alpha, const float *A,
                                int64_t lda, const float *B, int64_t ldb, float beta, float *C, int64_t ldc,
                                cudaStream_t s) {
    // Roles: the long output dimension is streamed (rows of C'), the short one
    // (<= SKINNY_MAX) is resident.  N short: C' = C, A' = op(A), B' = op(B).
    // M short: C' = C^T = op(B)^T op(A)^T, A' = op(B)^T, B' = op(A)^T.
    bool TA, TB;
    int64_t Mr, lda2, ldb2, rs, cs;
    int Nc;
    const float *Ap, *Bp;
    if (N <= SKINNY_MAX) {
        Mr = M; Nc = (int)N;
        Ap = A; lda2 = lda; TA = tA;          // op(A)(r,p): tA ? A[p + r*lda] : A[r + p*lda]
        Bp = B; ldb2 = ldb; TB = tB;          // op(B)(p,c): tB ? B[c + p*ldb] : B[p + c*ldb]
        rs = 1; cs = ldc;
    } else {
        Mr = N; Nc = (int)M;
        // A'(r,p) = op(B)(p,r): tB ? B[r + p*ldb] (r contiguous: !TA) : B[p + r*ldb] (TA)
        Ap = B; lda2 = ldb; TA = !tB;
        // B'(p,c) = op(A)(c,p): tA ? A[p + c*lda] (!TB form) : A[c + p*lda] (TB form)
        Bp = A; ldb2 = lda; TB = !tA;
        rs = ldc; cs = 1;
    }
    if ((Mr + 127) / 128 > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    cudaEvent_t ev = nullptr;
    prof_begin(s, true, &ev);
    cudaError_t e;
    const bool tma = tma_legal(Ap, lda2) && tma_legal(Bp, ldb2) && !getenv("EMM_SKINNY_NO_TMA") && K > 0;
    if (tma) {
        if (!TA && !TB) e = launch_tma<false, false>(Mr, Nc, K, alpha, Ap, lda2, Bp, ldb2, beta, C, rs, cs, s);
        else if (!TA && TB) e = launch_tma<false, true>(Mr, Nc, K, alpha, Ap, lda2, Bp, ldb2, beta, C, rs, cs, s);
        else if (TA && !TB) e = launch_tma<true, false>(Mr, Nc, K, alpha, Ap, lda2, Bp, ldb2, beta, C, rs, cs, s);
        else e = launch_tma<true, true>(Mr, Nc, K, alpha, Ap, lda2, Bp, ldb2, beta, C, rs, cs, s);
    } else if (!TA && !TB) e = launch_nc<false, false>(Mr, Nc, K, alpha, Ap, lda2, Bp, ldb2, beta, C, rs, cs, s);
    else if (!TA && TB) e = launch_nc<false, true>(Mr, Nc, K, alpha, Ap, lda2, Bp, ldb2, beta, C, rs, cs, s);
    else if (TA && !TB) e = launch_nc<true, false>(Mr, Nc, K, alpha, Ap, lda2, Bp, ldb2, beta, C, rs, cs, s);
    else e = launch_nc<true, true>(Mr, Nc, K, alpha, Ap, lda2, Bp, ldb2, beta, C, rs, cs, s);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    prof_end(s, true, ev);
    return e;
}

}  // namespace emm
