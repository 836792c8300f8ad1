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

#include <algorithm>
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
    float cin[NC];   // C_in loads before the stores (see skinny_tma_kernel)
#pragma unroll
    for (int c = 0; c < NC; ++c) cin[c] = (beta != 0.0f && c < Nc) ? C[row * rs + (int64_t)c * cs] : 0.0f;
#pragma unroll
    for (int c = 0; c < NC; ++c)
        if (c < Nc) C[row * rs + (int64_t)c * cs] = beta == 0.0f ? alpha * master[c] : fmaf(beta, cin[c], alpha * master[c]);
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

// RPT rows of C' per compute thread (RPT = 1: row tid; RPT = 2: rows 2 tid,
// 2 tid + 1 as an FFMA2 pair): the B' broadcast loads are shared by RPT rows.
template <bool TA, bool TB, int NC, int RPT, int TPB>
__global__ void __launch_bounds__(TPB + 32, 1)
    skinny_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int64_t Mr,
                      int Nc, int64_t K, float alpha, float beta, float *__restrict__ C, int64_t rs, int64_t cs,
                      int splits, float *__restrict__ partial) {
    using namespace ptx;
    constexpr int SKT_ROWS = TPB * RPT;
    constexpr int SKT_STAGES = RPT == 1 ? 4 : 3;
    constexpr int SKT_A_BYTES = SKT_ROWS * SKT_KC * 4;
    constexpr int B_BYTES = SKT_KC * NC * 4;
    constexpr int STAGE = SKT_A_BYTES + ((B_BYTES + 1023) / 1024) * 1024;
    extern __shared__ uint8_t skt_raw[];
    // offset arithmetic on the shared array (an integer round trip would turn
    // the operand reads into generic LD, long-scoreboard loads)
    uint8_t *smem = skt_raw + ((1024u - (ptx::smem_u32(skt_raw) & 1023u)) & 1023u);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + SKT_STAGES * STAGE);
    uint64_t *empty = full + SKT_STAGES;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t nblocks = (Mr + SKT_ROWS - 1) / SKT_ROWS;
    const int64_t nchunks = (K + SKT_KC - 1) / SKT_KC;
    // split-K (few row blocks, long K): unit u = (row block u % nblocks,
    // split u / nblocks); split sp runs the 256-of-K promotion groups
    // [sp*ng/S, (sp+1)*ng/S) and stores its raw master to partial slab sp
    constexpr int PROM = 256 / SKT_KC;
    const int64_t ngroups = (nchunks + PROM - 1) / PROM, nunits = nblocks * splits;
    auto unit = [&](int64_t u, int64_t &rb, int &sp, int64_t &c0, int64_t &c1) {
        rb = u % nblocks;
        sp = (int)(u / nblocks);
        c0 = min(nchunks, sp * ngroups / splits * PROM);
        c1 = min(nchunks, (sp + 1) * ngroups / splits * PROM);
    };
    auto store = [&](int64_t row, int c, int sp, float v, float cin) {
        if (partial) partial[((size_t)sp * Nc + c) * Mr + row] = v;
        else C[row * rs + (int64_t)c * cs] = beta == 0.0f ? alpha * v : fmaf(beta, cin, alpha * v);
    };
    // beta != 0: a thread's C_in values (rows row0 + h*step) loaded before any
    // of its stores (a store could alias a later load through ldc, so they
    // would otherwise run one round trip each)
    auto load_cin = [&](int64_t row0, int64_t step, auto &cin) {
        constexpr int H = sizeof(cin) / sizeof(cin[0]);
#pragma unroll
        for (int h = 0; h < H; ++h) {
            const int64_t row = row0 + h * step;
#pragma unroll
            for (int c = 0; c < NC; ++c)
                cin[h][c] = (!partial && beta != 0.0f && row < Mr && c < Nc) ? C[row * rs + (int64_t)c * cs] : 0.0f;
        }
    };
    if (tid == 0) {
        for (int s = 0; s < SKT_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], TPB / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == TPB / 32) {
        // ===== producer =====
        if (lane == 0) {
            prefetch_tmap(&tmA);
            prefetch_tmap(&tmB);
            const uint64_t pa = policy_evict_first(), pb = policy_evict_last();
            int64_t it = 0;
            for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
                int64_t rb, ch0, ch1;
                int sp;
                unit(u, rb, sp, ch0, ch1);
                for (int64_t ch = ch0; ch < ch1; ++ch, ++it) {
                    const int s = (int)(it % SKT_STAGES);
                    mbar_wait(&empty[s], ((uint32_t)(it / SKT_STAGES) & 1u) ^ 1u);
                    mbar_arrive_expect_tx(&full[s], (uint32_t)(SKT_A_BYTES + B_BYTES));
                    const uint32_t st = smem_u32(smem + s * STAGE);
                    const int32_t r0 = (int32_t)(rb * SKT_ROWS), k0 = (int32_t)(ch * SKT_KC);
#pragma unroll
                    for (int h = 0; h < RPT; ++h) {   // 256-row boxes
                        if (!TA) tma_load_2d(st + h * TPB * SKT_KC * 4, &tmA, &full[s], r0 + h * TPB, k0, pa);
                        else tma_load_2d(st + h * TPB * SKT_KC * 4, &tmA, &full[s], k0, r0 + h * TPB, pa);
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
    if (RPT == 2 && !TA) {
        // rows 2t and 2t+1 of the 512-row block: one float2 of A' per k is
        // an FFMA2 operand pair (the two rows), the column value of B' the
        // broadcast one — two FP32 FMAs per issue slot, each entry's sum in
        // increasing k exactly as the scalar form (same bits)
        const int rl = 2 * tid;                                 // row pair within the block
        const int hb = rl / TPB, rb_l = rl % TPB;       // its TPB-row box, row in the box
        for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
            int64_t rb, ch0, ch1;
            int sp;
            unit(u, rb, sp, ch0, ch1);
            float2 acc[NC], master[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) acc[c] = master[c] = make_float2(0.0f, 0.0f);
            for (int64_t ch = ch0; ch < ch1; ++ch, ++it) {
                const int s = (int)(it % SKT_STAGES);
                mbar_wait(&full[s], (uint32_t)(it / SKT_STAGES) & 1u);
                const float *Ah = reinterpret_cast<const float *>(smem + s * STAGE) + hb * TPB * SKT_KC;
                const float *Bs = reinterpret_cast<const float *>(smem + s * STAGE + SKT_A_BYTES);
#pragma unroll 1
                for (int j = 0; j < SKT_KC / 4; ++j) {   // not unrolled: B' values of one j only (no spills)
                    float2 a[4];
                    if (!TA) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            a[kk] = *reinterpret_cast<const float2 *>(Ah + (4 * j + kk) * TPB + rb_l);
                    } else {   // 128B swizzle: 16-byte chunk j of row r sits at chunk j ^ (r & 7)
                        const float4 x0 = *reinterpret_cast<const float4 *>(Ah + rb_l * SKT_KC + 4 * (j ^ (rb_l & 7)));
                        const float4 x1 =
                            *reinterpret_cast<const float4 *>(Ah + (rb_l + 1) * SKT_KC + 4 * (j ^ ((rb_l + 1) & 7)));
                        a[0] = make_float2(x0.x, x1.x);
                        a[1] = make_float2(x0.y, x1.y);
                        a[2] = make_float2(x0.z, x1.z);
                        a[3] = make_float2(x0.w, x1.w);
                    }
#pragma unroll
                    for (int c = 0; c < NC; ++c) {
                        float b[4];
                        if (!TB) {
                            const float4 v = *reinterpret_cast<const float4 *>(Bs + c * SKT_KC + 4 * j);
                            b[0] = v.x; b[1] = v.y; b[2] = v.z; b[3] = v.w;
                        } else {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) b[kk] = Bs[(4 * j + kk) * NC + c];
                        }
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) acc[c] = __ffma2_rn(a[kk], make_float2(b[kk], b[kk]), acc[c]);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                if ((ch + 1) % PROM == 0 || ch + 1 == ch1) {
#pragma unroll
                    for (int c = 0; c < NC; ++c) {
                        master[c].x += acc[c].x;
                        master[c].y += acc[c].y;
                        acc[c] = make_float2(0.0f, 0.0f);
                    }
                }
            }
            float cin[2][NC];
            load_cin(rb * SKT_ROWS + rl, 1, cin);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t row = rb * SKT_ROWS + rl + h;
                if (row < Mr) {
#pragma unroll
                    for (int c = 0; c < NC; ++c)
                        if (c < Nc) store(row, c, sp, h ? master[c].y : master[c].x, cin[h][c]);
                }
            }
        }
        return;
    }
    if (RPT == 2 && TA && TB) {
        // K-contiguous long operand, B' tile [32 k][NC]: rows tid and tid+TPB
        // (one float4 along k each), column pairs (c, c+1) as FFMA2 operand
        // pairs from one 128-bit broadcast of B' — same per-entry order
        for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
            int64_t rb, ch0, ch1;
            int sp;
            unit(u, rb, sp, ch0, ch1);
            float2 acc[2][NC / 2], master[2][NC / 2];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int c = 0; c < NC / 2; ++c) acc[h][c] = master[h][c] = make_float2(0.0f, 0.0f);
            for (int64_t ch = ch0; ch < ch1; ++ch, ++it) {
                const int s = (int)(it % SKT_STAGES);
                mbar_wait(&full[s], (uint32_t)(it / SKT_STAGES) & 1u);
                const float *As = reinterpret_cast<const float *>(smem + s * STAGE);
                const float *Bs = reinterpret_cast<const float *>(smem + s * STAGE + SKT_A_BYTES);
#pragma unroll 1
                for (int j = 0; j < SKT_KC / 4; ++j) {
                    float a[2][4];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {   // 128B swizzle: chunk j of row tid sits at chunk j ^ (tid & 7)
                        const float4 x = *reinterpret_cast<const float4 *>(As + h * TPB * SKT_KC + tid * SKT_KC +
                                                                            4 * (j ^ (tid & 7)));
                        a[h][0] = x.x; a[h][1] = x.y; a[h][2] = x.z; a[h][3] = x.w;
                    }
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        float b[NC];
#pragma unroll
                        for (int c = 0; c < NC; c += 4) {
                            const float4 v = *reinterpret_cast<const float4 *>(Bs + (4 * j + kk) * NC + c);
                            b[c] = v.x; b[c + 1] = v.y; b[c + 2] = v.z; b[c + 3] = v.w;
                        }
#pragma unroll
                        for (int h = 0; h < 2; ++h)
#pragma unroll
                            for (int c = 0; c < NC / 2; ++c)
                                acc[h][c] = __ffma2_rn(make_float2(a[h][kk], a[h][kk]), make_float2(b[2 * c], b[2 * c + 1]),
                                                       acc[h][c]);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                if ((ch + 1) % PROM == 0 || ch + 1 == ch1) {
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                        for (int c = 0; c < NC / 2; ++c) {
                            master[h][c].x += acc[h][c].x;
                            master[h][c].y += acc[h][c].y;
                            acc[h][c] = make_float2(0.0f, 0.0f);
                        }
                }
            }
            float cin[2][NC];
            load_cin(rb * SKT_ROWS + tid, TPB, cin);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t row = rb * SKT_ROWS + h * TPB + tid;
                if (row < Mr) {
#pragma unroll
                    for (int c = 0; c < NC; ++c)
                        if (c < Nc) store(row, c, sp, (c & 1) ? master[h][c >> 1].y : master[h][c >> 1].x, cin[h][c]);
                }
            }
        }
        return;
    }
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
        int64_t rb, ch0, ch1;
        int sp;
        unit(u, rb, sp, ch0, ch1);
        float acc[RPT][NC], master[RPT][NC];
#pragma unroll
        for (int h = 0; h < RPT; ++h)
#pragma unroll
            for (int c = 0; c < NC; ++c) acc[h][c] = master[h][c] = 0.0f;
        for (int64_t ch = ch0; ch < ch1; ++ch, ++it) {
            const int s = (int)(it % SKT_STAGES);
            mbar_wait(&full[s], (uint32_t)(it / SKT_STAGES) & 1u);
            const float *As = reinterpret_cast<const float *>(smem + s * STAGE);
            const float *Bs = reinterpret_cast<const float *>(smem + s * STAGE + SKT_A_BYTES);
#pragma unroll
            for (int j = 0; j < SKT_KC / 4; ++j) {
                float4 a[RPT];
#pragma unroll
                for (int h = 0; h < RPT; ++h) {
                    const float *Ah = As + h * TPB * SKT_KC;   // box h
                    if (!TA) {
                        a[h].x = Ah[(4 * j + 0) * TPB + tid];
                        a[h].y = Ah[(4 * j + 1) * TPB + tid];
                        a[h].z = Ah[(4 * j + 2) * TPB + tid];
                        a[h].w = Ah[(4 * j + 3) * TPB + tid];
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
            if ((ch + 1) % PROM == 0 || ch + 1 == ch1) {
#pragma unroll
                for (int h = 0; h < RPT; ++h)
#pragma unroll
                    for (int c = 0; c < NC; ++c) {
                        master[h][c] += acc[h][c];
                        acc[h][c] = 0.0f;
                    }
            }
        }
        float cin[RPT][NC];
        load_cin(rb * SKT_ROWS + tid, TPB, cin);
#pragma unroll
        for (int h = 0; h < RPT; ++h) {
            const int64_t row = rb * SKT_ROWS + h * TPB + tid;
            if (row < Mr) {
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    if (c < Nc) store(row, c, sp, master[h][c], cin[h][c]);
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

// Fixed-order reduce of the split-K slabs: C'(r, c) <- alpha * (P_0 + ... +
// P_{S-1})(r, c) (+ beta * C'), slab layout [c][r] (r contiguous).
__global__ void __launch_bounds__(256) skinny_splitk_reduce_kernel(const float *__restrict__ P, int S, int64_t Mr,
                                                                   int Nc, float alpha, float beta, float *C,
                                                                   int64_t rs, int64_t cs) {
    const int64_t total = Mr * Nc;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        float v = __ldcs(P + idx);
        for (int sp = 1; sp < S; ++sp) v += __ldcs(P + (size_t)sp * total + idx);
        const int64_t c = idx / Mr, r = idx - c * Mr;
        float *d = C + r * rs + c * cs;
        *d = beta == 0.0f ? alpha * v : fmaf(beta, *d, alpha * v);
    }
}

// Launch plan of the TMA streaming kernel: compute threads per CTA (rows per
// block = 2 TPB) and K splits.  Row blocks < SMs and K long: split K over
// whole 256-of-K promotion groups (>= 2 per split) so that blocks * S fill
// the SMs (16384 x 16 x 16384: 32 blocks x 4 splits).
struct SkPlan {
    int tpb = SKT_TPB, splits = 1;
};
static SkPlan skinny_plan(bool TA, int64_t Mr, int64_t K) {
    SkPlan P;
    const int64_t sms = tc_num_sms();
    auto span = [&](int64_t rows) { return ((Mr + rows - 1) / rows + sms - 1) / sms * rows; };
    // rows per CTA 2 * TPB: 512 or 448, whichever finishes the persistent
    // grid in fewer row-slots per SM (65536 rows: 128 blocks of 512 leave 20
    // SMs idle, 147 blocks of 448 fill them)
    P.tpb = span(448) < span(512) ? 224 : 256;
    if (const char *e = getenv("EMM_SKINNY_TPB")) P.tpb = atoi(e) == 224 ? 224 : 256;   // experiments
    const int64_t nb = (Mr + 2 * P.tpb - 1) / (2 * P.tpb);
    const int64_t ngroups = ((K + SKT_KC - 1) / SKT_KC + 7) / 8;
    int64_t S = nb < sms ? std::min<int64_t>(sms / nb, ngroups / 2) : 1;
    if (const char *e = getenv("EMM_SKINNY_SPLITS")) {   // > 0: forced (0: the policy)
        if (atoi(e) > 0) S = std::min<int64_t>(atoi(e), std::max<int64_t>(ngroups, 1));
    }
    P.splits = (int)std::max<int64_t>(1, std::min<int64_t>(S, 64));
    return P;
}

template <bool TA, bool TB, int NC, int RPT, int TPB = SKT_TPB>
static cudaError_t launch_tma_nc(int64_t Mr, int Nc, int64_t K, float alpha, const float *Ap, int64_t lda,
                                 const float *Bp, int64_t ldb, float beta, float *C, int64_t rs, int64_t cs,
                                 cudaStream_t s, int splits = 1, float *partial = nullptr) {
    constexpr int ROWS = TPB * RPT;
    constexpr int STAGES = RPT == 1 ? 4 : 3;
    constexpr int B_BYTES = SKT_KC * NC * 4;
    constexpr int STAGE = ROWS * SKT_KC * 4 + ((B_BYTES + 1023) / 1024) * 1024;
    constexpr int SMEM = STAGES * STAGE + 1024 + 128;
    static cudaError_t attr = cudaFuncSetAttribute(skinny_tma_kernel<TA, TB, NC, RPT, TPB>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (attr != cudaSuccess) return attr;
    CUtensorMap ta, tb;
    const bool ok_a = !TA ? skinny_tmap(&ta, Ap, lda, (uint64_t)Mr, (uint64_t)K, TPB, SKT_KC, false)
                          : skinny_tmap(&ta, Ap, lda, (uint64_t)K, (uint64_t)Mr, SKT_KC, TPB, true);
    const bool ok_b = !TB ? skinny_tmap(&tb, Bp, ldb, (uint64_t)K, (uint64_t)Nc, SKT_KC, NC, false)
                          : skinny_tmap(&tb, Bp, ldb, (uint64_t)Nc, (uint64_t)K, NC, SKT_KC, false);
    if (!ok_a || !ok_b) return cudaErrorInvalidValue;
    const int64_t units = (Mr + ROWS - 1) / ROWS * splits;
    const int64_t grid = units < tc_num_sms() ? units : tc_num_sms();
    skinny_tma_kernel<TA, TB, NC, RPT, TPB><<<(unsigned)grid, TPB + 32, SMEM, s>>>(
        ta, tb, Mr, Nc, K, alpha, beta, C, rs, cs, splits, splits > 1 ? partial : nullptr);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || splits == 1) return e;
    const int64_t total = Mr * Nc;
    const unsigned rg = (unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)tc_num_sms() * 8);
    skinny_splitk_reduce_kernel<<<rg, 256, 0, s>>>(partial, splits, Mr, Nc, alpha, beta, C, rs, cs);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

template <bool TA, bool TB>
static cudaError_t launch_tma(int64_t Mr, int Nc, int64_t K, float alpha, const float *Ap, int64_t lda,
                              const float *Bp, int64_t ldb, float beta, float *C, int64_t rs, int64_t cs,
                              cudaStream_t s, float *ws, size_t ws_bytes) {
    int rpt = 2;
    if (const char *e = getenv("EMM_SKINNY_RPT")) rpt = atoi(e);   // experiments
    if (rpt == 1) {
        if (Nc <= 4) return launch_tma_nc<TA, TB, 4, 1>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C, rs, cs, s);
        if (Nc <= 8) return launch_tma_nc<TA, TB, 8, 1>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C, rs, cs, s);
        return launch_tma_nc<TA, TB, 16, 1>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C, rs, cs, s);
    }
    SkPlan P = skinny_plan(TA, Mr, K);
    if (P.splits > 1 && (!ws || ws_bytes < (size_t)P.splits * Mr * Nc * 4)) P.splits = 1;
    const int S = P.splits;
    if (P.tpb == 224) {
        if (Nc <= 4) return launch_tma_nc<TA, TB, 4, 2, 224>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C, rs, cs, s, S, ws);
        if (Nc <= 8) return launch_tma_nc<TA, TB, 8, 2, 224>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C, rs, cs, s, S, ws);
        return launch_tma_nc<TA, TB, 16, 2, 224>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C, rs, cs, s, S, ws);
    }
    if (Nc <= 4) return launch_tma_nc<TA, TB, 4, 2>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C, rs, cs, s, S, ws);
    if (Nc <= 8) return launch_tma_nc<TA, TB, 8, 2>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C, rs, cs, s, S, ws);
    return launch_tma_nc<TA, TB, 16, 2>(Mr, Nc, K, alpha, Ap, lda, Bp, ldb, beta, C, rs, cs, s, S, ws);
}

// The skinny call's roles (see launch_skinny_sgemm).
struct SkRoles {
    bool TA, TB;
    int64_t Mr, lda2, ldb2, rs, cs;
    int Nc;
    const float *Ap, *Bp;
};
static SkRoles skinny_roles(bool tA, bool tB, int64_t M, int64_t N, const float *A, int64_t lda, const float *B,
                            int64_t ldb, int64_t ldc) {
    SkRoles R;
    if (N <= SKINNY_MAX) {
        R.Mr = M; R.Nc = (int)N;
        R.Ap = A; R.lda2 = lda; R.TA = tA;    // op(A)(r,p): tA ? A[p + r*lda] : A[r + p*lda]
        R.Bp = B; R.ldb2 = ldb; R.TB = tB;    // op(B)(p,c): tB ? B[c + p*ldb] : B[p + c*ldb]
        R.rs = 1; R.cs = ldc;
    } else {
        R.Mr = N; R.Nc = (int)M;
        // A'(r,p) = op(B)(p,r): tB ? B[r + p*ldb] (r contiguous: !TA) : B[p + r*ldb] (TA)
        R.Ap = B; R.lda2 = ldb; R.TA = !tB;
        // B'(p,c) = op(A)(c,p): tA ? A[p + c*lda] (!TB form) : A[c + p*lda] (TB form)
        R.Bp = A; R.ldb2 = lda; R.TB = !tA;
        R.rs = ldc; R.cs = 1;
    }
    return R;
}

static bool skinny_tma_ok(const SkRoles &R, int64_t K) {
    return tma_legal(R.Ap, R.lda2) && tma_legal(R.Bp, R.ldb2) && !getenv("EMM_SKINNY_NO_TMA") && K > 0;
}

// K-contiguous B' (!TB): B' is first transposed (PK_RAWT, 32 floats a row,
// zero padded) so the kernel reads [32 k][NC] tiles — with a K-contiguous
// long operand (TA) it pairs columns for FFMA2; with an MN-contiguous one
// (!TA, N' > 8) the row-pair kernel reads 4 columns per broadcast instead of
// 4 k.  EMM_SKINNY_BT=0 disables both.
static bool skinny_bt(const SkRoles &R, int64_t K) {
    const char *e = getenv("EMM_SKINNY_BT");
    if (e && e[0] == '0') return false;
    if (!R.TA && !R.TB) {
        // MN-contiguous long operand: the [32 k][NC] B' tiles measured ~4 %
        // faster for N' > 8 (c6 N = 16: 209 -> 202 us incl. the transpose
        // launch) and slower for N' <= 8 (65536 x 8 x 4096: 173 -> 179 us);
        // the extra launch pays only on a long operand of >= 2^26 elements.
        // EMM_SKINNY_BT_NN=0 / 1 forces it off / on.
        const char *n = getenv("EMM_SKINNY_BT_NN");
        return n ? n[0] == '1' : R.Nc > 8 && R.Mr * K >= ((int64_t)1 << 26);
    }
    return R.TA && !R.TB;
}
static size_t skinny_slab_bytes(const SkRoles &R, int64_t K) {
    const SkPlan P = skinny_plan(R.TA, R.Mr, K);
    return P.splits > 1 ? align_up((size_t)P.splits * R.Mr * R.Nc * 4, 1024) : 0;
}

// Workspace of this call's FFMA skinny path: split-K slabs + the transposed
// B' copy (0: none).  Upper bound without pointers (A = B = null: assumes
// the TMA path).
size_t skinny_split_bytes(bool tA, bool tB, int64_t M, int64_t N, int64_t K, const float *A, int64_t lda,
                          const float *B, int64_t ldb) {
    const SkRoles R = skinny_roles(tA, tB, M, N, A, lda, B, ldb, 1);
    if (A && B && !skinny_tma_ok(R, K)) return 0;
    return skinny_slab_bytes(R, K) + (skinny_bt(R, K) ? (size_t)K * 32 * 4 : 0);
}

cudaError_t launch_skinny_sgemm(bool tA, bool tB, int64_t M, int64_t N, int64_t K, float alpha, const float *A,
                                int64_t lda, const float *B, int64_t ldb, float beta, float *C, int64_t ldc,
                                cudaStream_t s, float *ws, size_t ws_bytes) {
    // Roles: the long output dimension is streamed (rows of C'), the short one
    // (<= SKINNY_MAX) is resident.  N short: C' = C, A' = op(A), B' = op(B).
    // M short: C' = C^T = op(B)^T op(A)^T, A' = op(B)^T, B' = op(A)^T.
    const SkRoles R = skinny_roles(tA, tB, M, N, A, lda, B, ldb, ldc);
    const bool TA = R.TA, TB = R.TB;
    const int64_t Mr = R.Mr, lda2 = R.lda2, ldb2 = R.ldb2, rs = R.rs, cs = R.cs;
    const int Nc = R.Nc;
    const float *Ap = R.Ap, *Bp = R.Bp;
    if ((Mr + 127) / 128 > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    cudaEvent_t ev = nullptr;
    prof_begin(s, true, &ev);
    cudaError_t e;
    if (skinny_tma_ok(R, K)) {
        const size_t slab = skinny_slab_bytes(R, K);
        if (skinny_bt(R, K) && ws && ws_bytes >= slab + (size_t)K * 32 * 4) {
            // B'(p, c) = Bp[p + c*ldb2] -> Bt[p*32 + c], then the TA x TB kernel
            float *Bt = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(ws) + slab);
            PackArgs x;
            x.X = Bp; x.ld = ldb2; x.R = K; x.kcontig = false; x.out0 = Bt; x.ld0 = 32;
            e = launch_pack(PK_RAWT_, x, nullptr, Nc, nullptr, s, 0);
            if (e == cudaSuccess)
                e = TA ? launch_tma<true, true>(Mr, Nc, K, alpha, Ap, lda2, Bt, 32, beta, C, rs, cs, s, ws, slab)
                       : launch_tma<false, true>(Mr, Nc, K, alpha, Ap, lda2, Bt, 32, beta, C, rs, cs, s, ws, slab);
        } else if (!TA && !TB) e = launch_tma<false, false>(Mr, Nc, K, alpha, Ap, lda2, Bp, ldb2, beta, C, rs, cs, s, ws, ws_bytes);
        else if (!TA && TB) e = launch_tma<false, true>(Mr, Nc, K, alpha, Ap, lda2, Bp, ldb2, beta, C, rs, cs, s, ws, ws_bytes);
        else if (TA && !TB) e = launch_tma<true, false>(Mr, Nc, K, alpha, Ap, lda2, Bp, ldb2, beta, C, rs, cs, s, ws, ws_bytes);
        else e = launch_tma<true, true>(Mr, Nc, K, alpha, Ap, lda2, Bp, ldb2, beta, C, rs, cs, s, ws, ws_bytes);
    } else if (!TA && !TB) e = launch_nc<false, false>(Mr, Nc, K, alpha, Ap, lda2, Bp, ldb2, beta, C, rs, cs, s);
    else if (!TA && TB) e = launch_nc<false, true>(Mr, Nc, K, alpha, Ap, lda2, Bp, ldb2, beta, C, rs, cs, s);
    else if (TA && !TB) e = launch_nc<true, false>(Mr, Nc, K, alpha, Ap, lda2, Bp, ldb2, beta, C, rs, cs, s);
    else e = launch_nc<true, true>(Mr, Nc, K, alpha, Ap, lda2, Bp, ldb2, beta, C, rs, cs, s);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    prof_end(s, true, ev);
    return e;
}

}  // namespace emm
