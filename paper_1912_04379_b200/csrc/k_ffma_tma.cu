// k_ffma_tma.cu — KN3b: warp-specialised FP32 FFMA SGEMM (EMM_MATH_FFMA).
//
// Same arithmetic as KN3 (k_ffma.cu): an 8x8 register tile per thread (the
// paper's L0 register blocking), FFMA2 (two FP32 FMAs per
// issue slot), sequential FP32 accumulation along K with promotion into a
// master copy every 256 of K.  What changes is the operand staging, the part
// KN3 spends its non-FMA issue slots and barriers on:
//   * one producer warp streams the 128 x 32 A and B tiles of each K-stage
//     into a 4-stage SMEM ring with TMA (cp.async.bulk.tensor, OOB = zero,
//     the paper's zero-padded K tail PAPER.md:449-451), full/empty mbarriers;
//   * 8 consumer warps never stage through registers or meet at
//     __syncthreads: they wait on the stage's full barrier, run 32 x 32
//     FFMA2 per thread from SMEM, and release the stage.
// SMEM tiles keep each operand's own majorness (no transpose anywhere):
//   MN-contiguous (A transA=N, B transB=T): four [32 k][32 mn] TMA boxes,
//     128B swizzle; a thread reads float4 along mn (rows 4t..4t+3, 64+4t..).
//   K-contiguous  (A transA=T, B transB=N): one [128 rows][32 k] box, 128B
//     swizzle; a thread owns rows t, t+16, ..., t+112 and reads float4
//     along k (4 k-steps per load).
// FFMA2 pairs two accumulators that share one operand value: adjacent
// columns when B is MN-contiguous, else adjacent rows (A MN-contiguous).
// The TN case (both K-contiguous) and non-TMA-legal layouts stay on KN3.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "emm_internal.h"
#include "ptx.cuh"

namespace emm {

using namespace ptx;

namespace {
constexpr int FT_M = 128, FT_N = 128, FT_K = 32;
constexpr int FT_TILE_FLOATS = 128 * FT_K;                  // one operand tile: 16 KB
constexpr int FT_STAGE_BYTES = 2 * FT_TILE_FLOATS * 4;      // A + B: 32 KB
constexpr int FT_CONSUMERS = 256, FT_THREADS = FT_CONSUMERS + 32;
constexpr int FT_PROMOTE = 256 / FT_K;                      // stages per promotion (256 of K)
constexpr int FT_MASTER_FLOATS = 64 * FT_CONSUMERS;
constexpr int FT_GROUP_M = 16;                              // raster: 16 tile-rows per group (L2 reuse of B)
// Two ways to feed the ring:
//  SEP = true:  a dedicated producer warp (288 threads -> 168 registers per
//               thread), 4 stages, promotion master in SMEM;
//  SEP = false: no producer warp — the LAST warp to finish a stage refills
//               its slot (a shared counter per slot, nobody waits for it) —
//               256 threads, up to 255 registers, master in registers,
//               6 stages.  Measured slower (c2-8192 19.79 vs 19.06 ms, c4-i
//               9.42 vs 8.98; profiles/r01_ab_ffma_kn3b_noprodwarp2.jsonl):
//               the extra registers buy nothing and the refilling warp
//               stalls; an earlier "thread 0 refills" form was slower still.
template <bool SEP>
struct FtCfg {
    static constexpr int STAGES = SEP ? 4 : 6;
    static constexpr int BLOCK = SEP ? FT_THREADS : FT_CONSUMERS;
    static constexpr int SMEM = STAGES * FT_STAGE_BYTES + (SEP ? FT_MASTER_FLOATS * 4 : 0) + 1024 + 256;
};
#ifndef EMM_FT_SEP
#define EMM_FT_SEP 1
#endif
constexpr bool FT_SEP = EMM_FT_SEP != 0;
#ifndef EMM_FT_GK
#define EMM_FT_GK 2
#endif
constexpr int FT_GK = EMM_FT_GK;                            // k per operand group (2 or 4)

// float index of the float4 holding (mn = 4q..4q+3, k) in an MN-contiguous tile
__device__ __forceinline__ int mn_idx(int q, int k) { return (q >> 3) * 1024 + k * 32 + (((q & 7) ^ (k & 7)) << 2); }
// float index of (row r, k) in a K-contiguous tile (k % GK == 0: the start
// of an aligned float2 / float4 along k)
__device__ __forceinline__ int kc_idx(int r, int k) { return r * 32 + (((k >> 2) ^ (r & 7)) << 2) + (k & 3); }

// The 8 operand values of one thread for GK consecutive k (k = GK*g + kk):
// v[kk][e], e = the thread's row (A) / column (B) slot.
//   MN-contiguous: slot e -> mn = 4t + e (e < 4), 64 + 4t + (e - 4)
//   K-contiguous:  slot e -> row t + 16 e (one float2 / float4 along k)
template <bool MN, int GK>
__device__ __forceinline__ void load_group(const float *__restrict__ T, int t, int g, float (&v)[GK][8]) {
    if (MN) {
#pragma unroll
        for (int kk = 0; kk < GK; ++kk) {
            const float4 x0 = *reinterpret_cast<const float4 *>(T + mn_idx(t, GK * g + kk));
            const float4 x1 = *reinterpret_cast<const float4 *>(T + mn_idx(16 + t, GK * g + kk));
            v[kk][0] = x0.x; v[kk][1] = x0.y; v[kk][2] = x0.z; v[kk][3] = x0.w;
            v[kk][4] = x1.x; v[kk][5] = x1.y; v[kk][6] = x1.z; v[kk][7] = x1.w;
        }
    } else if (GK == 4) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const float4 x = *reinterpret_cast<const float4 *>(T + kc_idx(t + 16 * e, 4 * g));
            v[0][e] = x.x; v[1 % GK][e] = x.y; v[2 % GK][e] = x.z; v[3 % GK][e] = x.w;
        }
    } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const float2 x = *reinterpret_cast<const float2 *>(T + kc_idx(t + 16 * e, GK * g));
            v[0][e] = x.x; v[1 % GK][e] = x.y;
        }
    }
}
__device__ __forceinline__ int slot_pos(bool mn, int t, int e) { return mn ? (e < 4 ? 4 * t + e : 60 + 4 * t + e) : t + 16 * e; }
}  // namespace

// PAIR_J (B MN-contiguous): acc[i*4 + j/2] holds (i, j), (i, j+1);
// else (A MN-contiguous):   acc[(i/2)*8 + j] holds (i, j), (i+1, j).
template <bool A_MN, bool B_MN, bool SEP>
__global__ void __launch_bounds__(FtCfg<SEP>::BLOCK, 1)
    ffma_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                    int K, float alpha, float beta, float *__restrict__ C, int64_t ldc, int tiles_m, int tiles_n,
                    int splits, float *__restrict__ partial) {
    static_assert(A_MN || B_MN, "TN (both K-contiguous) runs on KN3");
    constexpr bool PAIR_J = B_MN;
    constexpr int STAGES = FtCfg<SEP>::STAGES;
    extern __shared__ __align__(1024) uint8_t ft_raw[];
    // 1024-B aligned base for the 128B-swizzled TMA boxes; offset arithmetic
    // on the shared array (not via an integer cast) keeps the reads LDS
    uint8_t *smem = ft_raw + ((1024u - (smem_u32(ft_raw) & 1023u)) & 1023u);
    float *master_s = reinterpret_cast<float *>(smem + STAGES * FT_STAGE_BYTES);   // SEP only
    uint64_t *full = reinterpret_cast<uint64_t *>(master_s + (SEP ? FT_MASTER_FLOATS : 0));
    uint64_t *empty = full + STAGES;                                               // SEP only
    unsigned int *done_cnt = reinterpret_cast<unsigned int *>(empty + STAGES);    // !SEP only

    // split-K (sub-wave problems, splits > 1): block = (split sp, tile),
    // split-major; split sp runs the promotion chunks [sp*nch/S, (sp+1)*nch/S)
    // of K and stores its raw master to partial slab sp (the fixed-order
    // reduce launch adds the slabs)
    const int ntiles = tiles_m * tiles_n;
    const int sp = (int)blockIdx.x / ntiles;
    // grouped raster: FT_GROUP_M tile-rows share each B panel while it is in L2
    const int bid = (int)blockIdx.x - sp * ntiles;
    const int per_group = FT_GROUP_M * tiles_n;
    const int first_m = (bid / per_group) * FT_GROUP_M;
    const int gsize = min(tiles_m - first_m, FT_GROUP_M);
    const int m0 = (first_m + (bid % per_group) % gsize) * FT_M;
    const int n0 = ((bid % per_group) / gsize) * FT_N;
    const int nk_all = (K + FT_K - 1) / FT_K;
    const int nch = (nk_all + FT_PROMOTE - 1) / FT_PROMOTE;
    const int kt0 = min(nk_all, (int)((long long)sp * nch / splits) * FT_PROMOTE);
    const int nk = min(nk_all, (int)((long long)(sp + 1) * nch / splits) * FT_PROMOTE);   // end stage

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], FT_CONSUMERS / 32);
            done_cnt[s] = 0;
        }
        fence_mbar_init();
    }
    __syncthreads();

    const uint64_t pol = policy_evict_normal();
    // loads of K-stage kt into ring slot kt % STAGES (one thread; the slot
    // is known to be free)
    auto issue = [&](int kt) {
        const int s = (kt - kt0) % STAGES;
        mbar_arrive_expect_tx(&full[s], FT_STAGE_BYTES);
        const uint32_t st = smem_u32(smem + s * FT_STAGE_BYTES);
        const uint32_t sb = st + FT_TILE_FLOATS * 4;
        const int k0 = kt * FT_K;
        if (A_MN) {
#pragma unroll
            for (int b = 0; b < 4; ++b) tma_load_2d(st + b * 4096, &tmA, &full[s], m0 + 32 * b, k0, pol);
        } else {
            tma_load_2d(st, &tmA, &full[s], k0, m0, pol);
        }
        if (B_MN) {
#pragma unroll
            for (int b = 0; b < 4; ++b) tma_load_2d(sb + b * 4096, &tmB, &full[s], n0 + 32 * b, k0, pol);
        } else {
            tma_load_2d(sb, &tmB, &full[s], k0, n0, pol);
        }
    };
    if (SEP) {
        if (warp == FT_CONSUMERS / 32) {
            // ===== producer warp: one lane issues the TMA loads =====
            if (lane == 0) {
                prefetch_tmap(&tmA);
                prefetch_tmap(&tmB);
                for (int kt = kt0; kt < nk; ++kt) {
                    mbar_wait(&empty[(kt - kt0) % STAGES], ((uint32_t)((kt - kt0) / STAGES) & 1u) ^ 1u);
                    issue(kt);
                }
            }
            return;
        }
    } else if (threadIdx.x == 0) {
        for (int kt = kt0; kt < kt0 + STAGES && kt < nk; ++kt) issue(kt);   // fill the ring
    }

    // ===== consumers =====
    const int c = threadIdx.x;
    const int tm = c & 15, tn = c >> 4;
    float2 acc[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) acc[e] = make_float2(0.0f, 0.0f);
    float master_r[SEP ? 1 : 64];   // !SEP: promotion master in registers
#pragma unroll
    for (int e = 0; e < (SEP ? 1 : 64); ++e) master_r[e] = 0.0f;
    if (SEP) {
#pragma unroll
        for (int e = 0; e < 64; ++e) master_s[e * FT_CONSUMERS + c] = 0.0f;
    }

    for (int kt = kt0; kt < nk; ++kt) {
        const int s = (kt - kt0) % STAGES;
        mbar_wait(&full[s], (uint32_t)((kt - kt0) / STAGES) & 1u);
        const float *As = reinterpret_cast<const float *>(smem + s * FT_STAGE_BYTES);
        const float *Bs = As + FT_TILE_FLOATS;
        // operand groups double-buffered: group g+1 is read from SMEM while
        // group g's FFMA2s run
        float av[2][FT_GK][8], bv[2][FT_GK][8];
        load_group<A_MN, FT_GK>(As, tm, 0, av[0]);
        load_group<B_MN, FT_GK>(Bs, tn, 0, bv[0]);
#pragma unroll
        for (int g = 0; g < FT_K / FT_GK; ++g) {
            if (g + 1 < FT_K / FT_GK) {
                load_group<A_MN, FT_GK>(As, tm, g + 1, av[(g + 1) & 1]);
                load_group<B_MN, FT_GK>(Bs, tn, g + 1, bv[(g + 1) & 1]);
            }
            const int u = g & 1;
#pragma unroll
            for (int kk = 0; kk < FT_GK; ++kk) {
                // the pair operand stays fixed over 8 consecutive FFMA2s (operand
                // reuse cache) while the broadcast scalar varies: 125 vs 108
                // FMA/clk/SM for the other order (tools/ffma2_probe.cu)
                if (PAIR_J) {
#pragma unroll
                    for (int jp = 0; jp < 4; ++jp)
#pragma unroll
                        for (int i = 0; i < 8; ++i)
                            acc[i * 4 + jp] = __ffma2_rn(make_float2(av[u][kk][i], av[u][kk][i]),
                                                         make_float2(bv[u][kk][2 * jp], bv[u][kk][2 * jp + 1]),
                                                         acc[i * 4 + jp]);
                } else {
#pragma unroll
                    for (int ip = 0; ip < 4; ++ip)
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            acc[ip * 8 + j] = __ffma2_rn(make_float2(av[u][kk][2 * ip], av[u][kk][2 * ip + 1]),
                                                         make_float2(bv[u][kk][j], bv[u][kk][j]), acc[ip * 8 + j]);
                }
            }
        }
        __syncwarp();
        if (SEP) {
            if (lane == 0) mbar_arrive(&empty[s]);
        } else if (lane == 0) {
            // the last of the 8 warps to finish this stage refills its slot
            unsigned int old;
            asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                         : "=r"(old) : "r"(smem_u32(&done_cnt[s])) : "memory");
            if (old == FT_CONSUMERS / 32 - 1) {
                done_cnt[s] = 0;
                fence_proxy_async_smem();   // generic reads of the slot before the async-proxy overwrite
                if (kt + STAGES < nk) issue(kt + STAGES);
            }
        }
        if ((kt + 1) % FT_PROMOTE == 0 || kt + 1 == nk) {
            // promotion: master += register partials (round-to-nearest adds)
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float2 &p = PAIR_J ? acc[i * 4 + (j >> 1)] : acc[(i >> 1) * 8 + j];
                    const float v = PAIR_J ? ((j & 1) ? p.y : p.x) : ((i & 1) ? p.y : p.x);
                    if (SEP)
                        master_s[(i * 8 + j) * FT_CONSUMERS + c] += v;
                    else
                        master_r[(i * 8 + j) % (SEP ? 1 : 64)] += v;
                }
#pragma unroll
            for (int e = 0; e < 32; ++e) acc[e] = make_float2(0.0f, 0.0f);
        }
    }

    // epilogue: alpha*acc + beta*C (C not read when beta == 0), predicated.
    // beta != 0: the C_in loads of two columns (16 values) are issued before
    // their stores — a store could alias a later load through ldc, so the
    // compiler would otherwise serialise 64 load round trips per thread.
#pragma unroll
    for (int j0 = 0; j0 < 8; j0 += 2) {
        float cin[2][8];
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const int col = n0 + slot_pos(B_MN, tn, j0 + jj);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int row = m0 + slot_pos(A_MN, tm, i);
                cin[jj][i] = (!partial && beta != 0.0f && col < N && row < M) ? C[row + (int64_t)col * ldc] : 0.0f;
            }
        }
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const int j = j0 + jj;
            const int col = n0 + slot_pos(B_MN, tn, j);
            if (col >= N) continue;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int row = m0 + slot_pos(A_MN, tm, i);
                if (row < M) {
                    const float v = SEP ? master_s[(i * 8 + j) * FT_CONSUMERS + c] : master_r[(i * 8 + j) % (SEP ? 1 : 64)];
                    if (partial) {
                        partial[((size_t)sp * N + col) * M + row] = v;
                    } else {
                        C[row + (int64_t)col * ldc] = beta == 0.0f ? alpha * v : fmaf(beta, cin[jj][i], alpha * v);
                    }
                }
            }
        }
    }
}

// Fixed-order split-K reduce of KN3b: C <- alpha*(P_0 + ... + P_{S-1}) (+ beta*C),
// the slabs column-major M x N (ld = M); consecutive threads take
// consecutive rows (coalesced slab reads and C accesses).
__global__ void __launch_bounds__(256) ffma_splitk_reduce_kernel(const float *__restrict__ P, int S, int64_t M,
                                                                 int64_t N, float alpha, float beta, float *C,
                                                                 int64_t ldc) {
    const int64_t total = M * N, slab = M * N;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        float r = __ldcs(P + idx);
        for (int sp = 1; sp < S; ++sp) r += __ldcs(P + (size_t)sp * slab + idx);
        const int64_t col = idx / M, row = idx - col * M;
        float *d = C + row + col * ldc;
        *d = beta == 0.0f ? alpha * r : fmaf(beta, *d, alpha * r);
    }
}

// Split-K factor for sub-wave KN3b grids (one 288-thread CTA per SM):
// minimise waves(S) * stages_per_split(S) * t_stage + the reduce's HBM
// round trip ((2S + 1) M N 4 bytes at ~5 TB/s + a launch), with splits of
// whole promotion chunks (256 of K).  t_stage ~ 2.7 us (128 x 128 x 32 FFMA
// per SM at ~80 % of the FP32 pipe).  EMM_FFMA_SPLITS overrides.
int ffma_splits(int64_t M, int64_t N, int64_t K) {
    const int64_t tiles = ((M + FT_M - 1) / FT_M) * ((N + FT_N - 1) / FT_N);
    const int64_t nk = (K + FT_K - 1) / FT_K, nch = (nk + FT_PROMOTE - 1) / FT_PROMOTE;
    const int64_t slots = tc_num_sms();
    if (const char *e = getenv("EMM_FFMA_SPLITS")) {   // > 0: forced (0: the policy below)
        const int64_t v = atoi(e);
        if (v > 0) return (int)std::max<int64_t>(1, std::min<int64_t>({v, nch, 16}));
    }
    if (tiles >= slots || nch < 2) return 1;
    const double t_stage = 2.7e-6;
    double best = 0.0;
    int bs = 1;
    for (int S = 1; S <= 16 && S <= nch; ++S) {
        const int64_t waves = (tiles * S + slots - 1) / slots;
        int64_t st = 0;   // stages of the longest split
        for (int q = 0; q < S; ++q)
            st = std::max<int64_t>(st, std::min<int64_t>(nk, (int64_t)(q + 1) * nch / S * FT_PROMOTE) -
                                           std::min<int64_t>(nk, (int64_t)q * nch / S * FT_PROMOTE));
        double t = (double)waves * (double)st * t_stage;
        if (S > 1) t += (double)(2 * S + 1) * (double)M * (double)N * 4.0 / 5.0e12 + 3.0e-6;
        if (S == 1 || t < best) best = t, bs = S;
    }
    return bs;
}

size_t ffma_splitk_bytes(int64_t M, int64_t N, int splits) {
    return splits > 1 ? (size_t)splits * (size_t)M * (size_t)N * sizeof(float) : 0;
}

bool ffma_tma_eligible(bool tA, bool tB, const float *A, int64_t lda, const float *B, int64_t ldb) {
    // KN3b needs one MN-contiguous operand (not TN) and TMA-legal layouts
    return !(tA && !tB) && tma_legal(A, lda) && tma_legal(B, ldb);
}

cudaError_t launch_ffma_tma_sgemm(bool tA, bool tB, int64_t M, int64_t N, int64_t K, float alpha, const float *A,
                                  int64_t lda, const float *B, int64_t ldb, float beta, float *C, int64_t ldc,
                                  cudaStream_t s, int splits, float *partial) {
    const bool a_mn = !tA, b_mn = tB;
    if (splits < 1 || (splits > 1 && !partial)) return cudaErrorInvalidValue;
    if (splits == 1) partial = nullptr;
    if (!a_mn && !b_mn) return cudaErrorInvalidValue;
    if (M > 0x7fffff00LL || N > 0x7fffff00LL || K > 0x7fffff00LL) return cudaErrorInvalidValue;
    const int64_t tiles_m = (M + FT_M - 1) / FT_M, tiles_n = (N + FT_N - 1) / FT_N;
    if (tiles_m * tiles_n > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    // A: transA=N stored M x K (MN-contiguous), T stored K x M; B: transB=N
    // stored K x N (K-contiguous), T stored N x K.
    CUtensorMap ta, tb;
    const bool ok_a = a_mn ? encode_tmap_f32_2d(&ta, A, M, K, lda, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B)
                           : encode_tmap_f32_2d(&ta, A, K, M, lda, 32, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    const bool ok_b = b_mn ? encode_tmap_f32_2d(&tb, B, N, K, ldb, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B)
                           : encode_tmap_f32_2d(&tb, B, K, N, ldb, 32, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    if (!ok_a || !ok_b) return cudaErrorInvalidValue;
    static cudaError_t attr = [] {
        cudaError_t e = cudaSuccess;
        auto set = [&](const void *f) {
            cudaError_t r = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, FtCfg<FT_SEP>::SMEM);
            if (r != cudaSuccess) e = r;
        };
        set((const void *)ffma_tma_kernel<true, false, FT_SEP>);
        set((const void *)ffma_tma_kernel<true, true, FT_SEP>);
        set((const void *)ffma_tma_kernel<false, true, FT_SEP>);
        return e;
    }();
    if (attr != cudaSuccess) return attr;
    if (tiles_m * tiles_n * splits > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    const unsigned grid = (unsigned)(tiles_m * tiles_n * splits);
    cudaEvent_t ev = nullptr;
    prof_begin(s, true, &ev);
    if (a_mn && !b_mn)
        ffma_tma_kernel<true, false, FT_SEP><<<grid, FtCfg<FT_SEP>::BLOCK, FtCfg<FT_SEP>::SMEM, s>>>(ta, tb, (int)M, (int)N, (int)K, alpha, beta, C,
                                                                       ldc, (int)tiles_m, (int)tiles_n, splits, partial);
    else if (a_mn)
        ffma_tma_kernel<true, true, FT_SEP><<<grid, FtCfg<FT_SEP>::BLOCK, FtCfg<FT_SEP>::SMEM, s>>>(ta, tb, (int)M, (int)N, (int)K, alpha, beta, C,
                                                                      ldc, (int)tiles_m, (int)tiles_n, splits, partial);
    else
        ffma_tma_kernel<false, true, FT_SEP><<<grid, FtCfg<FT_SEP>::BLOCK, FtCfg<FT_SEP>::SMEM, s>>>(ta, tb, (int)M, (int)N, (int)K, alpha, beta, C,
                                                                       ldc, (int)tiles_m, (int)tiles_n, splits, partial);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    prof_end(s, true, ev);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || !partial) return e;
    const int64_t total = M * N;
    const unsigned rg = (unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)tc_num_sms() * 8);
    prof_begin(s, false, &ev);
    ffma_splitk_reduce_kernel<<<rg, 256, 0, s>>>(partial, splits, M, N, alpha, beta, C, ldc);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    prof_end(s, false, ev);
    return cudaGetLastError();
}

}  // namespace emm
