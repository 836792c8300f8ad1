// k_tc1w.cu — KN2w: 1xTF32 GEMM with a 256 x 512 output tile per CTA pair.
//
// The 1xTF32 kernel on 256 x 256 tiles is operand-fill-bound: one K8 MMA
// (128 clk per SM) needs 8 KB of fresh operands per SM, 64 B/clk, and the
// tensor pipe runs ~62% busy (profiles/r01_ncu_configs.md)
// where the 3xTF32 kernel, with 3 MMAs per byte, is not.  1xTF32 needs no
// FP32 promotion (its 5e-3 bound leaves the truncating TMEM accumulation
// ~30x headroom, Q7), so the whole 512-column TMEM can hold ONE
// accumulator: each CTA of the pair owns 128 rows x 512 columns, two N=256
// MMAs per K8 share the A tile, and a K-stage is A (16 KB) + two B halves
// (2 x 16 KB) per CTA — 48 KB for 2x the flops of the 32 KB stage, i.e. 25%
// fewer operand bytes per flop (the paper's "maximise reuse of the buffered
// panel" at the L1 level, applied to the SMEM ring).
//
// Without a second TMEM buffer the epilogue cannot run under the next
// tile's MMAs wholesale; instead it moves the N-half 0 columns to registers
// and releases them at once (then scales and stores them), and the MMA
// issuer starts the next tile with the half-0 MMAs of the first W_STAGES
// stages (already in SMEM) while half 1 drains.  (Prefetching the tile's C_in
// into L2 while its MMAs run was measured: c4-ii 1.030 -> 1.016 ms but c4-i
// 0.764 -> 0.782 ms — the prefetched C crowds the wave's operand panels out
// of L2 — so it is not done.)
// Warp roles as in KN1/KN2: warp 0 TMA producer, warp 1 MMA issuer (leader
// CTA), warps 2-9 epilogue (lane quarter q = warp % 4, column half).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "emm_internal.h"
#include "ptx.cuh"
#include "tc_common.cuh"

namespace emm {

using namespace ptx;

namespace {
constexpr int W_BN = 512;                              // C columns per pair
constexpr int W_STAGE_BYTES = 3 * TC_TILE_BYTES;      // A | B half 0 | B half 1 (per CTA)
// beta != 0 with a TMA-legal C (TMAC): the epilogue reads C_in through TMA
// into a ring of 4 x (128 rows x 16 columns) buffers per column group — many
// more bytes in flight than per-thread loads (the beta = 1 epilogue was
// load-latency-bound: c4-ii 1.03 ms vs 0.79 ms at beta = 0) — so the operand
// ring shrinks to 3 stages.
constexpr int W_CB_COLS = 16, W_CB_N = 4;
constexpr int W_CB_BYTES = 128 * W_CB_COLS * 4;       // 8 KB
template <bool TMAC>
struct WCfg {
    static constexpr int STAGES = TMAC ? 3 : 4;
    static constexpr int CBUF = TMAC ? 2 * W_CB_N * W_CB_BYTES : 0;   // two column groups
    static constexpr int SMEM = STAGES * W_STAGE_BYTES + CBUF + 1024 + 512;
};
constexpr int W_GROUP_M = 8;
}  // namespace

template <bool A_MN, bool B_MN, bool TMAC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(32 * (TC_EPI_WARPS + 2), 1)
    tc1w_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmC, int M, int N, int Kp, float alpha, float beta,
                float *__restrict__ C, int64_t ldc, int tiles_m, int tiles_n) {
    constexpr int W_STAGES = WCfg<TMAC>::STAGES;
    extern __shared__ __align__(1024) uint8_t w_raw[];
    uint8_t *smem = w_raw + ((1024u - (smem_u32(w_raw) & 1023u)) & 1023u);
    float *cbuf = reinterpret_cast<float *>(smem + W_STAGES * W_STAGE_BYTES);   // TMAC: [2 groups][W_CB_N][16][128]
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + W_STAGES * W_STAGE_BYTES + WCfg<TMAC>::CBUF);
    uint64_t *empty = full + W_STAGES;
    uint64_t *acc_full = empty + W_STAGES;   // [1]
    uint64_t *acc_empty = acc_full + 1;      // [2]: N-half 0 / 1 drained (both CTAs' epilogue warps)
    uint64_t *cfull = acc_empty + 2;         // TMAC: [2 groups][W_CB_N] C-chunk landed
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(cfull + 2 * W_CB_N);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int nclus = (int)(gridDim.x >> 1), cid = (int)(blockIdx.x >> 1);
    const int tiles = tiles_m * tiles_n;
    const int nkb = Kp / TC_BK;
    auto origin = [&](int t, int &m0, int &n0) {   // grouped raster along M
        const int per_group = W_GROUP_M * tiles_n;
        const int first_m = (t / per_group) * W_GROUP_M;
        const int gsize = min(tiles_m - first_m, W_GROUP_M);
        m0 = (first_m + (t % per_group) % gsize) * (2 * TC_BM);
        n0 = ((t % per_group) / gsize) * W_BN;
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < W_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(&acc_full[0], 1);
        mbar_init(&acc_empty[0], 2 * TC_EPI_WARPS);
        mbar_init(&acc_empty[1], 2 * TC_EPI_WARPS);
        for (int i = 0; i < 2 * W_CB_N; ++i) mbar_init(&cfull[i], 1);
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
        if (TMAC) prefetch_tmap(&tmC);
    }
    if (warp == 1) tmem_alloc_2sm<TC_TMEM_COLS>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp == 0) {
        // ===== TMA producer (both CTAs: own A rows, own 128 columns of each B half) =====
        if (lane == 0) {
            uint32_t leader_full0;
            asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(leader_full0) : "r"(smem_u32(&full[0])));
            const uint64_t pol = policy_evict_normal();
            int it = 0;
            for (int t = cid; t < tiles; t += nclus) {
                int m0, n0;
                origin(t, m0, n0);
                const int arow = m0 + (int)rank * TC_BM;
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = it % W_STAGES;
                    mbar_wait(&empty[s], ((uint32_t)(it / W_STAGES) & 1u) ^ 1u);
                    const uint32_t fb = leader_full0 + (uint32_t)(s * sizeof(uint64_t));
                    if (rank == 0) mbar_arrive_expect_tx(&full[s], 2u * W_STAGE_BYTES);
                    const uint32_t st = smem_u32(smem + s * W_STAGE_BYTES);
                    auto load = [&](const CUtensorMap *tm, uint32_t dst, int row0, bool mn) {
                        if (mn) {
#pragma unroll
                            for (int c = 0; c < 4; ++c)
                                tma_load_2d_2sm(dst + c * 4096, tm, fb, row0 + 32 * c, kb * TC_BK, pol);
                        } else {
                            tma_load_2d_2sm(dst, tm, fb, kb * TC_BK, row0, pol);
                        }
                    };
                    load(&tmA, st, arow, A_MN);
                    load(&tmB, st + TC_TILE_BYTES, n0 + (int)rank * TC_BM, B_MN);
                    load(&tmB, st + 2 * TC_TILE_BYTES, n0 + 256 + (int)rank * TC_BM, B_MN);
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer (leader CTA, one thread) =====
        if (rank == 0 && lane == 0) {
            constexpr uint32_t idesc = idesc_tf32_major<2 * TC_BM, 256, A_MN, B_MN>();
            auto dsc = [](uint32_t addr, bool mn, int k) -> uint64_t {
                return mn ? desc_mnmajor_sw128_32b(addr + (uint32_t)(k * 1024))
                          : desc_kmajor_sw128(addr + (uint32_t)(k * 32));
            };
            // the 4 K8 MMAs of N-half h of the stage in ring slot s
            auto issue_half = [&](int s, int h, bool first_stage) {
                const uint32_t st = smem_u32(smem + s * W_STAGE_BYTES);
                const uint32_t b = st + (uint32_t)((1 + h) * TC_TILE_BYTES);
#pragma unroll
                for (int k = 0; k < TC_BK / 8; ++k)
                    mma_tf32_2sm(tmem_base + (uint32_t)(h * 256), dsc(st, A_MN, k), dsc(b, B_MN, k), idesc,
                                 (first_stage && k == 0) ? 0u : 1u);
            };
            int it = 0, tl = 0;   // global stage counter, local tile counter
            for (int t = cid; t < tiles; t += nclus, ++tl) {
                const int look = min(W_STAGES, nkb);
                // half 0 of the first `look` stages as soon as the epilogue
                // has drained half 0 of the previous tile ...
                mbar_wait(&acc_empty[0], ((uint32_t)tl & 1u) ^ 1u);
                tc_fence_after();
                for (int j = 0; j < look; ++j) {
                    const int s = (it + j) % W_STAGES;
                    mbar_wait(&full[s], (uint32_t)((it + j) / W_STAGES) & 1u);
                    tc_fence_after();
                    issue_half(s, 0, j == 0);
                }
                // ... then half 1 once it is drained too
                mbar_wait(&acc_empty[1], ((uint32_t)tl & 1u) ^ 1u);
                tc_fence_after();
                for (int j = 0; j < look; ++j) {
                    const int s = (it + j) % W_STAGES;
                    issue_half(s, 1, j == 0);
                    mma_commit_2sm_mc(&empty[s], (uint16_t)0x3);
                }
                it += look;
                for (int kb = look; kb < nkb; ++kb, ++it) {
                    const int s = it % W_STAGES;
                    mbar_wait(&full[s], (uint32_t)(it / W_STAGES) & 1u);
                    tc_fence_after();
                    issue_half(s, 0, false);
                    issue_half(s, 1, false);
                    mma_commit_2sm_mc(&empty[s], (uint16_t)0x3);
                }
                mma_commit_2sm_mc(&acc_full[0], (uint16_t)0x3);
            }
        }
    } else {
        // ===== epilogue: TMEM -> alpha*acc (+ beta*C) -> C, N-half 0 first =====
        const int q = warp & 3, hh = (warp - 2) >> 2;   // lane quarter, 128-column part of each half
        uint32_t leader_empty0;
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(leader_empty0) : "r"(smem_u32(&acc_empty[0])));
        int tl = 0, cph = 0;   // tile counter, C-chunk counter (TMAC ring phases)
        for (int t = cid; t < tiles; t += nclus, ++tl) {
            int m0, n0;
            origin(t, m0, n0);
            const int row = m0 + (int)rank * TC_BM + 32 * q + lane;
            mbar_wait(&acc_full[0], (uint32_t)tl & 1u);
            tc_fence_after();
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                const int col0 = n0 + h * 256 + hh * 128;
                const uint32_t tb = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(h * 256 + hh * 128);
                // this warp's 32 rows x 128 columns of half h -> registers, then
                // release the half at once: the next tile's MMAs may start on it
                // while the values are scaled and stored
                float acc[128];
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    uint32_t v[16];
                    tmem_ld_32x32b_x16(tb + (uint32_t)(16 * c), v);
#pragma unroll
                    for (int j = 0; j < 16; ++j) acc[16 * c + j] = __uint_as_float(v[j]);
                }
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    const uint32_t eb = leader_empty0 + (uint32_t)(h * sizeof(uint64_t));
                    mbar_arrive_remote(eb);
                }
                float *cp = C + (int64_t)row + (int64_t)col0 * ldc;
                const int jmax = min(128, N - col0);
                if (TMAC) {
                    // C_in chunks of 16 columns x this group's 128 rows through
                    // TMA into a 4-deep ring; stores stay per thread (coalesced)
                    const int rl = 32 * q + lane;                      // row within the CTA's 128
                    float *gb = cbuf + hh * (W_CB_N * W_CB_BYTES / 4);
                    uint64_t *gf = cfull + hh * W_CB_N;
                    const bool leader_t = q == (TC_EPI_WARP0 & 3) && lane == 0;   // first warp of the group
                    const int crow = m0 + (int)rank * TC_BM;
                    auto issue = [&](int c) {
                        const int b = c % W_CB_N;
                        mbar_arrive_expect_tx(&gf[b], W_CB_BYTES);
                        tma_load_2d(smem_u32(gb + b * (W_CB_BYTES / 4)), &tmC, &gf[b], crow, col0 + W_CB_COLS * c,
                                    policy_evict_first());
                    };
                    if (leader_t)
                        for (int c = 0; c < W_CB_N; ++c) issue(c);
#pragma unroll
                    for (int c = 0; c < 128 / W_CB_COLS; ++c, ++cph) {
                        const int b = c % W_CB_N;
                        mbar_wait(&gf[b], (uint32_t)((cph / W_CB_N) & 1));
                        const float *bp = gb + b * (W_CB_BYTES / 4) + rl;
                        float *sp = cp + (int64_t)(W_CB_COLS * c) * ldc;
#pragma unroll
                        for (int j = 0; j < W_CB_COLS; ++j, sp += ldc) {
                            const int jj = W_CB_COLS * c + j;
                            if (row < M && jj < jmax) __stcs(sp, fmaf(beta, bp[j * 128], alpha * acc[jj]));
                        }
                        // the group's 128 threads are done with buffer b
                        if (hh == 0)
                            asm volatile("bar.sync 1, 128;" ::: "memory");
                        else
                            asm volatile("bar.sync 2, 128;" ::: "memory");
                        if (leader_t && c + W_CB_N < 128 / W_CB_COLS) issue(c + W_CB_N);
                    }
                    continue;
                }
                if (row >= M) continue;
                if (beta == 0.0f) {
                    float *sp = cp;
#pragma unroll
                    for (int j = 0; j < 128; ++j, sp += ldc)
                        if (j < jmax) __stcs(sp, alpha * acc[j]);
                } else {
                    // 16 independent C loads before the 16 stores of a group
                    // (a store may alias a later load through ldc)
#pragma unroll
                    for (int g = 0; g < 8; ++g) {
                        float cin[16];
                        const float *lp = cp + (int64_t)(16 * g) * ldc;
#pragma unroll
                        for (int j = 0; j < 16; ++j, lp += ldc) cin[j] = (16 * g + j < jmax) ? __ldcs(lp) : 0.0f;
                        float *sp = cp + (int64_t)(16 * g) * ldc;
#pragma unroll
                        for (int j = 0; j < 16; ++j, sp += ldc)
                            if (16 * g + j < jmax) __stcs(sp, fmaf(beta, cin[j], alpha * acc[16 * g + j]));
                    }
                }
            }
        }
    }

    tc_fence_before();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_2sm<TC_TMEM_COLS>(tmem_base);
    }
}

// Policy: 1xTF32 problems of at least one full wave of 256 x 512 tiles
// (smaller ones keep KN2's split-K / finer tiles) and K >= 1024 (measured:
// 8192^3 1.72 -> 1.34 ms, 4096^3 0.256 -> 0.186, c4-i 0.95 -> 0.77; c4-ii,
// K = 1024 with beta = 1, 1.03 -> 0.94 ms once C_in comes through TMA, and
// 0.96 -> 0.79 ms at beta = 0: profiles/r01_ab_1x_wide*.txt).
// EMM_WIDE=0 / 1 forces.
bool tc1w_wanted(int64_t M, int64_t N, int64_t K) {
    const char *e = getenv("EMM_WIDE");
    if (e && e[0] == '0') return false;
    const int64_t tiles = ((M + 255) / 256) * ((N + W_BN - 1) / W_BN);
    if (e && e[0] == '1') return tiles <= 0x7fffffffLL;
    return N > 256 && K >= 1024 && tiles >= tc_num_sms() / 2 && tiles <= 0x7fffffffLL;
}

template <bool A_MN, bool B_MN, bool TMAC>
static cudaError_t launch_w(const TcOperands &ops, int64_t M, int64_t N, int64_t Kp, float alpha, float beta,
                            float *C, int64_t ldc, cudaStream_t s) {
    constexpr int SMEM = WCfg<TMAC>::SMEM;
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    static int max_clusters = 0;
    std::call_once(once, [] {
        attr_err = cudaFuncSetAttribute(tc1w_kernel<A_MN, B_MN, TMAC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        SMEM);
        cudaLaunchConfig_t oc{};
        oc.gridDim = dim3(2 * 64);
        oc.blockDim = dim3(32 * (TC_EPI_WARPS + 2));
        oc.dynamicSmemBytes = SMEM;
        int n = 0;
        if (attr_err == cudaSuccess &&
            cudaOccupancyMaxActiveClusters(&n, tc1w_kernel<A_MN, B_MN, TMAC>, &oc) != cudaSuccess)
            n = 0;
        max_clusters = n;
        cudaGetLastError();
    });
    if (attr_err != cudaSuccess) return attr_err;
    CUtensorMap ta, tb, tc;
    if (!tc_make_tmap(&ta, ops.a0, M) || !tc_make_tmap(&tb, ops.b0, N)) return cudaErrorInvalidValue;
    if (TMAC) {   // C_in tiles of 128 rows x 16 columns, no swizzle
        if (!encode_tmap_f32_2d(&tc, C, M, N, ldc, 128, W_CB_COLS, CU_TENSOR_MAP_SWIZZLE_NONE))
            return cudaErrorInvalidValue;
    } else {
        tc = ta;
    }
    const int tiles_m = (int)((M + 255) / 256), tiles_n = (int)((N + W_BN - 1) / W_BN);
    const int64_t tiles = (int64_t)tiles_m * tiles_n;
    int64_t clusters = tc_num_sms() / 2;
    if (max_clusters > 0 && clusters > max_clusters) clusters = max_clusters;
    if (clusters > tiles) clusters = tiles;
    cudaEvent_t ev = nullptr;
    prof_begin(s, true, &ev);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(2 * clusters));
    cfg.blockDim = dim3(32 * (TC_EPI_WARPS + 2));
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t le = cudaLaunchKernelEx(&cfg, tc1w_kernel<A_MN, B_MN, TMAC>, ta, tb, tc, (int)M, (int)N, (int)Kp,
                                        alpha, beta, C, ldc, tiles_m, tiles_n);
    if (le != cudaSuccess) return le;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    prof_end(s, true, ev);
    return cudaGetLastError();
}

template <bool A_MN, bool B_MN>
static cudaError_t launch_w2(const TcOperands &ops, int64_t M, int64_t N, int64_t Kp, float alpha, float beta,
                             float *C, int64_t ldc, cudaStream_t s) {
    const char *e = getenv("EMM_WIDE_TMAC");
    const bool tmac = beta != 0.0f && tma_legal(C, ldc) && !(e && e[0] == '0');
    return tmac ? launch_w<A_MN, B_MN, true>(ops, M, N, Kp, alpha, beta, C, ldc, s)
                : launch_w<A_MN, B_MN, false>(ops, M, N, Kp, alpha, beta, C, ldc, s);
}

cudaError_t launch_tc1w_sgemm(const TcOperands &ops, int64_t M, int64_t N, int64_t K, float alpha, float beta,
                              float *C, int64_t ldc, cudaStream_t s) {
    if (M > 0x7fffffffLL || N > 0x7fffffffLL || K > 0x7fffffffLL - 32) return cudaErrorInvalidValue;
    const int64_t Kp = tc_kpad(K);
    const bool am = ops.a0.mn, bm = ops.b0.mn;
    if (!am && !bm) return launch_w2<false, false>(ops, M, N, Kp, alpha, beta, C, ldc, s);
    if (!am && bm) return launch_w2<false, true>(ops, M, N, Kp, alpha, beta, C, ldc, s);
    if (am && !bm) return launch_w2<true, false>(ops, M, N, Kp, alpha, beta, C, ldc, s);
    return launch_w2<true, true>(ops, M, N, Kp, alpha, beta, C, ldc, s);
}

}  // namespace emm
