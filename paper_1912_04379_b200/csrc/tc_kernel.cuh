// tc_kernel.cuh — KN1/KN2 (tcgen05 GEMM on CTA pairs) and its launch
// templates; included by k_tc_t1.cu / k_tc_t2.cu / k_tc_t3.cu, one
// translation unit per split so the (many) kernel instantiations compile in
// parallel.  Host helpers (tensor maps, schedules, the split pass, the
// split-K reduce) live in k_tc.cu.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "emm_internal.h"
#include "ptx.cuh"
#include "tc_common.cuh"

namespace emm {

using namespace ptx;

// =====================================================================
// KN1/KN2: tcgen05 GEMM, CTA pair per 256x256 tile.  Four 2-D tensor maps:
// A plane 0/1, B plane 0/1; plane 0 (big) and, for 3xTF32, plane 1 (small)
// are K-major or MN-major per A_MN / B_MN; the TF32+BF16 cross plane is
// always K-major.
//
// Accumulation precision (Q7, measured on B200): the tensor core
// adds each MMA's result into the TMEM accumulator with truncation, which on
// same-sign data biases a K=16384 sum by ~1.8e-4 relative.  So the K loop is
// cut into chunks of `kc_stages` stages: each chunk accumulates in one of two
// TMEM buffers (ping-pong, 2 x 256 columns) and the epilogue warps drain the
// finished buffer into FP32 registers with round-to-nearest adds while the
// MMAs run on the other buffer ("promotion"), bounding the truncation bias
// to one chunk.
// =====================================================================
// Cluster size from the launch (2, or a preferred 4 = two CTA pairs sharing
// B by TMA multicast for data-parallel launches); tmB0h/tmB1h:
// the K-major B planes with 64-row boxes for the multicast half-loads.
template <int TERMS, bool A_MN, bool B_MN, bool MC, bool TMAC>
__global__ void __launch_bounds__(TC_THREADS_P, 1)
    tc_sgemm_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
                    const __grid_constant__ CUtensorMap tmB0, const __grid_constant__ CUtensorMap tmB1,
                    const __grid_constant__ CUtensorMap tmB0h, const __grid_constant__ CUtensorMap tmB1h,
                    const __grid_constant__ CUtensorMap tmC, int M, int N,
                    int Kp, float alpha, float beta, float *C, int64_t ldc, int tiles_m, int tiles_n,
                    int group_m, int kc_stages, unsigned int *__restrict__ wave_ctr, int splits,
                    float *__restrict__ partial, const TcSk sk, const __grid_constant__ PeerOut peers,
                    const float *acc_init, int64_t ld_init) {   // acc_init may equal C (K-phased calls)
    if (threadIdx.x == 0) EMM_TL(0);
    using Cfg = TcCfg<TERMS>;
    constexpr bool A1_MN = TERMS == 3 ? A_MN : false;   // cross planes are K-major
    constexpr bool B1_MN = TERMS == 3 ? B_MN : false;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    float *cbuf = reinterpret_cast<float *>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);   // TMAC: C_in ring
    uint64_t *full =
        reinterpret_cast<uint64_t *>(smem + Cfg::STAGES * Cfg::STAGE_BYTES + (TMAC ? TC_CBUF_BYTES : 0));
    uint64_t *empty = full + Cfg::STAGES;
    uint64_t *acc_full = empty + Cfg::STAGES;     // [2]
    uint64_t *acc_empty = acc_full + 2;           // [2] (leader's counts both CTAs' epilogue warps)
    uint64_t *cfull = acc_empty + 2;              // TMAC: [2 halves][TC_CB_N]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(cfull + 2 * TC_CB_N);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = cluster_ctarank();
    const int cl = MC ? (int)cluster_nctarank() : 2;   // 2, or 4 (two pairs; MC launches only)
    const uint32_t rank = crank & 1u;                // rank in the CTA pair
    const uint32_t leader = crank & ~1u;             // the pair leader's cluster rank
    const int pair = (int)(crank >> 1);              // pair in the cluster

    const int nclus = (int)(gridDim.x >> 1);         // CTA pairs
    const int cid = (int)(blockIdx.x >> 1);
    const TcSched S(tiles_m, tiles_n, group_m, Kp, splits, sk.dp_tiles, TC_SK_CHUNK, nclus, cid);
    const int n_it = tc_n_items(S, cl);

    if (threadIdx.x == 0) {
        for (int s = 0; s < Cfg::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], (uint32_t)(cl / 2));   // one stage-release commit per pair
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 2 * TC_EPI_WARPS);
        }
        if (TMAC)
            for (int b = 0; b < 2 * TC_CB_N; ++b) mbar_init(&cfull[b], 1);
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmA0);
        prefetch_tmap(&tmB0);
        if (TMAC) prefetch_tmap(&tmC);
        if (Cfg::PLANES == 2) {
            prefetch_tmap(&tmA1);
            prefetch_tmap(&tmB1);
        }
    }
    if (warp == 1) tmem_alloc_2sm<TC_TMEM_COLS>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0) EMM_TL(1);
    // PDL: everything above overlapped the previous kernel (the pack pass);
    // from here on this grid reads its outputs (and C, wave counter).
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) EMM_TL(2);

    if (warp == 0) {
        // ===== TMA producer (both CTAs; each loads its half of A and B) =====
        if (lane == 0) {
            uint32_t leader_full0;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                         : "=r"(leader_full0)
                         : "r"(smem_u32(&full[0])), "r"(leader));
            const uint64_t pol = policy_evict_normal();
            int it = 0;
            unsigned int done_target = 0;   // CTAs that finished issuing waves 0..w-1
            int cur_wave = 0;
            bool lockstep = wave_ctr != nullptr;
            for (int i = 0; i < n_it; ++i) {
                const int w = S.wave_of(i);
                if (w != cur_wave || i == 0) {
                    if (w > 0 && lockstep) {
                        // Wave lockstep: start loading wave w only when every CTA
                        // has issued all loads of wave w-1, so the ~17 operand
                        // panels a wave shares stream through L2 once.  It is an
                        // L2 optimisation, not a correctness barrier: when the
                        // grid is not fully co-resident (another kernel holds
                        // SMs, e.g. concurrent GEMMs on other streams) the wait
                        // gives up after ~1 ms and this CTA drops the lockstep
                        // for the rest of the launch (no cross-kernel deadlock).
                        for (int v = cur_wave; v < w; ++v) done_target += 2u * (unsigned)S.pairs_in_wave(v);
                        const long long t0 = clock64();
                        while (true) {
                            unsigned int v;
                            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(wave_ctr) : "memory");
                            if (v >= done_target) break;
                            __nanosleep(128);
                            if (clock64() - t0 > TC_LOCKSTEP_TIMEOUT) {
                                lockstep = false;
                                break;
                            }
                        }
                    }
                    cur_wave = w;
                }
                TcItem ti;
                tc_get_item(S, cl, i, ti);
                const TcWork &wk = ti.w;
                const int m0 = wk.m0, n0 = wk.n0, kb0 = wk.kb0, kb1 = wk.kb1;
                const int arow = m0 + (int)rank * TC_BM;
                const int brow = n0 + (int)rank * TC_BM;
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const int s = it % Cfg::STAGES;
                    const uint32_t ph = (uint32_t)(it / Cfg::STAGES) & 1u;
                    mbar_wait(&empty[s], ph ^ 1u);
                    const uint32_t fb = leader_full0 + (uint32_t)(s * sizeof(uint64_t));
                    if (rank == 0) mbar_arrive_expect_tx(&full[s], 2u * Cfg::STAGE_BYTES);
                    const uint32_t st = smem_u32(smem + s * Cfg::STAGE_BYTES);
                    // a 128 (rows) x 32 (K) tile of one plane: one K-major box, or
                    // four MN-major 32x32 boxes (transpose in the TMA box)
                    auto load_plane = [&](const CUtensorMap *tm, uint32_t dst, int row0, bool mn) {
                        if (mn) {
#pragma unroll
                            for (int c = 0; c < 4; ++c)
                                tma_load_2d_2sm(dst + c * 4096, tm, fb, row0 + 32 * c, kb * TC_BK, pol);
                        } else {
                            tma_load_2d_2sm(dst, tm, fb, kb * TC_BK, row0, pol);
                        }
                    };
                    // multicast (4-cluster, shared B): half of this CTA's B
                    // half-tile, to the same-rank CTA of both pairs; completion on
                    // each destination pair leader's barrier at this offset
                    const uint32_t fbm = smem_u32(&full[s]) & 0xFEFFFFFFu;
                    const uint16_t mask = (uint16_t)((1u << rank) | (1u << (2 + rank)));
                    auto load_b = [&](const CUtensorMap *tm, const CUtensorMap *tmh, uint32_t dst, bool mn) {
                        if (!ti.mc) {
                            load_plane(tm, dst, brow, mn);
                        } else if (mn) {
#pragma unroll
                            for (int c = 2 * pair; c < 2 * pair + 2; ++c)
                                tma_load_2d_2sm_mc(dst + c * 4096, tm, fbm, brow + 32 * c, kb * TC_BK, mask, pol);
                        } else {
                            tma_load_2d_2sm_mc(dst + pair * 8192, tmh, fbm, kb * TC_BK, brow + 64 * pair, mask, pol);
                        }
                    };
                    load_plane(&tmA0, st, arow, A_MN);
                    load_b(&tmB0, &tmB0h, st + Cfg::PLANES * TC_TILE_BYTES, B_MN);
                    if (Cfg::PLANES == 2) {
                        load_plane(&tmA1, st + TC_TILE_BYTES, arow, A1_MN);
                        load_b(&tmB1, &tmB1h, st + 3 * TC_TILE_BYTES, B1_MN);
                    }
                }
                // this CTA has issued every load of its current wave
                if (wave_ctr && (i + 1 == n_it || S.wave_of(i + 1) != cur_wave))
                    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(wave_ctr) : "memory");
            }
        }
    } else if (warp == 1) {
        if (rank == 0 && lane == 0)
            tc_mma_loop<TERMS, A_MN, B_MN, A1_MN, B1_MN, Cfg::PLANES, Cfg::STAGES, Cfg::STAGE_BYTES, MC>(
                S, smem, full, empty, acc_full, acc_empty, tmem_base, kc_stages, cl, pair);
    } else if (warp >= TC_EPI_WARP0) {
        tc_epilogue_loop<MC, TMAC>(S, rank, warp & 3, (warp - TC_EPI_WARP0) >> 2, lane, tmem_base, acc_full,
                                   acc_empty, kc_stages, M, N, alpha, beta, C, ldc, partial, sk, peers, cl, leader,
                                   acc_init, ld_init, TcCin{&tmC, cbuf, cfull});
    }

    tc_fence_before();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_2sm<TC_TMEM_COLS>(tmem_base);
    }
    if (threadIdx.x == 0) EMM_TL(7);
}


// Preferred clusters of 4 (B multicast between two CTA pairs) for the
// data-parallel 3xTF32 / TF32+BF16 schedule at K >= 4096 (measured, one
// B200: c5 260.0 -> 262.3 / 263.6 TFLOP/s, c2-8192 +0.6% (3x) / +1.2%
// (TF32+BF16); c4-ii, K = 1024, -5%: profiles/r01_ab_pref4.txt).
// EMM_PREF4=0 / 1 forces.
static bool tc_pref4_wanted(int terms, int64_t K) {
    const char *e = getenv("EMM_PREF4");
    if (e && e[0] == '0') return false;
    if (e && e[0] == '1') return true;
    return terms >= 2 && K >= 4096;
}

template <int TERMS, bool A_MN, bool B_MN>
static cudaError_t launch_tc_t(const TcOperands &ops, int64_t M, int64_t N, int64_t Kp, float alpha, float beta,
                               float *C, int64_t ldc, unsigned int *ctrl, int splits, float *partial, cudaStream_t s,
                               const PeerOut &peers, void *sk_ws, const float *acc_init, int64_t ld_init) {
    if (acc_init && splits != 1) return cudaErrorInvalidValue;
    if (acc_init) sk_ws = nullptr;   // whole tiles only
    using Cfg = TcCfg<TERMS>;
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    constexpr int SMEM_T = Cfg::SMEM_BYTES + TC_CBUF_BYTES;   // TMAC variants: + the C_in ring
    std::call_once(once, [] {
        auto set = [](const void *f, int smem, bool cl4) {
            cudaError_t r = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (r == cudaSuccess && cl4) r = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            if (r != cudaSuccess && attr_err == cudaSuccess) attr_err = r;
        };
        set((const void *)tc_sgemm_kernel<TERMS, A_MN, B_MN, false, false>, Cfg::SMEM_BYTES, false);
        set((const void *)tc_sgemm_kernel<TERMS, A_MN, B_MN, false, TERMS >= 2>, SMEM_T, false);
        set((const void *)tc_sgemm_kernel<TERMS, A_MN, B_MN, TERMS >= 2, false>, Cfg::SMEM_BYTES, true);
        set((const void *)tc_sgemm_kernel<TERMS, A_MN, B_MN, TERMS >= 2, TERMS >= 2>, SMEM_T, true);
    });
    if (attr_err != cudaSuccess) return attr_err;
    CUtensorMap ta0, ta1, tb0, tb1, tb0h, tb1h;
    if (!tc_make_tmap(&ta0, ops.a0, M) || !tc_make_tmap(&tb0, ops.b0, N)) return cudaErrorInvalidValue;
    if (Cfg::PLANES == 2) {
        if (!tc_make_tmap(&ta1, ops.a1, M) || !tc_make_tmap(&tb1, ops.b1, N)) return cudaErrorInvalidValue;
    } else {
        ta1 = ta0;
        tb1 = tb0;
    }
    // beta != 0, TMA-legal C (3xTF32 / TF32+BF16): C_in through TMA (EMM_TMAC=0: off)
    const char *etc = getenv("EMM_TMAC");
    const bool tmac = TERMS >= 2 && beta != 0.0f && tma_legal(C, ldc) && !(etc && etc[0] == '0');
    CUtensorMap tcm;
    if (tmac) {
        if (!encode_tmap_f32_2d(&tcm, C, M, N, ldc, 128, TC_CB_COLS, CU_TENSOR_MAP_SWIZZLE_NONE))
            return cudaErrorInvalidValue;
    } else {
        tcm = ta0;
    }
    // K-major B planes with 64-row boxes: the multicast half-loads of 4-clusters
    if (!tc_make_tmap_rows(&tb0h, ops.b0, N, TC_BM / 2) ||
        !tc_make_tmap_rows(&tb1h, Cfg::PLANES == 2 ? ops.b1 : ops.b0, N, TC_BM / 2))
        return cudaErrorInvalidValue;
    const int tiles_m = (int)((M + 2 * TC_BM - 1) / (2 * TC_BM));
    const int tiles_n = (int)((N + TC_BN - 1) / TC_BN);
    const int group_m = 8;
    // 1xTF32 is operand-fill-bound: the wave lockstep's boundary stalls cost
    // more than its L2 reuse buys (c4-ii +4.7%, c4-i +2.4% without it;
    // 3xTF32 -1%, profiles/r01_ab_1x_lockstep_group.txt)
    if (TERMS == 1) ctrl = nullptr;
    const int64_t units = (int64_t)tiles_m * tiles_n * splits;
    if (units > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    const int64_t pairs = tc_num_sms() / 2;
    TcSk sk{0x7fffffff, nullptr, nullptr};   // dp_tiles >= tiles: stream-K off
    int dp = 0;
    if (sk_ws && tc_sk_plan(M, N, Kp, splits, TERMS, &dp)) {
        sk.dp_tiles = dp;
        sk.flags = reinterpret_cast<unsigned int *>(sk_ws);
        sk.slots = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(sk_ws) + TC_SK_FLAG_BYTES);
    }
    // persistent: one pair per 2 SMs (all of them when stream-K spreads the last wave)
    int64_t clusters = sk.slots ? pairs : (units < pairs ? units : pairs);
    // The persistent schedule (wave lockstep, stream-K flags) needs every
    // cluster co-resident; clusters live inside one GPC, so cap the grid at
    // what the occupancy API says fits (all 74 pairs on a B200).
    static std::once_flag occ_once;
    static int max_clusters = 0;
    std::call_once(occ_once, [] {
        cudaLaunchConfig_t oc{};
        oc.gridDim = dim3(2 * 64);
        oc.blockDim = dim3(TC_THREADS_P);
        oc.dynamicSmemBytes = TcCfg<TERMS>::SMEM_BYTES;
        cudaLaunchAttribute ca[1];
        ca[0].id = cudaLaunchAttributeClusterDimension;
        ca[0].val.clusterDim.x = 2;
        ca[0].val.clusterDim.y = 1;
        ca[0].val.clusterDim.z = 1;
        oc.attrs = ca;
        oc.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, tc_sgemm_kernel<TERMS, A_MN, B_MN, false, false>, &oc) != cudaSuccess)
            n = 0;
        max_clusters = n;
        cudaGetLastError();
    });
    if (max_clusters > 0 && clusters > max_clusters) {
        if (sk.slots) sk = TcSk{0x7fffffff, nullptr, nullptr};   // stream-K ranges assume every pair resident
        clusters = max_clusters;
    }
    const int64_t blocks = 2 * clusters;
    cudaEvent_t ev = nullptr;
    prof_begin(s, true, &ev);
    // promotion chunk: 256 of K for the FP32-accurate splits (8 stages)
    const int kc_stages = TERMS >= 2 ? 256 / TC_BK : 0x3fffffff;
    {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)blocks);
        cfg.blockDim = dim3(TC_THREADS_P);
        cfg.dynamicSmemBytes = tmac ? SMEM_T : Cfg::SMEM_BYTES;
        cfg.stream = s;
        // clusters of one CTA pair; for data-parallel schedules a PREFERRED
        // size of 4 (two pairs sharing B by multicast; the B200 forms as many
        // 4-clusters as its GPCs hold and pairs on the remaining SMs)
        cudaLaunchAttribute at[3];
        cudaLaunchAttribute at_sk[3];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = 2;
        at[1].val.clusterDim.y = 1;
        at[1].val.clusterDim.z = 1;
        at[2].id = cudaLaunchAttributePreferredClusterDimension;
        at[2].val.preferredClusterDim.x = 4;
        at[2].val.preferredClusterDim.y = 1;
        at[2].val.preferredClusterDim.z = 1;
        cfg.attrs = at;
        const bool mc = TERMS >= 2 && tc_pref4_wanted(TERMS, Kp) && splits == 1 && !sk.slots && blocks % 4 == 0;
        cfg.numAttrs = mc ? 3 : 2;
        constexpr bool T2 = TERMS >= 2;
        auto kern = mc ? (tmac ? tc_sgemm_kernel<TERMS, A_MN, B_MN, T2, T2> : tc_sgemm_kernel<TERMS, A_MN, B_MN, T2, false>)
                       : (tmac ? tc_sgemm_kernel<TERMS, A_MN, B_MN, false, T2>
                               : tc_sgemm_kernel<TERMS, A_MN, B_MN, false, false>);
        // Stream-K: an owner CTA waits for pieces published by other CTAs of
        // the grid, so the grid must be co-resident even when other kernels
        // (e.g. a concurrent GEMM on another stream) hold SMs: launch it
        // cooperatively (the driver then starts it only as a whole).  If the
        // cooperative launch is refused, run the data-parallel schedule.
        if (sk.slots) {
            at_sk[0] = at[0];
            at_sk[1] = at[1];
            at_sk[2].id = cudaLaunchAttributeCooperative;
            at_sk[2].val.cooperative = 1;
            cfg.attrs = at_sk;
            cfg.numAttrs = 3;
        }
        auto launch = [&]() {
            return cudaLaunchKernelEx(&cfg, kern, ta0, ta1, tb0, tb1, tb0h, tb1h, tcm, (int)M, (int)N, (int)Kp,
                                      alpha, beta, C, ldc, tiles_m, tiles_n, group_m, kc_stages, ctrl, splits,
                                      splits > 1 ? partial : nullptr, sk, peers, acc_init, ld_init);
        };
        cudaError_t le = launch();
        if (le != cudaSuccess && sk.slots) {
            cudaGetLastError();
            sk = TcSk{0x7fffffff, nullptr, nullptr};
            const int64_t dp_clusters = units < pairs ? units : pairs;
            cfg.gridDim = dim3((unsigned)(2 * (max_clusters > 0 && dp_clusters > max_clusters ? max_clusters
                                                                                                : dp_clusters)));
            cfg.attrs = at;
            cfg.numAttrs = 2;
            le = launch();
        }
        if (le != cudaSuccess) return le;
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    prof_end(s, true, ev);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || splits <= 1) return e;
    return launch_splitk_reduce(partial, splits, M, N, alpha, beta, C, ldc, s);
}

template <int TERMS>
static cudaError_t launch_tc_m(const TcOperands &ops, int64_t M, int64_t N, int64_t Kp, float alpha, float beta,
                               float *C, int64_t ldc, unsigned int *ctrl, int splits, float *partial, cudaStream_t s,
                               const PeerOut &pe, void *sk, const float *ai, int64_t ldi) {
    const bool am = ops.a0.mn, bm = ops.b0.mn;
    if (!am && !bm)
        return launch_tc_t<TERMS, false, false>(ops, M, N, Kp, alpha, beta, C, ldc, ctrl, splits, partial, s, pe, sk,
                                                ai, ldi);
    if (!am && bm)
        return launch_tc_t<TERMS, false, true>(ops, M, N, Kp, alpha, beta, C, ldc, ctrl, splits, partial, s, pe, sk,
                                               ai, ldi);
    if (am && !bm)
        return launch_tc_t<TERMS, true, false>(ops, M, N, Kp, alpha, beta, C, ldc, ctrl, splits, partial, s, pe, sk,
                                               ai, ldi);
    return launch_tc_t<TERMS, true, true>(ops, M, N, Kp, alpha, beta, C, ldc, ctrl, splits, partial, s, pe, sk, ai,
                                          ldi);
}

}  // namespace emm
