// k_tcx.cu — KN1X: tcgen05 3xTF32 GEMM with the operand split INSIDE the
// kernel, fed by TMA (the "TMA way").
//
// The tensor core truncates FP32 operands to TF32 (measured, R7b),
// so the raw operand tile IS the big part.  Per K-stage each CTA's producer
// TMAs only the raw 128x32 A and B tiles of the caller's arrays (in place:
// K-major or MN-major per trans flag, the transpose in the TMA box and the
// UMMA descriptor, OOB rows / columns / k read as zero), and a transform
// warpgroup writes
//     small = rn_tf32(x - trunc_tf32(x))     (x - trunc exact; 0 for non-finite x)
// element by element into the stage's second tile at the SAME offset — the
// 128B swizzle permutes 16-byte chunks identically in both tiles, so the
// transform never needs to know the layout.  That is exactly the plane the
// split pass KN4 writes for the direct path (PK_DSMALL), so this kernel and
// "split pass + KN1 direct" add the same products in the same order: bitwise
// identical results (tests/test_gpu_xs.py).  It removes the split pass
// launch, its HBM round trip of the small planes and the workspace for them,
// and halves the L2 -> SMEM operand traffic per flop (one raw FP32 copy
// instead of two planes).  The price is SMEM port traffic: MMA operand reads
// 64 B/clk + TMA fill 21 + transform read/write 43 = ~128 B/clk per SM at the
// full tensor rate (KN1 pre-split: 107).  (Paper analogue: B' "re-buffering"
// and A' prefetch, done on chip per stage.)
//
// Warp roles (512 threads, 4 warpgroups; setmaxnreg re-balances registers):
//   warpgroup 0: warp 0 = TMEM owner + MMA issuer (leader CTA, one lane);
//                warp 1 = TMA producer (one lane, each CTA); warps 2-3 idle
//   warpgroup 1: 4 transform warps (LDS raw -> small -> STS, each CTA)
//   warpgroups 2-3: 8 promotion/epilogue warps (tc_common.cuh)
// Barriers per stage s: rawfull[s] (each CTA: its TMA bytes landed),
// full[s] (leader: both CTAs' transform warps done), empty[s] (each CTA:
// the pair's MMAs finished reading the stage).
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

constexpr int TX_STAGES = 3;
constexpr int TX_STAGE_BYTES = 4 * TC_TILE_BYTES;   // A raw | A small | B raw | B small
constexpr int TX_XF_WARP0 = 4, TX_XF_WARPS = 4;
constexpr int TX_EPI_WARP0 = 8;
constexpr int TX_THREADS = 512;
constexpr int TX_SMEM_BYTES = TX_STAGES * TX_STAGE_BYTES + 1024 /*align*/ + 512 /*barriers*/;
constexpr int TX_REGS_WG0 = 48, TX_REGS_XF = 96, TX_REGS_EPI = 184;
static_assert(128 * TX_REGS_WG0 + 128 * TX_REGS_XF + 256 * TX_REGS_EPI <= 65536, "register budget");

__device__ __forceinline__ float tx_small(float x) {
    const uint32_t u = __float_as_uint(x);
    if ((u & 0x7F800000u) == 0x7F800000u) return 0.0f;   // inf / NaN: big*big alone carries it
    const float lo = x - __uint_as_float(u & 0xFFFFE000u);   // exact
    return __uint_as_float(cvt_tf32_rn(lo));
}

__device__ __forceinline__ void tx_split_rn(float x, float &big, float &small) {
    big = __uint_as_float(cvt_tf32_rn(x));
    small = isfinite(x) ? __uint_as_float(cvt_tf32_rn(x - big)) : 0.0f;   // x - big exact
}

// RN: the transform also rounds the big part in place (big = rn_tf32(x) over
// the raw tile, small = rn_tf32(x - big)): the re-buffered planes' numerics
// (bitwise equal to PK_FULL3 + KN1), with zeroed low mantissa bits in the
// tensor core's operands (lower switching power under the 1 kW cap) for
// 21 B/clk more SMEM writes.  EMM_XS_RN=1.
// CSK (cluster split-K, sub-wave shapes): the grid is one cluster of S CTA
// pairs per output tile, pair p computing K split p; each CTA keeps its raw
// partial in its (then idle) SMEM ring and the cluster reduces the tile over
// DSMEM — CTA (p, r) sums the S partials of its 128 rows on the column range
// p*256/S .. (p+1)*256/S in the fixed order s = 0..S-1 (KN8's order: bitwise
// equal to global split-K + the reduce launch), applies alpha/beta and stores
// C.  No partial slots in HBM, no reduce launch.
template <bool A_MN, bool B_MN, bool TMAC, bool RN, bool CSK>
__global__ void __launch_bounds__(TX_THREADS, 1)
    tc_xs_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmC, int M, int N, int Kp, float alpha, float beta, float *C,
                 int64_t ldc, int tiles_m, int tiles_n, int group_m, int kc_stages,
                 unsigned int *__restrict__ wave_ctr, int splits, float *__restrict__ partial, const TcSk sk,
                 const __grid_constant__ PeerOut peers, const float *acc_init, int64_t ld_init, int early) {
    if (threadIdx.x == 0) EMM_TL(0);
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    float *cbuf = reinterpret_cast<float *>(smem + TX_STAGES * TX_STAGE_BYTES);   // TMAC: C_in ring
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + TX_STAGES * TX_STAGE_BYTES + (TMAC ? TC_CBUF_BYTES : 0));
    uint64_t *empty = full + TX_STAGES;
    uint64_t *rawfull = empty + TX_STAGES;
    uint64_t *acc_full = rawfull + TX_STAGES;     // [2]
    uint64_t *acc_empty = acc_full + 2;           // [2]
    uint64_t *cfull = acc_empty + 2;              // TMAC: [2 halves][TC_CB_N]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(cfull + 2 * TC_CB_N);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = cluster_ctarank();
    const uint32_t rank = crank & 1u;                 // rank in the CTA pair
    const uint32_t leader = crank & ~1u;              // the pair leader's cluster rank
    const int pairc = CSK ? (int)(crank >> 1) : 0;    // CSK: the pair's K split
    // CSK: pair p of cluster k runs unit (split p, tile k) of the split-K schedule
    const int ntile = tiles_m * tiles_n;
    const int nclus = CSK ? ntile * splits : (int)(gridDim.x >> 1);
    const int cid = CSK ? pairc * ntile + (int)(blockIdx.x / (2 * splits)) : (int)(blockIdx.x >> 1);
    const TcSched S(tiles_m, tiles_n, group_m, Kp, splits, sk.dp_tiles, TC_SK_CHUNK, nclus, cid);

    const int n_it = S.n_items;
    // ===== TMA producer state (warp 1, one lane; each CTA: its 128 rows of A
    // and of B, raw).  The producer's barriers are its own CTA's, so it
    // issues the first ring pass between the cluster barrier's arrive and its
    // wait, overlapping the pair's TMEM allocation / cluster handshake
    // (griddepcontrol.wait first: A and B may be written by the previous
    // kernel).  EMM_XS_EARLY=0 issues after the full handshake.
    const bool producer = warp == 1 && lane == 0;
    const uint64_t pol = policy_evict_normal();
    int p_i = 0, p_kb = 0, p_kb1 = 0, p_it = 0, cur_wave = 0;
    unsigned int done_target = 0;
    bool lockstep = wave_ctr != nullptr, p_open = false;
    int arow = 0, brow = 0;
    // one K-stage of loads; false when the unit list is exhausted
    auto produce = [&]() -> bool {
        while (!p_open || p_kb >= p_kb1) {
            if (p_open) {
                // the item is done: wave counter, next item
                if (wave_ctr && (p_i + 1 == n_it || S.wave_of(p_i + 1) != cur_wave))
                    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(wave_ctr) : "memory");
                ++p_i;
                p_open = false;
            }
            if (p_i >= n_it) return false;
            const int w = S.wave_of(p_i);
            if (w != cur_wave || p_i == 0) {
                if (w > 0 && lockstep) {
                    // wave lockstep (tc_kernel.cuh): an L2 optimisation, dropped
                    // after ~1 ms if the grid is not co-resident
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
            TcWork wk;
            S.item(p_i, wk);
            arow = wk.m0 + (int)rank * TC_BM;
            brow = wk.n0 + (int)rank * TC_BM;
            p_kb = wk.kb0;
            p_kb1 = wk.kb1;
            p_open = true;
        }
        const int s = p_it % TX_STAGES;
        const uint32_t ph = (uint32_t)(p_it / TX_STAGES) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        mbar_arrive_expect_tx(&rawfull[s], 2u * TC_TILE_BYTES);
        const uint32_t st = smem_u32(smem + s * TX_STAGE_BYTES);
        auto load = [&](const CUtensorMap *tm, uint32_t dst, int row0, bool mn) {
            if (mn) {
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    tma_load_2d(dst + c * 4096, tm, &rawfull[s], row0 + 32 * c, p_kb * TC_BK, pol);
            } else {
                tma_load_2d(dst, tm, &rawfull[s], p_kb * TC_BK, row0, pol);
            }
        };
        load(&tmA, st, arow, A_MN);
        load(&tmB, st + 2 * TC_TILE_BYTES, brow, B_MN);
        ++p_kb;
        ++p_it;
        return true;
    };

    if (producer) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
        if (TMAC) prefetch_tmap(&tmC);
        for (int s = 0; s < TX_STAGES; ++s) {
            mbar_init(&full[s], 2 * TX_XF_WARPS);   // leader's: transform warps of both CTAs
            mbar_init(&empty[s], 1);                // the pair's stage-release commit
            mbar_init(&rawfull[s], 1);              // this CTA's TMA bytes
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 2 * TC_EPI_WARPS);
        }
        if (TMAC)
            for (int b = 0; b < 2 * TC_CB_N; ++b) mbar_init(&cfull[b], 1);
        fence_mbar_init();
        EMM_TL(8);
    }
    if (warp == 0) tmem_alloc_2sm<TC_TMEM_COLS>(tmem_slot);
    if (warp == 0 && lane == 0) EMM_TL(9);
    tc_fence_before();
    __syncwarp();
    cluster_arrive();
    if (producer && early) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        for (int k = 0; k < TX_STAGES; ++k)
            if (!produce()) break;
    }
    __syncwarp();
    cluster_wait();
    if (threadIdx.x == 0) EMM_TL(10);
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0) EMM_TL(1);
    // PDL: the prologue above may overlap the previous kernel on the stream
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) EMM_TL(2);

    if (warp < TX_XF_WARP0) {
        setmaxnreg_dec<TX_REGS_WG0>();
        if (warp == 0 && rank == 0 && lane == 0) {
            tc_mma_loop<3, A_MN, B_MN, A_MN, B_MN, 2, TX_STAGES, TX_STAGE_BYTES, CSK>(
                S, smem, full, empty, acc_full, acc_empty, tmem_base, kc_stages, 2, pairc);
        } else if (producer) {
            while (produce()) {
            }
        }
    } else if (warp < TX_EPI_WARP0) {
        setmaxnreg_dec<TX_REGS_XF>();
        // ===== transform: small = rn_tf32(x - trunc(x)) beside each raw tile =====
        const int t = threadIdx.x - 32 * TX_XF_WARP0;   // 0..127
        uint32_t leader_full0;   // the pair leader's full[0]
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(leader_full0) : "r"(smem_u32(&full[0])), "r"(leader));
        int it = 0;
        for (int i = 0; i < n_it; ++i) {
            TcWork wk;
            S.item(i, wk);
            for (int kb = wk.kb0; kb < wk.kb1; ++kb, ++it) {
                const int s = it % TX_STAGES;
                const uint32_t ph = (uint32_t)(it / TX_STAGES) & 1u;
                mbar_wait(&rawfull[s], ph);
                uint8_t *st = smem + s * TX_STAGE_BYTES;
                float4 v[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int off = (j < 8 ? 0 : 2 * TC_TILE_BYTES) + (t + 128 * (j & 7)) * 16;
                    v[j] = *reinterpret_cast<const float4 *>(st + off);
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int off = (j < 8 ? 0 : 2 * TC_TILE_BYTES) + (t + 128 * (j & 7)) * 16;
                    if (RN) {
                        float4 b, sm;
                        tx_split_rn(v[j].x, b.x, sm.x);
                        tx_split_rn(v[j].y, b.y, sm.y);
                        tx_split_rn(v[j].z, b.z, sm.z);
                        tx_split_rn(v[j].w, b.w, sm.w);
                        *reinterpret_cast<float4 *>(st + off) = b;
                        *reinterpret_cast<float4 *>(st + off + TC_TILE_BYTES) = sm;
                    } else {
                        *reinterpret_cast<float4 *>(st + off + TC_TILE_BYTES) =
                            make_float4(tx_small(v[j].x), tx_small(v[j].y), tx_small(v[j].z), tx_small(v[j].w));
                    }
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive_remote(leader_full0 + (uint32_t)(s * sizeof(uint64_t)));
            }
        }
    } else {
        setmaxnreg_inc<TX_REGS_EPI>();
        tc_epilogue_loop<CSK, TMAC>(S, rank, warp & 3, (warp - TX_EPI_WARP0) >> 2, lane, tmem_base, acc_full,
                                    acc_empty, kc_stages, M, N, alpha, beta, C, ldc, partial, sk, peers, 2, leader,
                                    acc_init, ld_init, TcCin{&tmC, cbuf, cfull},
                                    CSK ? reinterpret_cast<float *>(smem) : nullptr);
    }

    tc_fence_before();
    cluster_sync();
    if (CSK && warp >= TX_EPI_WARP0) {
        // ===== cluster reduce of the tile's S partials (DSMEM), alpha/beta, C =====
        TcWork w;
        S.item(0, w);
        const int t = threadIdx.x - 32 * TX_EPI_WARP0;   // 0..255
        const int rl = t & 127, par = t >> 7;
        const int row = w.m0 + (int)rank * TC_BM + rl;
        const int c0 = pairc * TC_BN / splits, c1 = (pairc + 1) * TC_BN / splits;
        const uint32_t lbase = smem_u32(smem) + (uint32_t)rl * 4u;
        uint32_t rb[4];
#pragma unroll
        for (int sp = 0; sp < 4; ++sp) {
            const uint32_t target = (uint32_t)(2 * (sp < splits ? sp : 0)) + rank;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb[sp]) : "r"(lbase), "r"(target));
        }
        for (int col = c0 + par; col < c1; col += 8) {
            float v[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int cc = col + 2 * u;
#pragma unroll
                for (int sp = 0; sp < 4; ++sp) {
                    v[u][sp] = 0.0f;
                    if (sp < splits && cc < c1)
                        asm volatile("ld.shared::cluster.f32 %0, [%1];"
                                     : "=f"(v[u][sp])
                                     : "r"(rb[sp] + (uint32_t)(cc * 128 * 4))
                                     : "memory");
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int cc = col + 2 * u, gc = w.n0 + cc;
                float acc = v[u][0];
#pragma unroll
                for (int sp = 1; sp < 4; ++sp)
                    if (sp < splits) acc += v[u][sp];
                if (cc < c1 && row < M && gc < N) {
                    float *cp = C + (int64_t)row + (int64_t)gc * ldc;
                    *cp = beta == 0.0f ? alpha * acc : fmaf(beta, *cp, alpha * acc);
                }
            }
        }
    }
    if (CSK) cluster_sync();   // no CTA leaves while others read its SMEM
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc_2sm<TC_TMEM_COLS>(tmem_base);
    }
    if (threadIdx.x == 0) EMM_TL(7);
}

template <bool A_MN, bool B_MN>
static cudaError_t launch_tx_t(const TcPlane &pa, const TcPlane &pb, int64_t M, int64_t N, int64_t Kp, float alpha,
                               float beta, float *C, int64_t ldc, unsigned int *ctrl, int splits, float *partial,
                               cudaStream_t s, const PeerOut &peers, void *sk_ws, const float *acc_init,
                               int64_t ld_init) {
    if (acc_init && splits != 1) return cudaErrorInvalidValue;
    if (acc_init) sk_ws = nullptr;   // whole tiles only
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
        const void *fs[5] = {(const void *)tc_xs_kernel<A_MN, B_MN, false, false, false>,
                             (const void *)tc_xs_kernel<A_MN, B_MN, true, false, false>,
                             (const void *)tc_xs_kernel<A_MN, B_MN, false, true, false>,
                             (const void *)tc_xs_kernel<A_MN, B_MN, true, true, false>,
                             (const void *)tc_xs_kernel<A_MN, B_MN, false, false, true>};
        for (int i = 0; i < 5 && attr_err == cudaSuccess; ++i)
            attr_err = cudaFuncSetAttribute(fs[i], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            TX_SMEM_BYTES + ((i & 1) ? TC_CBUF_BYTES : 0));
    });
    if (attr_err != cudaSuccess) return attr_err;
    CUtensorMap ta, tb, tcm;
    if (!tc_make_tmap(&ta, pa, M) || !tc_make_tmap(&tb, pb, N)) return cudaErrorInvalidValue;
    const char *etc = getenv("EMM_TMAC");
    const bool tmac = beta != 0.0f && tma_legal(C, ldc) && !(etc && etc[0] == '0');
    if (tmac) {
        if (!encode_tmap_f32_2d(&tcm, C, M, N, ldc, 128, TC_CB_COLS, CU_TENSOR_MAP_SWIZZLE_NONE))
            return cudaErrorInvalidValue;
    } else {
        tcm = ta;
    }
    const int tiles_m = (int)((M + 2 * TC_BM - 1) / (2 * TC_BM));
    const int tiles_n = (int)((N + TC_BN - 1) / TC_BN);
    const int64_t units = (int64_t)tiles_m * tiles_n * splits;
    if (units > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    const int64_t pairs = tc_num_sms() / 2;
    TcSk sk{0x7fffffff, nullptr, nullptr};
    int dp = 0;
    if (sk_ws && tc_sk_plan(M, N, Kp, splits, 3, &dp)) {
        sk.dp_tiles = dp;
        sk.flags = reinterpret_cast<unsigned int *>(sk_ws);
        sk.slots = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(sk_ws) + TC_SK_FLAG_BYTES);
    }
    const int64_t clusters = sk.slots ? pairs : (units < pairs ? units : pairs);
    const int kc_stages = 256 / TC_BK;
    const char *eearly = getenv("EMM_XS_EARLY");
    const int early = (eearly && eearly[0] == '0') ? 0 : 1;
    cudaEvent_t ev = nullptr;
    prof_begin(s, true, &ev);
    {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)(2 * clusters));
        cfg.blockDim = dim3(TX_THREADS);
        cfg.dynamicSmemBytes = TX_SMEM_BYTES + (tmac ? TC_CBUF_BYTES : 0);
        cfg.stream = s;
        cudaLaunchAttribute at[3];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = 2;
        at[1].val.clusterDim.y = 1;
        at[1].val.clusterDim.z = 1;
        // stream-K owners wait for other CTAs' pieces: co-resident grid only
        at[2].id = cudaLaunchAttributeCooperative;
        at[2].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = sk.slots ? 3 : 2;
        // the wave lockstep only matters for multi-wave problems (ctrl zeroed by the caller)
        unsigned int *wc = units > clusters ? ctrl : nullptr;
        const char *ern = getenv("EMM_XS_RN");
        const bool rn = ern && ern[0] == '1';
        auto kern = tmac ? (rn ? tc_xs_kernel<A_MN, B_MN, true, true, false> : tc_xs_kernel<A_MN, B_MN, true, false, false>)
                         : (rn ? tc_xs_kernel<A_MN, B_MN, false, true, false>
                               : tc_xs_kernel<A_MN, B_MN, false, false, false>);
        auto launch = [&]() {
            return cudaLaunchKernelEx(&cfg, kern, ta, tb, tcm, (int)M, (int)N, (int)Kp, alpha, beta, C, ldc, tiles_m,
                                      tiles_n, 8, kc_stages, wc, splits, splits > 1 ? partial : nullptr, sk, peers,
                                      acc_init, ld_init, early);
        };
        // cluster split-K (sub-wave shapes, S <= 4 splits): one cluster of S
        // pairs per tile, reduced over DSMEM in the same kernel.  Opt-in
        // (EMM_CSK=1): measured slower on B200 (profiles/r02_ab_csk.md) —
        // clusters of 6-8 CTAs do not all fit at once (1024^3: 16 clusters of
        // 8, c3: 24 of 6 ran in two rounds, 27.6 -> 45 us, 44 -> 106 us) and
        // even where they fit (512^3: 4 clusters of 8) 19.4 -> 21.5 us.
        const char *ecs = getenv("EMM_CSK");
        if (splits > 1 && splits <= 4 && !sk.slots && !rn && peers.n == 0 && ecs && ecs[0] == '1') {
            cudaLaunchConfig_t c2 = cfg;
            cudaLaunchAttribute a2[2];
            a2[0] = at[0];
            a2[1] = at[1];
            a2[1].val.clusterDim.x = (unsigned)(2 * splits);
            c2.attrs = a2;
            c2.numAttrs = 2;
            c2.gridDim = dim3((unsigned)(2 * units));
            c2.dynamicSmemBytes = TX_SMEM_BYTES;
            cudaError_t ce = cudaLaunchKernelEx(&c2, tc_xs_kernel<A_MN, B_MN, false, false, true>, ta, tb, tcm, (int)M,
                                                (int)N, (int)Kp, alpha, beta, C, ldc, tiles_m, tiles_n, 8, kc_stages,
                                                (unsigned int *)nullptr, splits, (float *)nullptr, sk, peers,
                                                (const float *)nullptr, (int64_t)0, early);
            if (ce == cudaSuccess) {
                g_launches.fetch_add(1, std::memory_order_relaxed);
                prof_end(s, true, ev);
                return cudaGetLastError();
            }
            cudaGetLastError();   // cluster shape not schedulable: global split-K below
        }
        cudaError_t le = launch();
        if (le != cudaSuccess && sk.slots) {   // cooperative launch refused: data-parallel schedule
            cudaGetLastError();
            sk = TcSk{0x7fffffff, nullptr, nullptr};
            cfg.gridDim = dim3((unsigned)(2 * (units < pairs ? units : pairs)));
            cfg.numAttrs = 2;
            wc = units > pairs ? ctrl : nullptr;
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

cudaError_t launch_tc_xs_sgemm(const TcPlane &a, const TcPlane &b, int64_t M, int64_t N, int64_t K, float alpha,
                               float beta, float *C, int64_t ldc, unsigned int *ctrl, int splits, float *partial,
                               cudaStream_t s, const PeerOut *peers, void *sk_ws, const float *acc_init,
                               int64_t ld_init) {
    if (M > 0x7fffffffLL || N > 0x7fffffffLL || K > 0x7fffffffLL - 32) return cudaErrorInvalidValue;
    if (splits < 1 || (splits > 1 && !partial)) return cudaErrorInvalidValue;
    if (peers && (peers->n < 0 || peers->n > 8 || splits > 1)) return cudaErrorInvalidValue;
    const PeerOut pe = peers ? *peers : PeerOut{};
    const int64_t Kp = tc_kpad(K);
    if (!a.mn && !b.mn) return launch_tx_t<false, false>(a, b, M, N, Kp, alpha, beta, C, ldc, ctrl, splits, partial, s, pe, sk_ws, acc_init, ld_init);
    if (!a.mn && b.mn) return launch_tx_t<false, true>(a, b, M, N, Kp, alpha, beta, C, ldc, ctrl, splits, partial, s, pe, sk_ws, acc_init, ld_init);
    if (a.mn && !b.mn) return launch_tx_t<true, false>(a, b, M, N, Kp, alpha, beta, C, ldc, ctrl, splits, partial, s, pe, sk_ws, acc_init, ld_init);
    return launch_tx_t<true, true>(a, b, M, N, Kp, alpha, beta, C, ldc, ctrl, splits, partial, s, pe, sk_ws, acc_init, ld_init);
}

}  // namespace emm

#ifdef EMM_TIMELINE
// the timeline buffer of this translation unit (KN1X launches)
extern "C" int emm_debug_timeline_xs(unsigned long long *out, int n) {
    const int m = n < 512 * emm::TL_SLOTS ? n : 512 * emm::TL_SLOTS;
    return (int)cudaMemcpyFromSymbol(out, emm::g_emm_timeline, (size_t)m * 8);
}
#endif
