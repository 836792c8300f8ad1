// tc_common.cuh — pieces shared by the two tcgen05 GEMM kernels:
//   * k_tc.cu  tc_sgemm_kernel      operands staged by TMA (planes prepared
//                                   in global memory by the split pass)
//   * k_tcl.cu tc_split_sgemm_kernel operands loaded with LDG by producer
//                                   warps that split them in registers
//                                   (in-kernel 3xTF32 split)
// Both use a CTA pair (cta_group::2) per 256 x 256 output tile, a ring of
// K-stages of four 128 x 32 FP32 operand tiles per CTA (128B-swizzled,
// K-major or MN-major), one elected thread issuing tcgen05.mma into a
// double-buffered TMEM accumulator, and 8 epilogue warps that promote the
// TMEM partials into FP32 registers every 256 of K (R7) and apply
// alpha/beta.
#pragma once
#include <cstdint>

#include "emm_internal.h"
#include "ptx.cuh"

namespace emm {

constexpr int TC_BK = 32;            // K per stage: one 128-byte swizzle row of FP32
constexpr int TC_BM = 128;           // rows of A per CTA (UMMA M = 256 per pair)
constexpr int TC_BN = 256;           // columns of C per pair (UMMA N)
constexpr int TC_TILE_BYTES = 128 * TC_BK * 4;   // one 128 x 32 FP32 operand tile
constexpr int TC_EPI_WARPS = 8;      // 2 per TMEM lane quarter, 128 columns each
constexpr int TC_TMEM_COLS = 512;    // 2 accumulator buffers of 256 columns

// Persistent schedule: cluster `cid` walks work units cid, cid + nclus, ...
// Units are (split, tile), split-major, tiles in grouped raster order along M
// (GPU-L2 analogue of the paper's L2 blocking): one "wave"
// of clusters covers a compact group_m x ~(nclus / group_m) block of tiles.
struct TcSched {
    int tiles_m, tiles_n, group_m, nkb, splits, nkb_s, total_tiles, total_units;
    __device__ __forceinline__ TcSched(int tm, int tn, int gm, int Kp, int sp)
        : tiles_m(tm), tiles_n(tn), group_m(gm), nkb(Kp / TC_BK), splits(sp) {
        nkb_s = (nkb + splits - 1) / splits;
        total_tiles = tiles_m * tiles_n;
        total_units = total_tiles * splits;
    }
    __device__ __forceinline__ void tile_origin(int t, int &m0, int &n0) const {
        const int per_group = group_m * tiles_n;
        const int g = t / per_group;
        const int first_m = g * group_m;
        const int gsize = min(tiles_m - first_m, group_m);
        const int tm = first_m + (t % per_group) % gsize;
        const int tn = (t % per_group) / gsize;
        m0 = tm * (2 * TC_BM);
        n0 = tn * TC_BN;
    }
    // unit u covers K stages [kb0, kb1) of its tile, split index sp
    __device__ __forceinline__ void unit(int u, int &m0, int &n0, int &kb0, int &kb1, int &sp) const {
        sp = u / total_tiles;
        tile_origin(u - sp * total_tiles, m0, n0);
        kb0 = sp * nkb_s;
        kb1 = min(nkb, kb0 + nkb_s);
    }
};

// ===== MMA issuer: one thread of the leader CTA drives the pair =====
// Stage s holds [A plane0 | A plane1 | B plane0 | B plane1] (PLANES == 2) or
// [A | B] (PLANES == 1).  TERMS: 3 = 3xTF32 (small*big + big*small +
// big*big), 2 = TF32+BF16 (bf16 cross pair as one K16 MMA + big*big), 1.
template <int TERMS, bool A_MN, bool B_MN, bool A1_MN, bool B1_MN, int PLANES, int STAGES, int STAGE_BYTES>
__device__ __forceinline__ void tc_mma_loop(const TcSched &S, int cid, int nclus, uint8_t *smem, uint64_t *full,
                                            uint64_t *empty, uint64_t *acc_full, uint64_t *acc_empty,
                                            uint32_t tmem_base, int kc_stages) {
    using namespace ptx;
    constexpr uint32_t idesc = idesc_tf32_major<2 * TC_BM, TC_BN, A_MN, B_MN>();
    // K8 step k of a plane: K-major advances 32 B inside the swizzle row,
    // MN-major advances 8 K-rows = 1024 B
    auto dsc = [](uint32_t addr, bool mn, int k) -> uint64_t {
        return mn ? desc_mnmajor_sw128_32b(addr + (uint32_t)(k * 1024)) : desc_kmajor_sw128(addr + (uint32_t)(k * 32));
    };
    int it = 0, ch = 0;   // global stage / chunk counters (continue across tiles)
    for (int t = cid; t < S.total_units; t += nclus) {
        int m0, n0, kb0, kb1, sp;
        S.unit(t, m0, n0, kb0, kb1, sp);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
            const bool first = ((kb - kb0) % kc_stages) == 0;
            const bool last = ((kb - kb0) % kc_stages) == kc_stages - 1 || kb == kb1 - 1;
            const int b = ch & 1;
            const uint32_t dt = tmem_base + (uint32_t)(b * TC_BN);
            if (first) {   // the epilogue has drained this buffer (both CTAs)
                mbar_wait(&acc_empty[b], (((uint32_t)ch >> 1) & 1u) ^ 1u);
                tc_fence_after();
            }
            const int s = it % STAGES;
            const uint32_t ph = (uint32_t)(it / STAGES) & 1u;
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint32_t st = smem_u32(smem + s * STAGE_BYTES);
            const uint32_t a0 = st, a1 = st + TC_TILE_BYTES;
            const uint32_t b0 = st + PLANES * TC_TILE_BYTES, b1 = b0 + TC_TILE_BYTES;
#pragma unroll
            for (int k = 0; k < TC_BK / 8; ++k) {
                const uint32_t acc0 = (first && k == 0) ? 0u : 1u;
                if (TERMS == 3) {
                    // small terms first (they are the smaller magnitudes)
                    mma_tf32_2sm(dt, dsc(a1, A1_MN, k), dsc(b0, B_MN, k), idesc, acc0);
                    mma_tf32_2sm(dt, dsc(a0, A_MN, k), dsc(b1, B1_MN, k), idesc, 1u);
                    mma_tf32_2sm(dt, dsc(a0, A_MN, k), dsc(b0, B_MN, k), idesc, 1u);
                } else if (TERMS == 2) {
                    // cross terms: K=16 bf16 = the same 32 bytes of a K-major row
                    constexpr uint32_t idesc_x = idesc_bf16<2 * TC_BM, TC_BN>();
                    mma_f16_2sm(dt, dsc(a1, false, k), dsc(b1, false, k), idesc_x, acc0);
                    mma_tf32_2sm(dt, dsc(a0, A_MN, k), dsc(b0, B_MN, k), idesc, 1u);
                } else {
                    mma_tf32_2sm(dt, dsc(a0, A_MN, k), dsc(b0, B_MN, k), idesc, acc0);
                }
            }
            mma_commit_2sm_mc(&empty[s], (uint16_t)0x3);
            if (last) {
                mma_commit_2sm_mc(&acc_full[b], (uint16_t)0x3);
                ++ch;
            }
        }
    }
}

// ===== epilogue: TMEM -> FP32 registers (promotion) -> alpha/beta -> C =====
// Warp with TMEM lane quarter q (= warp % 4) and column half h.
__device__ __forceinline__ void tc_epilogue_loop(const TcSched &S, int cid, int nclus, uint32_t rank, int q, int h,
                                                 int lane, uint32_t tmem_base, uint64_t *acc_full,
                                                 uint64_t *acc_empty, int kc_stages, int M, int N, float alpha,
                                                 float beta, float *__restrict__ C, int64_t ldc,
                                                 float *__restrict__ partial, const PeerOut &peers) {
    using namespace ptx;
    uint32_t leader_empty0;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(leader_empty0) : "r"(smem_u32(&acc_empty[0])));
    int ch = 0;
    for (int t = cid; t < S.total_units; t += nclus) {
        int m0, n0, kb0, kb1, sp;
        S.unit(t, m0, n0, kb0, kb1, sp);
        const int nchunks = (kb1 - kb0 + kc_stages - 1) / kc_stages;
        const int row = m0 + (int)rank * TC_BM + 32 * q + lane;
        float acc[128];
#pragma unroll
        for (int j = 0; j < 128; ++j) acc[j] = 0.0f;
        for (int c2 = 0; c2 < nchunks; ++c2, ++ch) {
            const int b = ch & 1;
            mbar_wait(&acc_full[b], ((uint32_t)ch >> 1) & 1u);
            tc_fence_after();
            const uint32_t tb = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(b * TC_BN + h * 128);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                uint32_t v[16];
                tmem_ld_32x32b_x16(tb + (uint32_t)(16 * c), v);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 16; ++j) acc[16 * c + j] += __uint_as_float(v[j]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                const uint32_t eb = leader_empty0 + (uint32_t)(b * sizeof(uint64_t));
                asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(eb) : "memory");
            }
        }
        if (partial) {
            // split-K: publish the raw FP32 partial of split sp; the reduce
            // launch (KN8) sums the S partials in fixed order.
            if (row < M) {
                const int col0 = n0 + h * 128;
                float *pp = partial + (int64_t)sp * M * N + (int64_t)row + (int64_t)col0 * M;
                const int jmax = min(128, N - col0);
#pragma unroll
                for (int j = 0; j < 128; ++j, pp += M)
                    if (j < jmax) *pp = acc[j];
            }
            continue;
        }
        if (row < M) {
            const int col0 = n0 + h * 128;
            float *cp = C + (int64_t)row + (int64_t)col0 * ldc;
            const int jmax = min(128, N - col0);
            if (beta == 0.0f) {
                float *sp2 = cp;
#pragma unroll
                for (int j = 0; j < 128; ++j, sp2 += ldc) {
                    acc[j] *= alpha;
                    if (j < jmax) *sp2 = acc[j];
                }
            } else {
                // beta != 0: issue 16 independent C loads before the 16
                // stores (a store could alias a later load through ldc, so
                // the compiler would otherwise serialise them).
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    float cin[16];
                    const float *lp = cp + (int64_t)(16 * g) * ldc;
#pragma unroll
                    for (int j = 0; j < 16; ++j, lp += ldc) cin[j] = (16 * g + j < jmax) ? __ldcs(lp) : 0.0f;
                    float *sp2 = cp + (int64_t)(16 * g) * ldc;
#pragma unroll
                    for (int j = 0; j < 16; ++j, sp2 += ldc) {
                        acc[16 * g + j] = fmaf(beta, cin[j], alpha * acc[16 * g + j]);
                        if (16 * g + j < jmax) __stcs(sp2, acc[16 * g + j]);
                    }
                }
            }
            // fused all-gather: the same values into every rank's full C
            // (peer memory over NVLink)
            for (int p = 0; p < peers.n; ++p) {
                float *pp = peers.base[p] + (peers.row_off + row) + (peers.col_off + col0) * peers.ld;
#pragma unroll
                for (int j = 0; j < 128; ++j, pp += peers.ld)
                    if (j < jmax) *pp = acc[j];
            }
            if (peers.n) __threadfence_system();
        }
    }
}

}  // namespace emm
