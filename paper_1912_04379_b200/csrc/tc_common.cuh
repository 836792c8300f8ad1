// tc_common.cuh — pieces shared by the two tcgen05 GEMM kernels:
//   * tc_kernel.cuh (k_tc_t{1,2,3}.cu) tc_sgemm_kernel   operands staged by
//                                   TMA (user arrays in place, or planes
//                                   prepared by the split pass in k_tc.cu)
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

// Debug timeline (build with EMM_TIMELINE=1 -> libemm_tl.so; never in the
// product library): %globaltimer stamps per CTA at fixed points of the
// kernel, read back with emm_debug_timeline().
#ifdef EMM_TIMELINE
constexpr int TL_SLOTS = 12;
static __device__ unsigned long long g_emm_timeline[512][TL_SLOTS];
__device__ __forceinline__ void emm_tl_mark(int slot) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x < 512) g_emm_timeline[blockIdx.x][slot] = t;
}
#define EMM_TL(slot) emm_tl_mark(slot)
#else
#define EMM_TL(slot) ((void)0)
#endif

constexpr int TC_BK = 32;            // K per stage: one 128-byte swizzle row of FP32
constexpr int TC_BM = 128;           // rows of A per CTA (UMMA M = 256 per pair)
constexpr int TC_BN = 256;           // columns of C per pair (UMMA N)
constexpr int TC_TILE_BYTES = 128 * TC_BK * 4;   // one 128 x 32 FP32 operand tile
constexpr int TC_EPI_WARPS = 8;      // 2 per TMEM lane quarter, 128 columns each
constexpr int TC_TMEM_COLS = 512;    // 2 accumulator buffers of 256 columns

// warp 0 = TMA producer, warp 1 = MMA issuer + TMEM owner, warps 2-9 = 8
// promotion/epilogue warps (2 per TMEM lane quarter).
constexpr int TC_EPI_WARP0 = 2;
constexpr int TC_THREADS_P = 32 * (TC_EPI_WARP0 + TC_EPI_WARPS);   // 320

// TERMS: 3 = 3xTF32 (small*big + big*small + big*big, three kind::tf32 MMAs
// per K8), 2 = TF32+BF16 (big*big kind::tf32 + both cross terms in one K16
// kind::f16 BF16 MMA), 1 = 1xTF32.
template <int TERMS>
struct TcCfg {
    static constexpr int PLANES = TERMS >= 2 ? 2 : 1;
    static constexpr int TILES_PER_STAGE = 2 * PLANES;              // A planes + B planes
    static constexpr int STAGE_BYTES = TILES_PER_STAGE * TC_TILE_BYTES;
    static constexpr int STAGES = TERMS >= 2 ? 3 : 6;
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

// Per-call control block (zeroed by the pack launch, TC_CTRL_BYTES): word 0 =
// wave-lockstep counter.  A lockstep wait longer than this many SM cycles
// (~1 ms) means the grid is not fully resident: the CTA stops waiting.
constexpr long long TC_LOCKSTEP_TIMEOUT = 2000000LL;
constexpr int TC_SK_CHUNK = 256 / TC_BK;   // stream-K granularity: 8 stages = one promotion chunk

// Work item kinds.
enum { TW_FULL = 0,     // whole tile -> C (alpha/beta epilogue)
       TW_SPLITK = 1,   // split-K unit -> raw partial in slot (sp, tile) (fixed-order reduce launch, KN8)
       TW_PUB = 2,      // stream-K piece not starting at k = 0 -> raw partial in slot `cid`
       TW_OWN = 3 };    // stream-K piece starting at k = 0 -> C, after adding the partials
                        // of the same tile published by clusters cid+1 .. last (ascending k)
struct TcWork {
    int m0, n0, kb0, kb1, kind, sp, last, tile;
};

// Stream-K scratch: one partial slot per cluster (a
// cluster publishes at most one piece: the first of its range) + one flag
// per (slot, CTA, epilogue warp).  Slot layout [rank][warp][32 float4 groups][lane].
constexpr int TC_SK_SLOT_FLOATS = 2 * TC_EPI_WARPS * 32 * 32 * 4;   // 256 x 256 floats
constexpr int TC_SK_FLAGS_PER_SLOT = 2 * TC_EPI_WARPS;
struct TcSk {
    int dp_tiles;            // tiles of the data-parallel phase; >= tiles: stream-K off
    float *slots;            // [nclus][TC_SK_SLOT_FLOATS]
    unsigned int *flags;     // [nclus][TC_SK_FLAGS_PER_SLOT], zero at launch
};

// Persistent schedule.  Tiles are numbered in grouped raster order along M
// (GPU-L2 analogue of the paper's L2 blocking): one "wave"
// of clusters covers a compact group_m x ~(nclus / group_m) block of tiles.
//  * split-K (splits > 1, sub-wave problems): units (split, tile), split-
//    major; cluster cid takes units cid, cid + nclus, ...
//  * data-parallel + stream-K: the first dp_tiles tiles (whole waves) go
//    round-robin; the remaining tiles' K-chunks (kc stages each) are cut
//    into nclus equal contiguous ranges, one per cluster, so the last
//    (partial) wave keeps every SM busy.  A cluster's range is walked in
//    ascending order: its first piece may be the tail of a tile (TW_PUB, its
//    partial is published early), its last piece the head of another tile
//    (TW_OWN, finished last, when the tail pieces are already published).
//    The tile's sum is own + P(cid+1) + ... in ascending k: deterministic.
__host__ __device__ __forceinline__ int tc_imin(int a, int b) { return a < b ? a : b; }

struct TcSched {
    int tiles_m, tiles_n, group_m, nkb, splits, nkb_s, total_tiles, total_units;
    int nclus, cid;
    bool sk;
    int dp_tiles, kc, nch, Wsk, a, b, n_dp, n_items, dp_waves;
    __host__ __device__ __forceinline__ TcSched(int tm, int tn, int gm, int Kp, int sp, int dp, int kc_, int nclus_, int cid_)
        : tiles_m(tm), tiles_n(tn), group_m(gm), nkb(Kp / TC_BK), splits(sp), nclus(nclus_), cid(cid_) {
        nkb_s = (nkb + splits - 1) / splits;
        total_tiles = tiles_m * tiles_n;
        total_units = total_tiles * splits;
        sk = splits == 1 && dp < total_tiles;
        dp_tiles = sk ? dp : total_tiles;
        kc = kc_;
        nch = (nkb + kc - 1) / kc;
        Wsk = sk ? (total_tiles - dp_tiles) * nch : 0;
        a = (int)((long long)cid * Wsk / nclus);
        b = (int)((long long)(cid + 1) * Wsk / nclus);
        const int dpu = sk ? dp_tiles : total_units;
        n_dp = cid < dpu ? (dpu - cid + nclus - 1) / nclus : 0;
        n_items = n_dp + ((sk && a < b) ? (b - 1) / nch - a / nch + 1 : 0);
        dp_waves = dp_tiles / nclus;
    }
    __host__ __device__ __forceinline__ void tile_origin(int t, int &m0, int &n0) const {
        const int per_group = group_m * tiles_n;
        const int g = t / per_group;
        const int first_m = g * group_m;
        const int gsize = tc_imin(tiles_m - first_m, group_m);
        const int tm = first_m + (t % per_group) % gsize;
        const int tn = (t % per_group) / gsize;
        m0 = tm * (2 * TC_BM);
        n0 = tn * TC_BN;
    }
    __host__ __device__ __forceinline__ void item(int i, TcWork &w) const {
        w.sp = 0;
        w.last = 0;
        if (i < n_dp) {
            const int u = cid + i * nclus;
            w.sp = u / total_tiles;
            w.tile = u - w.sp * total_tiles;
            tile_origin(w.tile, w.m0, w.n0);
            w.kb0 = w.sp * nkb_s;
            w.kb1 = tc_imin(nkb, w.kb0 + nkb_s);
            w.kind = splits > 1 ? TW_SPLITK : TW_FULL;
            return;
        }
        const int j = i - n_dp;
        const int s0 = j == 0 ? a : (a / nch + j) * nch;   // later pieces start at tile boundaries
        const int tl = s0 / nch;
        const int e0 = tc_imin(b, (tl + 1) * nch);
        const int srel = s0 - tl * nch, erel = e0 - tl * nch;
        w.tile = dp_tiles + tl;
        tile_origin(w.tile, w.m0, w.n0);
        w.kb0 = srel * kc;
        w.kb1 = tc_imin(nkb, erel * kc);
        if (srel == 0 && erel == nch) {
            w.kind = TW_FULL;
        } else if (srel == 0) {
            w.kind = TW_OWN;
            const long long x = (long long)(tl + 1) * nch - 1;          // the tile's last chunk
            w.last = (int)(((x + 1) * nclus - 1) / Wsk);                 // the cluster holding it
        } else {
            w.kind = TW_PUB;
        }
    }
    // data-parallel schedule (no stream-K) of another pair `c` (the partner
    // pair of a 4-cluster): its item count and its item i
    __host__ __device__ __forceinline__ int n_items_of(int c) const {
        return c < total_units ? (total_units - c + nclus - 1) / nclus : 0;
    }
    __host__ __device__ __forceinline__ void item_of(int c, int i, TcWork &w) const {
        const int u = c + i * nclus;
        w.sp = u / total_tiles;
        w.tile = u - w.sp * total_tiles;
        tile_origin(w.tile, w.m0, w.n0);
        w.kb0 = w.sp * nkb_s;
        w.kb1 = tc_imin(nkb, w.kb0 + nkb_s);
        w.kind = splits > 1 ? TW_SPLITK : TW_FULL;
        w.last = 0;
    }
    // wave-lockstep bookkeeping (producers): wave of item i, CTA pairs in a wave
    __host__ __device__ __forceinline__ int wave_of(int i) const { return i < n_dp ? i : dp_waves; }
    __host__ __device__ __forceinline__ int pairs_in_wave(int w) const {
        return sk ? nclus : tc_imin(nclus, total_units - w * nclus);
    }
};

// Clusters of two CTA pairs (launched with a PREFERRED cluster size of 4,
// DESIGN.md §3): pair cid and its partner cid ^ 1 walk the same schedule
// positions, and with the grouped raster their data-parallel tiles at the
// same position are vertically adjacent (same B tile), so B is multicast.
// When the partner has fewer items (last, partial wave) this pair mirrors
// the partner's item as a dummy (computed, never stored) so both pairs run
// the same stage sequence — each stage slot is released by both pairs'
// MMAs.  A cluster of 2 (cl == 2) is the plain schedule.
struct TcItem {
    TcWork w;
    bool dummy;   // mirror of the partner's item: no epilogue stores
    bool mc;      // B shared with the partner pair (multicast loads)
};
// cl == 4 only for data-parallel launches (no stream-K, no split-K)
__host__ __device__ __forceinline__ int tc_n_items(const TcSched &S, int cl) {
    if (cl != 4) return S.n_items;
    const int pn = S.n_items_of(S.cid ^ 1);
    return pn > S.n_items ? pn : S.n_items;
}
// MMA issuer / epilogue: the item only (its own, or the partner's mirrored)
__host__ __device__ __forceinline__ void tc_get_work(const TcSched &S, int cl, int i, TcWork &w, bool &dummy) {
    dummy = cl == 4 && i >= S.n_items;
    if (dummy) S.item_of(S.cid ^ 1, i, w);
    else S.item(i, w);
}
// producer: also whether B is shared with the partner pair (multicast)
__host__ __device__ __forceinline__ void tc_get_item(const TcSched &S, int cl, int i, TcItem &it) {
    const bool have = i < S.n_items, phave = cl == 4 && i < S.n_items_of(S.cid ^ 1);
    TcWork pw;
    if (have) S.item(i, it.w);
    if (phave) S.item_of(S.cid ^ 1, i, pw);
    it.dummy = !have;
    if (!have) it.w = pw;
    if (!phave) pw = it.w;
    it.mc = cl == 4 && it.w.kind == TW_FULL && pw.kind == TW_FULL && pw.n0 == it.w.n0 && pw.kb0 == it.w.kb0 &&
            pw.kb1 == it.w.kb1;
}

// ===== MMA issuer: one thread of the leader CTA drives the pair =====
// Stage s holds [A plane0 | A plane1 | B plane0 | B plane1] (PLANES == 2) or
// [A | B] (PLANES == 1).  TERMS: 3 = 3xTF32 (small*big + big*small +
// big*big), 2 = TF32+BF16 (bf16 cross pair as one K16 MMA + big*big), 1.
template <int TERMS, bool A_MN, bool B_MN, bool A1_MN, bool B1_MN, int PLANES, int STAGES, int STAGE_BYTES,
          bool MC = false>
__device__ __forceinline__ void tc_mma_loop(const TcSched &S, uint8_t *smem, uint64_t *full,
                                            uint64_t *empty, uint64_t *acc_full, uint64_t *acc_empty,
                                            uint32_t tmem_base, int kc_stages, int cl = 2, int pair = 0) {
    using namespace ptx;
    constexpr uint32_t idesc = idesc_tf32_major<2 * TC_BM, TC_BN, A_MN, B_MN>();
    // K8 step k of a plane: K-major advances 32 B inside the swizzle row,
    // MN-major advances 8 K-rows = 1024 B
    auto dsc = [](uint32_t addr, bool mn, int k) -> uint64_t {
        return mn ? desc_mnmajor_sw128_32b(addr + (uint32_t)(k * 1024)) : desc_kmajor_sw128(addr + (uint32_t)(k * 32));
    };
    int it = 0, ch = 0;   // global stage / chunk counters (continue across tiles)
    // stage slots are released to both pairs of a 4-cluster (each slot
    // receives the partner's multicast B); the accumulator only to this pair
    if (!MC) cl = 2, pair = 0;   // compile-time plain schedule
    // (cluster split-K, KN1X: clusters of S pairs with cl == 2 — this pair only)
    const uint16_t rel_mask = (uint16_t)(cl == 4 ? 0xF : (0x3u << (2 * pair)));
    const uint16_t acc_mask = (uint16_t)(0x3u << (2 * pair));
    const int n_it = tc_n_items(S, cl);
    for (int i = 0; i < n_it; ++i) {
        TcWork w;
        bool dummy;
        tc_get_work(S, cl, i, w, dummy);
        const int kb0 = w.kb0, kb1 = w.kb1;
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
            if (it == 0) EMM_TL(3);
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
            mma_commit_2sm_mc(&empty[s], rel_mask);
            if (last) {
                mma_commit_2sm_mc(&acc_full[b], acc_mask);
                ++ch;
            }
        }
    }
    EMM_TL(4);
}

// ===== epilogue: TMEM -> FP32 registers (promotion) -> alpha/beta -> C =====
// Warp with TMEM lane quarter q (= warp % 4) and column half h.
// beta != 0 with a TMA-legal C (TMAC): C_in comes through TMA in chunks of
// 128 rows x 16 columns into a 2-deep ring per column half (group of 4
// warps); the first two chunks of a tile are requested while its last K
// chunk is still in the tensor pipe.
constexpr int TC_CB_COLS = 16, TC_CB_N = 2;
constexpr int TC_CB_BYTES = 128 * TC_CB_COLS * 4;          // 8 KB
constexpr int TC_CBUF_BYTES = 2 * TC_CB_N * TC_CB_BYTES;    // both halves: 32 KB
struct TcCin {
    const CUtensorMap *tm = nullptr;   // C as a 2-D tensor map, box {128 rows, 16 cols}
    float *buf = nullptr;              // [2 halves][TC_CB_N][16][128]
    uint64_t *full = nullptr;          // [2 halves][TC_CB_N]
};
template <bool MC = false, bool TMAC = false>
__device__ __forceinline__ void tc_epilogue_loop(const TcSched &S, uint32_t rank, int q, int h, int lane,
                                                 uint32_t tmem_base, uint64_t *acc_full, uint64_t *acc_empty,
                                                 int kc_stages, int M, int N, float alpha, float beta,
                                                 float *C, int64_t ldc, float *__restrict__ partial,
                                                 const TcSk &sk, const PeerOut &peers, int cl = 2,
                                                 uint32_t leader = 0, const float *acc_init = nullptr,
                                                 int64_t ld_init = 0, const TcCin cin_tma = TcCin{},
                                                 float *csk_part = nullptr) {
    using namespace ptx;
    if (!MC) cl = 2, leader = 0;   // compile-time plain schedule
    uint32_t leader_empty0;   // the pair leader's acc_empty[0]
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                 : "=r"(leader_empty0)
                 : "r"(smem_u32(&acc_empty[0])), "r"(leader));
    // this warp's stream-K slot part / flag index (warp id within the CTA's 8)
    const int wslot = (int)rank * TC_EPI_WARPS + h * 4 + q;
    int ch = 0, cph = 0;   // TMEM chunk counter, C_in chunk counter (TMAC ring phases)
    const bool tmac = TMAC && beta != 0.0f;
    const bool cleader = q == (TC_EPI_WARP0 & 3) && lane == 0;   // first warp of this column half
    float *gbuf = TMAC ? cin_tma.buf + h * (TC_CB_N * TC_CB_BYTES / 4) : nullptr;
    uint64_t *gfull = TMAC ? cin_tma.full + h * TC_CB_N : nullptr;
    const int n_it = tc_n_items(S, cl);
    for (int i = 0; i < n_it; ++i) {
        TcWork w;
        bool dummy;
        tc_get_work(S, cl, i, w, dummy);
        const int m0 = w.m0, n0 = w.n0, kb0 = w.kb0, kb1 = w.kb1, sp = w.sp;
        const int nchunks = (kb1 - kb0 + kc_stages - 1) / kc_stages;
        const int row = m0 + (int)rank * TC_BM + 32 * q + lane;
        float acc[128];
        if (acc_init && row < M) {
            // K-phased call (host pipeline): continue the FP32 promotion chain
            // from the raw partial of the earlier K range (same additions in
            // the same order as one call over all of K)
            const int col0 = n0 + h * 128;
            const float *ip = acc_init + (int64_t)row + (int64_t)col0 * ld_init;
            const int jmax = min(128, N - col0);
#pragma unroll
            for (int j = 0; j < 128; ++j) acc[j] = j < jmax ? __ldcs(ip + (int64_t)j * ld_init) : 0.0f;
        } else {
#pragma unroll
            for (int j = 0; j < 128; ++j) acc[j] = 0.0f;
        }
        const bool stores = !dummy && (w.kind == TW_FULL || w.kind == TW_OWN);
        const int crow = m0 + (int)rank * TC_BM, ccol0 = n0 + h * 128;
        auto cissue = [&](int c) {   // C_in chunk c of this item into ring slot c % TC_CB_N
            const int bb = c % TC_CB_N;
            mbar_arrive_expect_tx(&gfull[bb], TC_CB_BYTES);
            tma_load_2d(smem_u32(gbuf + bb * (TC_CB_BYTES / 4)), cin_tma.tm, &gfull[bb], crow,
                        ccol0 + TC_CB_COLS * c, policy_evict_first());
        };
        for (int c2 = 0; c2 < nchunks; ++c2, ++ch) {
            const int b = ch & 1;
            if (TMAC && tmac && stores && cleader && c2 == nchunks - 1)
                for (int c = 0; c < TC_CB_N; ++c) cissue(c);
            mbar_wait(&acc_full[b], ((uint32_t)ch >> 1) & 1u);
            tc_fence_after();
            if (ch == 0 && q == 0 && h == 0 && lane == 0) EMM_TL(5);
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
                mbar_arrive_remote(eb);
            }
        }
        if (dummy) continue;   // mirrored partner item: drained, never stored
        if (w.kind == TW_PUB) {
            // stream-K tail piece: raw partial -> slot cid (coalesced float4
            // layout, all 256 x 256 entries), then this warp's flag (release)
            float4 *slot = reinterpret_cast<float4 *>(sk.slots + (size_t)S.cid * TC_SK_SLOT_FLOATS) +
                           (size_t)wslot * 32 * 32 + lane;
#pragma unroll
            for (int g = 0; g < 32; ++g)
                __stcg(slot + g * 32, make_float4(acc[4 * g], acc[4 * g + 1], acc[4 * g + 2], acc[4 * g + 3]));
            __threadfence();
            __syncwarp();
            if (lane == 0) {
                unsigned int *f = sk.flags + (size_t)S.cid * TC_SK_FLAGS_PER_SLOT + wslot;
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(1u) : "memory");
            }
            continue;
        }
        if (w.kind == TW_OWN) {
            // stream-K head piece: add the tile's other pieces in ascending k
            for (int c = S.cid + 1; c <= w.last; ++c) {
                const unsigned int *f = sk.flags + (size_t)c * TC_SK_FLAGS_PER_SLOT + wslot;
                const long long t0 = clock64();
                while (true) {
                    unsigned int v;
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                    if (v) break;
                    __nanosleep(64);
                    if (clock64() - t0 > 40000000000LL) __trap();
                }
                const float4 *slot = reinterpret_cast<const float4 *>(sk.slots + (size_t)c * TC_SK_SLOT_FLOATS) +
                                     (size_t)wslot * 32 * 32 + lane;
#pragma unroll
                for (int g0 = 0; g0 < 32; g0 += 8) {
                    float4 v[8];
#pragma unroll
                    for (int g = 0; g < 8; ++g) v[g] = __ldcg(slot + (g0 + g) * 32);
#pragma unroll
                    for (int g = 0; g < 8; ++g) {
                        acc[4 * (g0 + g)] += v[g].x;
                        acc[4 * (g0 + g) + 1] += v[g].y;
                        acc[4 * (g0 + g) + 2] += v[g].z;
                        acc[4 * (g0 + g) + 3] += v[g].w;
                    }
                }
            }
        }
        if (w.kind == TW_SPLITK && csk_part) {
            // cluster split-K (KN1X): the raw partial stays in this CTA's SMEM
            // ([256 columns][128 rows]); the cluster reduces it over DSMEM
            float *pp = csk_part + h * 128 * 128 + 32 * q + lane;
#pragma unroll
            for (int j = 0; j < 128; ++j) pp[j * 128] = acc[j];
            continue;
        }
        if (w.kind == TW_SPLITK) {
            // split-K: publish the raw FP32 partial of split sp into its slot
            // (coalesced float4 layout, all 256 x 256 entries); the reduce
            // launch (KN8) sums the S slots of a tile in fixed order.
            float4 *slot = reinterpret_cast<float4 *>(partial + ((size_t)sp * S.total_tiles + w.tile) *
                                                                   TC_SK_SLOT_FLOATS) +
                           (size_t)wslot * 32 * 32 + lane;
#pragma unroll
            for (int g = 0; g < 32; ++g)
                __stcg(slot + g * 32, make_float4(acc[4 * g], acc[4 * g + 1], acc[4 * g + 2], acc[4 * g + 3]));
            continue;
        }
        if (TMAC && tmac) {
            // the 4 warps of this column half walk the 8 C_in chunks together
            const int col0 = n0 + h * 128;
            float *cp = C + (int64_t)row + (int64_t)col0 * ldc;
            const int jmax = min(128, N - col0);
            const int rl = 32 * q + lane;
#pragma unroll
            for (int c = 0; c < 128 / TC_CB_COLS; ++c, ++cph) {
                const int bb = c % TC_CB_N;
                mbar_wait(&gfull[bb], (uint32_t)((cph / TC_CB_N) & 1));
                const float *bp = gbuf + bb * (TC_CB_BYTES / 4) + rl;
                float *sp2 = cp + (int64_t)(TC_CB_COLS * c) * ldc;
#pragma unroll
                for (int j = 0; j < TC_CB_COLS; ++j, sp2 += ldc) {
                    const int jj = TC_CB_COLS * c + j;
                    acc[jj] = fmaf(beta, bp[j * 128], alpha * acc[jj]);
                    if (row < M && jj < jmax) __stcs(sp2, acc[jj]);
                }
                if (h == 0)
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                else
                    asm volatile("bar.sync 2, 128;" ::: "memory");
                if (cleader && c + TC_CB_N < 128 / TC_CB_COLS) cissue(c + TC_CB_N);
            }
        }
        if (row < M) {
            const int col0 = n0 + h * 128;
            float *cp = C + (int64_t)row + (int64_t)col0 * ldc;
            const int jmax = min(128, N - col0);
            if (TMAC && tmac) {
                // stored above
            } else if (beta == 0.0f) {
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
    if (q == 0 && h == 0 && lane == 0) EMM_TL(6);
}

}  // namespace emm
