// k_tc.cu — the tensor-core SGEMM path for sm_100a (KN1 3xTF32, KN2 1xTF32,
// TF32+BF16) and its operand split pass (KN4).
//
// Paper → B200 mapping:
//  * The operands are read IN PLACE by TMA whenever their leading dimension
//    is TMA-legal (16-byte strides, 16-byte aligned base): op(A) / op(B) are
//    K-major or MN-major tiles depending on transA / transB, and the
//    transpose lives in the TMA box + the UMMA descriptor's major mode, not
//    in a copy.  The tensor core truncates FP32 inputs to TF32 (measured,
//    DESIGN.md R7b), so the raw operand IS the "big" part; KN4 only writes
//    the second plane (3xTF32: small = rn_tf32(x - trunc(x)) in the
//    operand's own layout; TF32+BF16: the bf16 cross plane).
//  * "Re-buffering ... re-ordering B" and "padding with
//    zeros" for K survive as the FALLBACK for TMA-illegal
//    leading dimensions (e.g. N = 333): KN4 re-orders both planes into
//    K-major, 32-padded buffers.
//  * L1 blocking + A' prefetch → TMA loads of
//    128x32 K-major tiles into a multi-stage 128B-swizzled SMEM ring
//    (mbarrier full/empty pairs), a producer warp running ahead.
//  * L0 register blocking, 5 dot products accumulated in registers for the
//    whole dot product → tcgen05.mma accumulating
//    a 256x256 FP32 tile of a CTA pair in TMEM for the whole K loop; one
//    elected thread issues.  "shuffling and write back" deferred to the end
//    of the dot product → one epilogue per tile.
//  * N-edge special cases → predicated epilogue stores.
//  * B200-specific: persistent CTA pairs with a wave lockstep (L2 reuse of
//    the wave's panels), split-K / hybrid stream-K for partial waves, and for
//    data-parallel launches at K >= 4096 a PREFERRED cluster size of 4 (two
//    pairs on vertically adjacent tiles share B by TMA multicast; MC
//    template); `acc_init` lets a later call over the rest of K continue the
//    FP32 promotion chains of an earlier one (K-phased host pipeline).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "emm_internal.h"
#include "ptx.cuh"
#include "tc_common.cuh"

namespace emm {

using namespace ptx;

int64_t tc_kpad(int64_t K) { return (K + TC_BK - 1) / TC_BK * TC_BK; }

// Per-call control block (zeroed by the pack launch, TC_CTRL_BYTES): word 0 =
// wave-lockstep counter.  A lockstep wait longer than this many SM cycles
// (~1 ms) means the grid is not fully resident: the CTA stops waiting.
constexpr long long TC_LOCKSTEP_TIMEOUT = 2000000LL;
constexpr int TC_SK_CHUNK = 256 / TC_BK;   // stream-K granularity: 8 stages = one promotion chunk

// =====================================================================
// KN4: operand split pass, both operands in ONE launch (a flat grid: A's
// blocks, then B's).  Block 0 also zeroes the GEMM's per-call control block
// (stream-ordered before the GEMM).  HBM-bound: 16-byte vector loads and
// stores wherever the layout allows.
//
//   PK_FULL1  plane 0 = rn_tf32(x), K-major                (fallback 1xTF32)
//   PK_FULL3  + plane 1 = rn_tf32(x - big), K-major       (fallback 3xTF32)
//   PK_FULLX  + plane 1 = BF16 cross operand, K-major     (fallback TF32+BF16)
//   PK_DSMALL plane 1 only = rn_tf32(x - trunc(x)) in the SOURCE layout
//             (direct 3xTF32: the tensor core reads trunc(x) from the user array)
//   PK_DCROSS plane 1 only = BF16 cross operand with big = trunc(x), K-major
//             (direct TF32+BF16)
// BF16 cross operand: for every group of 8 along K, 16 bf16 = [bf16(big) x8 |
// bf16(x - big) x8] (A side) or the halves swapped (B side), so that ONE K16
// BF16 MMA computes a_big*b_small + a_small*b_big.
// Non-finite x: the second part is 0 (inf/NaN propagate through big*big).
//
// Two block kinds:
//  * element-wise ("lines"): the output keeps the source orientation —
//    K-contiguous sources (every mode) and PK_DSMALL of MN-contiguous
//    sources.  A line is one stored column (contiguous run) of the source;
//    a thread handles groups of 8 consecutive elements (two 16-B vectors).
//  * transpose: MN-contiguous source -> K-major planes (the re-buffered
//    FULL modes and PK_DCROSS): 64 (r) x 32 (p) tiles through shared memory.
// =====================================================================
enum { PK_FULL1 = PK_FULL1_, PK_FULL3 = PK_FULL3_, PK_FULLX = PK_FULLX_, PK_DSMALL = PK_DSMALL_, PK_DCROSS = PK_DCROSS_ };

constexpr int PK_THREADS = 256;
constexpr int PK_GROUPS = 2;                                   // 8-element groups per thread (element-wise)
constexpr int PK_CHUNK = PK_THREADS * PK_GROUPS * 8;           // elements of a line per block
constexpr int PK_TR = 64, PK_TP = 32;                          // transpose tile (r x p)

struct PackOperand {
    const float *X;
    int64_t ld, R;
    int kcontig;      // element (r, p) at X[p + r*ld] (1) or X[r + p*ld] (0)
    float *out0;      // FULL modes: big plane, K-major, row length ld0
    int64_t ld0;
    float *out1;      // second plane: K-major [R][ld1], or (PK_DSMALL, !kcontig) [K][ld1] MN-major
    int64_t ld1;
    int cross_swap;   // B side of the cross operand
    int raw_big;      // test hook (EMM_DEBUG_RAW_BIG): FULL big = x unrounded
    // launch geometry (host-computed)
    int transpose;    // 1: tile path, 0: element-wise lines
    int vec;          // 16-B vector loads legal on the source (aligned base, ld % 4 == 0)
    int64_t lines, L, Lext;   // element-wise: lines, valid / written elements per line
    int64_t nx;       // blocks along a line (element-wise) or r-tiles (transpose)
    int64_t nblocks;
};

__device__ __forceinline__ float trunc_tf32(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

template <int MODE>
__device__ __forceinline__ void split_one(const PackOperand &op, float x, float &big, float &lo) {
    const bool direct = MODE == PK_DSMALL || MODE == PK_DCROSS;
    big = direct ? trunc_tf32(x) : (op.raw_big ? x : __uint_as_float(cvt_tf32_rn(x)));
    lo = isfinite(x) ? x - big : 0.0f;   // exact
}

// One element (r, p) of op(X) -> its output position(s) (scalar tails).
template <int MODE>
__device__ __forceinline__ void pack_store(const PackOperand &op, int64_t r, int64_t p, float x) {
    float big, lo;
    split_one<MODE>(op, x, big, lo);
    const bool direct = MODE == PK_DSMALL || MODE == PK_DCROSS;
    if (!direct) op.out0[r * op.ld0 + p] = big;
    if (MODE == PK_FULL3) op.out1[r * op.ld1 + p] = __uint_as_float(cvt_tf32_rn(lo));
    if (MODE == PK_DSMALL) {
        const float sm = __uint_as_float(cvt_tf32_rn(lo));
        if (op.kcontig) op.out1[r * op.ld1 + p] = sm;
        else op.out1[r + p * op.ld1] = sm;
    }
    if (MODE == PK_FULLX || MODE == PK_DCROSS) {
        uint16_t *row = reinterpret_cast<uint16_t *>(op.out1 + r * op.ld1);
        const int64_t g = p >> 3, j = p & 7;
        const uint16_t hb = __bfloat16_as_ushort(__float2bfloat16_rn(isfinite(x) ? big : 0.0f));
        const uint16_t lb = __bfloat16_as_ushort(__float2bfloat16_rn(lo));
        row[g * 16 + j] = op.cross_swap ? lb : hb;
        row[g * 16 + 8 + j] = op.cross_swap ? hb : lb;
    }
}

// 4 consecutive output positions p0..p0+3 of line/row r (p0 % 4 == 0),
// vector stores.  FULL/cross: K-major row r; DSMALL: the line's own layout.
template <int MODE>
__device__ __forceinline__ void pack_store4(const PackOperand &op, float *o0, float *o1, int64_t e, const float (&x)[4]) {
    float big[4], lo[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) split_one<MODE>(op, x[i], big[i], lo[i]);
    if (MODE == PK_FULL1 || MODE == PK_FULL3 || MODE == PK_FULLX)
        *reinterpret_cast<float4 *>(o0 + e) = make_float4(big[0], big[1], big[2], big[3]);
    if (MODE == PK_FULL3 || MODE == PK_DSMALL)
        *reinterpret_cast<float4 *>(o1 + e) =
            make_float4(__uint_as_float(cvt_tf32_rn(lo[0])), __uint_as_float(cvt_tf32_rn(lo[1])),
                        __uint_as_float(cvt_tf32_rn(lo[2])), __uint_as_float(cvt_tf32_rn(lo[3])));
    if (MODE == PK_FULLX || MODE == PK_DCROSS) {
        uint32_t hw[2], lw[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const float b0 = isfinite(x[2 * i]) ? big[2 * i] : 0.0f, b1 = isfinite(x[2 * i + 1]) ? big[2 * i + 1] : 0.0f;
            hw[i] = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(b0)) |
                    ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(b1)) << 16);
            lw[i] = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(lo[2 * i])) |
                    ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(lo[2 * i + 1])) << 16);
        }
        uint16_t *row = reinterpret_cast<uint16_t *>(o1);
        const int64_t g = e >> 3, j = e & 7;   // j in {0, 4}
        uint2 *ph = reinterpret_cast<uint2 *>(row + g * 16 + j);
        uint2 *pl = reinterpret_cast<uint2 *>(row + g * 16 + 8 + j);
        const uint2 H = make_uint2(hw[0], hw[1]), Lw = make_uint2(lw[0], lw[1]);
        *ph = op.cross_swap ? Lw : H;
        *pl = op.cross_swap ? H : Lw;
    }
}

template <int MODE>
__device__ __forceinline__ void pack_lines(const PackOperand &op, int64_t blk) {
    const int64_t line = blk / op.nx;
    const int64_t e0 = (blk - line * op.nx) * PK_CHUNK;
    const float *__restrict__ src = op.X + line * op.ld;
    // output line: FULL / cross planes are K-major rows; DSMALL keeps the layout
    float *o0 = op.out0 ? op.out0 + line * op.ld0 : nullptr;
    float *o1 = op.out1 + line * op.ld1;
    const int64_t L = op.L, Lext = op.Lext;
    // direct modes: the GEMM re-reads the raw operand right after this pass,
    // so keep it in L2 (normal loads); FULL modes never read it again
    constexpr bool keep = MODE == PK_DSMALL || MODE == PK_DCROSS;
    auto ld4 = [](const float *p) {
        return keep ? __ldg(reinterpret_cast<const float4 *>(p)) : __ldcs(reinterpret_cast<const float4 *>(p));
    };
    auto ld1 = [](const float *p) { return keep ? __ldg(p) : __ldcs(p); };
    float v[PK_GROUPS][8];
#pragma unroll
    for (int g = 0; g < PK_GROUPS; ++g) {
        const int64_t e = e0 + ((int64_t)g * PK_THREADS + threadIdx.x) * 8;
        if (op.vec && e + 8 <= L) {
            const float4 a = ld4(src + e);
            const float4 b = ld4(src + e + 4);
            v[g][0] = a.x; v[g][1] = a.y; v[g][2] = a.z; v[g][3] = a.w;
            v[g][4] = b.x; v[g][5] = b.y; v[g][6] = b.z; v[g][7] = b.w;
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) v[g][i] = e + i < L ? ld1(src + e + i) : 0.0f;
        }
    }
#pragma unroll
    for (int g = 0; g < PK_GROUPS; ++g) {
        const int64_t e = e0 + ((int64_t)g * PK_THREADS + threadIdx.x) * 8;
        if (e + 8 <= Lext) {
            const float h0[4] = {v[g][0], v[g][1], v[g][2], v[g][3]};
            const float h1[4] = {v[g][4], v[g][5], v[g][6], v[g][7]};
            pack_store4<MODE>(op, o0, o1, e, h0);
            pack_store4<MODE>(op, o0, o1, e + 4, h1);
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (e + i >= Lext) break;
                if (op.kcontig) pack_store<MODE>(op, line, e + i, v[g][i]);
                else pack_store<MODE>(op, e + i, line, v[g][i]);   // PK_DSMALL only
            }
        }
    }
}

// MN-contiguous source (r, p) at X[r + p*ld] -> K-major row r.
template <int MODE>
__device__ __forceinline__ void pack_transpose(const PackOperand &op, int64_t blk, int64_t K, float (*tile)[PK_TR + 1]) {
    const int64_t tp = blk / op.nx;
    const int64_t r0 = (blk - tp * op.nx) * PK_TR, p0 = tp * PK_TP;
    const int64_t R = op.R, ld = op.ld;
    // load: 32 p-rows x 16 float4 along r = 512 vectors, 2 per thread
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int idx = threadIdx.x + i * PK_THREADS;
        const int pp = idx >> 4, rv = (idx & 15) * 4;
        const int64_t p = p0 + pp, r = r0 + rv;
        float x[4] = {0.f, 0.f, 0.f, 0.f};
        if (p < K) {
            const float *s = op.X + r + p * ld;
            if (op.vec && r + 4 <= R) {
                const float4 a = __ldcs(reinterpret_cast<const float4 *>(s));
                x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) x[j] = r + j < R ? __ldcs(s + j) : 0.0f;
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) tile[pp][rv + j] = x[j];
    }
    __syncthreads();
    // store: 64 rows r x 8 float4 along p, 2 per thread (8 lanes per 128-B row segment)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int idx = threadIdx.x + i * PK_THREADS;
        const int rr = idx >> 3, pv = (idx & 7) * 4;
        const int64_t r = r0 + rr;
        if (r >= R) continue;
        const float x[4] = {tile[pv][rr], tile[pv + 1][rr], tile[pv + 2][rr], tile[pv + 3][rr]};
        float *o0 = op.out0 ? op.out0 + r * op.ld0 : nullptr;
        pack_store4<MODE>(op, o0, op.out1 + r * op.ld1, p0 + pv, x);
    }
}

template <int MODE>
__global__ void __launch_bounds__(PK_THREADS) pack_split_kernel(PackOperand opA, PackOperand opB, int64_t K,
                                                                unsigned int *ctrl, int ctrl_words) {
    // Programmatic dependent launch: the GEMM may start its prologue (barrier
    // init, TMEM alloc, descriptor prefetch) now; it waits (griddepcontrol.
    // wait) for this grid's completion before its first operand load.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __shared__ float tile[PK_TP][PK_TR + 1];
    if (ctrl && blockIdx.x == 0)
        for (int i = threadIdx.x; i < ctrl_words; i += blockDim.x) ctrl[i] = 0u;
    int64_t blk = blockIdx.x;
    const bool isA = blk < opA.nblocks;
    const PackOperand &op = isA ? opA : opB;
    if (!isA) blk -= opA.nblocks;
    if (op.transpose) pack_transpose<MODE>(op, blk, K, tile);   // block-uniform branch
    else pack_lines<MODE>(op, blk);
}

static void pack_geometry(PackOperand &o, int mode, int64_t K) {
    const bool dsmall = mode == PK_DSMALL;
    const int64_t Kext = dsmall ? K : tc_kpad(K);        // FULL / cross planes are zero-padded to Kp
    o.vec = ((reinterpret_cast<uintptr_t>(o.X) & 15u) == 0 && (o.ld & 3) == 0) ? 1 : 0;
    if (o.kcontig || dsmall) {
        o.transpose = 0;
        o.lines = o.kcontig ? o.R : K;
        o.L = o.kcontig ? K : o.R;
        o.Lext = o.kcontig ? Kext : o.R;
        o.nx = (o.Lext + PK_CHUNK - 1) / PK_CHUNK;
        o.nblocks = o.lines * o.nx;
    } else {
        o.transpose = 1;
        o.nx = (o.R + PK_TR - 1) / PK_TR;
        o.nblocks = o.nx * (Kext / PK_TP);
    }
}

cudaError_t launch_pack(int mode, const PackArgs &a, const PackArgs *b, int64_t K, unsigned int *ctrl,
                        cudaStream_t s, int ctrl_words) {
    // EMM_DEBUG_RAW_BIG=1 (tests only): hand the tensor core raw FP32 bits as
    // the "big" part of the FULL modes, to probe its TF32 input conversion
    // (R7b).
    static const int raw = [] {
        const char *e = getenv("EMM_DEBUG_RAW_BIG");
        return e && e[0] == '1' ? 1 : 0;
    }();
    auto mk = [&](const PackArgs &x, bool b_side) {
        PackOperand o{};
        o.X = x.X; o.ld = x.ld; o.R = x.R; o.kcontig = x.kcontig ? 1 : 0;
        o.out0 = x.out0; o.ld0 = x.ld0; o.out1 = x.out1; o.ld1 = x.ld1;
        o.cross_swap = b_side ? 1 : 0; o.raw_big = raw;
        pack_geometry(o, mode, K);
        return o;
    };
    if (a.R <= 0 || K <= 0 || (b && b->R <= 0)) return cudaErrorInvalidConfiguration;
    const PackOperand oa = mk(a, a.b_side);
    PackOperand ob = b ? mk(*b, true) : oa;
    if (!b) ob.nblocks = 0;
    const int64_t nblk = oa.nblocks + ob.nblocks;
    if (nblk <= 0 || nblk > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    cudaEvent_t ev = nullptr;
    prof_begin(s, false, &ev);
    const dim3 grid((unsigned)nblk);
    switch (mode) {
        case PK_FULL1: pack_split_kernel<PK_FULL1><<<grid, PK_THREADS, 0, s>>>(oa, ob, K, ctrl, ctrl_words); break;
        case PK_FULL3: pack_split_kernel<PK_FULL3><<<grid, PK_THREADS, 0, s>>>(oa, ob, K, ctrl, ctrl_words); break;
        case PK_FULLX: pack_split_kernel<PK_FULLX><<<grid, PK_THREADS, 0, s>>>(oa, ob, K, ctrl, ctrl_words); break;
        case PK_DSMALL: pack_split_kernel<PK_DSMALL><<<grid, PK_THREADS, 0, s>>>(oa, ob, K, ctrl, ctrl_words); break;
        case PK_DCROSS: pack_split_kernel<PK_DCROSS><<<grid, PK_THREADS, 0, s>>>(oa, ob, K, ctrl, ctrl_words); break;
        default: return cudaErrorInvalidValue;
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    prof_end(s, false, ev);
    return cudaGetLastError();
}

// =====================================================================
// KN8: split-K reduction.  C <- alpha * (P_0 + ... + P_{S-1}) + beta*C, the
// partials summed in fixed order s = 0..S-1 (deterministic).  P_s of tile t
// is the 256 x 256 slot (s*tiles + t) in the epilogue's coalesced layout
// [rank][warp w = h*4 + q][32 float4 column groups][lane] (tc_common.cuh):
// row = m0 + 128 rank + 32 q + lane, columns n0 + 128 h + 4g .. +3.
// Block = one (tile, rank, warp) 32 x 128 part: 8 threads per lane-row set,
// thread handles 4 column groups; grid (tiles * 16, 1).
// =====================================================================
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float *__restrict__ P, int S, int M, int N,
                                                            float alpha, float beta, float *__restrict__ C,
                                                            int64_t ldc, int tiles_m, int tiles_n, int group_m) {
    asm volatile("griddepcontrol.wait;" ::: "memory");   // PDL: the GEMM's partials
    const int part = blockIdx.x & 15, t = blockIdx.x >> 4;
    const int rank = part >> 3, wslot = part & 7, h = wslot >> 2, q = wslot & 3;
    const int lane = threadIdx.x & 31, gq = threadIdx.x >> 5;   // 8 x 4 column groups
    // tile origin: the same grouped raster as the GEMM's schedule
    const int per_group = group_m * tiles_n;
    const int gidx = t / per_group, first_m = gidx * group_m;
    const int gsize = min(tiles_m - first_m, group_m);
    const int m0 = (first_m + (t % per_group) % gsize) * 256, n0 = ((t % per_group) / gsize) * 256;
    const int row = m0 + 128 * rank + 32 * q + lane;
    const int tiles = tiles_m * tiles_n;
    const float4 *base = reinterpret_cast<const float4 *>(P) + (size_t)t * (TC_SK_SLOT_FLOATS / 4) +
                         (size_t)wslot * 1024 + (size_t)rank * 8 * 1024 + lane;
    const size_t sstride = (size_t)tiles * (TC_SK_SLOT_FLOATS / 4);
    float4 acc[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j] = __ldcg(base + (4 * gq + j) * 32);
    for (int s = 1; s < S; ++s) {
        float4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = __ldcg(base + (size_t)s * sstride + (4 * gq + j) * 32);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            acc[j].x += v[j].x;
            acc[j].y += v[j].y;
            acc[j].z += v[j].z;
            acc[j].w += v[j].w;
        }
    }
    if (row >= M) return;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const float r[4] = {acc[j].x, acc[j].y, acc[j].z, acc[j].w};
        const int c0 = n0 + 128 * h + 4 * (4 * gq + j);
        float cin[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
            cin[e] = (beta != 0.0f && c0 + e < N) ? C[(int64_t)row + (int64_t)(c0 + e) * ldc] : 0.0f;
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (c0 + e < N)
                C[(int64_t)row + (int64_t)(c0 + e) * ldc] = beta == 0.0f ? alpha * r[e] : fmaf(beta, cin[e], alpha * r[e]);
    }
}

cudaError_t launch_splitk_reduce(const float *partial, int splits, int64_t M, int64_t N, float alpha, float beta,
                                 float *C, int64_t ldc, cudaStream_t s) {
    const int tiles_m = (int)((M + 2 * TC_BM - 1) / (2 * TC_BM)), tiles_n = (int)((N + TC_BN - 1) / TC_BN);
    const int64_t blocks = (int64_t)tiles_m * tiles_n * 16;
    if (blocks > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    cudaEvent_t ev = nullptr;
    prof_begin(s, false, &ev);
    {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)blocks);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t le = cudaLaunchKernelEx(&cfg, splitk_reduce_kernel, partial, splits, (int)M, (int)N, alpha, beta,
                                            C, ldc, tiles_m, tiles_n, 8);
        if (le != cudaSuccess) return le;
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    prof_end(s, false, ev);
    return cudaGetLastError();
}

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
template <int TERMS, bool A_MN, bool B_MN, bool MC>
__global__ void __launch_bounds__(TC_THREADS_P, 1)
    tc_sgemm_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
                    const __grid_constant__ CUtensorMap tmB0, const __grid_constant__ CUtensorMap tmB1,
                    const __grid_constant__ CUtensorMap tmB0h, const __grid_constant__ CUtensorMap tmB1h, int M, int N,
                    int Kp, float alpha, float beta, float *__restrict__ C, int64_t ldc, int tiles_m, int tiles_n,
                    int group_m, int kc_stages, unsigned int *__restrict__ wave_ctr, int splits,
                    float *__restrict__ partial, const TcSk sk, const __grid_constant__ PeerOut peers,
                    const float *__restrict__ acc_init, int64_t ld_init) {
    if (threadIdx.x == 0) EMM_TL(0);
    using Cfg = TcCfg<TERMS>;
    constexpr bool A1_MN = TERMS == 3 ? A_MN : false;   // cross planes are K-major
    constexpr bool B1_MN = TERMS == 3 ? B_MN : false;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
    uint64_t *empty = full + Cfg::STAGES;
    uint64_t *acc_full = empty + Cfg::STAGES;     // [2]
    uint64_t *acc_empty = acc_full + 2;           // [2] (leader's counts both CTAs' epilogue warps)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + 2);

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
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmA0);
        prefetch_tmap(&tmB0);
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
        tc_epilogue_loop<MC>(S, rank, warp & 3, (warp - TC_EPI_WARP0) >> 2, lane, tmem_base, acc_full, acc_empty,
                         kc_stages, M, N, alpha, beta, C, ldc, partial, sk, peers, cl, leader, acc_init,
                              ld_init);
    }

    tc_fence_before();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_2sm<TC_TMEM_COLS>(tmem_base);
    }
    if (threadIdx.x == 0) EMM_TL(7);
}

#ifdef EMM_TIMELINE
}  // namespace emm
extern "C" int emm_debug_timeline(unsigned long long *out, int n) {
    const int m = n < 512 * emm::TL_SLOTS ? n : 512 * emm::TL_SLOTS;
    return (int)cudaMemcpyFromSymbol(out, emm::g_emm_timeline, (size_t)m * 8);
}
namespace emm {
#endif

// ---------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// Plain 2-D FP32 tensor map (column-major array: dims {d0 = contiguous,
// d1}, row stride ld elements), out-of-bounds reads zero; used by the
// TMA-fed FFMA kernel (k_ffma_tma.cu).
bool encode_tmap_f32_2d(CUtensorMap *tm, const float *ptr, int64_t d0, int64_t d1, int64_t ld, int box0, int box1,
                        CUtensorMapSwizzle swz) {
    auto enc = get_encode_fn();
    if (!enc || !ptr) return false;
    cuuint64_t dims[2] = {(cuuint64_t)d0, (cuuint64_t)d1}, strides[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)box1}, estr[2] = {1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(ptr), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// One operand plane as a 2-D tensor map, out-of-bounds reads zero (the
// M/N/K tails).  K-major: dims {kext, R}, box {32, 128}, 128B swizzle.
// MN-major: dims {R, kext}, box {32, 32} (a 128-row tile is four boxes),
// 128B swizzle with 32B atoms (the only MN-major TF32 UMMA layout).
bool tc_make_tmap(CUtensorMap *tm, const TcPlane &p, int64_t R) { return tc_make_tmap_rows(tm, p, R, TC_BM); }

// Same with `box_rows` rows per K-major box (MN-major planes: 32x32 boxes).
bool tc_make_tmap_rows(CUtensorMap *tm, const TcPlane &p, int64_t R, int box_rows) {
    auto enc = get_encode_fn();
    if (!enc || !p.ptr) return false;
    cuuint64_t dims[2], strides[1] = {(cuuint64_t)p.ld * 4};
    cuuint32_t box[2], estr[2] = {1, 1};
    if (p.mn) {
        dims[0] = (cuuint64_t)R;
        dims[1] = (cuuint64_t)p.kext;
        box[0] = 32;
        box[1] = (cuuint32_t)TC_BK;
    } else {
        dims[0] = (cuuint64_t)p.kext;
        dims[1] = (cuuint64_t)R;
        box[0] = (cuuint32_t)TC_BK;
        box[1] = (cuuint32_t)box_rows;
    }
    CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(p.ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE,
                     p.mn ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool tma_legal(const void *ptr, int64_t ld) {
    return ptr && (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0 && ((ld * 4) & 15) == 0 && ld * 4 < (1LL << 40) &&
           ld > 0;
}

int tc_num_sms() {
    static int num_sms = 0;
    if (!num_sms) {
        int dev = 0, n = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
            num_sms = n;
        else
            return 148;   // host-only query without a device: B200
    }
    return num_sms;
}

// Split-K factor for sub-wave problems: enough (tile,
// split) units to fill the CTA pairs, each split >= 4 K-stages (128 of K).
// units = tiles * S <= CTA pairs (one wave).
int tc_splits(int64_t M, int64_t N, int64_t K) {
    const int64_t tiles = ((M + 2 * TC_BM - 1) / (2 * TC_BM)) * ((N + TC_BN - 1) / TC_BN);
    const int64_t nkb = tc_kpad(K) / TC_BK;
    const int64_t clusters = tc_num_sms() / 2;
    int64_t s;
    if (const char *e = getenv("EMM_SPLITS")) {   // experiments: force S (clamped below)
        s = atoi(e);
    } else {
        if (tiles <= 0 || tiles * 2 > clusters) return 1;
        s = clusters / tiles;
        if (s > nkb / 4) s = nkb / 4;
        if (s > 16) s = 16;
    }
    if (s < 1) s = 1;
    while (s > 1 && (tiles * s > clusters || ((nkb + s - 1) / s) * (s - 1) >= nkb)) --s;
    return (int)s;
}

size_t tc_splitk_bytes(int64_t M, int64_t N, int splits) {
    return splits > 1 ? (size_t)tc_units(M, N, splits) * TC_SK_SLOT_FLOATS * sizeof(float) : 0;
}

size_t tc_sk_slot_bytes() { return (size_t)(tc_num_sms() / 2) * TC_SK_SLOT_FLOATS * sizeof(float); }

// Stream-K policy (measured on B200): the remainder tiles of
// the last, partial wave are spread over all CTA pairs only when that
// recovers a real share of the time: >= 1 full data-parallel wave (those
// keep the wave lockstep), a remainder <= 0.6 wave, an estimated gain
// (idle share of the last wave / waves) >= 3%, and a split with 2-3 tensor
// passes (1xTF32 is fill-bandwidth-bound and measured slower).  E.g. 4096^3
// 3xTF32 (256 tiles = 3.46 waves) 553 -> 508 us; 8192^3 (13.8 waves) and
// 3072^3 (1.95 waves) lose a few % to the piece fix-ups.  EMM_SK=0 / 1
// forces it off / on (where legal).
bool tc_sk_plan(int64_t M, int64_t N, int64_t K, int splits, int terms, int *dp_tiles) {
    const char *e = getenv("EMM_SK");
    const bool force = e && e[0] == '1';
    if (e && e[0] == '0') return false;
    if (splits != 1 || K <= 0) return false;
    const int64_t tiles = ((M + 2 * TC_BM - 1) / (2 * TC_BM)) * ((N + TC_BN - 1) / TC_BN);
    const int64_t pairs = tc_num_sms() / 2;
    if (tiles * 2 <= pairs || tiles % pairs == 0 || tiles > 0x3fffffffLL) return false;
    const int64_t nch = (tc_kpad(K) / TC_BK + TC_SK_CHUNK - 1) / TC_SK_CHUNK;
    const int64_t waves = tiles / pairs, rem = tiles % pairs;
    if (!force) {
        const double gain = (1.0 - (double)rem / (double)pairs) / (double)(waves + 1);
        if (terms < 2 || waves < 1 || rem > 0.6 * pairs || gain < 0.03) return false;
    }
    // EMM_SK_DP=minus1: stream-K over the last full wave + the remainder;
    // default: every full wave stays data-parallel, only the remainder
    // tiles are spread over all pairs
    const char *dpm = getenv("EMM_SK_DP");
    const bool minus1 = dpm && !strcmp(dpm, "minus1");
    const int64_t dp = minus1 ? (waves >= 1 ? (waves - 1) * pairs : 0) : waves * pairs;
    if ((tiles - dp) * nch < pairs || (tiles - dp) * nch > 0x7fffffffLL) return false;   // every range non-empty
    *dp_tiles = (int)dp;
    return true;
}

}  // namespace emm

// Host replay of the device schedule (tests): the work items of every
// cluster for this shape, 7 ints each (cluster, m0, n0, kb0, kb1, kind,
// last); returns the item count (or -1 if `cap` is too small).
extern "C" int emm_debug_schedule(int64_t M, int64_t N, int64_t K, int use_sk, int terms, int *out, int cap) {
    using namespace emm;
    const int splits = tc_splits(M, N, K);
    int dp = 0x7fffffff;
    int d = 0;
    if (use_sk && tc_sk_plan(M, N, K, splits, terms, &d)) dp = d;
    const int tiles_m = (int)((M + 2 * TC_BM - 1) / (2 * TC_BM)), tiles_n = (int)((N + TC_BN - 1) / TC_BN);
    const int64_t units = tc_units(M, N, splits);
    const int pairs = tc_num_sms() / 2;
    const int nclus = dp < 0x7fffffff ? pairs : (int)(units < pairs ? units : pairs);
    int n = 0;
    for (int c = 0; c < nclus; ++c) {
        const TcSched S(tiles_m, tiles_n, 8, (int)tc_kpad(K), splits, dp, TC_SK_CHUNK, nclus, c);
        for (int i = 0; i < S.n_items; ++i) {
            TcWork w;
            S.item(i, w);
            if (n >= cap) return -1;
            int *o = out + 7 * n++;
            o[0] = c; o[1] = w.m0; o[2] = w.n0; o[3] = w.kb0; o[4] = w.kb1; o[5] = w.kind; o[6] = w.last;
        }
    }
    return n;
}

// Host replay of the 4-cluster pairing (preferred clusters, data-parallel
// schedule): for every CTA pair, the items it runs under cl = 4 — its own
// and the partner's mirrored ones — 8 ints each (pair, i, m0, n0, kb0, kb1,
// dummy, multicast); returns the count (-1 if `cap` is too small).
extern "C" int emm_debug_pair_schedule(int64_t M, int64_t N, int64_t K, int *out, int cap) {
    using namespace emm;
    const int tiles_m = (int)((M + 2 * TC_BM - 1) / (2 * TC_BM)), tiles_n = (int)((N + TC_BN - 1) / TC_BN);
    const int64_t units = (int64_t)tiles_m * tiles_n;
    const int pairs = tc_num_sms() / 2;
    const int nclus = (int)(units < pairs ? units : pairs);
    int n = 0;
    for (int c = 0; c < nclus; ++c) {
        const TcSched S(tiles_m, tiles_n, 8, (int)tc_kpad(K), 1, 0x7fffffff, TC_SK_CHUNK, nclus, c);
        const int cl = (c ^ 1) < nclus ? 4 : 2;   // an odd last pair has no partner
        const int n_it = tc_n_items(S, cl);
        for (int i = 0; i < n_it; ++i) {
            TcItem it;
            tc_get_item(S, cl, i, it);
            if (n >= cap) return -1;
            int *o = out + 8 * n++;
            o[0] = c; o[1] = i; o[2] = it.w.m0; o[3] = it.w.n0; o[4] = it.w.kb0; o[5] = it.w.kb1;
            o[6] = it.dummy ? 1 : 0; o[7] = it.mc ? 1 : 0;
        }
    }
    return n;
}

namespace emm {

int64_t tc_units(int64_t M, int64_t N, int splits) {
    return ((M + 2 * TC_BM - 1) / (2 * TC_BM)) * ((N + TC_BN - 1) / TC_BN) * splits;
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
    std::call_once(once, [] {
        attr_err = cudaFuncSetAttribute(tc_sgemm_kernel<TERMS, A_MN, B_MN, false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
        if (attr_err == cudaSuccess && TERMS >= 2)
            attr_err = cudaFuncSetAttribute(tc_sgemm_kernel<TERMS, A_MN, B_MN, TERMS >= 2>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
        if (attr_err == cudaSuccess && TERMS >= 2)
            attr_err = cudaFuncSetAttribute(tc_sgemm_kernel<TERMS, A_MN, B_MN, TERMS >= 2>,
                                            cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
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
        if (cudaOccupancyMaxActiveClusters(&n, tc_sgemm_kernel<TERMS, A_MN, B_MN, false>, &oc) != cudaSuccess) n = 0;
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
        cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
        cfg.stream = s;
        // clusters of one CTA pair; for data-parallel schedules a PREFERRED
        // size of 4 (two pairs sharing B by multicast; the B200 forms as many
        // 4-clusters as its GPCs hold and pairs on the remaining SMs)
        cudaLaunchAttribute at[3];
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
        auto kern = mc ? tc_sgemm_kernel<TERMS, A_MN, B_MN, TERMS >= 2> : tc_sgemm_kernel<TERMS, A_MN, B_MN, false>;
        cudaError_t le = cudaLaunchKernelEx(&cfg, kern, ta0, ta1, tb0, tb1, tb0h, tb1h, (int)M,
                                            (int)N, (int)Kp, alpha, beta, C, ldc, tiles_m, tiles_n, group_m,
                                            kc_stages, ctrl, splits, splits > 1 ? partial : nullptr, sk, peers,
                                            acc_init, ld_init);
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

cudaError_t launch_tc_sgemm(int terms, const TcOperands &ops, int64_t M, int64_t N, int64_t K, float alpha,
                            float beta, float *C, int64_t ldc, unsigned int *ctrl, int splits, float *partial,
                            cudaStream_t s, const PeerOut *peers, void *sk_ws, const float *acc_init,
                            int64_t ld_init) {
    if (M > 0x7fffffffLL || N > 0x7fffffffLL || K > 0x7fffffffLL - 32) return cudaErrorInvalidValue;
    if (splits < 1 || (splits > 1 && !partial)) return cudaErrorInvalidValue;
    if (peers && (peers->n < 0 || peers->n > 8 || splits > 1)) return cudaErrorInvalidValue;
    const PeerOut pe = peers ? *peers : PeerOut{};
    if (terms == 1 && splits == 1 && pe.n == 0 && !acc_init && tc1w_wanted(M, N, K))
        return launch_tc1w_sgemm(ops, M, N, K, alpha, beta, C, ldc, s);
    const int64_t Kp = tc_kpad(K);
    if (terms == 3)
        return launch_tc_m<3>(ops, M, N, Kp, alpha, beta, C, ldc, ctrl, splits, partial, s, pe, sk_ws, acc_init, ld_init);
    if (terms == 2)
        return launch_tc_m<2>(ops, M, N, Kp, alpha, beta, C, ldc, ctrl, splits, partial, s, pe, sk_ws, acc_init, ld_init);
    return launch_tc_m<1>(ops, M, N, Kp, alpha, beta, C, ldc, ctrl, splits, partial, s, pe, sk_ws, acc_init, ld_init);
}

}  // namespace emm
