// k_tc.cu — the tensor-core SGEMM path for sm_100a (KN1 3xTF32, KN2 1xTF32,
// TF32+BF16): its operand split pass (KN4), the split-K reduce (KN8), tensor
// maps, schedules and the launch dispatch; the GEMM kernel itself is in
// tc_kernel.cuh, compiled per split in k_tc_t{1,2,3}.cu.
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
//   PK_DCROSS plane 1 only = BF16 cross operand with big = rn_tf32(x), K-major
//             (direct TF32+BF16: the GEMM's TMA rounds x to that big part)
//   PK_RAW    plane 0 = x unchanged in the SOURCE layout with a 16-byte-
//             multiple leading dimension ld0 (re-pitch of a TMA-illegal
//             operand for the in-kernel-split GEMM KN1X)
//   PK_RAWT   plane 0 = x unchanged, K-major [R][ld0], zero padded to Kp
//             (transposing copy of an MN-contiguous source; the FFMA path
//             uses it to turn a TN call into one the TMA-fed KN3b covers)
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
enum { PK_FULL1 = PK_FULL1_, PK_FULL3 = PK_FULL3_, PK_FULLX = PK_FULLX_, PK_DSMALL = PK_DSMALL_, PK_DCROSS = PK_DCROSS_, PK_RAWT = PK_RAWT_,
       PK_RAW = PK_RAW_ };

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
    // PK_DSMALL: the tensor core truncates the raw user operand (R7b).
    // PK_DCROSS: the direct GEMM's TMA rounds the user operand to
    // rn_tf32(x) on load (TFLOAT32 tensor map, R7c), so the cross plane is
    // made against that same big part
    if (MODE == PK_RAWT) big = x;
    else if (MODE == PK_DSMALL) big = trunc_tf32(x);
    else big = op.raw_big ? x : __uint_as_float(cvt_tf32_rn(x));
    lo = isfinite(x) ? x - big : 0.0f;   // exact
}

// One element (r, p) of op(X) -> its output position(s) (scalar tails).
template <int MODE>
__device__ __forceinline__ void pack_store(const PackOperand &op, int64_t r, int64_t p, float x) {
    if (MODE == PK_RAW) {
        if (op.kcontig) op.out0[r * op.ld0 + p] = x;
        else op.out0[r + p * op.ld0] = x;
        return;
    }
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
    if (MODE == PK_RAW) {
        *reinterpret_cast<float4 *>(o0 + e) = make_float4(x[0], x[1], x[2], x[3]);
        return;
    }
    float big[4], lo[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) split_one<MODE>(op, x[i], big[i], lo[i]);
    if (MODE == PK_FULL1 || MODE == PK_FULL3 || MODE == PK_FULLX || MODE == PK_RAWT)
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
    if (MODE == PK_RAW && !op.vec) {
        // re-pitch of a line that is not 16-byte aligned: scalar copies with
        // consecutive threads on consecutive elements (one 128-B segment per
        // warp access, all 16 loads in flight before the stores); the 8-wide
        // groups below would touch each sector from 8 instructions
        float w[PK_GROUPS * 8];
#pragma unroll
        for (int i = 0; i < PK_GROUPS * 8; ++i) {
            const int64_t e = e0 + (int64_t)i * PK_THREADS + threadIdx.x;
            w[i] = e < L ? ld1(src + e) : 0.0f;
        }
#pragma unroll
        for (int i = 0; i < PK_GROUPS * 8; ++i) {
            const int64_t e = e0 + (int64_t)i * PK_THREADS + threadIdx.x;
            if (e < Lext) o0[e] = w[i];
        }
        return;
    }
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
    const bool dsmall = mode == PK_DSMALL || mode == PK_RAW;   // source orientation, K unpadded
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
        case PK_RAW: pack_split_kernel<PK_RAW><<<grid, PK_THREADS, 0, s>>>(oa, ob, K, ctrl, ctrl_words); break;
        case PK_RAWT: pack_split_kernel<PK_RAWT><<<grid, PK_THREADS, 0, s>>>(oa, ob, K, ctrl, ctrl_words); break;
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
// Block = a quarter of one (tile, rank, warp) 32 x 128 part: thread (lane,
// gq) owns the KN8_J = 2 column groups 8*J*sub + J*gq + j.  The kernel runs
// after the GEMM's last CTA (its register file leaves no room to co-reside),
// so its time is the L2 round trips it exposes: every thread issues ALL of
// its partial loads (S <= KN8_SMAX, one instantiation per S) and its C_in loads before the
// first add — one round trip instead of one per split — and the grid is
// 4x finer (a sub-wave GEMM's reduce fits in one wave of resident blocks).
// Round 2: c2-1024 / c3 reduce tails measured in DESIGN.md §4.
// =====================================================================
constexpr int KN8_J = 2, KN8_SUB = 32 / (8 * KN8_J), KN8_SMAX = 16;
template <int S>
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float *__restrict__ P, int M, int N,
                                                            float alpha, float beta, float *__restrict__ C,
                                                            int64_t ldc, int tiles_m, int tiles_n, int group_m) {
    asm volatile("griddepcontrol.wait;" ::: "memory");   // PDL: the GEMM's partials
    const int sub = blockIdx.x % KN8_SUB, part = (blockIdx.x / KN8_SUB) & 15, t = blockIdx.x / (16 * KN8_SUB);
    const int rank = part >> 3, wslot = part & 7, h = wslot >> 2, q = wslot & 3;
    const int lane = threadIdx.x & 31, gq = threadIdx.x >> 5;
    const int g0 = KN8_J * (8 * sub + gq);   // first of this thread's column groups
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
    const int c0 = n0 + 128 * h + 4 * g0;    // first column
    const bool live = row < M;
    float cin[4 * KN8_J];
#pragma unroll
    for (int e = 0; e < 4 * KN8_J; ++e)
        cin[e] = (live && beta != 0.0f && c0 + e < N) ? C[(int64_t)row + (int64_t)(c0 + e) * ldc] : 0.0f;
    float4 v[S][KN8_J];
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
        for (int j = 0; j < KN8_J; ++j) v[s][j] = __ldcg(base + (size_t)s * sstride + (g0 + j) * 32);
    float4 acc[KN8_J];
#pragma unroll
    for (int j = 0; j < KN8_J; ++j) acc[j] = v[0][j];
#pragma unroll
    for (int s = 1; s < S; ++s)
#pragma unroll
        for (int j = 0; j < KN8_J; ++j) {
            acc[j].x += v[s][j].x;
            acc[j].y += v[s][j].y;
            acc[j].z += v[s][j].z;
            acc[j].w += v[s][j].w;
        }
    if (!live) return;
#pragma unroll
    for (int j = 0; j < KN8_J; ++j) {
        const float r[4] = {acc[j].x, acc[j].y, acc[j].z, acc[j].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int c = c0 + 4 * j + e;
            if (c < N)
                C[(int64_t)row + (int64_t)c * ldc] = beta == 0.0f ? alpha * r[e] : fmaf(beta, cin[4 * j + e], alpha * r[e]);
        }
    }
}

cudaError_t launch_splitk_reduce(const float *partial, int splits, int64_t M, int64_t N, float alpha, float beta,
                                 float *C, int64_t ldc, cudaStream_t s) {
    if (splits < 1 || splits > KN8_SMAX) return cudaErrorInvalidValue;
    const int tiles_m = (int)((M + 2 * TC_BM - 1) / (2 * TC_BM)), tiles_n = (int)((N + TC_BN - 1) / TC_BN);
    const int64_t blocks = (int64_t)tiles_m * tiles_n * 16 * KN8_SUB;
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
        cudaError_t le = cudaErrorInvalidValue;
        switch (splits) {
#define EMM_KN8(S_)                                                                                            \
    case S_:                                                                                                   \
        le = cudaLaunchKernelEx(&cfg, splitk_reduce_kernel<S_>, partial, (int)M, (int)N, alpha, beta, C, ldc, \
                                tiles_m, tiles_n, 8);                                                          \
        break;
            EMM_KN8(1) EMM_KN8(2) EMM_KN8(3) EMM_KN8(4) EMM_KN8(5) EMM_KN8(6) EMM_KN8(7) EMM_KN8(8)
            EMM_KN8(9) EMM_KN8(10) EMM_KN8(11) EMM_KN8(12) EMM_KN8(13) EMM_KN8(14) EMM_KN8(15) EMM_KN8(16)
#undef EMM_KN8
        }
        if (le != cudaSuccess) return le;
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    prof_end(s, false, ev);
    return cudaGetLastError();
}


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
    CUresult r = enc(tm, p.rn ? CU_TENSOR_MAP_DATA_TYPE_TFLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                     const_cast<float *>(p.ptr), dims, strides, box, estr,
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
// split) units to fill the CTA pairs, each split >= 2 K-stages (64 of K;
// late round 2: 4 stages measured slower at 512^3 3xTF32, 19.4 vs 17.4 us
// with S = 8, profiles/r02_ab_kn8.md).
// units = tiles * S <= CTA pairs (one wave).
int tc_splits(int64_t M, int64_t N, int64_t K) {
    const int64_t tiles = ((M + 2 * TC_BM - 1) / (2 * TC_BM)) * ((N + TC_BN - 1) / TC_BN);
    const int64_t nkb = tc_kpad(K) / TC_BK;
    const int64_t clusters = tc_num_sms() / 2;
    int64_t s;
    const char *e = getenv("EMM_SPLITS");         // experiments: > 0 forces S (clamped below); 0: the policy
    if (e && atoi(e) > 0) {
        s = atoi(e);
    } else {
        if (tiles <= 0 || tiles * 2 > clusters) return 1;
        s = clusters / tiles;
        if (s > nkb / 2) s = nkb / 2;
    }
    if (s > 16) s = 16;   // KN8_SMAX: the reduce keeps every split's loads in flight
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
    // one translation unit per split (k_tc_t{1,2,3}.cu) keeps the build parallel
    if (terms == 3)
        return launch_tc_terms3(ops, M, N, Kp, alpha, beta, C, ldc, ctrl, splits, partial, s, pe, sk_ws, acc_init, ld_init);
    if (terms == 2)
        return launch_tc_terms2(ops, M, N, Kp, alpha, beta, C, ldc, ctrl, splits, partial, s, pe, sk_ws, acc_init, ld_init);
    return launch_tc_terms1(ops, M, N, Kp, alpha, beta, C, ldc, ctrl, splits, partial, s, pe, sk_ws, acc_init, ld_init);
}

}  // namespace emm
