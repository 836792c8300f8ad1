// k_skinny_tc.cu — KN9T: skinny / memory-bound SGEMM on the tensor cores
// (the FFMA version is k_skinny.cu).
//
// min(M, N) <= 16: C' (Mr x Nc, Nc <= 16) = A' (Mr x K, the long operand) *
// B' (K x Nc), with C' = C, A' = op(A), B' = op(B) when N is short and the
// operand-role swap C' = C^T = op(B)^T op(A)^T when M is short (the paper's
// "buffer the matrix with the largest non-common dimension", PAPER.md:421-
// 424).  Arithmetic intensity ~Nc/2 flop/B: HBM is the roofline, so A' must
// stream from DRAM once, at full bandwidth, and nothing per byte may cost
// more on chip than the bytes themselves.
//
// Why tensor cores for a memory-bound GEMM: the FFMA kernel has to broadcast
// the short operand to every thread from SMEM (2 LSU wavefronts per 128-bit
// broadcast at Nc = 16: SMEM-LSU-bound at ~50 % of HBM bandwidth, round 1).
// Here one tcgen05.mma M128 x N16 x K8 per term does that work, with A'
// taken from TENSOR MEMORY: per K-stage a transform warpgroup reads its
// rows of the raw A' tile (TMA-staged in SMEM, K-major 128B-swizzled or
// MN-major) once, splits each element (big = rn_tf32(x), small =
// rn_tf32(x - big)) and writes both into TMEM with tcgen05.st; the three
// 3xTF32 MMAs (small*big, big*small, big*big) read A' from TMEM and only the
// tiny B' planes (Nc x 32 per stage, split once by the KN4 pass) from SMEM.
// SMEM traffic per A' byte: one TMA write + one LDS read (vs four reads for
// SMEM-resident A' operands).  FP32 promotion of the TMEM accumulator every
// 256 of K (R7).  The split and the per-element MMA order are the
// re-buffered KN1's (PK_FULL3 + tc_sgemm_kernel<3>), so the results are
// bitwise equal to that path (tests/test_gpu_skinny_tc.py).
//
// Warps (one CTA per SM, persistent over 128-row tiles of C'):
//   0: TMA producer (one lane)   1: TMEM owner + MMA issuer (one lane)
//   4 .. 4+4*ST_XG-1: transform groups (thread = row of the tile = TMEM lane)
//   last 4: promotion + alpha/beta epilogue (thread = row)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "emm_internal.h"
#include "ptx.cuh"
#include "tc_common.cuh"

namespace emm {

using namespace ptx;

constexpr int ST_ROWS = 128;                     // rows of C' per tile (UMMA M)
constexpr int ST_NC = 16;                        // UMMA N (Nc <= 16, zero-padded)
constexpr int ST_SS = 8;                         // SMEM ring stages
constexpr int ST_TS = 4;                         // TMEM A' ring stages
constexpr int ST_A_BYTES = ST_ROWS * TC_BK * 4;  // 16 KB raw A' tile
constexpr int ST_B_BYTES = ST_NC * TC_BK * 4;    // 2 KB per B' plane
constexpr int ST_STAGE = ST_A_BYTES + 2 * ST_B_BYTES;
constexpr int ST_SMEM = ST_SS * ST_STAGE + 1024 + 256;
constexpr int ST_XG = 3;                         // transform groups (4 warps each) working on stages it % ST_XG
constexpr int ST_XF_WARP0 = 4, ST_EPI_WARP0 = ST_XF_WARP0 + 4 * ST_XG;
constexpr int ST_THREADS = 32 * (ST_EPI_WARP0 + 4);
constexpr int ST_ACC_COL = 0;                    // 2 accumulator buffers x 16 columns
constexpr int ST_A_COL = 64;                     // TMEM A' ring: ST_TS x (32 big + 32 second) columns
constexpr int ST_KC = 256 / TC_BK;               // stages per promotion chunk

// C'(r, c) at C[r*rs + c*cs].  TERMS (as KN1): 3 = 3xTF32 (A' big + small
// in TMEM, B' PK_FULL3 planes), 2 = TF32+BF16 (A' big as tf32 + the bf16
// cross pair [bf16(big) x8 | bf16(small) x8] per 8 of K, B' PK_FULLX planes:
// one tf32 and one K16 bf16 MMA per K8), 1 = 1xTF32 (A' big only, B' PK_FULL1).
template <bool A_MN, int TERMS>
__global__ void __launch_bounds__(ST_THREADS, 1)
    skinny_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB0,
                     const __grid_constant__ CUtensorMap tmB1, int64_t Mr, int Nc, int Kp, float alpha, float beta,
                     float *C, int64_t rs, int64_t cs) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t *rawfull = reinterpret_cast<uint64_t *>(smem + ST_SS * ST_STAGE);
    uint64_t *sempty = rawfull + ST_SS;
    uint64_t *tfull = sempty + ST_SS;
    uint64_t *tempty = tfull + ST_TS;
    uint64_t *acc_full = tempty + ST_TS;    // [2]
    uint64_t *acc_empty = acc_full + 2;     // [2]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ntiles = (Mr + ST_ROWS - 1) / ST_ROWS;
    const int nkb = Kp / TC_BK;
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST_SS; ++s) {
            mbar_init(&rawfull[s], 1);
            mbar_init(&sempty[s], 2);   // transform (A' read) + MMA commit (B' read)
        }
        for (int s = 0; s < ST_TS; ++s) {
            mbar_init(&tfull[s], 4);    // the 4 transform warps of the stage's group
            mbar_init(&tempty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 4);
        }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB0);
        prefetch_tmap(&tmB1);
    }
    if (warp == 1) tmem_alloc_1sm<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    asm volatile("griddepcontrol.wait;" ::: "memory");   // PDL: B' planes from the split pass
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp == 0) {
        if (lane == 0) {
            // ===== TMA producer: raw A' tile + B' big/small planes per stage =====
            const uint64_t pol_a = policy_evict_first(), pol_b = policy_evict_last();
            int it = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int row0 = (int)(t * ST_ROWS);
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = it % ST_SS;
                    mbar_wait(&sempty[s], (uint32_t)((it / ST_SS) & 1) ^ 1u);
                    mbar_arrive_expect_tx(&rawfull[s], ST_STAGE);
                    const uint32_t st = smem_u32(smem + s * ST_STAGE);
                    if (A_MN) tma_load_2d(st, &tmA, &rawfull[s], row0, kb * TC_BK, pol_a);
                    else tma_load_2d(st, &tmA, &rawfull[s], kb * TC_BK, row0, pol_a);
                    tma_load_2d(st + ST_A_BYTES, &tmB0, &rawfull[s], kb * TC_BK, 0, pol_b);
                    tma_load_2d(st + ST_A_BYTES + ST_B_BYTES, &tmB1, &rawfull[s], kb * TC_BK, 0, pol_b);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ===== MMA issuer: 3 MMAs per K8 (small*big, big*small, big*big) =====
            constexpr uint32_t idesc = idesc_tf32_major<ST_ROWS, ST_NC, false, false>();
            int it = 0, ch = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const bool first = (kb % ST_KC) == 0;
                    const bool last = (kb % ST_KC) == ST_KC - 1 || kb == nkb - 1;
                    const int b = ch & 1;
                    const uint32_t dt = tmem_base + (uint32_t)(ST_ACC_COL + b * ST_NC);
                    if (first) {
                        mbar_wait(&acc_empty[b], (((uint32_t)ch >> 1) & 1u) ^ 1u);
                        tc_fence_after();
                    }
                    const int s = it % ST_SS, ts = it % ST_TS;
                    mbar_wait(&tfull[ts], (uint32_t)((it / ST_TS) & 1));
                    tc_fence_after();
                    const uint32_t abig = tmem_base + (uint32_t)(ST_A_COL + ts * 64);
                    const uint32_t sb = smem_u32(smem + s * ST_STAGE + ST_A_BYTES);
#pragma unroll
                    for (int k = 0; k < TC_BK / 8; ++k) {
                        const uint64_t bb = desc_kmajor_sw128(sb + (uint32_t)(32 * k));
                        const uint64_t bs = desc_kmajor_sw128(sb + ST_B_BYTES + (uint32_t)(32 * k));
                        const uint32_t acc0 = (first && k == 0) ? 0u : 1u;
                        if (TERMS == 3) {
                            mma_tf32_1sm_ts(dt, abig + 32 + 8 * k, bb, idesc, acc0);
                            mma_tf32_1sm_ts(dt, abig + 8 * k, bs, idesc, 1u);
                            mma_tf32_1sm_ts(dt, abig + 8 * k, bb, idesc, 1u);
                        } else if (TERMS == 2) {
                            // cross terms first (as KN1): [a_b | a_s] . [b_s ; b_b] as one K16 bf16 MMA
                            constexpr uint32_t idesc_x = idesc_bf16<ST_ROWS, ST_NC>();
                            mma_f16_1sm_ts(dt, abig + 32 + 8 * k, bs, idesc_x, acc0);
                            mma_tf32_1sm_ts(dt, abig + 8 * k, bb, idesc, 1u);
                        } else {
                            mma_tf32_1sm_ts(dt, abig + 8 * k, bb, idesc, acc0);
                        }
                    }
                    mma_commit_1sm(&tempty[ts]);
                    mma_commit_1sm(&sempty[s]);
                    if (last) {
                        mma_commit_1sm(&acc_full[b]);
                        ++ch;
                    }
                }
            }
        }
    } else if (warp >= ST_XF_WARP0 && warp < ST_EPI_WARP0) {
        // ===== transform: row r of the raw tile -> big / small into TMEM lane r =====
        // group g (4 warps, one per TMEM lane quarter) takes the stages it % ST_XG == g,
        // so ST_XG stages are split / stored concurrently (the per-stage chain
        // LDS -> split -> tcgen05.st -> wait::st is latency-bound)
        const int q = warp & 3;
        const int g = (warp - ST_XF_WARP0) >> 2;
        const int r = 32 * q + lane;
        int it = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            for (int kb = 0; kb < nkb; ++kb, ++it) {
                if (it % ST_XG != g) continue;
                const int s = it % ST_SS, ts = it % ST_TS;
                mbar_wait(&rawfull[s], (uint32_t)((it / ST_SS) & 1));
                const uint8_t *st = smem + s * ST_STAGE;
                float x[32];
                if (A_MN) {
                    // [32 k][128 rows], no swizzle: lane-consecutive rows, conflict-free
                    const float *a = reinterpret_cast<const float *>(st);
#pragma unroll
                    for (int k = 0; k < 32; ++k) x[k] = a[k * ST_ROWS + r];
                } else {
                    // K-major 128B swizzle: row r, 16-B chunk c at r*128 + ((c ^ (r & 7)) << 4)
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const float4 v = *reinterpret_cast<const float4 *>(st + r * 128 + ((c ^ (r & 7)) << 4));
                        x[4 * c] = v.x;
                        x[4 * c + 1] = v.y;
                        x[4 * c + 2] = v.z;
                        x[4 * c + 3] = v.w;
                    }
                }
                // the raw A' of this stage is consumed (B' planes stay until the MMA commit)
                asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
                if (q == 0 && lane == 0) mbar_arrive(&sempty[s]);
                uint32_t big[32], second[32];   // second: small (3 terms) or the bf16 cross pairs (2)
#pragma unroll
                for (int k = 0; k < 32; ++k) big[k] = cvt_tf32_rn(x[k]);
                if (TERMS == 3) {
#pragma unroll
                    for (int k = 0; k < 32; ++k) {
                        const float lo = x[k] - __uint_as_float(big[k]);   // exact
                        second[k] = isfinite(x[k]) ? cvt_tf32_rn(lo) : 0u;
                    }
                } else if (TERMS == 2) {
                    // per 8 of K: columns 0-3 = bf16(big) pairs, 4-7 = bf16(x - big) pairs (PK_FULLX's A side)
#pragma unroll
                    for (int g8 = 0; g8 < 4; ++g8) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int k0 = 8 * g8 + 2 * j, k1 = k0 + 1;
                            const bool f0 = isfinite(x[k0]), f1 = isfinite(x[k1]);
                            const float h0 = f0 ? __uint_as_float(big[k0]) : 0.0f;
                            const float h1 = f1 ? __uint_as_float(big[k1]) : 0.0f;
                            const float l0 = f0 ? x[k0] - __uint_as_float(big[k0]) : 0.0f;
                            const float l1 = f1 ? x[k1] - __uint_as_float(big[k1]) : 0.0f;
                            second[8 * g8 + j] = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(h0)) |
                                                 ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(h1)) << 16);
                            second[8 * g8 + 4 + j] = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(l0)) |
                                                     ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(l1)) << 16);
                        }
                    }
                }
                mbar_wait(&tempty[ts], (uint32_t)((it / ST_TS) & 1) ^ 1u);
                tc_fence_after();
                const uint32_t ta = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(ST_A_COL + ts * 64);
                tmem_st_32x32b_x32(ta, big);
                if (TERMS >= 2) tmem_st_32x32b_x32(ta + 32, second);
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tfull[ts]);
            }
        }
    } else if (warp >= ST_EPI_WARP0) {
        // ===== promotion (FP32 RN adds every 256 of K) + alpha/beta epilogue =====
        const int q = warp & 3;
        int ch = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            float master[ST_NC];
#pragma unroll
            for (int c = 0; c < ST_NC; ++c) master[c] = 0.0f;
            const int nch = (nkb + ST_KC - 1) / ST_KC;
            for (int c2 = 0; c2 < nch; ++c2, ++ch) {
                const int b = ch & 1;
                mbar_wait(&acc_full[b], ((uint32_t)ch >> 1) & 1u);
                tc_fence_after();
                uint32_t v[16];
                tmem_ld_32x32b_x16(tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(ST_ACC_COL + b * ST_NC), v);
                tmem_ld_wait();
#pragma unroll
                for (int c = 0; c < ST_NC; ++c) master[c] += __uint_as_float(v[c]);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty[b]);
            }
            const int64_t row = t * ST_ROWS + 32 * q + lane;
            if (row < Mr) {
                float *cp = C + row * rs;
                float cin[ST_NC];   // all C_in loads before the stores (no aliasing-forced round trips)
#pragma unroll
                for (int c = 0; c < ST_NC; ++c) cin[c] = (beta != 0.0f && c < Nc) ? cp[c * cs] : 0.0f;
#pragma unroll
                for (int c = 0; c < ST_NC; ++c)
                    if (c < Nc) cp[c * cs] = beta == 0.0f ? alpha * master[c] : fmaf(beta, cin[c], alpha * master[c]);
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_1sm<512>(tmem_base);
    }
}

static bool st_encode(CUtensorMap *tm, const float *ptr, uint64_t d0, uint64_t d1, int64_t ld, uint32_t b0,
                      uint32_t b1, CUtensorMapSwizzle swz) {
    return encode_tmap_f32_2d(tm, ptr, (int64_t)d0, (int64_t)d1, ld, (int)b0, (int)b1, swz);
}

// Policy (measured on B200, profiles/r02_skinny_tc.md): a tcgen05.mma
// M128 x N16 costs the tensor pipe about as much as a wide one (ncu: pipe
// 6.6 % active at N = 16), so the stream rate falls with the MMAs per K8:
// 65536 x 16 x 4096 runs at 5.04 TB/s with one term (1xTF32), 3.43 with two
// (TF32+BF16) and 3.09 with three (3xTF32), against 3.25 TB/s for the FFMA
// kernel (5.45 at a short side of 8, where it stays the default).
bool skinny_tc_wanted(int terms, bool tA, bool tB, int64_t M, int64_t N, int64_t K, const float *A, int64_t lda,
                      const float *B, int64_t ldb) {
    const char *e = getenv("EMM_SKINNY_TC");
    if (e && e[0] == '0') return false;
    const bool nshort = N <= SKINNY_MAX;
    const int64_t Mr = nshort ? M : N;
    const float *Ap = nshort ? A : B;
    const int64_t lda2 = nshort ? lda : ldb;
    if (!tma_legal(Ap, lda2) || K < 1 || Mr > 0x7fffff00LL || K > 0x7fffff00LL) return false;
    if (e && e[0] == '1') return true;
    const int64_t Nc = nshort ? N : M;
    // Measured against the FFMA streaming kernel KN9 (round 2: LDS operand
    // reads, FFMA2 row pairs, 448-row blocks, split-K for few blocks;
    // profiles/r02_skinny_ffma.md): KN9 is as fast or faster (and FP32-
    // accurate) everywhere except 1xTF32 with a K-contiguous long operand
    // (65536 x 16 x 4096 TN: 218 vs 244 us).  Small problems: KN9 needs no
    // split pass (one launch).
    const bool a_kcontig = nshort ? tA : !tB;
    return terms == 1 && a_kcontig && Nc > 8 && (double)Mr * (double)K >= (double)(1 << 22);
}

size_t skinny_tc_workspace_bytes(int64_t M, int64_t N, int64_t K) {
    const int64_t Nc = N <= SKINNY_MAX ? N : M;
    return align_up((size_t)2 * Nc * tc_kpad(K) * 4, 1024);
}

cudaError_t launch_skinny_tc_sgemm(int terms, bool tA, bool tB, int64_t M, int64_t N, int64_t K, float alpha,
                                   const float *A, int64_t lda, const float *B, int64_t ldb, float beta, float *C,
                                   int64_t ldc, void *ws, cudaStream_t s) {
    // roles (as k_skinny.cu): N short: A' = op(A), B' = op(B), C' = C;
    // M short: A' = op(B)^T, B' = op(A)^T, C' = C^T
    const bool nshort = N <= SKINNY_MAX;
    const int64_t Mr = nshort ? M : N;
    const int Nc = (int)(nshort ? N : M);
    const float *Ap = nshort ? A : B;
    const int64_t lda2 = nshort ? lda : ldb;
    // A'(r, p) K-contiguous?  N short: op(A)(r,p) = tA ? A[p + r*lda] : A[r + p*lda];
    // M short: op(B)(p,r) = tB ? B[r + p*ldb] : B[p + r*ldb]
    const bool a_kc = nshort ? tA : !tB;
    const float *Bp = nshort ? B : A;
    const int64_t ldb2 = nshort ? ldb : lda;
    // B'(p, c) as an (Nc x K) op-matrix row c: N short: op(B)(p,c) = tB ? B[c + p*ldb] : B[p + c*ldb];
    // M short: op(A)(c,p) = tA ? A[p + c*lda] : A[c + p*lda]
    const bool b_kc = nshort ? !tB : tA;
    const int64_t rs = nshort ? 1 : ldc, cs = nshort ? ldc : 1;
    const int64_t Kp = tc_kpad(K);
    float *B0 = reinterpret_cast<float *>(ws);
    float *B1 = B0 + (size_t)Nc * Kp;
    // split B' once into K-major planes (the re-buffered KN1's: PK_FULL3 /
    // PK_FULLX (B side of the cross pair) / PK_FULL1)
    PackArgs pb;
    pb.X = Bp; pb.ld = ldb2; pb.R = Nc; pb.kcontig = b_kc;
    pb.out0 = B0; pb.ld0 = Kp; pb.out1 = B1; pb.ld1 = Kp; pb.b_side = true;
    const int mode = terms == 3 ? PK_FULL3_ : terms == 2 ? PK_FULLX_ : PK_FULL1_;
    cudaError_t e = launch_pack(mode, pb, nullptr, K, nullptr, s, 0);
    if (e != cudaSuccess) return e;
    static std::once_flag once;
    static cudaError_t attr = cudaSuccess;
    std::call_once(once, [] {
        const void *fs[6] = {(const void *)skinny_tc_kernel<false, 1>, (const void *)skinny_tc_kernel<true, 1>,
                             (const void *)skinny_tc_kernel<false, 2>, (const void *)skinny_tc_kernel<true, 2>,
                             (const void *)skinny_tc_kernel<false, 3>, (const void *)skinny_tc_kernel<true, 3>};
        for (int i = 0; i < 6 && attr == cudaSuccess; ++i)
            attr = cudaFuncSetAttribute(fs[i], cudaFuncAttributeMaxDynamicSharedMemorySize, ST_SMEM);
    });
    if (attr != cudaSuccess) return attr;
    CUtensorMap ta, tb0, tb1;
    const bool ok = (a_kc ? st_encode(&ta, Ap, (uint64_t)K, (uint64_t)Mr, lda2, TC_BK, ST_ROWS,
                                      CU_TENSOR_MAP_SWIZZLE_128B)
                          : st_encode(&ta, Ap, (uint64_t)Mr, (uint64_t)K, lda2, ST_ROWS, TC_BK,
                                      CU_TENSOR_MAP_SWIZZLE_NONE)) &&
                    st_encode(&tb0, B0, (uint64_t)Kp, (uint64_t)Nc, Kp, TC_BK, ST_NC, CU_TENSOR_MAP_SWIZZLE_128B) &&
                    st_encode(&tb1, B1, (uint64_t)Kp, (uint64_t)Nc, Kp, TC_BK, ST_NC, CU_TENSOR_MAP_SWIZZLE_128B);
    if (!ok) return cudaErrorInvalidValue;
    if (terms == 1) tb1 = tb0;   // (unused)
    const int64_t ntiles = (Mr + ST_ROWS - 1) / ST_ROWS;
    const int64_t grid = ntiles < tc_num_sms() ? ntiles : tc_num_sms();
    cudaEvent_t ev = nullptr;
    prof_begin(s, true, &ev);
    {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3(ST_THREADS);
        cfg.dynamicSmemBytes = ST_SMEM;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        auto kern = terms == 3 ? (a_kc ? skinny_tc_kernel<false, 3> : skinny_tc_kernel<true, 3>)
                    : terms == 2 ? (a_kc ? skinny_tc_kernel<false, 2> : skinny_tc_kernel<true, 2>)
                                 : (a_kc ? skinny_tc_kernel<false, 1> : skinny_tc_kernel<true, 1>);
        e = cudaLaunchKernelEx(&cfg, kern, ta, tb0, tb1, Mr, Nc, (int)Kp, alpha, beta, C, rs, cs);
        if (e != cudaSuccess) return e;
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    prof_end(s, true, ev);
    return cudaGetLastError();
}

}  // namespace emm
