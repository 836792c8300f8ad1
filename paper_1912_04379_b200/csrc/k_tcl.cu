// k_tcl.cu — KN11: tcgen05 3xTF32 GEMM with the operand split inside the
// kernel.  No split pass and no operand workspace: four
// producer warps per CTA read op(A) / op(B) with LDG straight from the
// caller's arrays (any transA / transB / leading dimension), split every
// element in registers
//     big   = rn_tf32(x)                      (low 13 mantissa bits zero)
//     small = rn_tf32(x - big)   (x - big exact; 0 for non-finite x)
// — the same planes the re-buffering pass KN4 (PK_FULL3) writes, so the two
// paths are bitwise identical — and store both planes K-major into the
// 128B-swizzled SMEM stage the UMMA descriptors expect.  The MMA issuer and
// the promotion/epilogue warps are the TMA kernel's (tc_common.cuh).
//
// Why LDG producers instead of TMA + an SMEM transform: per CTA and K-stage
// the MMAs read 96 KB of SMEM; TMA-then-transform would add 32 KB (TMA) +
// 32 KB (read) + 32 KB (write) = 125 B/clk of the 128 B/clk SMEM port, while
// LDG -> registers -> STS adds only the 64 KB of stores (104 B/clk, the same
// as the re-buffered TMA path), and L2 -> SM traffic is one FP32 copy of the
// operands instead of two planes.  (Paper analogue: "re-buffering" B' and
// prefetching A' done on the fly by the loading warps.)
//
// Warp roles (512 threads, 4 warpgroups; setmaxnreg re-balances registers):
//   warpgroup 0: warp 0 = TMEM owner + MMA issuer (one lane); warps 1-3 idle
//   warpgroup 1: 4 producer warps (LDG, split, STS)
//   warpgroups 2-3: 8 promotion/epilogue warps
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "emm_internal.h"
#include "ptx.cuh"
#include "tc_common.cuh"

namespace emm {

using namespace ptx;

constexpr int TL_STAGES = 3;
constexpr int TL_STAGE_BYTES = 4 * TC_TILE_BYTES;   // A big | A small | B big | B small
constexpr int TL_SMEM_BYTES = TL_STAGES * TL_STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int TL_PROD_WARP0 = 4;
constexpr int TL_PROD_WARPS = 4;
constexpr int TL_EPI_WARP0 = 8;
constexpr int TL_THREADS = 512;
// registers per thread after setmaxnreg (sum over the 16 warps = 64K)
constexpr int TL_REGS_WG0 = 48, TL_REGS_PROD = 96, TL_REGS_EPI = 184;
static_assert(128 * TL_REGS_WG0 + 128 * TL_REGS_PROD + 256 * TL_REGS_EPI <= 65536, "register budget");

// One operand as the producers read it: element (r, p) of op(X) (R x K) at
// X[p + r*ld] (KC, K contiguous) or X[r + p*ld].
struct TlOperand {
    const float *X;
    int64_t ld;
    int R;
};

__device__ __forceinline__ float4 f4zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }

// 4x4 transpose inside each quad of lanes: on entry lane j of the quad holds
// M[j][0..3]; on exit it holds M[0..3][j] (two xor-butterfly steps).
__device__ __forceinline__ void quad_transpose(float4 &v, int jq) {
    const bool odd = jq & 1, hi = jq & 2;
    float s = odd ? v.x : v.y;
    float r = __shfl_xor_sync(0xffffffffu, s, 1);
    if (odd) v.x = r; else v.y = r;
    s = odd ? v.z : v.w;
    r = __shfl_xor_sync(0xffffffffu, s, 1);
    if (odd) v.z = r; else v.w = r;
    s = hi ? v.x : v.z;
    r = __shfl_xor_sync(0xffffffffu, s, 2);
    if (hi) v.x = r; else v.z = r;
    s = hi ? v.y : v.w;
    r = __shfl_xor_sync(0xffffffffu, s, 2);
    if (hi) v.y = r; else v.w = r;
}

// Load this thread's 8 K-chunks (16 B = 4 consecutive k of one row) of the
// 128-row x 32-k tile (rows row0.., k k0..) into v[], zero outside op(X).
// Thread pt (0..127) owns:
//   KC:  rows (pt>>3) + 16j, chunk pt&7        (8 lanes cover one 128-B row)
//   !KC: row 4(pt>>2) + (pt&3), chunks j=0..7  (a quad loads 4 rows x 4 k as
//        four MN-contiguous float4 and transposes them in registers)
// VEC: the 16-B vector loads are legal (16-B aligned base, ld % 4 == 0);
// vectors crossing the R or K edge are loaded element-wise (never past op(X)).
template <bool KC, bool VEC>
__device__ __forceinline__ void tl_load(const TlOperand &op, int K, int row0, int k0, int pt, float4 (&v)[8]) {
    const float *__restrict__ X = op.X;
    const int64_t ld = op.ld;
    const int R = op.R;
    if (KC) {
        const int rr = row0 + (pt >> 3);
        const int kk = k0 + 4 * (pt & 7);
        const bool kfull = kk + 3 < K;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int row = rr + 16 * j;
            float4 x = f4zero();
            if (row < R) {
                const float *p = X + (int64_t)row * ld + kk;
                if (VEC && kfull) {
                    x = __ldg(reinterpret_cast<const float4 *>(p));
                } else {
                    if (kk < K) x.x = __ldg(p);
                    if (kk + 1 < K) x.y = __ldg(p + 1);
                    if (kk + 2 < K) x.z = __ldg(p + 2);
                    if (kk + 3 < K) x.w = __ldg(p + 3);
                }
            }
            v[j] = x;
        }
    } else {
        const int jq = pt & 3;
        const int rg = row0 + 4 * (pt >> 2);   // first row of the quad's 4-row group
        if (VEC) {
            const bool rfull = rg + 3 < R;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int k = k0 + 4 * j + jq;
                float4 x = f4zero();
                if (k < K && rg < R) {
                    const float *p = X + rg + (int64_t)k * ld;
                    if (rfull) {
                        x = __ldg(reinterpret_cast<const float4 *>(p));
                    } else {
                        x.x = __ldg(p);
                        if (rg + 1 < R) x.y = __ldg(p + 1);
                        if (rg + 2 < R) x.z = __ldg(p + 2);
                    }
                }
                v[j] = x;
            }
            // (the quad transpose happens in tl_store, after BOTH operands'
            // loads are in flight)
        } else {
            // element-wise, already in K-chunk order: lane jq reads its own row
            const int row = rg + jq;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int k = k0 + 4 * j;
                float4 x = f4zero();
                if (row < R) {
                    const float *p = X + row + (int64_t)k * ld;
                    if (k < K) x.x = __ldg(p);
                    if (k + 1 < K) x.y = __ldg(p + ld);
                    if (k + 2 < K) x.z = __ldg(p + 2 * ld);
                    if (k + 3 < K) x.w = __ldg(p + 3 * ld);
                }
                v[j] = x;
            }
        }
    }
}

__device__ __forceinline__ void split1(float x, float &big, float &small) {
    big = __uint_as_float(cvt_tf32_rn(x));
    small = isfinite(x) ? __uint_as_float(cvt_tf32_rn(x - big)) : 0.0f;
}

// Split v[] and store both planes into the stage's K-major SW128 tiles
// (row r, 16-B chunk c at r*128 + ((c ^ (r & 7)) << 4)).
template <bool KC, bool VEC>
__device__ __forceinline__ void tl_store(uint8_t *big_tile, uint8_t *small_tile, int pt, float4 (&v)[8]) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        if (!KC && VEC) quad_transpose(v[j], pt & 3);
        int r, c;
        if (KC) {
            r = (pt >> 3) + 16 * j;
            c = pt & 7;
        } else {
            r = 4 * (pt >> 2) + (pt & 3);
            c = j;
        }
        const int off = r * 128 + ((c ^ (r & 7)) << 4);
        float4 b, s;
        split1(v[j].x, b.x, s.x);
        split1(v[j].y, b.y, s.y);
        split1(v[j].z, b.z, s.z);
        split1(v[j].w, b.w, s.w);
        *reinterpret_cast<float4 *>(big_tile + off) = b;
        *reinterpret_cast<float4 *>(small_tile + off) = s;
    }
}

template <bool A_KC, bool B_KC, bool VEC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TL_THREADS, 1)
    tc_split_sgemm_kernel(const TlOperand opA, const TlOperand opB, int M, int N, int K, int Kp, float alpha,
                          float beta, float *__restrict__ C, int64_t ldc, int tiles_m, int tiles_n, int group_m,
                          int kc_stages, unsigned int *__restrict__ wave_ctr, int splits,
                          float *__restrict__ partial, const __grid_constant__ PeerOut peers) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // keeps LDS/STS (no generic)
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + TL_STAGES * TL_STAGE_BYTES);
    uint64_t *empty = full + TL_STAGES;
    uint64_t *acc_full = empty + TL_STAGES;     // [2]
    uint64_t *acc_empty = acc_full + 2;         // [2]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int nclus = (int)(gridDim.x >> 1);
    const int cid = (int)(blockIdx.x >> 1);
    const TcSched S(tiles_m, tiles_n, group_m, Kp, splits, 0x7fffffff /*no stream-K*/, 8, nclus, cid);

    if (threadIdx.x == 0) {
        for (int s = 0; s < TL_STAGES; ++s) {
            mbar_init(&full[s], 2 * TL_PROD_WARPS);   // leader's: producer warps of both CTAs
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 2 * TC_EPI_WARPS);
        }
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc_2sm<TC_TMEM_COLS>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // PDL: the prologue above may overlap the previous kernel on the stream
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp < TL_PROD_WARP0) {
        setmaxnreg_dec<TL_REGS_WG0>();
        if (warp == 0 && rank == 0 && lane == 0)
            tc_mma_loop<3, false, false, false, false, 2, TL_STAGES, TL_STAGE_BYTES>(
                S, smem, full, empty, acc_full, acc_empty, tmem_base, kc_stages);
    } else if (warp < TL_EPI_WARP0) {
        setmaxnreg_dec<TL_REGS_PROD>();
        // ===== producers: LDG -> split -> STS, both CTAs (each its 128 rows of A and of B) =====
        const int pt = threadIdx.x - 32 * TL_PROD_WARP0;
        const uint32_t leader_full0 = mapa_leader(&full[0]);
        int it = 0;
        unsigned int done_target = 0;
        bool lockstep = wave_ctr != nullptr;
        for (int i = 0; i < S.n_items; ++i) {
            const int w = i;   // no stream-K here: item i is wave i
            if (w > 0 && lockstep) {
                // wave lockstep (see tc_kernel.cuh): every producer warp of every CTA
                // finished loading wave w-1; bounded (~1 ms), then dropped
                int stop = 0;
                if (lane == 0) {
                    const long long t0 = clock64();
                    while (true) {
                        unsigned int v;
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(wave_ctr) : "memory");
                        if (v >= done_target) break;
                        __nanosleep(128);
                        if (clock64() - t0 > 2000000LL) {
                            stop = 1;
                            break;
                        }
                    }
                }
                if (__shfl_sync(0xffffffffu, stop, 0)) lockstep = false;
            }
            done_target += 2u * TL_PROD_WARPS * (unsigned)S.pairs_in_wave(w);
            TcWork wk;
            S.item(i, wk);
            const int m0 = wk.m0, n0 = wk.n0, kb0 = wk.kb0, kb1 = wk.kb1;
            const int arow = m0 + (int)rank * TC_BM;
            const int brow = n0 + (int)rank * TC_BM;
            for (int kb = kb0; kb < kb1; ++kb, ++it) {
                const int s = it % TL_STAGES;
                const uint32_t ph = (uint32_t)(it / TL_STAGES) & 1u;
                float4 va[8], vb[8];
                // global loads first: they fly while the MMA drains the stage
                tl_load<A_KC, VEC>(opA, K, arow, kb * TC_BK, pt, va);
                tl_load<B_KC, VEC>(opB, K, brow, kb * TC_BK, pt, vb);
                mbar_wait(&empty[s], ph ^ 1u);
                uint8_t *st = smem + s * TL_STAGE_BYTES;
                tl_store<A_KC, VEC>(st, st + TC_TILE_BYTES, pt, va);
                tl_store<B_KC, VEC>(st + 2 * TC_TILE_BYTES, st + 3 * TC_TILE_BYTES, pt, vb);
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive_remote(leader_full0 + (uint32_t)(s * sizeof(uint64_t)));
            }
            if (wave_ctr && lane == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(wave_ctr) : "memory");
        }
    } else {
        setmaxnreg_inc<TL_REGS_EPI>();
        tc_epilogue_loop(S, rank, warp & 3, (warp - TL_EPI_WARP0) >> 2, lane, tmem_base, acc_full, acc_empty,
                         kc_stages, M, N, alpha, beta, C, ldc, partial, TcSk{0x7fffffff, nullptr, nullptr}, peers);
    }

    tc_fence_before();
    cluster_sync();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc_2sm<TC_TMEM_COLS>(tmem_base);
    }
}

template <bool A_KC, bool B_KC, bool VEC>
static cudaError_t launch_tl_t(const TlOperand &a, const TlOperand &b, int64_t M, int64_t N, int64_t K, float alpha,
                               float beta, float *C, int64_t ldc, unsigned int *ctrl, int splits, float *partial,
                               cudaStream_t s, const PeerOut &peers) {
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
        attr_err = cudaFuncSetAttribute(tc_split_sgemm_kernel<A_KC, B_KC, VEC>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, TL_SMEM_BYTES);
    });
    if (attr_err != cudaSuccess) return attr_err;
    const int tiles_m = (int)((M + 2 * TC_BM - 1) / (2 * TC_BM));
    const int tiles_n = (int)((N + TC_BN - 1) / TC_BN);
    const int64_t units = (int64_t)tiles_m * tiles_n * splits;
    if (units > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    const int64_t pairs = tc_num_sms() / 2;
    const int64_t clusters = units < pairs ? units : pairs;
    const int kc_stages = 256 / TC_BK;
    const int Kp = (int)tc_kpad(K);
    cudaEvent_t ev = nullptr;
    prof_begin(s, true, &ev);
    {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)(2 * clusters));
        cfg.blockDim = dim3(TL_THREADS);
        cfg.dynamicSmemBytes = TL_SMEM_BYTES;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        // the wave lockstep only matters for multi-wave problems (and needs a
        // zeroed counter: ctrl == NULL disables it)
        unsigned int *wc = units > clusters ? ctrl : nullptr;
        cudaError_t le = cudaLaunchKernelEx(&cfg, tc_split_sgemm_kernel<A_KC, B_KC, VEC>, a, b, (int)M, (int)N,
                                            (int)K, Kp, alpha, beta, C, ldc, tiles_m, tiles_n, 8, kc_stages, wc,
                                            splits, splits > 1 ? partial : nullptr, peers);
        if (le != cudaSuccess) return le;
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    prof_end(s, true, ev);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || splits <= 1) return e;
    return launch_splitk_reduce(partial, splits, M, N, alpha, beta, C, ldc, s);
}

bool tl_vec_ok(const void *p, int64_t ld) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0 && (ld & 3) == 0; }

cudaError_t launch_tc_split_sgemm(bool a_kc, bool b_kc, const float *A, int64_t lda, const float *B, int64_t ldb,
                                  int64_t M, int64_t N, int64_t K, float alpha, float beta, float *C, int64_t ldc,
                                  unsigned int *ctrl, int splits, float *partial, cudaStream_t s,
                                  const PeerOut *peers) {
    if (M > 0x7fffffffLL || N > 0x7fffffffLL || K > 0x7fffffffLL - 32) return cudaErrorInvalidValue;
    if (splits < 1 || (splits > 1 && !partial)) return cudaErrorInvalidValue;
    if (peers && (peers->n < 0 || peers->n > 8 || splits > 1)) return cudaErrorInvalidValue;
    const PeerOut pe = peers ? *peers : PeerOut{};
    const TlOperand a{A, lda, (int)M}, b{B, ldb, (int)N};
    const bool vec = tl_vec_ok(A, lda) && tl_vec_ok(B, ldb);
#define EMM_TLX(AK, BK, V) \
    return launch_tl_t<AK, BK, V>(a, b, M, N, K, alpha, beta, C, ldc, ctrl, splits, partial, s, pe)
    if (vec) {
        if (a_kc && b_kc) EMM_TLX(true, true, true);
        if (a_kc && !b_kc) EMM_TLX(true, false, true);
        if (!a_kc && b_kc) EMM_TLX(false, true, true);
        EMM_TLX(false, false, true);
    }
    if (a_kc && b_kc) EMM_TLX(true, true, false);
    if (a_kc && !b_kc) EMM_TLX(true, false, false);
    if (!a_kc && b_kc) EMM_TLX(false, true, false);
    EMM_TLX(false, false, false);
#undef EMM_TLX
}

}  // namespace emm
